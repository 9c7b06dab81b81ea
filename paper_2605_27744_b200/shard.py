"""Hash-sharded pool: the shard exchange transports and the owner function.

A pool of global budget N is split over G <= 8 GPUs; block key k lives on shard
(k >> 40) % G. Each shard scans and k-selects its own slots; per admission the shards allgather
their probe results and per-class candidate lists and replay the same exact evict_one loop
(cs_shard.cuh). The transports (include/cachesage_b200.h):

  NcclComm      ncclAllGather on the engine stream, one process per GPU (the production path)
  local_group   G shards driven by G threads of one process (device-to-device copies); the
                shards may share one GPU, which is how the single-GPU tests exercise G > 1
  TorchComm     host allgather through a torch.distributed group (gloo): G processes that may
                share one GPU
  peer_group /  the fused exchange over peer memory (NVLink / NVSwitch stores + flags, one kernel
  PeerComm      per exchange): G threads of one process, or one process per GPU via CUDA IPC
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib

ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


def shard_owner(keys, world):
    """owner(key) = (key >> 40) % world, vectorised (matches cs_shard_owner)."""
    k = np.asarray(keys, dtype=np.uint64)
    return ((k >> np.uint64(40)) % np.uint64(world)).astype(np.int64)


class Comm:
    """A shard exchange handle (cs_comm_t). Borrowed by the engines that use it."""

    def __init__(self, h, rank, world, keep=None):
        self.h = h
        self.rank, self.world = rank, world
        self._keep = keep

    def close(self):
        if getattr(self, "h", None):
            lib().cs_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def local_group(world):
    """world Comms for world shards driven by world threads of this process."""
    hs = (C.c_void_p * world)()
    check(lib().cs_comm_local_group(world, hs))
    return [Comm(C.c_void_p(hs[r]), r, world) for r in range(world)]


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    check(lib().cs_nccl_unique_id(buf))
    return bytes(buf)


def NcclComm(uid, rank, world, device):
    """NCCL transport (one process per GPU). uid: 128 bytes from nccl_unique_id() on rank 0."""
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    h = C.c_void_p()
    check(lib().cs_comm_nccl(buf, rank, world, device, C.byref(h)))
    return Comm(h, rank, world)


PEER_CAP = 1 << 18  # bytes per rank and exchange (the shard lists are 74,400 B)


def peer_group(world, devices=None, cap=PEER_CAP):
    """world Comms over peer memory for world shards driven by world threads of this process
    (the fused exchange: one kernel stores each shard's bytes into its peers' windows)."""
    hs = (C.c_void_p * world)()
    devs = None if devices is None else (C.c_int * world)(*devices)
    check(lib().cs_comm_peer_group(world, devs, cap, hs))
    return [Comm(C.c_void_p(hs[r]), r, world) for r in range(world)]


def PeerComm(rank, world, device, allgather_bytes, cap=PEER_CAP):
    """Peer-memory transport for one shard per process. allgather_bytes(b: bytes) -> list of
    every rank's bytes in rank order (e.g. torch.distributed.all_gather_object): exchanges the
    ranks' CUDA IPC handles once."""
    h = C.c_void_p()
    mine = (C.c_uint8 * 128)()
    check(lib().cs_comm_peer_create(rank, world, device, cap, mine, C.byref(h)))
    comm = Comm(h, rank, world)
    allh = allgather_bytes(bytes(mine))
    buf = (C.c_uint8 * (128 * world)).from_buffer_copy(b"".join(allh))
    check(lib().cs_comm_peer_connect(comm.h, buf))
    return comm


def CallbackComm(rank, world, allgather):
    """allgather(send: np.uint8 array, world) -> np.uint8 array of world * send.size bytes."""

    def fn(ctx, send, recv, nbytes):
        try:
            src = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), shape=(nbytes,)).copy()
            out = np.ascontiguousarray(allgather(src, world), dtype=np.uint8)
            if out.size != nbytes * world:
                return -1
            C.memmove(recv, out.ctypes.data, out.size)
            return 0
        except Exception:  # an exception must not cross the C boundary
            return -1

    cb = ALLGATHER_FN(fn)
    h = C.c_void_p()
    check(lib().cs_comm_callback(rank, world, cb, None, C.byref(h)))
    return Comm(h, rank, world, keep=cb)


def TorchComm(group=None):
    """Host allgather over a torch.distributed process group (e.g. gloo)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)

    def allgather(send, w):
        t = torch.from_numpy(send)
        out = torch.empty(w * send.size, dtype=torch.uint8)
        dist.all_gather_into_tensor(out, t, group=group)
        return out.numpy()

    return CallbackComm(rank, world, allgather)


def snapshot_shard(n_local, world, rank, n_agents, seed=11, mode="realistic", t0=1 << 20):
    """This shard's part of a global snapshot of world * n_local resident blocks (cfg5
    composition): keys owned by `rank`, last_touch a permutation interleaved across shards
    (globally distinct ticks), ~13 A agent-carrying slots and 0.01% pinned overall."""
    from .workloads import pool_snapshot

    keys, lt, agents, refs = pool_snapshot(n_local, n_agents, seed=seed + 7919 * rank, mode=mode)
    # force ownership: replace the owner bits (key >> 40) % world by rank, keep the rest
    hi = keys >> np.uint64(40)
    hi = hi - (hi % np.uint64(world)) + np.uint64(rank)
    keys = (hi << np.uint64(40)) | (keys & np.uint64((1 << 40) - 1))
    lt = (lt - lt.min()) * np.uint64(world) + np.uint64(rank) + np.uint64(t0)
    if mode == "realistic" and world > 1:  # ~13 A agent blocks in total, not per shard
        ag = agents != np.uint32(0xFFFFFFFF)
        drop = ag & (np.arange(agents.size) % world != 0)
        agents = np.where(drop, np.uint32(0xFFFFFFFF), agents).astype(np.uint32)
    return keys, lt, agents, refs
