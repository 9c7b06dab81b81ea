"""Hash-sharded pool on the GPU: G shards of one pool, each scanning and
k-selecting its own slots, exchanging candidates, replaying the same evict_one loop. Every
shard must return exactly the decisions of ONE pool of the same global budget: the reference
fixtures (tests/golden, produced by the unmodified reference) are the bar, bit-exact.

The shards share the test box's single B200: `local` shards are G threads of this process
(device-to-device exchange), `torch` shards are G processes exchanging through a gloo group,
`nccl` is the production transport at world 1.
"""
import json
import os
import threading

import numpy as np
import pytest

import refshim

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RUNS = {g["name"] + "-" + g["kw"]["policy"]: g for g in json.load(open(os.path.join(GOLD, "runs.json")))["runs"]}

pytestmark = pytest.mark.gpu

ENGINE_KW = ("budget", "concurrency", "block_size", "prefetch", "skip", "take")
CASES = ["supervisor-a-cachesage", "supervisor-b-lru", "synthetic-chain-cachesage", "cfg1@128-cachesage",
         "oversized-mixed-cachesage", "pins-defer-lru", "supervisor-a-emax3-cachesage"]


def fnv(a):
    return hex(refshim.fnv1a64(np.ascontiguousarray(a, dtype="<u8")))


def _kw(g):
    kw = dict(g["kw"])
    ekw = {k: kw.pop(k) for k in list(kw) if k in ENGINE_KW}
    return ekw, kw.pop("policy"), kw


def _run_shards(g, world, grid=None, shard_slots=0, transport="local"):
    from paper_2605_27744_b200 import api, shard

    ekw, pol, kw = _kw(g)
    comms = shard.local_group(world) if transport == "local" else shard.peer_group(world)
    # the G cooperative scan grids must be co-resident; with the peer exchange the shards' streams
    # also run concurrently, and an exchange kernel waiting for a peer must never hold the SM a
    # peer's cooperative scan needs (one GPU per shard in deployment): leave SMs free for them
    grid = grid or max(1, 148 // world - (4 if transport == "peer" else 0))
    out = [None] * world
    err = []

    def work(r):
        try:
            eng = api.Engine(g["spec"], policy=pol, agent_capacity=1024, comm=comms[r], shard_slots=shard_slots,
                             grid_ctas=grid, **ekw, **kw)
            try:
                res = eng.run()
                out[r] = (res, eng.turns(), eng.evictions(), eng.warmups(), eng.pool_stats())
            finally:
                eng.close()
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        c.close()
    if err:
        raise err[0]
    return out


def _check_golden(g, res, t, ev, w):
    ws, wt, wk = w
    assert t["cached_tokens"].size == g["turns"]
    assert repr(res["hit_rate"]) == g["hit_rate"]
    assert ev.size == g["evictions"]
    assert [hex(int(x)) for x in ev[:16]] == g["first_evictions"]
    assert fnv(ev) == g["evictions_fnv"]
    assert fnv(t["cached_tokens"]) == g["cached_fnv"]
    assert fnv(t["end_us"].view(np.uint64)) == g["end_us_fnv"]
    assert ws.size == g["n_warmups"]
    assert fnv(wt) == g["warmups_fnv"]
    assert repr(res["sim_us"]) == g["sim_us"]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("name", CASES)
def test_sharded_engine_matches_reference(name, world):
    """Every shard of a G-way sharded pool reproduces the reference run bit-exactly."""
    g = RUNS[name]
    out = _run_shards(g, world)
    residents = []
    for res, t, ev, w, ps in out:
        _check_golden(g, res, t, ev, w)
        residents.append(ps["resident"])
    # the shards partition the pool: their residents add up to the single pool's
    assert sum(residents) <= g["kw"].get("budget", 10**12)
    if world > 1:
        assert min(residents) > 0


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", ["supervisor-a-cachesage", "cfg1@128-cachesage", "pins-defer-lru",
                                  "supervisor-a-emax3-cachesage"])
def test_sharded_engine_peer_exchange(name, world):
    """The fused exchange (the admission kernels store into the peers' windows and wait on their
    flags; no exchange kernel, no NCCL, no host round trip): every shard reproduces the reference
    run bit-exactly."""
    g = RUNS[name]
    for res, t, ev, w, ps in _run_shards(g, world, transport="peer"):
        _check_golden(g, res, t, ev, w)


@pytest.mark.parametrize("name", ["supervisor-a-cachesage", "pins-defer-lru"])
def test_sharded_engine_peer_unfused(name, monkeypatch):
    """The peer transport exchanging between kernels (CS_PEER_UNFUSED: the stand-alone
    8-CTA-per-peer allgather kernel between probe and decide, and between scan and replay)."""
    monkeypatch.setenv("CS_PEER_UNFUSED", "1")
    g = RUNS[name]
    for res, t, ev, w, ps in _run_shards(g, 2, transport="peer"):
        _check_golden(g, res, t, ev, w)


def _peer_worker(rank, world, port, name, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_27744_b200 import api, shard

        def allgather_bytes(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        g = RUNS[name]
        ekw, pol, kw = _kw(g)
        comm = shard.PeerComm(rank, world, 0, allgather_bytes)
        eng = api.Engine(g["spec"], policy=pol, agent_capacity=1024, comm=comm, grid_ctas=148 // world - 4, **ekw,
                         **kw)
        res = eng.run()
        q.put((rank, fnv(eng.evictions()), repr(res["hit_rate"]), fnv(eng.turns()["cached_tokens"])))
        eng.close()
        comm.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e), ""))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_processes_cuda_ipc():
    """One shard per process, the windows shared through CUDA IPC handles (the multi-GPU
    deployment's wiring; here both processes share this box's GPU)."""
    import multiprocessing as mp
    import random

    name = "supervisor-b-cachesage"
    g = RUNS[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=_peer_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, ev_fnv, hr, cached in got:
        assert ev_fnv == g["evictions_fnv"], (rank, hr)
        assert hr == g["hit_rate"]
        assert cached == g["cached_fnv"]


def test_sharded_tight_shards_error_loudly():
    """A shard too small for its share of the pool fails with CS_ERR_CAPACITY, never silently."""
    from paper_2605_27744_b200 import CacheSageError

    g = RUNS["supervisor-a-cachesage"]
    with pytest.raises(CacheSageError):
        _run_shards(g, 2, shard_slots=64)


def test_sharded_snapshot_matches_single_pool():
    """A 1M-slot realistic snapshot + a mixed trace: 4 shards vs one pool, same victims."""
    from paper_2605_27744_b200 import api, shard, workloads as W

    pool = 1 << 20
    spec = W.cfg4_mixed(sessions=300, budget=pool, seed=2608)
    keys, lt, agents, refs = W.pool_snapshot(pool, 256, seed=11, mode="adversarial")

    def single():
        eng = api.Engine(spec, policy="cachesage", budget=pool, agent_capacity=1024)
        eng.restore(keys, lt, agents=agents, refs=refs)
        eng.run_for(150)
        r = (eng.evictions(), eng.turns()["cached_tokens"], eng.warmups()[1], eng.result())
        eng.close()
        return r

    ref_ev, ref_cached, ref_w, ref_res = single()
    assert ref_ev.size > 1000
    world = 4
    comms = shard.local_group(world)
    out = [None] * world
    err = []

    def work(r):
        try:
            eng = api.Engine(spec, policy="cachesage", budget=pool, agent_capacity=1024, comm=comms[r],
                             grid_ctas=148 // world)
            eng.restore(keys, lt, agents=agents, refs=refs)  # each shard keeps what it owns
            eng.run_for(150)
            out[r] = (eng.evictions(), eng.turns()["cached_tokens"], eng.warmups()[1], eng.pool_stats())
            eng.close()
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    owners = shard.shard_owner(ref_ev, world)
    for r, (ev, cached, wt, ps) in enumerate(out):
        assert np.array_equal(ev, ref_ev)
        assert np.array_equal(cached, ref_cached)
        assert np.array_equal(wt, ref_w)
        assert ps["scans"] > 0
    assert len(set(owners.tolist())) == world  # victims came from every shard


def test_nccl_transport_world1():
    """The production transport (ncclAllGather) at world 1 on this box's one GPU."""
    from paper_2605_27744_b200 import api, shard

    g = RUNS["supervisor-a-cachesage"]
    ekw, pol, kw = _kw(g)
    comm = shard.NcclComm(shard.nccl_unique_id(), 0, 1, 0)
    eng = api.Engine(g["spec"], policy=pol, agent_capacity=1024, comm=comm, **ekw, **kw)
    try:
        res = eng.run()
        _check_golden(g, res, eng.turns(), eng.evictions(), eng.warmups())
    finally:
        eng.close()
        comm.close()


def _torch_worker(rank, world, port, name, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_27744_b200 import api, shard

        g = RUNS[name]
        ekw, pol, kw = _kw(g)
        comm = shard.TorchComm()
        eng = api.Engine(g["spec"], policy=pol, agent_capacity=1024, comm=comm, grid_ctas=148 // world, **ekw, **kw)
        res = eng.run()
        q.put((rank, fnv(eng.evictions()), repr(res["hit_rate"]), fnv(eng.turns()["cached_tokens"])))
        eng.close()
        comm.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e), ""))
    finally:
        dist.destroy_process_group()


def test_torch_gloo_processes_share_one_gpu():
    """Two processes (one shard each) exchanging through a torch.distributed gloo group."""
    import multiprocessing as mp
    import random

    name = "supervisor-b-cachesage"
    g = RUNS[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=_torch_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, ev_fnv, hr, cached in got:
        assert ev_fnv == g["evictions_fnv"], (rank, hr)
        assert hr == g["hit_rate"]
        assert cached == g["cached_fnv"]


def _nccl_worker(rank, world, uid, name, q):
    try:
        from paper_2605_27744_b200 import api, shard

        g = RUNS[name]
        ekw, pol, kw = _kw(g)
        comm = shard.NcclComm(uid, rank, world, rank)  # one GPU per rank
        eng = api.Engine(g["spec"], policy=pol, agent_capacity=1024, comm=comm, device=rank, **ekw, **kw)
        res = eng.run()
        q.put((rank, fnv(eng.evictions()), repr(res["hit_rate"]), fnv(eng.turns()["cached_tokens"])))
        eng.close()
        comm.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e), ""))


def _visible_gpus():
    import ctypes

    try:
        n = ctypes.c_int(0)
        cu = ctypes.CDLL("libcudart.so.12")
        return n.value if cu.cudaGetDeviceCount(ctypes.byref(n)) == 0 else 0
    except OSError:
        return 0


@pytest.mark.skipif(_visible_gpus() < 2, reason="needs two GPUs: NCCL runs one rank per device")
def test_nccl_world2_processes_two_gpus():
    """The production exchange at world 2: two processes, one GPU and one shard each, ncclAllGather
    over NVLink; both ranks must reproduce the reference fixture."""
    import multiprocessing as mp

    from paper_2605_27744_b200 import shard

    name = "supervisor-a-cachesage"
    g = RUNS[name]
    uid = shard.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_nccl_worker, args=(r, 2, uid, name, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, ev_fnv, hr, cached in got:
        assert ev_fnv == g["evictions_fnv"], (rank, hr)
        assert hr == g["hit_rate"]
        assert cached == g["cached_fnv"]


@pytest.mark.parametrize("transport", ["local", "peer"])
@pytest.mark.parametrize("world", [1, 2, 4])
def test_exchange_transport_allgather(transport, world):
    """The exchange itself, outside any admission: world threads, many rounds of odd and
    16-byte-multiple sizes, every rank must receive every rank's bytes in rank order."""
    import ctypes as C

    from paper_2605_27744_b200 import shard
    from paper_2605_27744_b200._lib import check, lib

    comms = shard.local_group(world) if transport == "local" else shard.peer_group(world)
    err = []

    def work(r):
        try:
            rng = np.random.default_rng(r)
            for it in range(40):
                nb = [8, 16, 808, 74400, 1000][it % 5]
                mine = ((np.arange(nb) * 7 + it * 131 + r * 17) % 251).astype(np.uint8)
                out = np.zeros(nb * world, np.uint8)
                check(lib().cs_comm_allgather_host(comms[r].h, mine.ctypes.data, out.ctypes.data, nb))
                for p in range(world):
                    want = ((np.arange(nb) * 7 + it * 131 + p * 17) % 251).astype(np.uint8)
                    assert np.array_equal(out[p * nb:(p + 1) * nb], want), (r, it, p)
                rng.random()
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        c.close()
    if err:
        raise err[0]
