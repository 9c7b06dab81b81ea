// Shard exchange for the hash-sharded pool: one allgather per exchange step.
// Three transports behind one interface:
//   nccl     ncclAllGather on the pool's stream (one process per GPU, NVLink / NVSwitch);
//            libnccl is loaded at run time (the copy torch already loaded, else the system one)
//   local    G shards driven by G host threads of one process (one or several devices):
//            device-to-device copies between the shards' buffers, host barriers around them
//   callback the bytes go through host memory to a caller-supplied allgather (e.g. a
//            torch.distributed gloo group); used to test the N>1 path with processes that
//            share one GPU
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace csb {
struct PeerTable;
}

struct cs_comm {
    int rank = 0, world = 1;
    virtual ~cs_comm() {}
    // drecv receives world * bytes: rank r's dsend at offset r * bytes. Stream-ordered after
    // the work already queued on s; the pool's next kernel on s may read drecv.
    virtual void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) = 0;
    virtual const char* kind() const = 0;
    // this shard failed mid-admission: release (with an error) the peers waiting on it
    virtual void abort() {}
    // The fused exchange (peer transport only): the admission kernels store into the peers'
    // windows and wait on their flags themselves (csb::ShardX). fused() fills the table and the
    // window bytes per rank; fused_next() numbers the next exchange; fused_meet() precedes the
    // kernel that waits and fused_end() follows it (shards that share a GPU in one process
    // drain their stream and meet there, so no kernel that waits is queued behind another
    // shard's cooperative scan).
    virtual bool fused(csb::PeerTable*, size_t*) { return false; }
    virtual unsigned long long fused_next() { return 0; }
    virtual void fused_meet(cudaStream_t) {}
    virtual void fused_end(cudaStream_t) {}
};
