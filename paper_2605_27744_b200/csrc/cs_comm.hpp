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

struct cs_comm {
    int rank = 0, world = 1;
    virtual ~cs_comm() {}
    // drecv receives world * bytes: rank r's dsend at offset r * bytes. Stream-ordered after
    // the work already queued on s; the pool's next kernel on s may read drecv.
    virtual void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) = 0;
    virtual const char* kind() const = 0;
    // this shard failed mid-admission: release (with an error) the peers waiting on it
    virtual void abort() {}
};
