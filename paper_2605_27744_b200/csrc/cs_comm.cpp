// Shard exchange transports (cs_comm.hpp) and their C ABI.
#include "cs_comm.hpp"

#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "cs_pool.hpp"

using csb::ck;
using csb::CsError;

void cs_set_error(const std::string& m);  // cs_pool.cpp

namespace {

template <class F>
int cguard(F&& f) {
    try {
        f();
        return CS_OK;
    } catch (const CsError& e) {
        cs_set_error(e.what());
        return e.code;
    } catch (const std::invalid_argument& e) {
        cs_set_error(e.what());
        return CS_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        cs_set_error(e.what());
        return CS_ERR_RUNTIME;
    }
}

// ------------------------------------------------------------------ local (threads of one process)
struct LocalGroup {
    int world;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    bool broken = false;
    std::vector<const void*> send;
    explicit LocalGroup(int w) : world(w), send(w, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        if (broken) throw CsError(CS_ERR_RUNTIME, "shard exchange: a peer shard failed");
        const unsigned long long my = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return;
        }
        // a peer that died (threw) would leave the others waiting forever: time out instead
        if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != my || broken; }) || broken) {
            broken = true;
            cv.notify_all();
            throw CsError(CS_ERR_RUNTIME, "shard exchange: peer shards did not arrive (timeout)");
        }
    }
};

struct LocalComm : cs_comm {
    std::shared_ptr<LocalGroup> g;
    const char* kind() const override { return "local"; }
    void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) override {
        ck(cudaStreamSynchronize(s), "shard exchange: send ready");
        g->send[rank] = dsend;
        g->barrier();
        for (int p = 0; p < world; ++p)
            ck(cudaMemcpyAsync(static_cast<char*>(drecv) + (size_t)p * bytes, g->send[p], bytes, cudaMemcpyDefault, s),
               "shard exchange: peer copy");
        ck(cudaStreamSynchronize(s), "shard exchange: peer copy");
        g->barrier();  // no shard rewrites its send buffer while a peer still copies from it
    }
    void abort() override {
        std::lock_guard<std::mutex> lk(g->m);
        g->broken = true;
        g->cv.notify_all();
    }
    ~LocalComm() override {
        std::lock_guard<std::mutex> lk(g->m);
        g->broken = true;  // a destroyed shard releases anyone still waiting on it
        g->cv.notify_all();
    }
};

// ------------------------------------------------------------------ callback (host allgather)
struct CallbackComm : cs_comm {
    cs_allgather_fn fn = nullptr;
    void* ctx = nullptr;
    void* hsend = nullptr;
    void* hrecv = nullptr;
    size_t cap = 0;
    const char* kind() const override { return "callback"; }
    void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) override {
        if (bytes > cap) {
            if (hsend) cudaFreeHost(hsend);
            if (hrecv) cudaFreeHost(hrecv);
            hsend = hrecv = nullptr;
            cap = 0;
            ck(cudaMallocHost(&hsend, bytes), "cudaMallocHost");
            ck(cudaMallocHost(&hrecv, bytes * world), "cudaMallocHost");
            cap = bytes;
        }
        ck(cudaMemcpyAsync(hsend, dsend, bytes, cudaMemcpyDeviceToHost, s), "shard exchange D2H");
        ck(cudaStreamSynchronize(s), "shard exchange D2H");
        if (fn(ctx, hsend, hrecv, bytes) != 0) throw CsError(CS_ERR_RUNTIME, "shard exchange: allgather callback failed");
        ck(cudaMemcpyAsync(drecv, hrecv, bytes * world, cudaMemcpyHostToDevice, s), "shard exchange H2D");
        ck(cudaStreamSynchronize(s), "shard exchange H2D");  // hrecv is reused by the next exchange
    }
    ~CallbackComm() override {
        if (hsend) cudaFreeHost(hsend);
        if (hrecv) cudaFreeHost(hrecv);
    }
};

// ------------------------------------------------------------------ NCCL (loaded at run time)
typedef struct {
    char internal[128];
} NcclUid;
typedef void* NcclComm;
struct NcclApi {
    void* h = nullptr;
    int (*get_unique_id)(NcclUid*) = nullptr;
    int (*comm_init_rank)(NcclComm*, int, NcclUid, int) = nullptr;
    int (*all_gather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
    int (*comm_destroy)(NcclComm) = nullptr;
    const char* (*error_string)(int) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = std::getenv("CS_NCCL_LIB");
        const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            if (!n) continue;
            api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
        api.get_unique_id = reinterpret_cast<int (*)(NcclUid*)>(dlsym(api.h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<int (*)(NcclComm*, int, NcclUid, int)>(dlsym(api.h, "ncclCommInitRank"));
        api.all_gather = reinterpret_cast<int (*)(const void*, void*, size_t, int, NcclComm, cudaStream_t)>(
            dlsym(api.h, "ncclAllGather"));
        api.comm_destroy = reinterpret_cast<int (*)(NcclComm)>(dlsym(api.h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(api.h, "ncclGetErrorString"));
    });
    if (!api.h || !api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.comm_destroy)
        throw CsError(CS_ERR_CUDA, "libnccl.so.2 not loadable (set CS_NCCL_LIB)");
    return api;
}

void nck(int r, const char* what) {
    if (r != 0) {
        const char* m = nccl().error_string ? nccl().error_string(r) : "?";
        throw CsError(CS_ERR_CUDA, std::string(what) + ": " + m);
    }
}

constexpr int kNcclUint8 = 1;  // ncclDataType_t ncclUint8

struct NcclCommImpl : cs_comm {
    NcclComm c = nullptr;
    const char* kind() const override { return "nccl"; }
    void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) override {
        nck(nccl().all_gather(dsend, drecv, bytes, kNcclUint8, c, s), "ncclAllGather");
    }
    ~NcclCommImpl() override {
        if (c) nccl().comm_destroy(c);
    }
};

}  // namespace

extern "C" {

int cs_comm_local_group(int world, cs_comm_t* out) {
    return cguard([&] {
        if (world < 1 || world > csb::kMaxShards || !out) throw std::invalid_argument("cs_comm_local_group: bad world");
        auto g = std::make_shared<LocalGroup>(world);
        for (int r = 0; r < world; ++r) {
            auto* c = new LocalComm();
            c->rank = r;
            c->world = world;
            c->g = g;
            out[r] = c;
        }
    });
}

int cs_comm_callback(int rank, int world, cs_allgather_fn fn, void* ctx, cs_comm_t* out) {
    return cguard([&] {
        if (world < 1 || world > csb::kMaxShards || rank < 0 || rank >= world || !fn || !out)
            throw std::invalid_argument("cs_comm_callback: bad argument");
        auto* c = new CallbackComm();
        c->rank = rank;
        c->world = world;
        c->fn = fn;
        c->ctx = ctx;
        *out = c;
    });
}

int cs_nccl_unique_id(uint8_t* id128) {
    return cguard([&] {
        if (!id128) throw std::invalid_argument("cs_nccl_unique_id: null argument");
        NcclUid u;
        nck(nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id128, u.internal, 128);
    });
}

int cs_comm_nccl(const uint8_t* id128, int rank, int world, int device, cs_comm_t* out) {
    return cguard([&] {
        if (!id128 || world < 1 || world > csb::kMaxShards || rank < 0 || rank >= world || !out)
            throw std::invalid_argument("cs_comm_nccl: bad argument");
        ck(cudaSetDevice(device), "cudaSetDevice");
        NcclUid u;
        std::memcpy(u.internal, id128, 128);
        auto* c = new NcclCommImpl();
        c->rank = rank;
        c->world = world;
        try {
            nck(nccl().comm_init_rank(&c->c, world, u, rank), "ncclCommInitRank");
        } catch (...) {
            c->c = nullptr;
            delete c;
            throw;
        }
        *out = c;
    });
}

int cs_comm_destroy(cs_comm_t c) {
    return cguard([&] { delete c; });
}

int cs_shard_owner(uint64_t key, int world) { return world > 0 ? csb::shard_owner(key, world) : -1; }

}  // extern "C"
