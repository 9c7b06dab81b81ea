// Shard exchange transports (cs_comm.hpp) and their C ABI.
#include "cs_comm.hpp"

#include <dlfcn.h>

#include <chrono>
#include <cstdio>
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

// ------------------------------------------------------------------ peer memory (fused exchange)
// Each rank owns a window (2 parity slots x world x cap bytes) and one flag word per source rank
// and message part on its own device; every rank maps every peer's window and flags (same
// process: plain pointers with peer access enabled between distinct devices; other processes:
// CUDA IPC handles). An exchange is one
// stream-ordered kernel (csb::launch_peer_allgather): no host round trip, no NCCL.
struct PeerComm : cs_comm {
    int device = 0;
    size_t cap = 0;
    unsigned long long seq = 0;
    unsigned char* my_win = nullptr;         // owned
    unsigned long long* my_flags = nullptr;  // owned
    csb::PeerTable t{};
    std::vector<void*> ipc_opened;           // peers' mappings to close
    bool connected = false;
    // Shards that are threads of one process share one CUDA context (and, in the tests, one
    // GPU): a device-wide synchronizing call of one thread (cudaFree, ...) would wait for another
    // shard's exchange kernel, itself waiting for the first thread's next exchange, and a
    // cooperative grid queued behind one shard's exchange kernel can hold back the dispatch of a
    // peer's exchange kernel on the shared GPU. Those shards drain their own stream and meet at a
    // host rendezvous before each exchange kernel is enqueued, and drain it again after, so the
    // group's exchange kernels always run together with nothing queued behind them. Shards in
    // different processes (one per GPU in deployment) need none: their exchange is fully
    // stream-ordered on the device.
    std::shared_ptr<LocalGroup> g;
    const char* kind() const override { return "peer"; }
    void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) override {
        if (!connected) throw CsError(CS_ERR_LOGIC, "peer exchange: not connected");
        if (bytes > cap) throw CsError(CS_ERR_CAPACITY, "peer exchange: message exceeds the window capacity");
        if (g) {
            ck(cudaStreamSynchronize(s), "peer exchange: send ready");
            g->barrier();
        }
        ++seq;
        static const bool trace = std::getenv("CS_DEBUG_PEER") != nullptr;
        if (trace) std::fprintf(stderr, "[peer] rank %d seq %llu bytes %zu\n", rank, seq, bytes);
        ck(csb::launch_peer_allgather(dsend, drecv, bytes, t, rank, world, seq, cap, s), "peer allgather");
        if (g) ck(cudaStreamSynchronize(s), "peer exchange");
    }
    bool fused(csb::PeerTable* out, size_t* c) override {
        if (!connected || std::getenv("CS_PEER_UNFUSED")) return false;
        *out = t;
        *c = cap;
        return true;
    }
    unsigned long long fused_next() override { return ++seq; }
    void fused_meet(cudaStream_t s) override {
        if (g) {
            ck(cudaStreamSynchronize(s), "fused exchange: send ready");
            g->barrier();
        }
    }
    void fused_end(cudaStream_t s) override {
        if (g) ck(cudaStreamSynchronize(s), "fused exchange");
    }
    // a failing shard must not leave its peers spinning: poison its flag in every peer (their
    // exchange kernels then trap with an error instead of waiting forever)
    void abort() override {
        if (g) {
            std::lock_guard<std::mutex> lk(g->m);
            g->broken = true;
            g->cv.notify_all();
        }
        if (!connected) return;
        const unsigned long long poison = ~0ull;
        for (int p = 0; p < world; ++p)
            if (t.flags[p])
                for (int q = 0; q < csb::kPeerParts; ++q)
                    cudaMemcpy(t.flags[p] + rank * csb::kPeerParts + q, &poison, 8, cudaMemcpyHostToDevice);
    }
    ~PeerComm() override {
        for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
        if (my_win) cudaFree(my_win);
        if (my_flags) cudaFree(my_flags);
    }
};

PeerComm* peer_new(int rank, int world, int device, size_t cap) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new PeerComm();
    c->rank = rank;
    c->world = world;
    c->device = device;
    c->cap = (cap + 15) & ~size_t(15);
    try {
        ck(cudaMalloc(reinterpret_cast<void**>(&c->my_win), 2 * (size_t)world * c->cap), "cudaMalloc(peer window)");
        const size_t fbytes = 8 * (size_t)csb::kMaxShards * csb::kPeerParts;
        ck(cudaMalloc(reinterpret_cast<void**>(&c->my_flags), fbytes), "cudaMalloc(peer flags)");
        ck(cudaMemset(c->my_flags, 0, fbytes), "memset");
        ck(cudaDeviceSynchronize(), "peer window");
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}

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

int cs_comm_peer_group(int world, const int* devices, size_t cap, cs_comm_t* out) {
    return cguard([&] {
        if (world < 1 || world > csb::kMaxShards || !out || cap == 0)
            throw std::invalid_argument("cs_comm_peer_group: bad argument");
        std::vector<PeerComm*> cs;
        try {
            auto grp = std::make_shared<LocalGroup>(world);
            for (int r = 0; r < world; ++r) {
                cs.push_back(peer_new(r, world, devices ? devices[r] : 0, cap));
                cs.back()->g = grp;
            }
            for (int r = 0; r < world; ++r) {
                ck(cudaSetDevice(cs[r]->device), "cudaSetDevice");
                for (int p = 0; p < world; ++p) {
                    if (cs[p]->device != cs[r]->device) {
                        int can = 0;
                        ck(cudaDeviceCanAccessPeer(&can, cs[r]->device, cs[p]->device), "cudaDeviceCanAccessPeer");
                        if (!can) throw CsError(CS_ERR_CUDA, "peer exchange: no peer access between the shards' GPUs");
                        const cudaError_t e = cudaDeviceEnablePeerAccess(cs[p]->device, 0);
                        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "cudaDeviceEnablePeerAccess");
                        cudaGetLastError();
                    }
                    cs[r]->t.win[p] = cs[p]->my_win;
                    cs[r]->t.flags[p] = cs[p]->my_flags;
                }
                cs[r]->connected = true;
            }
        } catch (...) {
            for (auto* c : cs) delete c;
            throw;
        }
        for (int r = 0; r < world; ++r) out[r] = cs[r];
    });
}

int cs_comm_peer_create(int rank, int world, int device, size_t cap, uint8_t* handle_out, cs_comm_t* out) {
    return cguard([&] {
        if (world < 1 || world > csb::kMaxShards || rank < 0 || rank >= world || !handle_out || !out || cap == 0)
            throw std::invalid_argument("cs_comm_peer_create: bad argument");
        PeerComm* c = peer_new(rank, world, device, cap);
        try {
            cudaIpcMemHandle_t hw, hf;
            ck(cudaIpcGetMemHandle(&hw, c->my_win), "cudaIpcGetMemHandle(window)");
            ck(cudaIpcGetMemHandle(&hf, c->my_flags), "cudaIpcGetMemHandle(flags)");
            static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
            std::memcpy(handle_out, &hw, 64);
            std::memcpy(handle_out + 64, &hf, 64);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int cs_comm_peer_connect(cs_comm_t comm, const uint8_t* handles) {
    return cguard([&] {
        auto* c = dynamic_cast<PeerComm*>(comm);
        if (!c || !handles) throw std::invalid_argument("cs_comm_peer_connect: not a peer comm");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        for (int p = 0; p < c->world; ++p) {
            if (p == c->rank) {
                c->t.win[p] = c->my_win;
                c->t.flags[p] = c->my_flags;
                continue;
            }
            cudaIpcMemHandle_t hw, hf;
            std::memcpy(&hw, handles + 128 * (size_t)p, 64);
            std::memcpy(&hf, handles + 128 * (size_t)p + 64, 64);
            void* w = nullptr;
            void* f = nullptr;
            ck(cudaIpcOpenMemHandle(&w, hw, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(window)");
            c->ipc_opened.push_back(w);
            ck(cudaIpcOpenMemHandle(&f, hf, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(flags)");
            c->ipc_opened.push_back(f);
            c->t.win[p] = static_cast<unsigned char*>(w);
            c->t.flags[p] = static_cast<unsigned long long*>(f);
        }
        c->connected = true;
    });
}

int cs_comm_allgather_host(cs_comm_t comm, const void* send, void* recv, size_t bytes) {
    return cguard([&] {
        if (!comm || !send || !recv) throw std::invalid_argument("cs_comm_allgather_host: null argument");
        cudaStream_t s;
        ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        void* ds = nullptr;
        void* dr = nullptr;
        try {
            ck(cudaMalloc(&ds, bytes), "cudaMalloc");
            ck(cudaMalloc(&dr, bytes * (size_t)comm->world), "cudaMalloc");
            ck(cudaMemcpyAsync(ds, send, bytes, cudaMemcpyHostToDevice, s), "H2D");
            comm->allgather(ds, dr, bytes, s);
            ck(cudaMemcpyAsync(recv, dr, bytes * (size_t)comm->world, cudaMemcpyDeviceToHost, s), "D2H");
            ck(cudaStreamSynchronize(s), "allgather");
        } catch (...) {
            cudaFree(ds);
            cudaFree(dr);
            cudaStreamDestroy(s);
            throw;
        }
        cudaFree(ds);
        cudaFree(dr);
        cudaStreamDestroy(s);
    });
}

int cs_comm_destroy(cs_comm_t c) {
    return cguard([&] { delete c; });
}

int cs_shard_owner(uint64_t key, int world) { return world > 0 ? csb::shard_owner(key, world) : -1; }

}  // extern "C"
