// Standalone device TransitionLearner (cs_learner_t): the reference's learner API
// (transition_learner.hpp:19-60, bound in py_module.cpp:103-123), its reachability rebuild
// (reachability.cpp:39-81), argmax_row (transition_learner.cpp:79-96) and the horizon-k survival
// oracle exact_survival_prob (survival_oracle.cpp:9-62), on the GPU. Paths relative to
// /root/reference/proj. The pool's own learner lives inside the admission kernel; this handle
// serves callers that drive the learner directly (the reference's Python API and tests).
//
// Layout: dense u32 counts over agent indices (first-seen order, note_agent), u32 row totals,
// the window as an index-pair ring. A zero cell is the reference's erased map entry.
#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "cs_block.cuh"
#include "cs_pool.hpp"

using csb::ck;
using csb::CsError;

void cs_set_error(const std::string& m);  // cs_pool.cpp

namespace csb {

// K3 batch record: the window after the batch is the last W pairs of (old window ++ batch).
// Element e of that concatenation is popped iff e < pops; a batch pair adds +1, a popped pair
// -1 (a batch pair popped within its own batch nets 0). Deltas are warp-aggregated per cell.
__global__ void learner_record_kernel(unsigned int* counts, unsigned int* totals, int* win_a, int* win_b, int acap,
                                      long long W, long long head0, long long size0, long long pops,
                                      const int* ba, const int* bb, long long n) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned int act = __ballot_sync(0xffffffffu, e < size0 + n);
    if (e >= size0 + n) return;
    int a, b, d;
    if (e < size0) {
        const long long q = (head0 + e) % W;
        a = win_a[q];
        b = win_b[q];
        d = e < pops ? -1 : 0;
    } else {
        const long long j = e - size0;
        a = ba[j];
        b = bb[j];
        d = e < pops ? 0 : 1;
    }
    const long long cell = (long long)a * acap + b;
    const unsigned long long key = (unsigned long long)cell * 4ull + (unsigned long long)(d + 1);
    const unsigned int peers = __match_any_sync(act, key);
    if (d != 0 && (threadIdx.x & 31) == __ffs(peers) - 1) {
        const unsigned int m = (unsigned int)__popc(peers);
        if (d > 0) {
            atomicAdd(counts + cell, m);
            atomicAdd(totals + a, m);
        } else {
            atomicSub(counts + cell, m);
            atomicSub(totals + a, m);
        }
    }
}

// The surviving batch pairs into the ring (after learner_record_kernel read the popped ones).
__global__ void learner_window_kernel(int* win_a, int* win_b, long long W, long long head0, long long size0,
                                      long long pops, const int* ba, const int* bb, long long n) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n || size0 + j < pops) return;
    const long long q = (head0 + size0 + j) % W;
    win_a[q] = ba[j];
    win_b[q] = bb[j];
}

// nonzero cells and nonzero rows (state_bytes accounting)
__global__ void learner_nonzero_kernel(const unsigned int* counts, const unsigned int* totals, int acap, int n,
                                       unsigned long long* out) {
    unsigned long long c = 0, r = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)n * n;
         i += (long long)gridDim.x * blockDim.x) {
        const int a = (int)(i / n), b = (int)(i % n);
        c += counts[(long long)a * acap + b] != 0u;
        if (b == 0) r += totals[a] != 0u;
    }
    for (int o = 16; o; o >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, o);
        r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, c);
        atomicAdd(out + 1, r);
    }
}

// K3b rebuild_reachability over the window pairs (every positive cell is a window pair):
// level-synchronous BFS, edge iff !(count/total < tau) in fp64, expansion while depth+1 < e_max.
__global__ void learner_bfs_kernel(const unsigned int* counts, const unsigned int* totals, const int* win_a,
                                   const int* win_b, int acap, long long W, long long head, long long size, int n,
                                   int current, double tau, int e_max, int* hops) {
    extern __shared__ unsigned char sm[];
    unsigned char* hop = sm;  // n <= kMaxAgents
    const int tid = threadIdx.x, T = blockDim.x;
    for (int x = tid; x < n; x += T) hop[x] = (unsigned char)min(e_max, 255);
    __syncthreads();
    if (tid == 0 && current >= 0) hop[current] = 0;
    __syncthreads();
    for (int d = 0; d + 1 < e_max; ++d) {
        int any = 0;
        for (long long j = tid; j < size; j += T) {
            const long long q = (head + j) % W;
            const int a = win_a[q], b = win_b[q];
            if (hop[a] != d) continue;
            if (__ddiv_rn((double)counts[(long long)a * acap + b], (double)totals[a]) < tau) continue;
            if (hop[b] > d + 1) {
                hop[b] = (unsigned char)(d + 1);
                any = 1;
            }
        }
        if (!__syncthreads_or(any)) break;
    }
    for (int x = tid; x < n; x += T) hops[x] = hop[x];
}

// K6 argmax_row: max count, ties -> the smaller 64-bit AgentId. out: best index or -1.
__global__ void learner_argmax_kernel(const unsigned int* counts, const unsigned long long* ids, int acap, int n,
                                      int a, int* out) {
    __shared__ unsigned long long bc[32], bi[32];
    __shared__ int bb[32];
    unsigned long long best_c = 0, best_id = ~0ull;
    int best = -1;
    for (int b = threadIdx.x; b < n; b += blockDim.x) {
        const unsigned int c = counts[(long long)a * acap + b];
        if (c == 0u) continue;
        if (best < 0 || c > best_c || (c == best_c && ids[b] < best_id)) {
            best_c = c;
            best_id = ids[b];
            best = b;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long oc = __shfl_xor_sync(0xffffffffu, best_c, o);
        const unsigned long long oi = __shfl_xor_sync(0xffffffffu, best_id, o);
        const int ob = __shfl_xor_sync(0xffffffffu, best, o);
        if (ob >= 0 && (best < 0 || oc > best_c || (oc == best_c && oi < best_id))) {
            best_c = oc;
            best_id = oi;
            best = ob;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        bc[threadIdx.x >> 5] = best_c;
        bi[threadIdx.x >> 5] = best_id;
        bb[threadIdx.x >> 5] = best;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        best = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            if (bb[w] < 0) continue;
            if (best < 0 || bc[w] > best_c || (bc[w] == best_c && bi[w] < best_id)) {
                best_c = bc[w];
                best_id = bi[w];
                best = bb[w];
            }
        }
        *out = best;
    }
}

// a21 exact_survival_prob: the probability that a walk from `current` on the MLE matrix visits
// `target` within k steps (step 0 excluded; mass on a row with no observations dies). Thread b
// owns next[b] and adds the rows in alphabet order, so every fp64 operation happens in the
// reference's order: next[b] += dist[i] * count / total, i ascending.
__global__ void learner_survival_kernel(const unsigned int* counts, const unsigned int* totals, int acap, int n,
                                        int current, int target, int k, double* out) {
    __shared__ double dist[64], nxt[64];
    __shared__ double absorbed;
    const int t = threadIdx.x;
    if (t < n) dist[t] = t == current ? 1.0 : 0.0;
    if (t == 0) absorbed = 0.0;
    __syncthreads();
    for (int step = 0; step < k; ++step) {
        if (t < n) {
            double acc = 0.0;
            for (int i = 0; i < n; ++i) {
                const double di = dist[i];
                const unsigned int tot = totals[i];
                if (di == 0.0 || tot == 0u) continue;
                const unsigned int c = counts[(long long)i * acap + t];
                if (c == 0u) continue;
                acc = __dadd_rn(acc, __ddiv_rn(__dmul_rn(di, (double)c), (double)tot));
            }
            nxt[t] = acc;
        }
        __syncthreads();
        if (t == 0) {
            absorbed = __dadd_rn(absorbed, nxt[target]);
            nxt[target] = 0.0;
        }
        __syncthreads();
        if (t < n) dist[t] = nxt[t];
        __syncthreads();
    }
    if (t == 0) *out = absorbed;
}

}  // namespace csb

struct cs_learner {
    int device = 0;
    int acap = 0;
    long long W = 0, head = 0, size = 0;
    unsigned long long recorded = 0;
    unsigned int* counts = nullptr;
    unsigned int* totals = nullptr;
    int* win_a = nullptr;
    int* win_b = nullptr;
    unsigned long long* ids_dev = nullptr;
    std::vector<uint64_t> ids;  // alphabet, first-seen order (TransitionLearner::agents)
    std::unordered_map<uint64_t, int> index;
    cudaStream_t stream = nullptr;
    csb::DevBuf scratch, scratch2;

    int note(uint64_t id) {  // TransitionLearner::note_agent (transition_learner.cpp:16-20)
        auto it = index.find(id);
        if (it != index.end()) return it->second;
        if ((int)ids.size() >= acap) throw CsError(CS_ERR_CAPACITY, "TransitionLearner: agent capacity exceeded");
        const int k = (int)ids.size();
        index.emplace(id, k);
        ids.push_back(id);
        ck(cudaMemcpyAsync(ids_dev + k, &ids.back(), 8, cudaMemcpyHostToDevice, stream), "H2D");
        return k;
    }
    int find(uint64_t id) const {
        auto it = index.find(id);
        return it == index.end() ? -1 : it->second;
    }
    void sync() { ck(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }
};

namespace {
template <class F>
int lguard(F&& f) {
    try {
        f();
        return CS_OK;
    } catch (const CsError& e) {
        cs_set_error(e.what());
        return e.code;
    } catch (const std::invalid_argument& e) {
        cs_set_error(e.what());
        return CS_ERR_INVALID_ARGUMENT;
    } catch (const std::logic_error& e) {
        cs_set_error(e.what());
        return CS_ERR_LOGIC;
    } catch (const std::exception& e) {
        cs_set_error(e.what());
        return CS_ERR_RUNTIME;
    }
}
}  // namespace

extern "C" {

int cs_learner_create(int64_t window, int agent_capacity, int device, cs_learner_t* out) {
    return lguard([&] {
        if (!out) throw std::invalid_argument("cs_learner_create: null argument");
        if (window <= 0) throw std::invalid_argument("TransitionLearner: window capacity must be positive");
        if (agent_capacity < 1 || agent_capacity > csb::kMaxAgents)
            throw CsError(CS_ERR_CAPACITY, "agent_capacity must be in [1, 4096]");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw CsError(CS_ERR_CUDA, "no CUDA device: cachesage_b200 has no CPU fallback");
        auto* L = new cs_learner();
        try {
            L->device = device;
            L->acap = agent_capacity;
            L->W = window;
            ck(cudaSetDevice(device), "cudaSetDevice");
            ck(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            const size_t A = (size_t)agent_capacity;
            ck(cudaMalloc(&L->counts, 4 * A * A), "cudaMalloc");
            ck(cudaMalloc(&L->totals, 4 * A), "cudaMalloc");
            ck(cudaMalloc(&L->win_a, 4 * (size_t)window), "cudaMalloc");
            ck(cudaMalloc(&L->win_b, 4 * (size_t)window), "cudaMalloc");
            ck(cudaMalloc(&L->ids_dev, 8 * A), "cudaMalloc");
            ck(cudaMemsetAsync(L->counts, 0, 4 * A * A, L->stream), "memset");
            ck(cudaMemsetAsync(L->totals, 0, 4 * A, L->stream), "memset");
            L->sync();
        } catch (...) {
            cs_learner_destroy(L);
            throw;
        }
        *out = L;
    });
}

int cs_learner_destroy(cs_learner_t L) {
    return lguard([&] {
        if (!L) return;
        for (void* p : {(void*)L->counts, (void*)L->totals, (void*)L->win_a, (void*)L->win_b, (void*)L->ids_dev})
            if (p) cudaFree(p);
        L->scratch.release();
        L->scratch2.release();
        if (L->stream) cudaStreamDestroy(L->stream);
        delete L;
    });
}

int cs_learner_record(cs_learner_t L, const uint64_t* prev, const uint64_t* next, int64_t n) {
    return lguard([&] {
        if (!L || n < 0 || (n > 0 && (!prev || !next))) throw std::invalid_argument("cs_learner_record: null argument");
        if (n == 0) return;
        std::vector<int> a(n), b(n);
        for (int64_t i = 0; i < n; ++i) {  // note_agent(prev), note_agent(next), in record order
            a[i] = L->note(prev[i]);
            b[i] = L->note(next[i]);
        }
        L->scratch.ensure(4 * (size_t)n);
        L->scratch2.ensure(4 * (size_t)n);
        ck(cudaMemcpyAsync(L->scratch.p, a.data(), 4 * n, cudaMemcpyHostToDevice, L->stream), "H2D");
        ck(cudaMemcpyAsync(L->scratch2.p, b.data(), 4 * n, cudaMemcpyHostToDevice, L->stream), "H2D");
        const long long pops = std::max(0ll, L->size + n - L->W);
        const long long tot = L->size + n;
        csb::learner_record_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, L->stream>>>(
            L->counts, L->totals, L->win_a, L->win_b, L->acap, L->W, L->head, L->size, pops,
            L->scratch.as<int>(), L->scratch2.as<int>(), n);
        ck(cudaGetLastError(), "learner_record_kernel");
        csb::learner_window_kernel<<<(unsigned)((n + 255) / 256), 256, 0, L->stream>>>(
            L->win_a, L->win_b, L->W, L->head, L->size, pops, L->scratch.as<int>(), L->scratch2.as<int>(), n);
        ck(cudaGetLastError(), "learner_window_kernel");
        L->head = (L->head + pops) % L->W;
        L->size = tot - pops;
        L->recorded += (unsigned long long)n;
        L->sync();
    });
}

int cs_learner_prob(cs_learner_t L, uint64_t a, uint64_t b, double* p) {
    return lguard([&] {
        if (!L || !p) throw std::invalid_argument("cs_learner_prob: null argument");
        const int ia = L->find(a), ib = L->find(b);
        *p = 0.0;
        if (ia < 0 || ib < 0) return;
        unsigned int c = 0, t = 0;
        ck(cudaMemcpy(&c, L->counts + (size_t)ia * L->acap + ib, 4, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(&t, L->totals + ia, 4, cudaMemcpyDeviceToHost), "D2H");
        if (t == 0u || c == 0u) return;  // prob = 0 by convention on an empty row (transition_learner.cpp:53-67)
        *p = (double)c / (double)t;
    });
}

int cs_learner_row_total(cs_learner_t L, uint64_t a, uint64_t* total) {
    return lguard([&] {
        if (!L || !total) throw std::invalid_argument("cs_learner_row_total: null argument");
        const int ia = L->find(a);
        unsigned int t = 0;
        if (ia >= 0) ck(cudaMemcpy(&t, L->totals + ia, 4, cudaMemcpyDeviceToHost), "D2H");
        *total = t;
    });
}

int cs_learner_agents(cs_learner_t L, uint64_t* ids, int cap) {
    if (!L) {
        cs_set_error("cs_learner_agents: null learner");
        return CS_ERR_INVALID_ARGUMENT;
    }
    const int n = (int)L->ids.size();
    for (int i = 0; i < n && i < cap && ids; ++i) ids[i] = L->ids[i];
    return n;
}

int cs_learner_state_bytes(cs_learner_t L, uint64_t* bytes) {
    return lguard([&] {
        if (!L || !bytes) throw std::invalid_argument("cs_learner_state_bytes: null argument");
        // TransitionLearner::state_bytes (transition_learner.cpp:98-106)
        const int n = (int)L->ids.size();
        csb::DevBuf acc;
        acc.ensure(16);
        ck(cudaMemsetAsync(acc.p, 0, 16, L->stream), "memset");
        if (n > 0)
            csb::learner_nonzero_kernel<<<64, 256, 0, L->stream>>>(L->counts, L->totals, L->acap, n,
                                                                   acc.as<unsigned long long>());
        unsigned long long h[2] = {0, 0};
        ck(cudaMemcpyAsync(h, acc.p, 16, cudaMemcpyDeviceToHost, L->stream), "D2H");
        L->sync();
        *bytes = (uint64_t)(L->size * 4 + (long long)h[0] * 12 + (long long)h[1] * 10 + n * 8 + 8);
    });
}

int cs_learner_rebuild(cs_learner_t L, uint64_t current, double tau, int e_max, int* hops, int cap) {
    return lguard([&] {
        if (!L || (cap > 0 && !hops)) throw std::invalid_argument("cs_learner_rebuild: null argument");
        if (e_max <= 0) throw std::invalid_argument("rebuild_reachability: e_max must be positive");
        const int n = (int)L->ids.size();
        if (n == 0) return;
        csb::DevBuf out;
        out.ensure(4 * (size_t)n);
        csb::learner_bfs_kernel<<<1, 512, (size_t)n, L->stream>>>(L->counts, L->totals, L->win_a, L->win_b, L->acap,
                                                                  L->W, L->head, L->size, n, L->find(current), tau,
                                                                  e_max, out.as<int>());
        ck(cudaGetLastError(), "learner_bfs_kernel");
        std::vector<int> h(n);
        ck(cudaMemcpyAsync(h.data(), out.p, 4 * (size_t)n, cudaMemcpyDeviceToHost, L->stream), "D2H");
        L->sync();
        for (int i = 0; i < n && i < cap; ++i) hops[i] = h[i];
    });
}

int cs_learner_argmax(cs_learner_t L, uint64_t a, uint64_t* best, double* p, int* found) {
    return lguard([&] {
        if (!L || !best || !p || !found) throw std::invalid_argument("cs_learner_argmax: null argument");
        *found = 0;
        const int ia = L->find(a);
        if (ia < 0) return;
        csb::DevBuf out;
        out.ensure(4);
        csb::learner_argmax_kernel<<<1, 256, 0, L->stream>>>(L->counts, L->ids_dev, L->acap, (int)L->ids.size(), ia,
                                                            out.as<int>());
        int b = -1;
        unsigned int c = 0, t = 0;
        ck(cudaMemcpyAsync(&b, out.p, 4, cudaMemcpyDeviceToHost, L->stream), "D2H");
        ck(cudaMemcpyAsync(&t, L->totals + ia, 4, cudaMemcpyDeviceToHost, L->stream), "D2H");
        L->sync();
        if (b < 0 || t == 0u) return;
        ck(cudaMemcpy(&c, L->counts + (size_t)ia * L->acap + b, 4, cudaMemcpyDeviceToHost), "D2H");
        *best = L->ids[b];
        *p = (double)c / (double)t;
        *found = 1;
    });
}

int cs_exact_survival_prob(cs_learner_t L, uint64_t target, int k, uint64_t current, double* out) {
    return lguard([&] {
        if (!L || !out) throw std::invalid_argument("cs_exact_survival_prob: null argument");
        const int n = (int)L->ids.size();
        // survival_oracle.cpp:12-33, in order
        if (n > 64) throw std::invalid_argument("exact_survival_prob: alphabet too large (test-scale <= 64)");
        if (k > 32) throw std::invalid_argument("exact_survival_prob: horizon too deep (test-scale <= 32)");
        if (k < 0) throw std::invalid_argument("exact_survival_prob: negative horizon");
        if (target == current) {
            *out = 1.0;
            return;
        }
        const int it = L->find(target), ic = L->find(current);
        if (it < 0 || ic < 0) {
            *out = 0.0;
            return;
        }
        csb::DevBuf o;
        o.ensure(8);
        csb::learner_survival_kernel<<<1, 64, 0, L->stream>>>(L->counts, L->totals, L->acap, n, ic, it, k,
                                                             o.as<double>());
        ck(cudaGetLastError(), "learner_survival_kernel");
        ck(cudaMemcpyAsync(out, o.p, 8, cudaMemcpyDeviceToHost, L->stream), "D2H");
        L->sync();
    });
}

}  // extern "C"
