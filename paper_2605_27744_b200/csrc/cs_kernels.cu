// sm_100a kernels of the CacheSage per-step hot path.
//
//   K1  hash_prompts / hash_turns   chain_hash + block_keys_for + derive_agent_identity
//   K2  table_find / table_insert   block table probe, lookup touches, lock-free insert, erase
//   K3  observe_dispatch            transition-learner window update
//   K3b (same)                      level-synchronous BFS -> survival class per agent
//   K6  (same)                      prefetch gate: argmax of the current row, ties on AgentId
//   K4  scan_pass                   one HBM pass over the SoA pool: per survival class the
//                                   `keep` oldest unpinned slots + the keep+1 oldest resident
//   K5a finalize_list               per-list exact select over the CTAs' candidates, sorted
//   K5b replay_apply                exact sequential replay of admit_pinned/evict_one on the
//                                   class heads, then table/SoA updates
//
// K3..K5b run inside ONE cooperative launch per admission (admit_kernel); grid barriers
// separate the phases. Reference semantics: engine.cpp:102-195, cachesage_policy.cpp:50-130,
// transition_learner.cpp:22-96, reachability.cpp:39-81, runtime.cpp:23-32 (paths relative to
// /root/reference/proj). Why the per-class select is exact: DESIGN.md §4.
#include <cuda_runtime.h>

#include <algorithm>

#include "cs_launch.h"

namespace csb {

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

// ------------------------------------------------------------------ block helpers

struct RedSmem {
    long long v[32];
};

__device__ long long block_sum(long long x, RedSmem& R) {
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if (lane_id() == 0) R.v[warp_id()] = x;
    __syncthreads();
    if (warp_id() == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        long long y = lane_id() < nw ? R.v[lane_id()] : 0;
        for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
        if (lane_id() == 0) R.v[0] = y;
    }
    __syncthreads();
    const long long r = R.v[0];
    __syncthreads();
    return r;
}

__device__ long long block_min(long long x, RedSmem& R) {
    for (int o = 16; o; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
    __syncthreads();
    if (lane_id() == 0) R.v[warp_id()] = x;
    __syncthreads();
    if (warp_id() == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        long long y = lane_id() < nw ? R.v[lane_id()] : 0x7fffffffffffffffll;
        for (int o = 16; o; o >>= 1) y = min(y, __shfl_xor_sync(0xffffffffu, y, o));
        if (lane_id() == 0) R.v[0] = y;
    }
    __syncthreads();
    const long long r = R.v[0];
    __syncthreads();
    return r;
}

struct SelectSmem {
    unsigned int hist[256];
    unsigned long long or_diff;
    unsigned long long prefix;
    int k;
    int tmp;
};

// k-th smallest (1-based) of m values at v (shared or global), MSB-first 8-bit radix select.
// Values are distinct ticks, so the result is a value present in v with exactly k values <= it.
// Digits above the highest differing bit are skipped. All threads of the block must call.
__device__ unsigned long long block_kth(const unsigned long long* v, int m, int k, SelectSmem& S) {
    const unsigned long long x0 = v[0];
    if (threadIdx.x == 0) S.or_diff = 0ull;
    __syncthreads();
    unsigned long long d = 0;
    for (int j = threadIdx.x; j < m; j += blockDim.x) d |= v[j] ^ x0;
    for (int o = 16; o; o >>= 1) d |= __shfl_xor_sync(0xffffffffu, d, o);
    if (lane_id() == 0 && d) atomicOr(&S.or_diff, d);
    __syncthreads();
    d = S.or_diff;
    if (d == 0ull) {
        __syncthreads();
        return x0;
    }
    const int hb = 63 - __clzll((long long)d);
    int shift = (hb / 8) * 8;
    unsigned long long hmask = (shift + 8 >= 64) ? 0ull : ~((1ull << (shift + 8)) - 1ull);
    unsigned long long prefix = x0 & hmask;
    int kk = k;
    for (;;) {
        for (int b = threadIdx.x; b < 256; b += blockDim.x) S.hist[b] = 0u;
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
            const unsigned long long x = v[j];
            if ((x & hmask) == prefix) atomicAdd(&S.hist[(x >> shift) & 255ull], 1u);
        }
        __syncthreads();
        if (warp_id() == 0) {
            unsigned int c[8];
            unsigned int s = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = S.hist[lane_id() * 8 + q];
                s += c[q];
            }
            unsigned int inc = s;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane_id() >= o) inc += t;
            }
            const unsigned int exc = inc - s;
            if (exc < (unsigned)kk && (unsigned)kk <= inc) {
                unsigned int cum = exc;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (cum + c[q] >= (unsigned)kk) {
                        S.prefix = prefix | ((unsigned long long)(lane_id() * 8 + q) << shift);
                        S.k = kk - (int)cum;
                        break;
                    }
                    cum += c[q];
                }
            }
        }
        __syncthreads();
        prefix = S.prefix;
        kk = S.k;
        hmask |= (255ull << shift);
        if (shift == 0) break;
        shift -= 8;
    }
    __syncthreads();
    return prefix;
}

// In-place: keep the (lt, slot) pairs with lt <= v. m <= 4 * blockDim.x. Returns the count.
__device__ int block_compact_le(unsigned long long* blt, unsigned int* bslot, int m, unsigned long long v,
                                SelectSmem& S) {
    unsigned long long l[4];
    unsigned int s[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int j = threadIdx.x + r * blockDim.x;
        if (j < m) {
            l[r] = blt[j];
            s[r] = bslot[j];
        }
    }
    if (threadIdx.x == 0) S.tmp = 0;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int j = threadIdx.x + r * blockDim.x;
        if (j < m && l[r] <= v) {
            const int p = atomicAdd(&S.tmp, 1);
            blt[p] = l[r];
            bslot[p] = s[r];
        }
    }
    __syncthreads();
    const int n = S.tmp;
    __syncthreads();
    return n;
}

// ------------------------------------------------------------------ shared state

struct ScanSmem {
    int cnt[kMaxLists];
    unsigned long long thr[kMaxLists];
    unsigned long long gbw[kMaxLists];
    int wcnt[kMaxLists];
    int wbase[kMaxLists];
    int wpos[kMaxLists];
};

// Per-admission state of CTA 0 (persists across phases of one launch).
struct AdmSmem {
    unsigned long long tick;        // engine clock
    unsigned long long first_touch; // earliest tick touched by admit_pinned in this admission
    long long cached;
    long long n_ev_adm;
    long long resident, pinned, free_top;
    int first_miss, admit_n, anchor, chunk, started, error, needed, warm_issued, scans;
};

// Replay-phase view of the (re-used) dynamic scan region.
struct ReplaySmem {
    unsigned long long L_lt[kMaxLists][kChunk + 2];
    unsigned int L_slot[kMaxLists][kChunk + 2];
    int L_n[kMaxLists];
    unsigned int rs_key[1024];
    unsigned char rs_flag[1024];
    unsigned int c_slot[kChunk];
    unsigned int c_refs0[kChunk];
    unsigned int out_slot[kChunk];
    unsigned long long out_lt[kChunk];
    unsigned char out_new[kChunk];
    unsigned int victims[kChunk];
    unsigned int lfree[kChunk];
    int n_vict, n_lfree, n_reused;
};

constexpr unsigned char kRsTouched = 1, kRsEvicted = 2;

__device__ __forceinline__ unsigned int rs_hash(unsigned int s) { return (s * 2654435761u) >> 22; }  // 10 bits

__device__ __forceinline__ unsigned char rs_get(const ReplaySmem& R, unsigned int s) {
    unsigned int h = rs_hash(s);
    for (int n = 0; n < 1024; ++n) {
        const unsigned int k = R.rs_key[h];
        if (k == kNoSlot) return 0;
        if (k == s) return R.rs_flag[h];
        h = (h + 1) & 1023u;
    }
    __trap();
    return 0;
}

__device__ __forceinline__ void rs_put(ReplaySmem& R, unsigned int s, unsigned char f) {
    unsigned int h = rs_hash(s);
    for (int n = 0; n < 1024; ++n) {
        const unsigned int k = R.rs_key[h];
        if (k == kNoSlot || k == s) {
            R.rs_key[h] = s;
            R.rs_flag[h] = f;
            return;
        }
        h = (h + 1) & 1023u;
    }
    __trap();
}

// ------------------------------------------------------------------ K3 / K3b / K6

// CacheSagePolicy::observe(AgentDispatch) (cachesage_policy.cpp:57-72). CTA 0, all threads.
__device__ void observe_dispatch(const DevPool& P, int prev, int next, unsigned long long tick, int n_agents,
                                 unsigned char* hop_s, RedSmem& R, AdmSmem& A) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const long long W = P.window;
    const int Acap = P.a_cap;
    if (P.policy == 0) return;  // LruPolicy::observe is a no-op (baselines.cpp:10)
    // K3: TransitionLearner::record (transition_learner.cpp:22-51), one pair per dispatch
    if (prev >= 0 && tid == 0) {
        const long long head = C->win_head, size = C->win_size;
        P.counts[(long long)prev * Acap + next] += 1u;
        P.totals[prev] += 1u;
        if (size == W) {
            const int oa = P.win_a[head], ob = P.win_b[head];
            P.win_a[head] = prev;
            P.win_b[head] = next;
            P.counts[(long long)oa * Acap + ob] -= 1u;
            P.totals[oa] -= 1u;
            C->win_head = (head + 1) % W;
        } else {
            const long long pos = (head + size) % W;
            P.win_a[pos] = prev;
            P.win_b[pos] = next;
            C->win_size = size + 1;
        }
    }
    __syncthreads();
    const bool changed = C->cur_agent != next;
    __syncthreads();
    if (tid == 0) C->cur_agent = next;
    if (changed) {
        // K3b: rebuild_reachability (reachability.cpp:39-81) as a level-synchronous BFS over
        // the window's pairs (every positive count cell is in the window). Depth d expands only
        // while d + 1 < e_max; edge iff !(count/total < tau) in fp64.
        const int e = P.e_max;
        for (int x = tid; x < n_agents; x += T) hop_s[x] = (unsigned char)e;
        __syncthreads();
        if (tid == 0) hop_s[next] = 0;
        __syncthreads();
        const long long head = C->win_head, size = C->win_size;
        for (int d = 0; d + 1 < e; ++d) {
            int any = 0;
            for (long long j = tid; j < size; j += T) {
                const long long q = (head + j) % W;
                const int a = P.win_a[q], b = P.win_b[q];
                if (hop_s[a] != d) continue;
                const double c = (double)P.counts[(long long)a * Acap + b];
                const double t = (double)P.totals[a];
                if (__ddiv_rn(c, t) < P.tau) continue;
                if (hop_s[b] > d + 1) {
                    hop_s[b] = (unsigned char)(d + 1);
                    any = 1;
                }
            }
            if (!__syncthreads_or(any)) break;
        }
        for (int x = tid; x < n_agents; x += T) {
            P.hop[x] = hop_s[x];
            P.cls[x] = hop_s[x];
        }
        if (tid == 0) {
            C->rebuilds += 1ull;
            C->reach_built = 1;
        }
        __syncthreads();
    }
    // K6: maybe_prefetch (cachesage_policy.cpp:109-123) with argmax_row
    // (transition_learner.cpp:79-96): max count, ties -> smaller 64-bit AgentId.
    const int budget_ok = C->step_warmups < P.budget_per_step;
    const unsigned int total = P.totals[next];
    if (budget_ok && (unsigned long long)total >= P.min_row && total > 0u) {
        unsigned long long best_c = 0ull, best_id = ~0ull;
        int best_b = -1;
        for (int b = tid; b < n_agents; b += T) {
            const unsigned int c = P.counts[(long long)next * Acap + b];
            if (c == 0u) continue;
            const unsigned long long id = P.agent_ids[b];
            if (best_b < 0 || c > best_c || (c == best_c && id < best_id)) {
                best_c = c;
                best_id = id;
                best_b = b;
            }
        }
        // block arg-reduction on (count desc, id asc)
        for (int o = 16; o; o >>= 1) {
            const unsigned long long oc = __shfl_xor_sync(0xffffffffu, best_c, o);
            const unsigned long long oi = __shfl_xor_sync(0xffffffffu, best_id, o);
            const int ob = __shfl_xor_sync(0xffffffffu, best_b, o);
            if (ob >= 0 && (best_b < 0 || oc > best_c || (oc == best_c && oi < best_id))) {
                best_c = oc;
                best_id = oi;
                best_b = ob;
            }
        }
        __shared__ unsigned long long s_c[32], s_i[32];
        __shared__ int s_b[32];
        if (lane_id() == 0) {
            s_c[warp_id()] = best_c;
            s_i[warp_id()] = best_id;
            s_b[warp_id()] = best_b;
        }
        __syncthreads();
        if (tid == 0) {
            const int nw = (T + 31) >> 5;
            for (int w = 1; w < nw; ++w) {
                if (s_b[w] >= 0 && (best_b < 0 || s_c[w] > best_c || (s_c[w] == best_c && s_i[w] < best_id))) {
                    best_c = s_c[w];
                    best_id = s_i[w];
                    best_b = s_b[w];
                }
            }
            if (best_b >= 0) {
                const double p = __ddiv_rn((double)best_c, (double)total);
                if (!(p < P.min_conf)) {
                    C->step_warmups += 1;
                    if (C->n_pend < kMaxPending) {
                        C->pend_target[C->n_pend] = best_b;
                        C->pend_tick[C->n_pend] = tick;
                        C->n_pend += 1;
                    }
                    A.warm_issued = best_b;
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ K4: the pool scan

__device__ void trim_lists(const DevPool& P, int NL, int keep, unsigned long long* blt, unsigned int* bslot,
                           int CAP, ScanSmem& S, SelectSmem& Sel) {
    for (int l = 0; l < NL; ++l) {
        const int kl = (l == NL - 1) ? keep + 1 : keep;
        const int m = S.cnt[l];
        if (m > kl) {
            const unsigned long long v = block_kth(blt + (long long)l * CAP, m, kl, Sel);
            const int n = block_compact_le(blt + (long long)l * CAP, bslot + (long long)l * CAP, m, v, Sel);
            if (threadIdx.x == 0) {
                S.cnt[l] = n;
                if (v < S.thr[l]) S.thr[l] = v;
                atomicMin(P.gbound + l, v);
            }
            __syncthreads();
        }
    }
}

// One streaming pass over this CTA's contiguous slot range. Reads lt/agent/refs (16 B per
// slot) exactly once with 4 tiles of loads in flight per thread; everything else is on-chip.
__device__ void scan_pass(const DevPool& P, int NL, int keep, const unsigned char* cls_s, unsigned long long* blt,
                          unsigned int* bslot, int CAP, ScanSmem& S, SelectSmem& Sel) {
    const int T = blockDim.x, tid = threadIdx.x;
    long long per = (P.cap + gridDim.x - 1) / gridDim.x;
    per = (per + 31) / 32 * 32;
    const long long lo = (long long)blockIdx.x * per;
    const long long hi = min(P.cap, lo + per);
    const int R = NL - 1;
    const int e_max = P.e_max;
    if (tid < NL) {
        S.cnt[tid] = 0;
        S.thr[tid] = ld_relaxed_u64(P.gbound + tid);
    }
    __syncthreads();
    volatile unsigned long long* thr = S.thr;
    constexpr int D = 4;
    unsigned long long rl[D];
    unsigned int ra[D], rr[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const long long i = lo + (long long)d * T + tid;
        if (i < hi) {
            rl[d] = __ldcs(P.lt + i);
            ra[d] = __ldcs(P.agent + i);
            rr[d] = __ldcs(P.refs + i);
        }
    }
    unsigned long long gbn = ~0ull;
    for (long long base = lo; base < hi; base += (long long)D * T) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const long long tb = base + (long long)d * T;
            if (tb >= hi) break;
            if (tid < NL) gbn = ld_relaxed_u64(P.gbound + tid);
            const long long i = tb + tid;
            int over = 0;
            if (i < hi) {
                const unsigned long long x = rl[d];
                if (x != kFreeTick) {
                    if (x <= thr[R]) {
                        const int p = atomicAdd(&S.cnt[R], 1);
                        blt[(long long)R * CAP + p] = x;
                        bslot[(long long)R * CAP + p] = (unsigned int)i;
                        over |= p >= keep + 1 + kSlack;
                    }
                    if (rr[d] == 0u) {
                        const unsigned int a = ra[d];
                        const int c = (a == kNoAgent) ? e_max : (int)cls_s[a];
                        if (x <= thr[c]) {
                            const int p = atomicAdd(&S.cnt[c], 1);
                            blt[(long long)c * CAP + p] = x;
                            bslot[(long long)c * CAP + p] = (unsigned int)i;
                            over |= p >= keep + kSlack;
                        }
                    }
                }
            }
            const long long j = tb + (long long)D * T + tid;
            if (j < hi) {
                rl[d] = __ldcs(P.lt + j);
                ra[d] = __ldcs(P.agent + j);
                rr[d] = __ldcs(P.refs + j);
            }
            if (tid < NL && gbn < thr[tid]) thr[tid] = gbn;
            if (__syncthreads_or(over)) {
                trim_lists(P, NL, keep, blt, bslot, CAP, S, Sel);
            }
        }
    }
    __syncthreads();
    trim_lists(P, NL, keep, blt, bslot, CAP, S, Sel);
    // publish this CTA's survivors that can still be in the global keep-set
    if (tid < NL) {
        S.gbw[tid] = ld_relaxed_u64(P.gbound + tid);
        S.wcnt[tid] = 0;
        S.wpos[tid] = 0;
    }
    __syncthreads();
    for (int l = 0; l < NL; ++l) {
        const int m = S.cnt[l];
        for (int q = tid; q < m; q += T)
            if (blt[(long long)l * CAP + q] <= S.gbw[l]) atomicAdd(&S.wcnt[l], 1);
    }
    __syncthreads();
    if (tid < NL) S.wbase[tid] = S.wcnt[tid] ? atomicAdd(P.gcount + tid, S.wcnt[tid]) : 0;
    __syncthreads();
    for (int l = 0; l < NL; ++l) {
        const int m = S.cnt[l];
        for (int q = tid; q < m; q += T) {
            const unsigned long long x = blt[(long long)l * CAP + q];
            if (x <= S.gbw[l]) {
                const long long o = (long long)l * P.gcap + S.wbase[l] + atomicAdd(&S.wpos[l], 1);
                P.gbuf_lt[o] = x;
                P.gbuf_slot[o] = bslot[(long long)l * CAP + q];
            }
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------------ K5a: exact per-list select

__device__ void finalize_list(const DevPool& P, int l, int NL, int keep, unsigned long long* t_lt,
                              unsigned int* t_slot, SelectSmem& Sel) {
    const int T = blockDim.x, tid = threadIdx.x;
    const int kl = (l == NL - 1) ? keep + 1 : keep;
    const int m = *(volatile int*)(P.gcount + l);
    const unsigned long long* g = P.gbuf_lt + (long long)l * P.gcap;
    const unsigned int* gs = P.gbuf_slot + (long long)l * P.gcap;
    unsigned long long v = ~0ull;
    if (m > kl) v = block_kth(g, m, kl, Sel);
    if (tid == 0) Sel.tmp = 0;
    __syncthreads();
    for (int j = tid; j < m; j += T) {
        const unsigned long long x = g[j];
        if (x <= v) {
            const int p = atomicAdd(&Sel.tmp, 1);
            t_lt[p] = x;
            t_slot[p] = gs[j];
        }
    }
    __syncthreads();
    const int n = Sel.tmp;
    for (int j = tid; j < 256; j += T)
        if (j >= n) {
            t_lt[j] = ~0ull;
            t_slot[j] = kNoSlot;
        }
    __syncthreads();
    for (int k = 2; k <= 256; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = tid; i < 256; i += T) {
                const int ixj = i ^ jj;
                if (ixj > i) {
                    const bool asc = (i & k) == 0;
                    const unsigned long long a = t_lt[i], b = t_lt[ixj];
                    if ((a > b) == asc) {
                        t_lt[i] = b;
                        t_lt[ixj] = a;
                        const unsigned int sa = t_slot[i];
                        t_slot[i] = t_slot[ixj];
                        t_slot[ixj] = sa;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int j = tid; j < n; j += T) {
        P.fin_lt[(long long)l * (kChunk + 2) + j] = t_lt[j];
        P.fin_slot[(long long)l * (kChunk + 2) + j] = t_slot[j];
    }
    if (tid == 0) P.fin_n[l] = n;
    __syncthreads();
}

// ------------------------------------------------------------------ K5b: replay + apply

// Exact replay of admit_pinned over prompt blocks [lo, hi) (engine.cpp:141-168). Each
// eviction is evict_one (engine.cpp:102-125): the argmin of (score, last_touch) over the
// class heads, where a class head is the oldest not-yet-removed candidate of that class, and
// oldest_live_touch comes from the resident-oldest list (engine.cpp:90-100).
__device__ void replay_apply(const DevPool& P, const AdmitArgs& a, ReplaySmem& R, AdmSmem& A, int NL, bool scanned) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int lo = A.chunk * kChunk;
    const int hi = min(A.admit_n, lo + kChunk);
    const int len = hi - lo;
    for (int j = tid; j < 1024; j += T) R.rs_key[j] = kNoSlot;
    for (int l = 0; l < NL; ++l) {
        const int n = scanned ? P.fin_n[l] : 0;
        for (int j = tid; j < n; j += T) {
            R.L_lt[l][j] = P.fin_lt[(long long)l * (kChunk + 2) + j];
            R.L_slot[l][j] = P.fin_slot[(long long)l * (kChunk + 2) + j];
        }
        if (tid == 0) R.L_n[l] = n;
    }
    for (int i = tid; i < len; i += T) {
        R.c_slot[i] = P.p_slot[lo + i];
        R.c_refs0[i] = P.p_refs0[lo + i];
    }
    if (tid == 0) {
        R.n_vict = 0;
        R.n_lfree = 0;
        R.n_reused = 0;
    }
    __syncthreads();

    if (warp_id() == 0) {
        const int lane = lane_id();
        const int Rl = NL - 1;
        int cursor = 0;
        const int my_n = lane < NL ? R.L_n[lane] : 0;
        const double my_surv = survival_of_class(lane, P.e_max);
        unsigned long long tick = A.tick;
        unsigned long long first_touch = A.first_touch;
        long long resident = C->resident;
        long long pinned = C->pinned;
        long long free_top = C->free_top;
        int error = 0;
        for (int i = 0; i < len && !error; ++i) {
            unsigned int s = R.c_slot[i];
            if (s != kNoSlot && rs_get(R, s) == kRsEvicted) s = kNoSlot;
            if (s != kNoSlot) {
                ++tick;
                if (lane == 0) {
                    R.out_slot[i] = s;
                    R.out_lt[i] = tick;
                    R.out_new[i] = 0;
                    rs_put(R, s, kRsTouched);
                }
                if (R.c_refs0[i] == 0u) ++pinned;
                if (first_touch == ~0ull) first_touch = tick;
                __syncwarp();
                continue;
            }
            while (resident >= P.cap) {
                // advance each list past removed entries (touched / evicted / pinned this admission)
                if (lane < NL) {
                    while (cursor < my_n && rs_get(R, R.L_slot[lane][cursor]) != 0) ++cursor;
                }
                const unsigned long long rhead =
                    __shfl_sync(0xffffffffu, (lane == Rl && cursor < my_n) ? R.L_lt[Rl][cursor] : ~0ull, Rl);
                unsigned long long old = tick;
                if (rhead < old) old = rhead;
                if (first_touch < old) old = first_touch;
                double sc = __longlong_as_double(0x7ff0000000000000ll);  // +inf: no head
                unsigned long long hl = ~0ull;
                int has = 0;
                if (lane < Rl && cursor < my_n) {
                    hl = R.L_lt[lane][cursor];
                    sc = score_of(P.policy, P.w_pred, my_surv, hl, tick, old);
                    has = 1;
                }
                int best = has ? lane : -1;
                for (int o = 16; o; o >>= 1) {
                    const double os = __shfl_xor_sync(0xffffffffu, sc, o);
                    const unsigned long long ol = __shfl_xor_sync(0xffffffffu, hl, o);
                    const int ob = __shfl_xor_sync(0xffffffffu, best, o);
                    if (ob >= 0 && (best < 0 || os < sc || (os == sc && ol < hl))) {
                        sc = os;
                        hl = ol;
                        best = ob;
                    }
                }
                if (best < 0) {
                    error = 1;  // evict_one: all resident blocks are pinned
                    break;
                }
                unsigned int v = 0;
                if (lane == best) {
                    v = R.L_slot[lane][cursor];
                    ++cursor;
                }
                v = __shfl_sync(0xffffffffu, v, best);
                if (lane == 0) {
                    rs_put(R, v, kRsEvicted);
                    R.victims[R.n_vict++] = v;
                    R.lfree[R.n_lfree++] = v;
                }
                --resident;
                __syncwarp();
            }
            if (error) break;
            unsigned int ns = 0;
            if (lane == 0) {
                if (R.n_lfree > 0) {
                    ns = R.lfree[--R.n_lfree];
                } else {
                    ns = P.free_stack[--free_top];
                }
            }
            ns = __shfl_sync(0xffffffffu, ns, 0);
            free_top = __shfl_sync(0xffffffffu, free_top, 0);
            ++tick;
            if (lane == 0) {
                R.out_slot[i] = ns;
                R.out_lt[i] = tick;
                R.out_new[i] = 1;
            }
            ++resident;
            ++pinned;
            if (first_touch == ~0ull) first_touch = tick;
            __syncwarp();
        }
        if (lane == 0) {
            A.tick = tick;
            A.first_touch = first_touch;
            A.resident = resident;
            A.pinned = pinned;
            A.free_top = free_top;
            if (error) A.error = 1;
        }
    }
    __syncthreads();
    const bool err = A.error != 0;
    const int nv = R.n_vict;
    // apply: victims first (erase key, free slot), then inserts and touches
    const unsigned long long ev0 = C->n_ev;
    for (int k = tid; k < nv; k += T) {
        const unsigned int v = R.victims[k];
        const unsigned long long kk = P.key[v];
        table_erase(P, kk);
        P.evlog[(ev0 + k) % (unsigned long long)P.evlog_cap] = kk;  // ring; the host drains it
        P.lt[v] = kFreeTick;
        P.refs[v] = 0u;
        P.agent[v] = kNoAgent;
    }
    __syncthreads();
    const int done_len = err ? 0 : len;  // on error the partially replayed chunk is not applied
    for (int i = tid; i < done_len; i += T) {
        const unsigned int s = R.out_slot[i];
        if (R.out_new[i]) {
            const int gi = lo + i;
            P.key[s] = a.keys[gi];
            P.tokens[s] = a.counts[gi];
            P.agent[s] = (a.agent != kNoAgent && gi < A.anchor) ? a.agent : kNoAgent;
            P.lt[s] = R.out_lt[i];
            P.refs[s] = 1u;
            if (table_insert(P, a.keys[gi], s)) atomicAdd(&R.n_reused, 1);
        } else {
            P.lt[s] = R.out_lt[i];
            atomicAdd(&P.refs[s], 1u);
        }
        P.p_slot[lo + i] = s;
    }
    // later chunks: blocks evicted here are absent when reached
    if (nv > 0) {
        for (int j = hi + tid; j < A.admit_n; j += T) {
            const unsigned int s = P.p_slot[j];
            if (s != kNoSlot && rs_get(R, s) == kRsEvicted) P.p_slot[j] = kNoSlot;
        }
    }
    __syncthreads();
    if (tid == 0) {
        for (int k = 0; k < R.n_lfree; ++k) P.free_stack[A.free_top++] = R.lfree[k];
        C->resident = A.resident;
        C->pinned = A.pinned;
        C->free_top = A.free_top;
        C->n_ev = ev0 + nv;
        C->tombstones += (long long)nv - R.n_reused;
        A.n_ev_adm += nv;
    }
    __syncthreads();
}

// ------------------------------------------------------------------ the admission kernel

__device__ void write_status(const DevPool& P, const AdmitArgs& a, const AdmSmem& A) {
    Ctrl* C = P.ctrl;
    AdmitStatus* st = a.status;
    st->started = A.started;
    st->error = A.error;
    st->first_miss = A.first_miss;
    st->admit_n = A.admit_n;
    st->cached = A.cached;
    st->n_evicted = A.n_ev_adm;
    st->resident = C->resident;
    st->pinned = C->pinned;
    st->tick_after = A.tick;
    st->ev_total = C->n_ev;
    st->warm_issued = A.warm_issued;
    st->needed = A.needed;
    st->scans = A.scans;
    st->tombstones = C->tombstones;
    st->n_pend = C->n_pend;
    for (int k = 0; k < C->n_pend && k < kMaxPending; ++k) {
        st->pend_target[k] = C->pend_target[k];
        st->pend_tick[k] = C->pend_tick[k];
    }
    __threadfence_system();
}

__global__ void __launch_bounds__(1024, 1) admit_kernel(DevPool P, AdmitArgs a, int CAP) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ ScanSmem S;
    __shared__ SelectSmem Sel;
    __shared__ RedSmem Red;
    __shared__ AdmSmem A;
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int NL = P.n_lists;
    unsigned long long* blt = reinterpret_cast<unsigned long long*>(dsm);
    unsigned int* bslot = reinterpret_cast<unsigned int*>(dsm + (size_t)NL * CAP * 8);
    unsigned char* cls_s = dsm + (size_t)NL * CAP * 12;
    ReplaySmem& Rp = *reinterpret_cast<ReplaySmem*>(dsm);

    // ---- phase 0 (CTA 0): poll reset, probe, feasibility, dispatch, lookup
    if (blockIdx.x == 0) {
        if (tid == 0) {
            A.started = 1;
            A.error = 0;
            A.cached = 0;
            A.n_ev_adm = 0;
            A.first_miss = 0;
            A.admit_n = 0;
            A.chunk = 0;
            A.needed = 0;
            A.warm_issued = -1;
            A.scans = 0;
            A.first_touch = ~0ull;
            A.tick = a.tick_base;
            C->done = 0;
            C->error = 0;
            if (a.flags & kPollReset) {
                C->step_warmups = 0;
                C->n_pend = 0;
            }
        }
        __syncthreads();
        const int n = a.n;
        long long miss_min = n, need = 0;
        for (int i = tid; i < n; i += T) {
            const unsigned int s = table_find(P, a.keys[i]);
            const unsigned int r0 = s == kNoSlot ? 0u : P.refs[s];
            P.p_slot[i] = s;
            P.p_refs0[i] = r0;
            if (s == kNoSlot && i < miss_min) miss_min = i;
            if (s == kNoSlot || r0 == 0u) ++need;
        }
        need = block_sum(need, Red);
        miss_min = block_min(miss_min, Red);
        if (tid == 0) A.needed = (int)need;
        if ((a.flags & kFeasible) && C->pinned + need > P.cap) {
            if (tid == 0) A.started = 0;  // try_start_head: wait for in-flight pins to clear
        }
        __syncthreads();
        if (A.started) {
            if (a.flags & kDispatch) {
                if (tid == 0) A.tick = A.tick + 1;
                __syncthreads();
                observe_dispatch(P, a.prev, a.next, A.tick, a.n_agents, dsm, Red, A);
            }
            if (a.flags & kLookup) {
                const int f = (int)miss_min;
                long long cached = 0;
                for (int i = tid; i < f; i += T) {
                    cached += a.counts[i];
                    P.lt[P.p_slot[i]] = A.tick + 1 + (unsigned long long)i;  // EngineSim::touch
                }
                cached = block_sum(cached, Red);
                if (tid == 0) {
                    A.first_miss = f;
                    A.cached = cached;
                    A.tick += (unsigned long long)f;
                }
            }
            if (tid == 0) {
                int an = (a.flags & kAdmit) ? n : 0;
                const long long room = P.cap - C->pinned;
                if (a.flags & kTruncate) an = (int)room;
                if (a.flags & kWarmupRoom) an = (int)min((long long)n, room);
                A.admit_n = an;
                A.anchor = a.anchor < 0 ? an : a.anchor;
            }
        }
        __syncthreads();
    }

    // ---- chunk loop: prep (CTA 0) | scan (all) | finalize (one CTA per list) | replay (CTA 0)
    for (;;) {
        if (blockIdx.x == 0) {
            const bool stop = !A.started || A.error || A.chunk * kChunk >= A.admit_n;
            if (stop) {
                if (tid == 0) C->done = 1;
            } else {
                const int lo = A.chunk * kChunk, hi = min(A.admit_n, lo + kChunk);
                long long absent = 0;
                for (int j = lo + tid; j < hi; j += T) absent += P.p_slot[j] == kNoSlot ? 1 : 0;
                absent = block_sum(absent, Red);
                const int need_scan = C->resident + absent > P.cap ? 1 : 0;
                if (tid < NL && need_scan) {
                    P.gbound[tid] = ~0ull;
                    P.gcount[tid] = 0;
                }
                if (tid == 0) {
                    C->need_scan = need_scan;
                    C->keep = hi - lo;
                    if (need_scan) {
                        A.scans += 1;
                        C->scans += 1;
                        C->scanned_slots += P.cap;
                    }
                }
            }
            // lists (and hop classes) must be visible before the scan reads them
            for (int x = tid; x < a.n_agents; x += T) cls_s[x] = P.cls[x];
            __threadfence();
        }
        grid_barrier(C);
        if (*(volatile int*)&C->done) break;
        const int need_scan = *(volatile int*)&C->need_scan;
        const int keep = *(volatile int*)&C->keep;
        if (need_scan) {
            if (blockIdx.x != 0) {
                for (int x = tid; x < a.n_agents; x += T) cls_s[x] = P.cls[x];
                __syncthreads();
            }
            scan_pass(P, NL, keep, cls_s, blt, bslot, CAP, S, Sel);
            grid_barrier(C);
            for (int l = blockIdx.x; l < NL; l += gridDim.x)
                finalize_list(P, l, NL, keep, blt, bslot, Sel);
            grid_barrier(C);
        }
        if (blockIdx.x == 0) {
            replay_apply(P, a, Rp, A, NL, need_scan != 0);
            if (tid == 0) A.chunk += 1;
            __syncthreads();
        }
    }

    // ---- epilogue (CTA 0): EngineSim::admit unpins at once; pins out; status
    if (blockIdx.x == 0) {
        if (A.started && !A.error) {
            long long dec = 0;
            for (int i = tid; i < A.admit_n; i += T) {
                const unsigned int s = P.p_slot[i];
                if (a.pins_out) a.pins_out[i] = s;
                if (a.flags & kUnpinAfter) {
                    if (atomicSub(&P.refs[s], 1u) == 1u) ++dec;
                }
            }
            dec = block_sum(dec, Red);
            if (tid == 0) C->pinned -= dec;
        }
        __syncthreads();
        if (tid == 0) write_status(P, a, A);
    }
}

// ------------------------------------------------------------------ small kernels

__global__ void init_pool_kernel(DevPool P) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long s = i; s < P.cap; s += stride) {
        P.lt[s] = kFreeTick;
        P.agent[s] = kNoAgent;
        P.refs[s] = 0u;
        P.key[s] = 0ull;
        P.tokens[s] = 0;
        P.free_stack[s] = (unsigned int)(P.cap - 1 - s);  // pops hand out slot 0 first
    }
    for (long long e = i; e <= (long long)P.tmask; e += stride) {
        P.table[e].key = 0ull;
        P.table[e].slot = kSlotEmpty;
        P.table[e].pad = 0u;
    }
    for (long long x = i; x < P.a_cap; x += stride) {
        P.cls[x] = (unsigned char)P.e_max;
        P.hop[x] = (unsigned char)P.e_max;
    }
    if (i == 0) {
        Ctrl* C = P.ctrl;
        C->resident = 0;
        C->pinned = 0;
        C->free_top = P.cap;
        C->tombstones = 0;
        C->n_ev = 0;
        C->scans = 0;
        C->scanned_slots = 0;
        C->rebuilds = 0;
        C->win_head = 0;
        C->win_size = 0;
        C->cur_agent = -1;
        C->reach_built = 0;
        C->step_warmups = 0;
        C->n_pend = 0;
        C->bar_count = 0;
        C->bar_gen = 0;
        C->done = 0;
    }
}

struct HashCursor {
    unsigned long long h, parent;
    long long pos, len, blk, bo;
    int in_blk, bs, has_parent;
    unsigned long long* keys;
    int* counts;
    __device__ __forceinline__ void start() {
        h = mix64(kHashSeed ^ kRootParent);
        in_blk = 0;
        blk = 0;
        pos = 0;
    }
    // chain_hash absorbs one token; a full (or final) block emits its key (hashing.cpp:26-51)
    __device__ __forceinline__ void eat(unsigned int t) {
        h = mix64(h ^ ((unsigned long long)t + kGolden));
        ++in_blk;
        ++pos;
        if (in_blk == bs || pos == len) {
            keys[bo + blk] = h;
            counts[bo + blk] = in_blk;
            ++blk;
            in_blk = 0;
            h = mix64(kHashSeed ^ h);
        }
    }
};

// derive_agent_identity (cachesage_policy.cpp:9-31) over this prompt's freshly written keys
__device__ __forceinline__ unsigned long long identity_of(const unsigned long long* k, long long nb, int skip,
                                                           int take) {
    long long lo = 0, hi = nb;
    if (nb >= (long long)skip + take) {
        lo = skip;
        hi = (long long)skip + take;
    } else if (nb > skip) {
        lo = skip;
    }
    unsigned long long h = mix64(kHashSeed ^ kIdentitySalt);
    for (long long j = lo; j < hi; ++j) h = mix64(h ^ k[j]);
    return h;
}

// K1 over explicit token streams: one thread per prompt (the chain is sequential within a
// prompt), tokens read as 128-bit vectors once 16-B aligned.
__global__ void hash_prompts_kernel(const unsigned int* __restrict__ tok, const long long* __restrict__ tok_off, int n,
                                    int bs, int skip, int take, const long long* __restrict__ blk_off,
                                    unsigned long long* keys, int* counts, unsigned long long* agents, int* err) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const long long off = tok_off[p];
    HashCursor c;
    c.len = tok_off[p + 1] - off;
    c.bs = bs;
    c.bo = blk_off[p];
    c.keys = keys;
    c.counts = counts;
    if (c.len <= 0) {
        atomicExch(err, 1);  // chain_hash: token sequence must be nonempty
        return;
    }
    c.start();
    const unsigned int* t = tok + off;
    long long i = 0;
    while (i < c.len && (reinterpret_cast<uintptr_t>(t + i) & 15u)) c.eat(t[i++]);
    for (; i + 4 <= c.len; i += 4) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(t + i));
        c.eat(q.x);
        c.eat(q.y);
        c.eat(q.z);
        c.eat(q.w);
    }
    while (i < c.len) c.eat(t[i++]);
    if (agents) agents[p] = identity_of(keys + c.bo, c.blk, skip, take);
}

// K1 for generated traces: token ids synthesised in registers from the turn descriptor
// (Trace::turn_tokens / warmup_tokens, workload.cpp:125-154), so no token stream crosses HBM.
__global__ void hash_turns_kernel(const TurnDesc* __restrict__ turns, int n, int bs, int skip, int take,
                                  unsigned int stride, int pos_bits, unsigned long long* keys, int* counts,
                                  unsigned long long* agents) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const TurnDesc d = turns[p];
    HashCursor c;
    c.len = (long long)d.template_tokens + d.anchor_tokens + (d.warmup ? 1 : d.history_tokens);
    c.bs = bs;
    c.bo = d.blk_off;
    c.keys = keys;
    c.counts = counts;
    c.start();
    for (int j = 0; j < d.template_tokens; ++j) c.eat(0x00100000u + (unsigned int)j);
    const unsigned int ab = 0x01000000u + (unsigned int)d.agent * stride;
    for (int j = 0; j < d.anchor_tokens; ++j) c.eat(ab + (unsigned int)j);
    if (d.warmup) {
        c.eat(0x02000000u);
    } else {
        const unsigned int hb = 0x80000000u | ((unsigned int)d.session << pos_bits);
        for (int q = 0; q < d.history_tokens; ++q) c.eat(hb | (unsigned int)q);
    }
    if (agents) agents[p] = identity_of(keys + c.bo, c.blk, skip, take);
}

__global__ void unpin_kernel(DevPool P, const unsigned int* slots, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int dec = 0;
    if (i < n) {
        if (atomicSub(&P.refs[slots[i]], 1u) == 1u) dec = 1;
    }
    dec = __reduce_add_sync(0xffffffffu, dec);
    if (lane_id() == 0 && dec) atomicAdd(reinterpret_cast<unsigned long long*>(&P.ctrl->pinned),
                                         (unsigned long long)(-(long long)dec));
}

__global__ void restore_kernel(DevPool P, const unsigned long long* keys, const unsigned long long* lt,
                               const unsigned int* agents, const unsigned int* refs, long long n,
                               unsigned long long* acc /* [pinned, reused] */) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long top = P.ctrl->free_top;
    const unsigned int s = P.free_stack[top - 1 - i];
    P.key[s] = keys[i];
    P.lt[s] = lt[i];
    P.agent[s] = agents ? agents[i] : kNoAgent;
    const unsigned int r = refs ? refs[i] : 0u;
    P.refs[s] = r;
    P.tokens[s] = 16;
    const int reused = table_insert(P, keys[i], s);
    if (r) atomicAdd(acc, 1ull);
    if (reused) atomicAdd(acc + 1, 1ull);
}

__global__ void restore_finish_kernel(DevPool P, long long n, const unsigned long long* acc) {
    Ctrl* C = P.ctrl;
    C->free_top -= n;
    C->resident += n;
    C->pinned += (long long)acc[0];
    C->tombstones -= (long long)acc[1];
}

__global__ void probe_kernel(DevPool P, const unsigned long long* keys, int n, int* needed) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int c = 0;
    if (i < n) {
        const unsigned int s = table_find(P, keys[i]);
        c = (s == kNoSlot || P.refs[s] == 0u) ? 1 : 0;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane_id() == 0 && c) atomicAdd(needed, c);
}

__global__ void min_lt_kernel(DevPool P, unsigned long long* out) {
    unsigned long long m = ~0ull;
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < P.cap;
         s += (long long)gridDim.x * blockDim.x) {
        const unsigned long long x = P.lt[s];
        if (x < m) m = x;
    }
    for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane_id() == 0) atomicMin(out, m);
}

__global__ void scores_kernel(DevPool P, unsigned long long now, const unsigned long long* minlt,
                              unsigned long long* keys, double* scores, long long* n_out) {
    const unsigned long long old = min(now, *minlt);
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < P.cap;
         s += (long long)gridDim.x * blockDim.x) {
        const unsigned long long x = P.lt[s];
        if (x == kFreeTick) continue;
        const unsigned int a = P.agent[s];
        const int c = (a == kNoAgent) ? P.e_max : (int)P.cls[a];
        const double sc = score_of(P.policy, P.w_pred, survival_of_class(c, P.e_max), x, now, old);
        const long long o = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(n_out), 1ull);
        keys[o] = P.key[s];
        scores[o] = sc;
    }
}

__global__ void table_clear_kernel(DevPool P) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e <= (long long)P.tmask;
         e += (long long)gridDim.x * blockDim.x) {
        P.table[e].slot = kSlotEmpty;
        P.table[e].key = 0ull;
    }
}

__global__ void table_fill_kernel(DevPool P) {
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < P.cap;
         s += (long long)gridDim.x * blockDim.x) {
        if (P.lt[s] != kFreeTick) table_insert(P, P.key[s], (unsigned int)s);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) P.ctrl->tombstones = 0;
}

// ------------------------------------------------------------------ host launchers

static size_t admit_smem_bytes(int NL, int CAP, int a_cap) {
    size_t scan = (size_t)NL * CAP * 12 + (size_t)a_cap;
    scan = (scan + 15) & ~size_t(15);
    size_t replay = sizeof(ReplaySmem);
    size_t need = std::max(scan, replay + (size_t)a_cap + 16);
    // cls_s sits right after the NL*CAP*12 candidate area; keep it clear of ReplaySmem
    if ((size_t)NL * CAP * 12 < replay) need = std::max(need, replay + (size_t)a_cap + 16);
    return need;
}

LaunchCfg admit_launch_config(const DevPool& P, int device, int want_grid) {
    LaunchCfg lc{0, 0, 0, 0};
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return lc;
    const size_t smem_max = prop.sharedMemPerBlockOptin;
    const size_t static_smem = sizeof(ScanSmem) + sizeof(SelectSmem) + sizeof(RedSmem) + sizeof(AdmSmem) + 1024;
    for (int threads = kScanThreads; threads >= 256; threads >>= 1) {
        int cap = kChunk + 1 + kSlack + threads;
        cap = (cap + 3) & ~3;
        if (cap > 4 * threads) continue;
        size_t smem = admit_smem_bytes(P.n_lists, cap, P.a_cap);
        // cls_s is placed at NL*CAP*12: when ReplaySmem is larger, move it past ReplaySmem
        if (smem + static_smem > smem_max) continue;
        if (cudaFuncSetAttribute(admit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return lc;
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, admit_kernel, threads, smem) != cudaSuccess || occ < 1)
            continue;
        int grid = prop.multiProcessorCount * occ;
        if (want_grid > 0 && want_grid < grid) grid = want_grid;
        lc.grid = grid;
        lc.threads = threads;
        lc.cap_per_list = cap;
        lc.smem = smem;
        return lc;
    }
    return lc;
}

cudaError_t launch_admit(const DevPool& P, const AdmitArgs& a, const LaunchCfg& lc, int grid, cudaStream_t s) {
    DevPool p = P;
    AdmitArgs aa = a;
    int cap = lc.cap_per_list;
    void* args[] = {&p, &aa, &cap};
    if (grid <= 1) {
        return cudaLaunchKernel((const void*)admit_kernel, dim3(1), dim3(lc.threads), args, lc.smem, s);
    }
    return cudaLaunchCooperativeKernel((const void*)admit_kernel, dim3(grid), dim3(lc.threads), args, lc.smem, s);
}

cudaError_t launch_init_pool(const DevPool& P, cudaStream_t s) {
    init_pool_kernel<<<1184, 256, 0, s>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_hash_prompts(const unsigned int* tokens, const long long* tok_off, int n, int bs, int skip,
                                int take, const long long* blk_off, unsigned long long* keys, int* counts,
                                unsigned long long* agents, int* err, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    hash_prompts_kernel<<<(n + 127) / 128, 128, 0, s>>>(tokens, tok_off, n, bs, skip, take, blk_off, keys, counts,
                                                         agents, err);
    return cudaGetLastError();
}

cudaError_t launch_hash_turns(const TurnDesc* turns, int n, int bs, int skip, int take, unsigned int anchor_stride,
                              int hist_pos_bits, unsigned long long* keys, int* counts, unsigned long long* agents,
                              cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    hash_turns_kernel<<<(n + 127) / 128, 128, 0, s>>>(turns, n, bs, skip, take, anchor_stride, hist_pos_bits, keys,
                                                       counts, agents);
    return cudaGetLastError();
}

cudaError_t launch_unpin(const DevPool& P, const unsigned int* slots, int n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    unpin_kernel<<<(n + 255) / 256, 256, 0, s>>>(P, slots, n);
    return cudaGetLastError();
}

cudaError_t launch_restore(const DevPool& P, const unsigned long long* keys, const unsigned long long* lt,
                           const unsigned int* agents, const unsigned int* refs, long long n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    unsigned long long* acc = nullptr;
    cudaError_t e = cudaMallocAsync(&acc, 16, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(acc, 0, 16, s);
    restore_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, keys, lt, agents, refs, n, acc);
    restore_finish_kernel<<<1, 1, 0, s>>>(P, n, acc);
    cudaFreeAsync(acc, s);
    return cudaGetLastError();
}

cudaError_t launch_probe(const DevPool& P, const unsigned long long* keys, int n, int* needed, cudaStream_t s) {
    cudaMemsetAsync(needed, 0, sizeof(int), s);
    if (n > 0) probe_kernel<<<(n + 255) / 256, 256, 0, s>>>(P, keys, n, needed);
    return cudaGetLastError();
}

cudaError_t launch_scores(const DevPool& P, unsigned long long now, unsigned long long* keys, double* scores,
                          long long* n_out, unsigned long long* scratch, cudaStream_t s) {
    cudaMemsetAsync(scratch, 0xff, 8, s);
    cudaMemsetAsync(n_out, 0, 8, s);
    min_lt_kernel<<<592, 256, 0, s>>>(P, scratch);
    scores_kernel<<<592, 256, 0, s>>>(P, now, scratch, keys, scores, n_out);
    return cudaGetLastError();
}

cudaError_t launch_table_rebuild(const DevPool& P, cudaStream_t s) {
    table_clear_kernel<<<1184, 256, 0, s>>>(P);
    table_fill_kernel<<<1184, 256, 0, s>>>(P);
    return cudaGetLastError();
}

}  // namespace csb
