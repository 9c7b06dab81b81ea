// The admission kernel: ONE cooperative launch per EngineSim admission
// (start_request / execute_warmup / admit, engine.cpp:141-323), paths relative to
// /root/reference/proj.
//
//   phase 0  (CTA 0)  poll reset, K2 probe of the prompt, try_start_head feasibility,
//                     K3/K3b/K6 observe(AgentDispatch), K2 lookup touches
//   per chunk of <= 128 prompt blocks:
//     prep   (CTA 0)  can this chunk evict? reset the per-list bounds
//     K4 scan (all)   one streaming pass over the SoA pool (16 B per slot): per survival
//                     class the `keep` oldest unpinned slots + the keep+1 oldest resident
//     K5a     (CTA l) exact select of list l over all CTAs' survivors, sorted by last_touch
//     K5b     (CTA 0) exact replay of admit_pinned with evict_one (engine.cpp:102-125) over
//                     the class heads, then block-table / SoA updates
//
// Why per-class heads are exact: inside one survival class the score w_pred*S + rho is a
// non-decreasing function of last_touch and ties break on last_touch (engine.cpp:111-114), so
// the class's oldest unpinned block is its best candidate; classes only lose members during an
// admission (new and reached blocks are pinned at once), at most one per prompt block, so the
// `keep` oldest per class at the start of a chunk contain every head the chunk needs. The
// resident-oldest list gives oldest_live_touch (engine.cpp:90-100) the same way. DESIGN.md §4.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>

#include "cs_block.cuh"
#include "cs_engine_state.h"
#include "cs_launch.h"

namespace csb {

constexpr int kThreads = 512;            // one CTA per SM (cooperative grid)
constexpr int kV = 4;                    // slots per thread per tile (2 x LDG.128 + 2 x LDG.128)
constexpr int kTile = kThreads * kV;     // 2048 slots = 16 KiB of packed scan words per tile
constexpr int kRing = 6;                 // TMA stages (16 KiB of packed words each) per CTA
constexpr int kStage = 6144;             // staged candidates per CTA (all lists share it)
constexpr int kFlushAt = kStage - 2 * kTile;  // a tile appends at most 2 entries per slot
constexpr int kSide = kMaxLists * (kChunk + 1);

// ------------------------------------------------------------------ shared state

constexpr int kBfsPre = 2048;  // window pairs phase 0 can prefetch for the BFS
constexpr int kPend = kMaxLists;  // staged agent-carrying slot whose class phase 0 has not fixed yet

struct ScanSmem {
    unsigned long long thr[kMaxLists + 1];  // inclusive acceptance bound per list (+ kPend)
    unsigned long long gbw[kMaxLists];
    int count;                          // staged entries
    int side_n;
    int lcnt[kMaxLists];
    int wcnt[kMaxLists], wbase[kMaxLists], wpos[kMaxLists];
    unsigned long long flush_ns, flushes;  // instrumentation (reported by CTA 0)
    unsigned long long hint[kMaxLists];
    unsigned long long lmin[kMaxLists];
    int overflow;
    int ovf_base;   // staging positions [0, ovf_base) were all written before an overflow
    int spec;       // speculative pass: phase 0 runs concurrently on CTA 0
    int hc, dc;     // ensure_cls compaction counters
    int prep_done;  // the producer warp already loaded the classes and built the change set
    unsigned char hinted[kMaxLists];  // CTA 0: the lists that had a hint in this launch's first pass
    int cls_ready;  // B.cls holds this launch's classes (else kPend for every agent)
    unsigned int xset[kXset];  // slots phase 0 may change: excluded here, restaged fresh by CTA 0
    __align__(8) unsigned long long mbar[kRing];        // TMA ring: stage filled
    __align__(8) unsigned long long mbar_empty[kRing];  // TMA ring: stage released by all consumers
};

struct AdmSmem {
    unsigned long long tick;         // engine clock (EngineSim::tick_)
    unsigned long long first_touch;  // earliest tick admit_pinned touched in this admission
    long long cached, n_ev_adm, resident, pinned, free_top;
    int first_miss, admit_n, anchor, chunk, started, error, needed, warm_issued, scans;
    int fin_want;  // lists finalized by CTAs other than 0 in the current pass
    int q_deleg;   // CTA kSvcQ applies the previous queue: wait for it before touching the counters
    int need_full; // a prescan-fed chunk needs the serial replay (every class list): scan instead
    double wsurv[kMaxLists];  // P.wsurv staged on chip (indexed kernel-parameter loads are slow)
    unsigned long long ph[kPhases], tl;  // phase timestamps (CTA 0, thread 0)
    long long pf_head, pf_size;  // the learner window at launch (BFS prefetch)
    int pf_on;
    unsigned long long srv_t0;  // admission server: when CTA 0 picked this admission up (else 0)
    int st_done;  // the status went out early (from the apply's idle warp), not in the epilogue
    int svc_b;    // observe(AgentDispatch) comes from the learner service (commit_observe)
    // CTA 0's own counters, kept on chip (their Ctrl copies are written through): the eviction
    // log length and the block-table queue lengths
    unsigned long long n_ev_c;
    int tq_e, tq_i;
    long long pin_c;  // pinned_count_ (its Ctrl copy written through)
};

// Dynamic shared memory, phase by phase (the regions alias across phases):
//   scan    : staging (lt, slot, list) x kStage | side (lt, slot, list) x kSide | cls table
//   select  : staging holds list l's candidates, side the sorted output
//   replay  : ReplaySmem
//   phase 0 : BFS window (pairs + edge flags) and hop table
struct ScanBufs {
    unsigned long long* st_lt;
    unsigned int* st_slot;
    unsigned char* st_list;
    unsigned long long* sd_lt;
    unsigned int* sd_slot;
    unsigned char* sd_list;
    unsigned char* cls;
};

constexpr size_t kOffStSlot = 8ull * kStage;
constexpr size_t kOffStList = kOffStSlot + 4ull * kStage;
constexpr size_t kOffSdLt = (kOffStList + kStage + 15) & ~size_t(15);
constexpr size_t kOffSdSlot = kOffSdLt + 8ull * kSide;
constexpr size_t kOffSdList = kOffSdSlot + 4ull * kSide;
constexpr size_t kOffCls = (kOffSdList + kSide + 15) & ~size_t(15);
constexpr size_t kOffRing = (kOffCls + kMaxAgents + 127) & ~size_t(127);  // TMA ring (128-B aligned)
constexpr size_t kRingStage = 8ull * kTile;  // 16 KiB: one packed word (pk) per slot
constexpr size_t kDynSmem = kOffRing + kRing * kRingStage;

__device__ __forceinline__ ScanBufs scan_bufs(unsigned char* d) {
    ScanBufs b;
    b.st_lt = reinterpret_cast<unsigned long long*>(d);
    b.st_slot = reinterpret_cast<unsigned int*>(d + kOffStSlot);
    b.st_list = d + kOffStList;
    b.sd_lt = reinterpret_cast<unsigned long long*>(d + kOffSdLt);
    b.sd_slot = reinterpret_cast<unsigned int*>(d + kOffSdSlot);
    b.sd_list = d + kOffSdList;
    b.cls = d + kOffCls;
    return b;
}

struct ReplaySmem {
    unsigned long long L_lt[kMaxLists][kChunk + 2];
    unsigned int L_slot[kMaxLists][kChunk + 2];
    short L_pidx[kMaxLists][kChunk + 2];  // chunk-relative prompt index of the slot, or -1
    short L_rpos[kMaxLists][kChunk + 2];  // position in the resident list, or -1
    int L_n[kMaxLists];
    unsigned char touched[kChunk];       // prompt block touched+pinned by this chunk
    unsigned char pevict[kChunk];        // prompt block evicted before it was reached
    unsigned char rremoved[kChunk + 2];  // resident-list entry evicted
    unsigned int c_slot[kChunk];
    unsigned int c_refs0[kChunk];
    unsigned int out_slot[kChunk];
    unsigned long long out_lt[kChunk];
    unsigned char out_new[kChunk];
    unsigned int victims[kChunk];
    unsigned long long vkey[kChunk];
    unsigned int freeslots[kChunk];
    unsigned int ph_key[512];  // slot -> chunk index hash of the chunk's resident prompt blocks
    short ph_val[512];
    unsigned int vh_key[512];  // victim-slot set for fixing up later chunks
    int n_vict, n_new_global, n_reused;
    int pdom;  // length of the class-E prefix whose heads beat every other class outright
    int bulk;  // this chunk was replayed in bulk (no serial loop)
    // list-independent prologue (replay_prologue), valid from phase 0 on
    long long res0, pinned0, ftop;
    int absent, pre_unpinned;
    int n_ins;  // queued inserts of this chunk
    int lists_ready;  // the consumer of a prescan wrote L_* (and E keys) directly
    unsigned long long E_key[kChunk + 2];  // keys of list E (lists_ready): victims need no key load
    unsigned char E_key_ok[kChunk + 2];
};
// The replay view lives in the TMA ring: free after a scan, and never used by CTA 0 during a
// speculative pass, so CTA 0 prepares the prologue while the other CTAs still stream.
static_assert(sizeof(ReplaySmem) <= kRing * kRingStage, "replay view must fit the TMA ring");

// The prescan consumer's view (CTA 0, pipelined launch): the list service's E and R lists, the
// set U re-read in phase 0 and the slots this launch's lookup touched. Lives in the TMA ring
// above the replay view.
constexpr int kTset = 1024;   // slots touched by this launch's lookup (hash)
struct EarlySmem {
    unsigned long long E_lt[kPreK], E_key[kPreK];
    unsigned int E_slot[kPreK];
    unsigned char E_ok[kPreK];
    unsigned long long R_lt[kPreK];
    unsigned int R_slot[kPreK];
    unsigned char R_ok[kPreK];
    unsigned long long U_lt[kXset];  // U re-read after the unpins, by xset position
    unsigned int U_agent[kXset];
    unsigned char U_ok[kXset];
    unsigned short xl[kXset];  // the xset positions phase 0 filled (U), in insertion order
    int xn;
    int efx[kPreK + 1];        // exclusive prefix count of the surviving E entries
    unsigned int tset[kTset];
    unsigned long long TE, TR, TP;
    int nE, nR, nP, ok, valid;
};
constexpr size_t kEarlyOff = 64 * 1024;
static_assert(sizeof(ReplaySmem) <= kEarlyOff, "replay view must stay below the early-validation view");
static_assert(kEarlyOff + sizeof(EarlySmem) <= kRing * kRingStage, "early-validation view must fit the TMA ring");

struct BfsSmem {
    unsigned short wa[8192];
    unsigned short wb[8192];
    unsigned char edge[8192];
    unsigned char hop[kMaxAgents];
    // prefetched by admit_body's phase 0 (window pairs in window order, their counts and row
    // totals before this admission's record): the BFS then runs without global round trips
    unsigned int pc[kBfsPre], pt[kBfsPre];
    int pf_size;
    unsigned int rec_c, rec_t;  // the record's counts[prev][next] and totals[prev] before it
};
static_assert(sizeof(BfsSmem) <= kOffCls, "BFS view must fit the scan region");
static_assert(sizeof(SelectSmem) <= 4096, "service_lists keeps its per-CTA offsets after a SelectSmem in the ring");

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void stamp(AdmSmem& A, int k) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long t = gtimer();
        A.ph[k] += t - A.tl;
        A.tl = t;
    }
}

// The admission server's trace ring (instrumentation, tools/cta0_timeline.py): per admission
// (seq % 8) 8 %globaltimer stamps: 0 pickup, 1 admit_body entry, 2 phase 0 end, 3 early status
// ready (CTA 0), 4 status published (CTA kSvcQ), 5 CTA 0 done, 6 streamers' verdict seen (CTA 4)
__device__ __forceinline__ void tstamp(const DevPool& P, unsigned long long seq, int k) {
    P.dbg[(size_t)gridDim.x * 16 + 192 + (seq & 7ull) * 8 + k] = gtimer();
}

// CTA-0 serial-chain timestamps (%globaltimer), after the per-CTA rows (instrumentation)
__device__ __forceinline__ void pstamp(const DevPool& P, int k) {
    if (blockIdx.x == 0 && threadIdx.x == 0) P.dbg[gridDim.x * 16 + k] = gtimer();
}

// CTA-0 sub-phase timestamps of the replay (instrumentation row 0, columns 10..15)
__device__ __forceinline__ void dstamp(const DevPool& P, int k) {
    if (blockIdx.x == 0 && threadIdx.x == 0) P.dbg[10 + k] = gtimer();
}

// CTA-0 sub-phase SM-clock stamps of finalize_list (instrumentation row 2, columns 10..15)
__device__ __forceinline__ void fstamp(const DevPool& P, int k) {
    if (blockIdx.x == 0 && threadIdx.x == 0) P.dbg[32 + 10 + k] = clock64();
}

// ------------------------------------------------------------------ K3 / K3b / K6

// CacheSagePolicy::observe(AgentDispatch) (cachesage_policy.cpp:57-72). CTA 0, all threads.
// K3b from a prefetched window (BfsSmem: pairs wa/wb, their counts pc and row totals pt before
// this dispatch's record, pf_size pairs, rec_c / rec_t = counts[prev][next] / totals[prev]
// before it): rebuild_reachability (reachability.cpp:39-81) on the learner state the record
// leaves. The record pushed (prev, next) and, with a full window, pushed out the oldest pair
// (oa, ob): counts and row totals move by +-1 exactly there (transition_learner.cpp:22-51).
// Writes B.hop[0, n_agents). All threads of the CTA.
__device__ void bfs_prefetched(const DevPool& P, BfsSmem& B, int prev, int next, int n_agents) {
    const int tid = threadIdx.x, T = blockDim.x;
    const long long W = P.window;
    const int e = P.e_max;
    const int sz0 = B.pf_size;
    const bool popped = prev >= 0 && (long long)sz0 == W;
    const int oa = popped ? (int)B.wa[0] : -1, ob = popped ? (int)B.wb[0] : -1;
    const int jlo = popped ? 1 : 0, jhi = sz0 + (prev >= 0 ? 1 : 0);
    for (int x = tid; x < n_agents; x += T) B.hop[x] = (unsigned char)e;
    for (int j = jlo + tid; j < jhi; j += T) {
        int aj, bj;
        unsigned int c, t;
        if (j < sz0) {
            aj = B.wa[j];
            bj = B.wb[j];
            c = B.pc[j] + (aj == prev && bj == next ? 1u : 0u) - (aj == oa && bj == ob ? 1u : 0u);
            t = B.pt[j] + (aj == prev ? 1u : 0u) - (aj == oa ? 1u : 0u);
        } else {  // the pair this record appended
            aj = prev;
            bj = next;
            B.wa[j] = (unsigned short)aj;
            B.wb[j] = (unsigned short)bj;
            c = B.rec_c + 1u - (aj == oa && bj == ob ? 1u : 0u);
            t = B.rec_t + 1u - (aj == oa ? 1u : 0u);
        }
        B.edge[j] = __ddiv_rn((double)c, (double)t) < P.tau ? 0 : 1;
    }
    __syncthreads();
    if (tid == 0) B.hop[next] = 0;
    __syncthreads();
    for (int d = 0; d + 1 < e; ++d) {
        int any = 0;
        for (int j = jlo + tid; j < jhi; j += T) {
            const int aj = B.wa[j], bj = B.wb[j];
            if (!B.edge[j] || B.hop[aj] != d) continue;
            if (B.hop[bj] > d + 1) {
                B.hop[bj] = (unsigned char)(d + 1);
                any = 1;
            }
        }
        if (!__syncthreads_or(any)) break;
    }
}

__device__ void observe_dispatch(const DevPool& P, int prev, int next, unsigned long long tick, int n_agents,
                                 unsigned char* dsm, RedSmem& Red, AdmSmem& A, unsigned char* cls_smem = nullptr,
                                 bool prefetched = false) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const long long W = P.window;
    const int Acap = P.a_cap;
    if (P.policy == 0) return;  // LruPolicy::observe is a no-op (baselines.cpp:10)
    // K3: TransitionLearner::record (transition_learner.cpp:22-51): one pair per dispatch
    if (prev >= 0 && tid == 0) {
        const long long head = C->win_head, size = C->win_size;
        atomicAdd(&C->recorded, 1ull);
        if (prefetched) {  // the new pair's count and row total (the BFS below needs them)
            BfsSmem& Bq = *reinterpret_cast<BfsSmem*>(dsm);
            Bq.rec_c = atomicAdd(&P.counts[(long long)prev * Acap + next], 1u);
            Bq.rec_t = atomicAdd(&P.totals[prev], 1u);
        } else {
            atomicAdd(&P.counts[(long long)prev * Acap + next], 1u);  // fire-and-forget (RED)
            atomicAdd(&P.totals[prev], 1u);
        }
        if (size == W) {
            const int oa = P.win_a[head], ob = P.win_b[head];
            P.win_a[head] = prev;
            P.win_b[head] = next;
            atomicSub(&P.counts[(long long)oa * Acap + ob], 1u);
            atomicSub(&P.totals[oa], 1u);
            C->win_head = head + 1 == W ? 0 : head + 1;
        } else {
            const long long pos = (head + size) % W;
            P.win_a[pos] = prev;
            P.win_b[pos] = next;
            C->win_size = size + 1;
        }
    }
    __syncthreads();
    pstamp(P, 13);
    const bool changed = C->cur_agent != next;
    __syncthreads();
    if (tid == 0) C->cur_agent = next;
    if (changed && prefetched) {
        BfsSmem& B = *reinterpret_cast<BfsSmem*>(dsm);
        bfs_prefetched(P, B, prev, next, n_agents);
        for (int x = tid; x < n_agents; x += T) {
            P.hop[x] = B.hop[x];
            P.cls[x] = B.hop[x];
            if (cls_smem) cls_smem[x] = B.hop[x];
        }
        if (tid == 0) {
            atomicAdd(&C->rebuilds, 1ull);
            C->reach_built = 1;
        }
        __syncthreads();
    } else if (changed) {
        // K3b: rebuild_reachability (reachability.cpp:39-81), level-synchronous over the
        // window's pairs (every positive count cell is a window pair). Edge iff
        // !(count/total < tau) in fp64; depth d expands only while d + 1 < e_max.
        const int e = P.e_max;
        const long long head = C->win_head, size = C->win_size;
        BfsSmem& B = *reinterpret_cast<BfsSmem*>(dsm);
        const bool in_smem = size <= 8192;
        for (int x = tid; x < n_agents; x += T) B.hop[x] = (unsigned char)e;
        for (long long j = tid; in_smem && j < size; j += T) {
            const long long q = (head + j) % W;
            const int a = P.win_a[q], b = P.win_b[q];
            const double c = (double)P.counts[(long long)a * Acap + b];
            const double t = (double)P.totals[a];
            B.wa[j] = (unsigned short)a;
            B.wb[j] = (unsigned short)b;
            B.edge[j] = __ddiv_rn(c, t) < P.tau ? 0 : 1;
        }
        __syncthreads();
        if (tid == 0) B.hop[next] = 0;
        __syncthreads();
        for (int d = 0; d + 1 < e; ++d) {
            int any = 0;
            for (long long j = tid; j < size; j += T) {
                int a, b, ok;
                if (in_smem) {
                    a = B.wa[j];
                    b = B.wb[j];
                    ok = B.edge[j];
                } else {
                    const long long q = (head + j) % W;
                    a = P.win_a[q];
                    b = P.win_b[q];
                    ok = !(__ddiv_rn((double)P.counts[(long long)a * Acap + b], (double)P.totals[a]) < P.tau);
                }
                if (!ok || B.hop[a] != d) continue;
                if (B.hop[b] > d + 1) {
                    B.hop[b] = (unsigned char)(d + 1);
                    any = 1;
                }
            }
            if (!__syncthreads_or(any)) break;
        }
        for (int x = tid; x < n_agents; x += T) {
            P.hop[x] = B.hop[x];
            P.cls[x] = B.hop[x];
            if (cls_smem) cls_smem[x] = B.hop[x];  // the admission kernel's class table on chip
        }
        if (tid == 0) {
            atomicAdd(&C->rebuilds, 1ull);
            C->reach_built = 1;
        }
        __syncthreads();
    }
    pstamp(P, 14);
    // K6: maybe_prefetch (cachesage_policy.cpp:109-123) with argmax_row
    // (transition_learner.cpp:79-96): max count, ties -> smaller 64-bit AgentId
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
        __syncthreads();
        if (lane_id() == 0) {
            Red.u[warp_id()] = best_c;
            Red.v[warp_id()] = (long long)best_b;
            Red.w[warp_id()] = best_id;
        }
        __syncthreads();
        if (tid == 0) {
            const int nw = (T + 31) >> 5;
            best_c = 0;
            best_b = -1;
            best_id = ~0ull;
            for (int w = 0; w < nw; ++w) {
                const int b = (int)Red.v[w];
                if (b < 0) continue;
                const unsigned long long c = Red.u[w], id = Red.w[w];
                if (best_b < 0 || c > best_c || (c == best_c && id < best_id)) {
                    best_c = c;
                    best_id = id;
                    best_b = b;
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

// The learner service (CTA kSvcB of a pipelined launch): CacheSagePolicy::observe(AgentDispatch
// {prev, next}) (cachesage_policy.cpp:50-77) computed speculatively, concurrently with CTA 0's
// probe, on the learner state this dispatch's record will leave (the record's +-1 applied on
// chip): the rebuilt reachability (K3b) when the agent changes and the prefetch gate's
// argmax_row(next) (K6, transition_learner.cpp:79-96). Nothing of the policy's state is written;
// CTA 0 commits it (commit_observe) only if the request starts, so a request that waits commits
// nothing. Runs only when CTA 0 uses it (the same predicate, evaluated on the same inputs).
__device__ void service_learner(const DevPool& P, const AdmitArgs& a, unsigned char* dsm, RedSmem& Red) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const long long W = P.window;
    const int Acap = P.a_cap, n_agents = a.n_agents, prev = a.prev, next = a.next;
    BfsSmem& B = *reinterpret_cast<BfsSmem*>(dsm);
    __shared__ long long s_head, s_size;
    __shared__ int s_changed;
    if (tid == 0) {
        P.dbg[blockIdx.x * 16 + 6] = gtimer();  // (instrumentation: service start / loads / BFS / done)
        s_head = __ldcg(&C->win_head);
        s_size = __ldcg(&C->win_size);
        s_changed = __ldcg(&C->cur_agent) != next ? 1 : 0;
    }
    // row `next` and the ids for the argmax: independent of the window, issued first
    unsigned long long best_c = 0ull, best_id = ~0ull;
    int best_b = -1;
    unsigned int rc[8];
    unsigned long long rid[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int b = tid + k * T;
        rc[k] = b < n_agents ? __ldcg(P.counts + (long long)next * Acap + b) : 0u;
        rid[k] = b < n_agents ? __ldcg(P.agent_ids + b) : 0ull;
    }
    __syncthreads();
    const long long head = s_head, size = s_size;
    const bool changed = s_changed != 0;
    // the window's pairs, then their counts and row totals (two dependent rounds), and the
    // record's own cell
    for (long long j = tid; j < size; j += T) {
        const long long q = (head + j) % W;
        const int aj = __ldcg(P.win_a + q), bj = __ldcg(P.win_b + q);
        B.wa[j] = (unsigned short)aj;
        B.wb[j] = (unsigned short)bj;
        B.pc[j] = __ldcg(P.counts + (long long)aj * Acap + bj);
        B.pt[j] = __ldcg(P.totals + aj);
    }
    unsigned int tot_next = 0u;
    if (tid == 0) {
        B.pf_size = (int)size;
        if (prev >= 0) {
            B.rec_c = __ldcg(P.counts + (long long)prev * Acap + next);
            B.rec_t = __ldcg(P.totals + prev);
        }
        tot_next = __ldcg(P.totals + next);
    }
    __syncthreads();
    const bool popped = prev >= 0 && size == W;
    const int oa = popped ? (int)B.wa[0] : -1, ob = popped ? (int)B.wb[0] : -1;
    if (tid == 0) P.dbg[blockIdx.x * 16 + 7] = gtimer();
    if (changed) bfs_prefetched(P, B, prev, next, n_agents);
    if (tid == 0) P.dbg[blockIdx.x * 16 + 8] = gtimer();
    // argmax_row(next) after the record: +1 at [next][next] when prev == next, -1 at [oa][ob]
    // when oa == next (the popped pair); ties -> the smaller 64-bit AgentId
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int b = tid + k * T;
        if (b >= n_agents) continue;
        const unsigned int c = rc[k] + (prev >= 0 && prev == next && b == next ? 1u : 0u) -
                               (oa == next && b == ob ? 1u : 0u);
        if (c == 0u) continue;
        if (best_b < 0 || c > best_c || (c == best_c && rid[k] < best_id)) {
            best_c = c;
            best_id = rid[k];
            best_b = b;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long oc = __shfl_xor_sync(0xffffffffu, best_c, o);
        const unsigned long long oi = __shfl_xor_sync(0xffffffffu, best_id, o);
        const int ob2 = __shfl_xor_sync(0xffffffffu, best_b, o);
        if (ob2 >= 0 && (best_b < 0 || oc > best_c || (oc == best_c && oi < best_id))) {
            best_c = oc;
            best_id = oi;
            best_b = ob2;
        }
    }
    __syncthreads();
    if (lane_id() == 0) {
        Red.u[warp_id()] = best_c;
        Red.v[warp_id()] = (long long)best_b;
        Red.w[warp_id()] = best_id;
    }
    if (changed)
        for (int w = tid; w * 8 < n_agents; w += T) {
            unsigned long long h8 = 0ull;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (w * 8 + k < n_agents) h8 |= (unsigned long long)B.hop[w * 8 + k] << (8 * k);
            P.spec_hop[w] = make_ulonglong2(a.seq, h8);
        }
    __syncthreads();
    if (tid == 0) {
        const int nw = (T + 31) >> 5;
        best_c = 0;
        best_b = -1;
        best_id = ~0ull;
        for (int w = 0; w < nw; ++w) {
            const int b = (int)Red.v[w];
            if (b < 0) continue;
            const unsigned long long c = Red.u[w], id = Red.w[w];
            if (best_b < 0 || c > best_c || (c == best_c && id < best_id)) {
                best_c = c;
                best_id = id;
                best_b = b;
            }
        }
        LearnSpec sp;
        sp.seq0 = sp.seq1 = sp.seq2 = a.seq;
        sp.changed = changed ? 1 : 0;
        sp.oa = oa;
        sp.ob = ob;
        sp.best_b = best_b;
        sp.best_c = (unsigned int)best_c;
        sp.total_next = tot_next + (prev >= 0 && prev == next ? 1u : 0u) - (oa == next ? 1u : 0u);
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(&sp);
        ulonglong2* dst = reinterpret_cast<ulonglong2*>(P.spec);
        for (int k = 0; k < 3; ++k) dst[k] = src[k];  // (16-byte stores: each word with its seq)
    }
    __syncthreads();  // (every thread's spec_hop stores before the release)
    if (tid == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&C->svc_b_seq), "l"(a.seq) : "memory");
        P.dbg[blockIdx.x * 16 + 9] = gtimer();
    }
}

// CTA 0: commits the learner service's observe(AgentDispatch{prev, next}) for a request that
// starts, exactly as observe_dispatch would have applied it: TransitionLearner::record (the
// count cells and the window ring, transition_learner.cpp:22-51), the rebuilt hops when the agent
// changed, and the prefetch gate (cachesage_policy.cpp:109-123).
__device__ void commit_observe(const DevPool& P, const AdmitArgs& a, unsigned long long tick, AdmSmem& A,
                               unsigned char* cls_smem) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x;
    const long long W = P.window;
    const int Acap = P.a_cap, prev = a.prev, next = a.next, n_agents = a.n_agents;
    __shared__ __align__(16) LearnSpec sp;
    // one round of 16-byte loads: the result and the hops, each word tagged with its admission;
    // only a service that has not finished yet costs a wait (then the words are read again)
    const int nw = (n_agents + 7) / 8;
    ulonglong2 hw = make_ulonglong2(0ull, 0ull);
    for (unsigned long long spins = 0;; ++spins) {
        int ok = 1;
        if (tid < 3) {
            const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(P.spec) + tid);
            reinterpret_cast<ulonglong2*>(&sp)[tid] = v;
            ok = v.x == a.seq;
        } else if (tid - 3 < nw && tid - 3 < kMaxAgents / 8) {
            hw = __ldcg(P.spec_hop + (tid - 3));
        }
        // (the hops are this admission's only if the BFS ran: checked once `changed` is known)
        if (__syncthreads_and(ok)) {
            const int need_hops = sp.changed;
            if (!need_hops || __syncthreads_and(!(tid >= 3 && tid - 3 < nw) || hw.x == a.seq)) break;
        }
        if (++spins > 64) __nanosleep(100);
        if (spins > (1ull << 28)) trap_at(101);
    }
    pstamp(P, 13);
    if (sp.changed && tid >= 3 && tid - 3 < nw) {
        const int w = tid - 3;
        for (int k = 0; k < 8 && w * 8 + k < n_agents; ++k) {
            const unsigned char h = (unsigned char)(hw.y >> (8 * k));
            P.hop[w * 8 + k] = h;
            P.cls[w * 8 + k] = h;
            if (cls_smem) cls_smem[w * 8 + k] = h;
        }
    }
    if (tid == 0) {
        if (prev >= 0) {  // record: fire-and-forget count updates, the window ring
            const long long head = A.pf_head, size = A.pf_size;
            atomicAdd(&C->recorded, 1ull);
            atomicAdd(&P.counts[(long long)prev * Acap + next], 1u);
            atomicAdd(&P.totals[prev], 1u);
            if (size == W) {
                P.win_a[head] = prev;
                P.win_b[head] = next;
                atomicSub(&P.counts[(long long)sp.oa * Acap + sp.ob], 1u);
                atomicSub(&P.totals[sp.oa], 1u);
                C->win_head = head + 1 == W ? 0 : head + 1;
            } else {
                const long long pos = (head + size) % W;
                P.win_a[pos] = prev;
                P.win_b[pos] = next;
                C->win_size = size + 1;
            }
        }
        C->cur_agent = next;
        if (sp.changed) {
            atomicAdd(&C->rebuilds, 1ull);
            C->reach_built = 1;
        }
        // maybe_prefetch on argmax_row(next) of the recorded learner
        const unsigned int total = sp.total_next;
        if (C->step_warmups < P.budget_per_step && (unsigned long long)total >= P.min_row && total > 0u &&
            sp.best_b >= 0) {
            const double p = __ddiv_rn((double)sp.best_c, (double)total);
            if (!(p < P.min_conf)) {
                C->step_warmups += 1;
                if (C->n_pend < kMaxPending) {
                    C->pend_target[C->n_pend] = sp.best_b;
                    C->pend_tick[C->n_pend] = tick;
                    C->n_pend += 1;
                }
                A.warm_issued = sp.best_b;
            }
        }
    }
    __syncthreads();
    pstamp(P, 14);
}

// ------------------------------------------------------------------ K4: the pool scan

__device__ __forceinline__ int keep_of(int l, int NL, int keep) { return l == NL - 1 ? keep + 1 : keep; }

// Per list: keep the keep_l smallest staged entries (exact select), tighten the list's bound,
// publish it grid-wide, and compact the staging pool.
// Small staging pools: rank of each entry among the same list's entries (ticks are distinct),
// O(m^2 / threads) compares and no multi-pass barriers. The entry of rank keep_l - 1 is the
// list's new bound; entries of rank < keep_l survive.
constexpr int kRankSelectMax = 768;

__device__ void stage_flush_rank(const DevPool& P, int NL, int keep, const ScanBufs& B, ScanSmem& S,
                                 bool final_flush) {
    const int tid = threadIdx.x, T = blockDim.x;
    const int m = S.count;
    if (tid == 0) S.side_n = 0;
    __syncthreads();
    for (int j0 = 0; j0 < m; j0 += T) {
        const int j = j0 + tid;
        bool keep_it = false;
        unsigned char l = 0;
        unsigned long long x = 0;
        if (j < m) {
            l = B.st_list[j];
            x = B.st_lt[j];
            int r = 0;
            for (int k = 0; k < m; ++k) r += (B.st_list[k] == l) & (B.st_lt[k] < x);
            const int kl = keep_of(l, NL, keep);
            keep_it = r < kl;
            if (r == kl - 1) {  // exactly kl entries of list l are <= x: a valid bound
                if (x < S.thr[l]) S.thr[l] = x;
                atomicMin(P.gbound + l, x);
                if (final_flush) atomicMax(P.gmaxk + l, x);  // next scan's hint
            }
        }
        const unsigned int ball = __ballot_sync(0xffffffffu, keep_it);
        int base = 0;
        if (lane_id() == 0 && ball) base = atomicAdd(&S.side_n, __popc(ball));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep_it) {
            const int p = base + __popc(ball & ((1u << lane_id()) - 1u));
            B.sd_lt[p] = x;
            B.sd_slot[p] = B.st_slot[j];
            B.sd_list[p] = l;
        }
    }
    __syncthreads();
    const int n2 = S.side_n;
    for (int j = tid; j < n2; j += T) {
        B.st_lt[j] = B.sd_lt[j];
        B.st_slot[j] = B.sd_slot[j];
        B.st_list[j] = B.sd_list[j];
    }
    __syncthreads();
    if (tid == 0) S.count = n2;
    __syncthreads();
}

__device__ void stage_flush(const DevPool& P, int NL, int keep, const ScanBufs& B, ScanSmem& S, SelectSmem& Sel,
                            bool final_flush) {
    const int tid = threadIdx.x, T = blockDim.x;
    const int m = S.count;
    const unsigned long long t_in = tid == 0 ? gtimer() : 0ull;
    if (m <= kRankSelectMax) {
        stage_flush_rank(P, NL, keep, B, S, final_flush);
        if (tid == 0) {
            S.flush_ns += gtimer() - t_in;
            S.flushes += 1;
        }
        return;
    }
    if (tid < NL) S.lcnt[tid] = 0;
    __syncthreads();
    for (int j0 = 0; j0 < m; j0 += T) {  // per-list counts, aggregated per warp (match_any)
        const int j = j0 + tid;
        const unsigned int act = __ballot_sync(0xffffffffu, j < m);
        if (j < m) {
            const unsigned int tg = B.st_list[j];
            const unsigned int peers = __match_any_sync(act, tg);
            if (lane_id() == __ffs(peers) - 1) atomicAdd(&S.lcnt[tg], __popc(peers));
        }
    }
    __syncthreads();
    for (int l = 0; l < NL; ++l) {
        const int kl = keep_of(l, NL, keep);
        if (S.lcnt[l] >= kl && (S.lcnt[l] > kl || final_flush)) {
            const unsigned long long v = block_kth(B.st_lt, B.st_list, (unsigned char)l, m, kl, Sel);
            if (tid == 0) {
                if (v < S.thr[l]) S.thr[l] = v;
                atomicMin(P.gbound + l, v);
                if (final_flush) atomicMax(P.gmaxk + l, v);  // next scan's hint
            }
        }
    }
    if (tid == 0) S.side_n = 0;
    __syncthreads();
    for (int j0 = 0; j0 < m; j0 += T) {  // compaction of the survivors, one atomic per warp
        const int j = j0 + tid;
        bool keep_it = false;
        unsigned char l = 0;
        unsigned long long x = 0;
        if (j < m) {
            l = B.st_list[j];
            x = B.st_lt[j];
            keep_it = x <= S.thr[l];
        }
        const unsigned int ball = __ballot_sync(0xffffffffu, keep_it);
        int base = 0;
        if (lane_id() == 0 && ball) base = atomicAdd(&S.side_n, __popc(ball));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep_it) {
            const int p = base + __popc(ball & ((1u << lane_id()) - 1u));
            B.sd_lt[p] = x;
            B.sd_slot[p] = B.st_slot[j];
            B.sd_list[p] = l;
        }
    }
    __syncthreads();
    const int n2 = S.side_n;
    for (int j = tid; j < n2; j += T) {
        B.st_lt[j] = B.sd_lt[j];
        B.st_slot[j] = B.sd_slot[j];
        B.st_list[j] = B.sd_list[j];
    }
    __syncthreads();
    if (tid == 0) {
        S.count = n2;
        S.flush_ns += gtimer() - t_in;
        S.flushes += 1;
    }
    __syncthreads();
}

// ---- TMA (cp.async.bulk) + mbarrier helpers for the SoA stream
__device__ __forceinline__ unsigned int smem_u32(const void* p) { return (unsigned int)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned int bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned int parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)),
        "r"(parity)
        : "memory");
}

// Cross-proxy ordering for the TMA stream, global and shared: (1) the pool slots the previous
// admission wrote with generic stores (on CTA 0, made visible by a grid barrier or a kernel
// boundary) must be what the async-proxy bulk reads see; (2) this CTA's earlier generic accesses
// to the ring (which doubles as the replay view, the prescan select buffer and the scheduler's
// staging area) must precede the async-proxy writes into it. Issued after a __syncthreads.
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async;" ::: "memory"); }

// 1-D bulk copy global -> this CTA's shared memory, completion counted on mbarrier m. The pool
// stream is read once per pass: it is marked evict-first in L2, so it does not flush the small
// hot state CTA 0's serial chain works on (block table entries, prescan lists, learner).
__device__ __forceinline__ unsigned long long l2_evict_first() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, unsigned int bytes, unsigned long long* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(m))
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned int bytes, unsigned long long* m) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(m)), "l"(l2_evict_first())
        : "memory");
}

// One streaming pass over this CTA's contiguous slot range: one 8-B packed word per slot, read once.
// The SoA arrives through a kRing-stage TMA ring (cp.async.bulk into shared memory, one
// elected thread issues, mbarrier transaction counts complete), so kRing-1 tiles of 16 KiB
// are in flight independently of the threads' progress and no registers hold in-flight data.
// Survivors go to a staging pool flushed (exact per-list select) only when it could overflow.
__device__ __forceinline__ void mbar_arrive(unsigned long long* m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(m)) : "memory");
}

// Classifies this thread's 4 slots of the current tile. Bit k: resident-oldest list R; bit
// 4+k: survival-class list cl[k] (unpinned only). Thresholds are < kFreeTick, so free slots
// never pass a compare. Branch-free except for agent-carrying slots (rare in real pools).
__device__ __forceinline__ unsigned int classify4(const unsigned long long (&x4)[kV], const unsigned int (&a4)[kV],
                                                  const unsigned int (&r4)[kV], unsigned long long thrR,
                                                  unsigned long long thrE, volatile unsigned long long* thr,
                                                  const unsigned char* cls, int E, int (&cl)[kV]) {
    unsigned int acc = 0u;
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const unsigned long long x = x4[k];
        acc |= (unsigned int)(x <= thrR) << k;
        cl[k] = E;
        if (a4[k] == kNoAgent) {
            acc |= (unsigned int)(r4[k] == 0u && x <= thrE) << (kV + k);
        } else if (r4[k] == 0u) {
            const int c = cls[a4[k]];
            cl[k] = c;
            acc |= (unsigned int)(x <= thr[c]) << (kV + k);
        }
    }
    return acc;
}

// Warp-aggregated append of the accepted entries (one shared atomic per warp). Returns the last
// reserved position (-1: none). With `bounded`, a reservation past the staging capacity sets
// S.overflow and writes nothing (the fast pass is then redone in safe mode).
__device__ __forceinline__ int append4(unsigned int acc, const unsigned long long (&x4)[kV], const int (&cl)[kV],
                                       long long i0, int R, const ScanBufs& B, ScanSmem& S, bool bounded) {
    if (!__any_sync(0xffffffffu, acc != 0u)) return -1;
    const int mine = __popc(acc);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane_id() >= o) incl += v;
    }
    const int wtot = __shfl_sync(0xffffffffu, incl, 31);
    int base = 0;
    if (lane_id() == 31) base = atomicAdd(&S.count, wtot);
    base = __shfl_sync(0xffffffffu, base, 31);
    if (bounded && base + wtot > kStage) {
        // this warp's reservation [base, base + wtot) stays unwritten, and so does every later
        // one: only [0, ovf_base) holds staged entries
        if (lane_id() == 31) atomicMin(&S.ovf_base, base);
        S.overflow = 1;
        return kStage;
    }
    int p = base + incl - mine;
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        if (acc & (1u << k)) {
            B.st_lt[p] = x4[k];
            B.st_slot[p] = (unsigned int)(i0 + k);
            B.st_list[p] = (unsigned char)R;
            ++p;
        }
        if (acc & (1u << (kV + k))) {
            B.st_lt[p] = x4[k];
            B.st_slot[p] = (unsigned int)(i0 + k);
            B.st_list[p] = (unsigned char)cl[k];
            ++p;
        }
    }
    return base + wtot - 1;
}

// Reads this thread's 4 slots of ring stage `st` (kFreeTick / no agent / pinned when the
// thread has no slots in the tile).
__device__ __forceinline__ void read4(const unsigned char* st, int tid, bool valid, unsigned long long (&x4)[kV],
                                      unsigned int (&a4)[kV], unsigned int (&r4)[kV]) {
    if (valid) {
        const ulonglong2 w01 = *reinterpret_cast<const ulonglong2*>(st + (size_t)tid * 32);
        const ulonglong2 w23 = *reinterpret_cast<const ulonglong2*>(st + (size_t)tid * 32 + 16);
        pk_decode(w01.x, x4[0], a4[0], r4[0]);
        pk_decode(w01.y, x4[1], a4[1], r4[1]);
        pk_decode(w23.x, x4[2], a4[2], r4[2]);
        pk_decode(w23.y, x4[3], a4[3], r4[3]);
    } else {
#pragma unroll
        for (int k = 0; k < kV; ++k) {
            x4[k] = kFreeTick;
            a4[k] = kNoAgent;
            r4[k] = 1u;
        }
    }
}

// ---- the unpin ranges of a launch as one flat index space: every thread loads its own entry,
// so a launch's ranges cost one round of loads instead of one per range
__device__ __forceinline__ int unpin_total(const AdmitArgs& a, bool with_prev) {
    int t = 0;
#pragma unroll
    for (int r = 0; r < kMaxUnpinRanges; ++r) t += r < a.n_unpin_ranges ? a.unpin_n[r] : 0;
    if (with_prev) {
#pragma unroll
        for (int r = 0; r < kMaxUnpinRanges + 1; ++r) t += r < a.n_prev_ranges ? a.prev_n[r] : 0;
    }
    return t;
}

__device__ __forceinline__ unsigned int unpin_at(const AdmitArgs& a, int i) {
#pragma unroll
    for (int r = 0; r < kMaxUnpinRanges; ++r) {
        if (r < a.n_unpin_ranges) {
            if (i < a.unpin_n[r]) return a.unpin_ptr[r][i];
            i -= a.unpin_n[r];
        }
    }
#pragma unroll
    for (int r = 0; r < kMaxUnpinRanges + 1; ++r) {
        if (r < a.n_prev_ranges) {
            if (i < a.prev_n[r]) return a.prev_ptr[r][i];
            i -= a.prev_n[r];
        }
    }
    return kNoSlot;
}

// The same 4 slots straight from global memory (L2, 128-bit loads): the persistent engine kernel
// streams this way (kFreeTick / no agent / pinned past the range end).
__device__ __forceinline__ void load4(const DevPool& P, long long i0, bool valid, unsigned long long (&x4)[kV],
                                      unsigned int (&a4)[kV], unsigned int (&r4)[kV]) {
    if (valid) {
        const ulonglong2 w01 = __ldcg(reinterpret_cast<const ulonglong2*>(P.pk + i0));
        const ulonglong2 w23 = __ldcg(reinterpret_cast<const ulonglong2*>(P.pk + i0 + 2));
        pk_decode(w01.x, x4[0], a4[0], r4[0]);
        pk_decode(w01.y, x4[1], a4[1], r4[1]);
        pk_decode(w23.x, x4[2], a4[2], r4[2]);
        pk_decode(w23.y, x4[3], a4[3], r4[3]);
    } else {
#pragma unroll
        for (int k = 0; k < kV; ++k) {
            x4[k] = kFreeTick;
            a4[k] = kNoAgent;
            r4[k] = 1u;
        }
    }
}

// ---- speculative pass support: the set of slots phase 0 may change (the prompt's resident
// blocks, touched by lookup / pinned by admit_pinned, and the slots unpinned first) and the
// deferred classification of agent-carrying slots (the BFS of phase 0 may move them).
__device__ __forceinline__ unsigned int xhash(unsigned int s) { return (s * 2654435761u) >> 22; }  // 10 bits

__device__ __forceinline__ bool xset_insert(ScanSmem& S, unsigned int s) {
    unsigned int h = xhash(s);
    for (int c = 0; c < kXset; ++c) {
        const unsigned int old = atomicCAS(&S.xset[h], kNoSlot, s);
        if (old == kNoSlot) return true;
        if (old == s) return false;
        h = (h + 1) & (kXset - 1);
    }
    return false;  // unreachable: at most kXsetMax entries
}

// The same, returning the hash position of a newly inserted slot (-1: already present).
__device__ __forceinline__ int xset_insert_pos(ScanSmem& S, unsigned int s) {
    unsigned int h = xhash(s);
    for (int c = 0; c < kXset; ++c) {
        const unsigned int old = atomicCAS(&S.xset[h], kNoSlot, s);
        if (old == kNoSlot) return (int)h;
        if (old == s) return -1;
        h = (h + 1) & (kXset - 1);
    }
    return -1;  // unreachable: at most kXsetMax entries
}

__device__ __forceinline__ bool xset_has(const ScanSmem& S, unsigned int s) {
    unsigned int h = xhash(s);
    for (int c = 0; c < kXset; ++c) {
        const unsigned int k = S.xset[h];
        if (k == s) return true;
        if (k == kNoSlot) return false;
        h = (h + 1) & (kXset - 1);
    }
    return false;
}

// All threads, after this launch's phase 0: the slots it may have changed, from the prompt
// slots CTA 0 probed (P.p_slot) and the unpin list.
__device__ void build_xset(const DevPool& P, const AdmitArgs& a, ScanSmem& S) {
    const int tid = threadIdx.x, T = blockDim.x;
    for (int j = tid; j < kXset; j += T) S.xset[j] = kNoSlot;
    __syncthreads();
    for (int i = tid; i < a.n; i += T) {
        const unsigned int s = __ldcg(P.p_slot + i);
        if (s != kNoSlot) xset_insert(S, s);
    }
    const int nu = unpin_total(a, false);
    for (int i = tid; i < nu; i += T) {
        const unsigned int us = unpin_at(a, i);
        if (us != kNoSlot) xset_insert(S, us);
    }
    __syncthreads();
}


// All threads of a scanning CTA, before its first flush (no bound has used a staged entry
// yet): waits for this launch's phase 0, loads the survival classes it fixed, drops the staged
// entries of slots phase 0 may have changed (CTA 0 restages those with their new state) and
// classifies the staged agent-carrying entries (phase 0 never changes a slot's agent).
__device__ void ensure_cls(const DevPool& P, const AdmitArgs& a, const ScanBufs& B, ScanSmem& S) {
    if (!S.spec || S.cls_ready) return;
    const int tid = threadIdx.x, T = blockDim.x;
    if (!S.prep_done) {
        if (tid == 0) {
            unsigned long long spins = 0;
            while (ld_acquire_u64(&P.ctrl->p0_seq) != a.seq) {
                if (++spins > 1024) __nanosleep(128);
                if (spins > (1ull << 27)) trap_at(102);
            }
        }
        __syncthreads();
        for (int x = tid; x < a.n_agents; x += T) B.cls[x] = __ldcg(P.cls + x);
        build_xset(P, a, S);
    }
    // Relabel, then drop (a) entries of the change set and (b) relabelled entries above their
    // class's bound: every staged entry then satisfies the bound its list would have applied,
    // which the hint check of finalize_list relies on. In-place compaction: the holes below the
    // new count are filled from the survivors above it.
    constexpr unsigned char kDrop = 0xFF;
    const int m = S.count;
    if (tid == 0) {
        S.side_n = 0;
        S.hc = 0;
        S.dc = 0;
    }
    __syncthreads();
    int dropped = 0;
    for (int j = tid; j < m; j += T) {
        const unsigned int sl = B.st_slot[j];
        unsigned char l = B.st_list[j];
        bool keep_it = !xset_has(S, sl);
        if (keep_it && l == kPend) l = B.cls[P.agent[sl]];
        if (keep_it && B.st_lt[j] > S.thr[l]) keep_it = false;
        B.st_list[j] = keep_it ? l : kDrop;
        dropped += keep_it ? 0 : 1;
    }
    dropped = __reduce_add_sync(0xffffffffu, dropped);
    if (lane_id() == 0 && dropped) atomicAdd(&S.side_n, dropped);
    __syncthreads();
    const int n2 = m - S.side_n;
    unsigned int* holes = reinterpret_cast<unsigned int*>(B.sd_lt);  // <= m / 2 each
    unsigned int* donors = holes + kSide;
    for (int j = tid; j < m; j += T) {
        const bool d = B.st_list[j] == kDrop;
        if (j < n2 && d) holes[atomicAdd(&S.hc, 1)] = (unsigned int)j;
        if (j >= n2 && !d) donors[atomicAdd(&S.dc, 1)] = (unsigned int)j;
    }
    __syncthreads();
    for (int i = tid; i < S.hc; i += T) {
        const unsigned int h = holes[i], d = donors[i];
        B.st_lt[h] = B.st_lt[d];
        B.st_slot[h] = B.st_slot[d];
        B.st_list[h] = B.st_list[d];
    }
    __syncthreads();
    if (tid == 0) {
        S.count = n2;
        S.cls_ready = 1;
    }
    __syncthreads();
}

// The producer warp of a fast speculative pass, once it has issued every tile: waits for phase
// 0, publishes the new survival classes to the consumers (a consumer that reads a class from
// now on stages the slot under it; earlier reads left kPend) and builds the change set, so the
// tail of the pass only filters.
__device__ void producer_prep(const DevPool& P, const AdmitArgs& a, const ScanBufs& B, ScanSmem& S) {
    const int lane = lane_id();
    if (lane == 0) {
        unsigned long long spins = 0;
        while (ld_acquire_u64(&P.ctrl->p0_seq) != a.seq) {
            if (++spins > 1024) __nanosleep(128);
            if (spins > (1ull << 27)) trap_at(103);
        }
    }
    __syncwarp();
    for (int x = lane; x < a.n_agents; x += 32) B.cls[x] = __ldcg(P.cls + x);
    for (int j = lane; j < kXset; j += 32) S.xset[j] = kNoSlot;
    __syncwarp();
    for (int i = lane; i < a.n; i += 32) {
        const unsigned int sl = __ldcg(P.p_slot + i);
        if (sl != kNoSlot) xset_insert(S, sl);
    }
    const int nu = unpin_total(a, false);
    for (int i = lane; i < nu; i += 32) {
        const unsigned int us = unpin_at(a, i);
        if (us != kNoSlot) xset_insert(S, us);
    }
    __syncwarp();
    if (lane == 0) S.prep_done = 1;
}

// One streaming pass over this CTA's contiguous slot range: one 8-B packed word per slot, read once.
// The SoA arrives through a kRing-stage TMA ring (cp.async.bulk into shared memory, mbarrier
// transaction counts), so the loads are independent of the threads' progress.
//   fast: warp-specialized. A producer warp refills a stage as soon as the 16 consumer warps
//         release it (per-stage "empty" mbarriers); no CTA-wide barrier per tile. Used when
//         every list has a hint (or is known small), so survivors fit the staging pool; an
//         overflow aborts the pass and the caller redoes it in safe mode.
//   safe: one CTA barrier per tile decides whether the staging pool must be flushed (exact
//         per-list select) before it could overflow; any threshold state works.
//   spec: (either of the above) runs while CTA 0 is still in phase 0; see ensure_cls.
// Returns with S.overflow set when a fast pass overflowed.
__device__ void scan_pass(const DevPool& P, int NL, int keep, const ScanBufs& B, ScanSmem& S, SelectSmem& Sel,
                          unsigned char* dsm, bool fast, const AdmitArgs& a) {
    const int tid = threadIdx.x;
    const long long TV = kTile;  // consumer threads (kThreads) x kV slots
    // speculative pass: CTA 0 runs phase 0 and restages the change set instead of a range
    const bool spec = S.spec != 0;
    const int nscan = spec ? (int)gridDim.x - 1 : (int)gridDim.x;
    const int me = spec ? (int)blockIdx.x - 1 : (int)blockIdx.x;
    long long per = (P.cap_scan + nscan - 1) / nscan;
    per = (per + kV - 1) / kV * kV;
    const long long lo = me < 0 ? 0 : min(P.cap_scan, (long long)me * per);
    const long long hi = me < 0 ? 0 : min(P.cap_scan, lo + per);  // multiple of 4 slots: 16-B granules
    const int ntiles = (int)((hi - lo + TV - 1) / TV);
    const int R = NL - 1;
    const int E = P.e_max;  // class of agentless / unreachable blocks (survival 0)
    const unsigned char* cls = B.cls;
    unsigned char* ring = dsm + kOffRing;
    if (tid < NL) {
        // start from the previous scan's hint: no accept-everything warm-up tiles
        const unsigned long long h = P.ghint[tid];
        S.hint[tid] = h;
        S.thr[tid] = min(ld_relaxed_u64(P.gbound + tid), h);
    }
    if (tid == 0) {
        S.count = 0;
        S.overflow = 0;
        S.ovf_base = kStage;
        S.prep_done = 0;
        S.flush_ns = 0;
        S.flushes = 0;
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&S.mbar[s], 1u);
            mbar_init(&S.mbar_empty[s], (unsigned int)(kThreads / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    fence_proxy_async_smem();
    if (tid == 0) {  // an unclassified agent slot may land in any survival class
        unsigned long long m = 0ull;
        for (int c = 0; c + 1 < NL; ++c) m = max(m, S.thr[c]);
        S.thr[kPend] = m;
    }
    __syncthreads();
    auto issue = [&](int t) {  // one elected thread
        const int s = t % kRing;
        const long long b0 = lo + (long long)t * TV;
        const unsigned int nsl = (unsigned int)min(TV, hi - b0);
        unsigned char* st = ring + (size_t)s * kRingStage;
        mbar_expect_tx(&S.mbar[s], nsl * 8u);
        bulk_g2s(st, P.pk + b0, nsl * 8u, &S.mbar[s]);  // the packed scan words
    };
    if (tid == 0) {
        P.dbg[blockIdx.x * 16 + 0] = gtimer();
        P.dbg[blockIdx.x * 16 + 7] = clock64();
    }
    volatile unsigned long long* thr = S.thr;
    const bool consumer = tid < kThreads;

    if (fast && !P.stream_generic) {
        if (!consumer) {  // producer warp
            if (lane_id() == 0) {
                for (int t = 0; t < ntiles; ++t) {
                    const int s = t % kRing;
                    if (t >= kRing) mbar_wait(&S.mbar_empty[s], (unsigned int)(((t / kRing) - 1) & 1));
                    issue(t);
                }
            }
            __syncwarp();
            if (spec && !S.cls_ready) producer_prep(P, a, B, S);
        } else {
            unsigned long long gbn = ~0ull;
            for (int t = 0; t < ntiles; ++t) {
                const int s = t % kRing;
                if (tid < NL && s == 0) {  // grid-wide bounds: refreshed every kRing tiles, applied a round later
                    if (gbn < thr[tid]) thr[tid] = gbn;
                    gbn = ld_relaxed_u64(P.gbound + tid);
                }
                const long long i0 = lo + (long long)t * TV + (long long)tid * kV;
                const unsigned char* st = ring + (size_t)s * kRingStage;
                mbar_wait(&S.mbar[s], (unsigned int)((t / kRing) & 1));
                // classify the packed words as they sit in the stage (no decode; thresholds
                // clamped below the free tick, so a free slot never passes a compare)
                const ulonglong2 w01 = *reinterpret_cast<const ulonglong2*>(st + (size_t)tid * 32);
                const ulonglong2 w23 = *reinterpret_cast<const ulonglong2*>(st + (size_t)tid * 32 + 16);
                __syncwarp();
                if (lane_id() == 0) mbar_arrive(&S.mbar_empty[s]);  // stage s consumed by this warp
                const unsigned long long w[kV] = {w01.x, w01.y, w23.x, w23.y};
                const unsigned long long cR = min(thr[R], kPkFree - 1ull), cE = min(thr[E], kPkFree - 1ull);
                unsigned long long x4[kV];
                int cl[kV];
                unsigned int acc = 0u;
#pragma unroll
                for (int k = 0; k < kV; ++k) {
                    const unsigned long long x = w[k] & kPkLtMask;
                    const unsigned int ag = (unsigned int)((w[k] >> 40) & kPkNoAgent);
                    x4[k] = x;
                    cl[k] = E;
                    acc |= (unsigned int)(x <= cR) << k;
                    if ((long long)w[k] >= 0) {  // unpinned
                        if (ag == (unsigned int)kPkNoAgent) {
                            acc |= (unsigned int)(x <= cE) << (kV + k);
                        } else {  // agent-carrying (rare in real pools)
                            const int c = cls[ag];
                            cl[k] = c;
                            acc |= (unsigned int)(x <= min(thr[c], kPkFree - 1ull)) << (kV + k);
                        }
                    }
                }
                if (i0 + kV > hi) acc = 0u;
                append4(acc, x4, cl, i0, R, B, S, true);
            }
        }
        __syncthreads();
        if (S.overflow) {
            if (tid == 0) atomicExch(&P.ctrl->rescan, 1);
            return;  // the caller redoes this pass in safe mode
        }
    } else {
        if (tid == 0 && !P.stream_generic)
            for (int t = 0; t < kRing && t < ntiles; ++t) issue(t);
        unsigned long long gbn = ~0ull;
        for (int t = 0; t < ntiles; ++t) {
            const int s = t % kRing;
            if (tid < NL && s == 0) {
                if (gbn < thr[tid]) thr[tid] = gbn;
                gbn = ld_relaxed_u64(P.gbound + tid);
            }
            const long long i0 = lo + (long long)t * TV + (long long)tid * kV;
            const unsigned char* st = ring + (size_t)s * kRingStage;
            unsigned long long x4[kV];
            unsigned int a4[kV], r4[kV];
            if (P.stream_generic) {
                load4(P, i0, consumer && i0 + kV <= hi, x4, a4, r4);
            } else {
                mbar_wait(&S.mbar[s], (unsigned int)((t / kRing) & 1));
                read4(st, tid, consumer && i0 + kV <= hi, x4, a4, r4);
            }
            int cl[kV];
            unsigned int acc = classify4(x4, a4, r4, thr[R], thr[E], thr, cls, E, cl);
            const int maxpos = append4(acc, x4, cl, i0, R, B, S, false);
            // every thread is done with stage s: refill it with tile t + kRing
            const int need_flush = __syncthreads_or(maxpos >= kFlushAt);
            if (tid == 0 && t + kRing < ntiles && !P.stream_generic) issue(t + kRing);
            if (need_flush) {
                ensure_cls(P, a, B, S);
                stage_flush(P, NL, keep, B, S, Sel, false);
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        P.dbg[blockIdx.x * 16 + 1] = gtimer();
        P.dbg[blockIdx.x * 16 + 5] = S.count;
        P.dbg[blockIdx.x * 16 + 6] = clock64() - P.dbg[blockIdx.x * 16 + 7];  // SM cycles of the stream
        P.dbg[blockIdx.x * 16 + 8] = fast ? 1 : 0;
    }
    if (spec && blockIdx.x == 0) {
        // CTA 0 (after its phase 0): the change set with its post-phase-0 state, unfiltered
        for (int j = tid; j < kXset; j += blockDim.x) {
            const unsigned int sl = S.xset[j];
            if (sl == kNoSlot) continue;
            const unsigned long long x = P.lt[sl];
            if (x == kFreeTick) continue;
            const unsigned int ag = P.agent[sl];
            const int c = ag == kNoAgent ? E : B.cls[ag];
            // the same bounds the scanning CTAs apply (finalize_list's hint check needs them)
            const bool in_r = x <= S.thr[R];
            const bool in_c = P.refs[sl] == 0u && x <= S.thr[c];
            if (!in_r && !in_c) continue;
            int p = atomicAdd(&S.count, (in_r ? 1 : 0) + (in_c ? 1 : 0));
            if (in_r) {
                B.st_lt[p] = x;
                B.st_slot[p] = sl;
                B.st_list[p] = (unsigned char)R;
                ++p;
            }
            if (in_c) {
                B.st_lt[p] = x;
                B.st_slot[p] = sl;
                B.st_list[p] = (unsigned char)c;
            }
        }
        __syncthreads();
    }
    if (S.count > 0) {
        ensure_cls(P, a, B, S);
        stage_flush(P, NL, keep, B, S, Sel, true);
    }
    if (tid == 0) P.dbg[blockIdx.x * 16 + 2] = gtimer();
    // publish this CTA's survivors that can still be among the global keep smallest
    if (tid < NL) {
        S.gbw[tid] = ld_relaxed_u64(P.gbound + tid);
        S.wcnt[tid] = 0;
        S.wpos[tid] = 0;
        S.lmin[tid] = kNoBound;
    }
    __syncthreads();
    const int m = S.count;
    const int T = blockDim.x;
    for (int j = tid; j < m; j += T) {
        const unsigned char l = B.st_list[j];
        atomicMin(&S.lmin[l], B.st_lt[j]);
        if (B.st_lt[j] <= S.gbw[l]) atomicAdd(&S.wcnt[l], 1);
    }
    __syncthreads();
    if (tid < NL) {
        S.wbase[tid] = S.wcnt[tid] ? atomicAdd(P.gcount + tid, S.wcnt[tid]) : 0;
        // this CTA's smallest candidate: the select bound is the keep-th smallest CTA minimum
        P.gmin[(long long)tid * gridDim.x + blockIdx.x] = S.lmin[tid];
    }
    __syncthreads();
    for (int j = tid; j < m; j += T) {
        const unsigned char l = B.st_list[j];
        const unsigned long long x = B.st_lt[j];
        if (x <= S.gbw[l]) {
            const long long o = (long long)l * P.gcap + S.wbase[l] + atomicAdd(&S.wpos[l], 1);
            P.gbuf_lt[o] = x;
            P.gbuf_slot[o] = B.st_slot[j];
        }
    }
    __syncthreads();
    if (tid == 0) P.dbg[blockIdx.x * 16 + 3] = gtimer();
}

// ------------------------------------------------------------------ K5a: exact per-list select

constexpr int kDirectRank = 384;  // finalize_list ranks up to this many candidates directly

// One thread: list l holds n sorted entries; hint bookkeeping for the next scan.
// The next scan's hint for a full list: the largest per-CTA keep-th value (mk). A list no CTA
// had to truncate (mk == 0: every CTA held fewer than keep of its members) is "small": the next
// fast pass stages all of its members (a staging overflow sends it to a safe rescan).
__device__ __forceinline__ void finish_list(const DevPool& P, int l, int n, int kl, unsigned long long hmax) {
    P.fin_n[l] = n;
    // Hint verification. Hints are only carried for lists that were full (n == keep) in the previous scan; a
    // hinted list that now comes up short may be missing members above its hint.
    const bool hinted = P.ghint[l] < kNoBound;
    if (n < kl && hinted) atomicExch(&P.ctrl->rescan, 1);
    const unsigned long long mk = *(volatile unsigned long long*)(P.gmaxk + l);
    P.ghint[l] = (n == kl && mk) ? mk : kNoBound;
    P.gsmall[l] = mk == 0ull ? 1 : 0;
    (void)hmax;
}

__device__ void finalize_list(const DevPool& P, int l, int NL, int keep, const ScanBufs& B, SelectSmem& Sel) {
    const int tid = threadIdx.x, T = blockDim.x;
    const int kl = keep_of(l, NL, keep);
    const int m = *(volatile int*)(P.gcount + l);
    const unsigned long long* g = P.gbuf_lt + (long long)l * P.gcap;
    const unsigned int* gs = P.gbuf_slot + (long long)l * P.gcap;
    // Pre-filter bound: the kl-th smallest of the CTAs' minima. At most kl CTAs can have a
    // minimum below the global kl-th smallest value v* (each such minimum is a distinct element
    // <= v*), so this bound is >= v* and keeps the whole answer, and at least kl written
    // candidates are <= it. It cuts the ~grid*kl written candidates to ~kl.
    const int G = gridDim.x;
    fstamp(P, 0);
    unsigned long long* mins = B.sd_lt;  // G <= kSide minima staged on chip
    if (tid == 0) {
        Sel.tmp = 0;
        Sel.prefix = kNoBound;
        Sel.hmax = 0ull;
    }
    for (int i = tid; i < G; i += T) mins[i] = P.gmin[(long long)l * G + i];
    __syncthreads();
    for (int i = tid; i < G; i += T) {
        const unsigned long long x = mins[i];
        if (x >= kNoBound) continue;  // that CTA had no candidate of this list
        int r = 0;
        for (int k = 0; k < G; ++k) r += mins[k] < x;  // CTA minima are distinct ticks
        if (r == kl - 1) Sel.prefix = x;
    }
    __syncthreads();
    fstamp(P, 1);
    const unsigned long long fb = Sel.prefix;
    // stage the filtered candidates on chip when they fit (the common case), else select from L2
    unsigned long long hm = 0ull;
    for (int j = tid; j < m; j += T) {
        const unsigned long long x = g[j];
        hm = max(hm, x);
        if (x <= fb) {
            const int p = atomicAdd(&Sel.tmp, 1);
            if (p < kStage) {
                B.st_lt[p] = x;
                B.st_slot[p] = gs[j];
            }
        }
    }
    for (int o = 16; o; o >>= 1) hm = max(hm, __shfl_xor_sync(0xffffffffu, hm, o));
    if (lane_id() == 0 && hm) atomicMax(&Sel.hmax, hm);
    __syncthreads();
    fstamp(P, 2);
    const int mf = Sel.tmp;
    const bool local = mf <= kStage;
    const unsigned long long* src = local ? B.st_lt : g;
    const unsigned int* srs = local ? B.st_slot : gs;
    const int ms = local ? mf : m;
    __syncthreads();
    if (local && mf <= kDirectRank) {
        // few candidates (the common case): every entry's rank directly, one pass (distinct ticks)
        for (int j = tid; j < mf; j += T) {
            const unsigned long long x = src[j];
            const int r = count_below(src, mf, x);
            if (r < kl) {
                P.fin_lt[(long long)l * (kChunk + 2) + r] = x;
                P.fin_slot[(long long)l * (kChunk + 2) + r] = srs[j];
            }
        }
        fstamp(P, 3);
        if (tid == 0) finish_list(P, l, min(mf, kl), kl, Sel.hmax);
        __syncthreads();
        fstamp(P, 4);
        if (blockIdx.x == 0 && tid == 0) P.dbg[32 + 15] = (unsigned long long)mf | ((unsigned long long)m << 32);
        return;
    }
    unsigned long long v = ~0ull;
    if (ms > kl) v = block_kth(src, nullptr, 0, ms, kl, Sel);
    unsigned long long* t_lt = B.sd_lt;
    unsigned int* t_slot = B.sd_slot;
    if (tid == 0) Sel.tmp = 0;
    __syncthreads();
    for (int j = tid; j < ms; j += T) {
        const unsigned long long x = src[j];
        if (x <= v) {
            const int p = atomicAdd(&Sel.tmp, 1);
            t_lt[p] = x;
            t_slot[p] = srs[j];
        }
    }
    __syncthreads();
    const int n = Sel.tmp;
    // rank sort of the (at most keep + 1) survivors: distinct ticks, one barrier
    for (int j = tid; j < n; j += T) {
        const unsigned long long x = t_lt[j];
        const int r = count_below(t_lt, n, x);
        P.fin_lt[(long long)l * (kChunk + 2) + r] = x;
        P.fin_slot[(long long)l * (kChunk + 2) + r] = t_slot[j];
    }
    if (tid == 0) finish_list(P, l, n, kl, Sel.hmax);
    __syncthreads();
}

// ------------------------------------------------------------------ prescan (pipelined K4/K5a)
//
// CTAs 1..grid-1 of launch k run the scoring pass of admission k+1 while CTA 0 serves admission
// k (phase 0, replay, apply), so the pool stream overlaps the serial part of the step. The pass
// reads a pool that CTA 0 is changing, so its lists are validated by their consumer (CTA 0 of
// launch k+1, after its phase 0):
//   * an entry is valid iff its slot's last_touch is unchanged: every change of a slot's list
//     membership except an unpin also changes its last_touch (a touch, pin+touch, eviction or
//     reuse); unpinned slots (this and the previous launch's, the set U) are dropped and re-read;
//   * acceptance is by fixed thresholds, so list l holds EVERY member of the read state below
//     its completeness bound T_l; after validation it holds every member of the current state
//     below T_l (new members are younger than any read tick, or are in U);
//   * agent-carrying slots are kept whole (class unknown until the consumer's BFS), so the
//     class lists are the consumer's and the survival classes may change freely in between.
// A prescan that cannot stand in for a scan (overflow, a list too short, a non-bulk replay)
// makes its consumer scan as before; decisions are never taken from an invalid list.

__device__ __forceinline__ unsigned long long sat_add(unsigned long long a, unsigned long long b) {
    return (a > kNoBound - 1 - b) ? kNoBound : a + b;
}

// The next acceptance threshold of a list from its sorted kept entries: ~2x the rank reached
// (the front moves by about one admission of victims before the next prescan reads it). Any
// threshold is safe: it only sizes the candidate set; completeness is tracked per list.
__device__ __forceinline__ unsigned long long next_hint(unsigned long long v1, unsigned long long base) {
    if (base >= kNoBound || base < v1) return kNoBound;
    const unsigned long long span = base - v1;
    return sat_add(v1, sat_add(span, span));
}

// The same target (about 2 kPreK candidates next pass) from the density just below the kPreK-th
// value: the span of the upper half of the list, doubled past it. A list whose oldest entries are
// far older than the rest (old snapshot blocks ahead of recently unpinned ones) would make the
// v1-based estimate overshoot by orders of magnitude. Any hint is safe; it only sizes the pass.
__device__ __forceinline__ unsigned long long next_hint_mid(unsigned long long vmid, unsigned long long base) {
    if (base >= kNoBound || vmid >= kNoBound || base < vmid) return kNoBound;
    const unsigned long long span = base - vmid;
    return sat_add(base, sat_add(span, span));
}

__device__ void prescan_pass(const DevPool& P, const ScanBufs& B, ScanSmem& S, unsigned char* dsm, int par,
                             bool after_writes, unsigned long long seq) {
    const int tid = threadIdx.x, T = blockDim.x;
    const long long TV = kTile;
    const int nscan = (int)gridDim.x - kStream0, me = (int)blockIdx.x - kStream0;
    long long per = (P.cap_scan + nscan - 1) / nscan;
    per = (per + kV - 1) / kV * kV;
    const long long lo = min(P.cap_scan, (long long)me * per);
    const long long hi = min(P.cap_scan, lo + per);
    const int ntiles = (int)((hi - lo + TV - 1) / TV);
    unsigned char* ring = dsm + kOffRing;
    if (tid == 0) {
        S.count = 0;
        S.overflow = 0;
        S.ovf_base = kStage;
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&S.mbar[s], 1u);
            mbar_init(&S.mbar_empty[s], (unsigned int)(kThreads / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        P.dbg[blockIdx.x * 16 + 0] = gtimer();
    }
    __syncthreads();
    if (after_writes) fence_proxy_async_smem();  // pool slots written earlier in this launch
    // (the thresholds load while the first tiles are in flight) agent-carrying slots share E's
    // threshold: the E members among them are complete to it, and the other classes' lists are
    // only needed non-empty (see consume_svc). This launch's parity slot: the list service of the
    // previous launch wrote it, the one of this launch writes the other slot.
    const unsigned long long hE = __ldcg(P.pre_hint + par * 3 + 0), hR = __ldcg(P.pre_hint + par * 3 + 1), hP = hE;
    // list ids: 0 = E (agentless unpinned), 1 = R (resident), 2 = pending (agent, unpinned)
    auto classify_append = [&](const unsigned long long (&x4)[kV], const unsigned int (&a4)[kV],
                               const unsigned int (&r4)[kV], long long i0) {
        unsigned int acc = 0u;
        int cl[kV];
#pragma unroll
        for (int k = 0; k < kV; ++k) {
            const unsigned long long x = x4[k];
            acc |= (unsigned int)(x <= hR) << k;
            const bool agentless = a4[k] == kNoAgent;
            cl[k] = agentless ? 0 : 2;
            acc |= (unsigned int)(r4[k] == 0u && x <= (agentless ? hE : hP)) << (kV + k);
        }
        if (!S.overflow) append4(acc, x4, cl, i0, 1, B, S, true);
    };
    // The same classification straight on the packed words (the TMA stream's hot loop, issue-
    // bound): thresholds clamped below the free tick, so a free slot never passes a compare
    static_assert(kV == 4, "the packed consumer reads two 16-B vectors per thread");
    const unsigned long long cE = min(hE, kPkFree - 1ull), cR = min(hR, kPkFree - 1ull), cP = cE;
    auto classify_append_pk = [&](const ulonglong2 w01, const ulonglong2 w23, bool valid, long long i0) {
        const unsigned long long w[kV] = {w01.x, w01.y, w23.x, w23.y};
        unsigned long long x4[kV];
        int cl[kV];
        unsigned int acc = 0u;
#pragma unroll
        for (int k = 0; k < kV; ++k) {
            const unsigned long long x = w[k] & kPkLtMask;
            x4[k] = x;
            const bool agentless = ((w[k] >> 40) & kPkNoAgent) == kPkNoAgent;
            cl[k] = agentless ? 0 : 2;
            acc |= (unsigned int)(x <= cR) << k;
            acc |= (unsigned int)((long long)w[k] >= 0 && x <= (agentless ? cE : cP)) << (kV + k);
        }
        if (!valid) acc = 0u;
        if (!S.overflow) append4(acc, x4, cl, i0, 1, B, S, true);
    };
    if (P.stream_generic) {
        // persistent engine kernel: L2-coherent 128-bit loads, one tile prefetched in registers
        if (tid < kThreads) {
            unsigned long long nx[kV];
            unsigned int na[kV], nr[kV];
            long long i0 = lo + (long long)tid * kV;
            load4(P, i0, i0 + kV <= hi, nx, na, nr);
            for (int t = 0; t < ntiles; ++t, i0 += TV) {
                unsigned long long x4[kV];
                unsigned int a4[kV], r4[kV];
#pragma unroll
                for (int k = 0; k < kV; ++k) {
                    x4[k] = nx[k];
                    a4[k] = na[k];
                    r4[k] = nr[k];
                }
                if (t + 1 < ntiles) load4(P, i0 + TV, i0 + TV + kV <= hi, nx, na, nr);
                classify_append(x4, a4, r4, i0);
            }
        }
    } else if (tid >= kThreads) {  // producer warp: one elected thread keeps kRing tiles in flight
        if (lane_id() == 0) {
            // generic-proxy writes to the pool that this thread has observed (a kernel boundary,
            // or the admission server's grid barrier) before the async-proxy bulk reads
            asm volatile("fence.proxy.async.global;" ::: "memory");
            for (int t = 0; t < ntiles; ++t) {
                const int s = t % kRing;
                if (t >= kRing) mbar_wait(&S.mbar_empty[s], (unsigned int)(((t / kRing) - 1) & 1));
                const long long b0 = lo + (long long)t * TV;
                const unsigned int nsl = (unsigned int)min(TV, hi - b0);
                unsigned char* st = ring + (size_t)s * kRingStage;
                mbar_expect_tx(&S.mbar[s], nsl * 8u);
                bulk_g2s(st, P.pk + b0, nsl * 8u, &S.mbar[s]);  // the packed scan words
            }
        }
        __syncwarp();
    } else {
        for (int t = 0; t < ntiles; ++t) {
            const int s = t % kRing;
            const long long i0 = lo + (long long)t * TV + (long long)tid * kV;
            const unsigned char* st = ring + (size_t)s * kRingStage;
            mbar_wait(&S.mbar[s], (unsigned int)((t / kRing) & 1));
            if (P.dbg_check == 2) {
                unsigned long long x4[kV];
                unsigned int a4[kV], r4[kV];
                read4(st, tid, i0 + kV <= hi, x4, a4, r4);
                if (i0 + kV <= hi) load4(P, i0, true, x4, a4, r4);  // debug: L2 values
                __syncwarp();
                if (lane_id() == 0) mbar_arrive(&S.mbar_empty[s]);
                classify_append(x4, a4, r4, i0);
                continue;
            }
            const ulonglong2 w01 = *reinterpret_cast<const ulonglong2*>(st + (size_t)tid * 32);
            const ulonglong2 w23 = *reinterpret_cast<const ulonglong2*>(st + (size_t)tid * 32 + 16);
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&S.mbar_empty[s]);
            classify_append_pk(w01, w23, i0 + kV <= hi, i0);
        }
    }
    __syncthreads();
    if (tid == 0) P.dbg[blockIdx.x * 16 + 1] = gtimer();
    // this CTA's staged candidates, as staged, into its own raw region (no global atomics, no
    // cross-CTA wait): the next launch's list service gathers and finalizes them
    const size_t base = ((size_t)par * P.raw_grid + me) * kRawCap;
    // (an overflowed pass keeps what it staged: a subset, from which the service derives a
    // tighter threshold for the next prescan; the lists themselves are then unusable)
    const int m = min(min(S.count, S.ovf_base), kRawCap);
    for (int j = tid; j < m; j += T) {
        const unsigned int l = B.st_list[j];
        const unsigned int s = B.st_slot[j];
        P.raw_lt[base + j] = B.st_lt[j];
        P.raw_slot[base + j] = s;
        P.raw_list[base + j] = (unsigned char)l;
        if (l == 2) P.raw_agent[base + j] = __ldcg(P.agent + s);  // agent-carrying: its agent index
    }
    if (tid == 0) {
        RawHdr h;
        h.seq = seq;
        h.n = m;
        h.bad = S.overflow ? 1 : 0;
        P.raw_hdr[(size_t)par * P.raw_grid + me] = h;  // (a kernel boundary orders it before the reader)
    }
}

// Barrier of the prescan CTAs (1..grid-1) only: CTA 0 is busy with this launch's admission.
__device__ void prescan_barrier(Ctrl* c) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = ld_acquire(&c->pbar_gen);
        __threadfence();
        if (atomicAdd(&c->pbar_count, 1u) == gridDim.x - 2) {
            c->pbar_count = 0;
            __threadfence();
            atomicAdd(&c->pbar_gen, 1u);
        } else {
            unsigned long long spins = 0;
            while (ld_acquire(&c->pbar_gen) == gen) {
                if (++spins > 4096) __nanosleep(64);
                if (spins > (1ull << 27)) trap_at(104);
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// The table service (CTA kSvcQ of a pipelined launch): applies the block-table updates the
// previous admission queued (every erase, then every insert: a key erased and re-admitted in one
// admission is inserted after its erase), concurrently with CTA 0's probe, which resolves the
// queued keys from its on-chip overlay (a table operation on one key never misleads a find of
// another: finds skip claimed and erased entries, and an erased entry's key is cleared first).
// CTA 0 owns the queue counters: it resets them once it has seen svc_q_seq.
__device__ void service_queue(const DevPool& P, const AdmitArgs& a, RedSmem& Red) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int ne = C->tq_erase, ni = C->tq_insert;
    if (tid == 0) P.dbg[blockIdx.x * 16 + 6] = gtimer();
    for (int k = tid; k < ne; k += T) table_erase(P, P.tq_key[k]);
    __syncthreads();
    long long reused = 0;
    for (int i = tid; i < ni; i += T) reused += table_insert(P, P.tq_key[P.p_cap + i], P.tq_slot[i]);
    reused = block_sum(reused, Red);
    if (tid == 0) {
        C->tombstones += (long long)ne - reused;
        __threadfence();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&C->svc_q_seq), "l"(a.seq) : "memory");
        P.dbg[blockIdx.x * 16 + 7] = gtimer();
    }
}

// Block-wide exclusive prefix sum of one int per thread; *total = the sum (all threads).
__device__ __forceinline__ int block_excl_scan(int v, RedSmem& Red, int* total) {
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane_id() >= o) incl += y;
    }
    __syncthreads();
    if (lane_id() == 31) Red.v[warp_id()] = incl;
    __syncthreads();
    int off = 0;
    const int nw = (int)blockDim.x >> 5;
    for (int w = 0; w < warp_id(); ++w) off += (int)Red.v[w];
    int tot = 0;
    for (int w = 0; w < nw; ++w) tot += (int)Red.v[w];
    *total = tot;
    __syncthreads();
    return off + incl - v;
}

constexpr int kSvcStage = kStage / 2;  // E and R candidates the list service stages on chip, each

// The list service (CTA kSvcL of a pipelined launch, all threads): the previous launch's prescan
// (parity par) for this launch's CTA 0. Gathers the raw candidates every streaming CTA wrote;
// keeps per list E (agentless unpinned) and R (resident) the kPreK oldest, sorted, with the
// completeness bound T_l (every member of the state the prescan read at or below T_l is among
// the candidates); keeps every agent-carrying unpinned candidate (pending, complete to E's
// threshold); validates each entry against the pool as this launch found it (its last_touch is
// unchanged: DESIGN.md §5.6; CTA 0 filters this launch's own touches and unpins) and loads the
// keys of E's head. Publishes through svc_l_seq; writes the acceptance thresholds of the next
// launch's prescan (the parity slot this prescan used).
__device__ void service_lists(const DevPool& P, const AdmitArgs& a, const ScanBufs& B, SelectSmem& Sel, RedSmem& Red,
                              unsigned char* dsm, int par) {
    int* off = reinterpret_cast<int*>(dsm + kOffRing + 4096);  // per streaming CTA (the ring is idle here)
    __shared__ int cntL[3];
    __shared__ int okf;
    __shared__ unsigned long long hused[2];
    __shared__ int ng[2];
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int ns = (int)gridDim.x - kStream0;
    if (tid == 0) {
        P.dbg[blockIdx.x * 16 + 6] = gtimer();
        okf = 1;
        cntL[0] = cntL[1] = cntL[2] = 0;
        hused[0] = __ldcg(P.pre_hint + par * 3 + 0);
        hused[1] = __ldcg(P.pre_hint + par * 3 + 1);
    }
    int nc = 0;
    bool mine_ok = true, mine_full = true;
    if (tid < ns) {
        const RawHdr h = P.raw_hdr[(size_t)par * P.raw_grid + tid];
        mine_ok = h.seq == a.seq - 1ull;
        mine_full = !h.bad;
        nc = mine_ok ? h.n : 0;
    }
    int M = 0;
    const int ex = block_excl_scan(nc, Red, &M);
    if (tid <= ns) off[tid] = ex;  // off[ns] = M (nc = 0 there)
    // produced: every streaming CTA of the previous launch wrote its candidates; overflowed:
    // some staged only a subset (the lists are unusable, the next threshold tightens)
    const bool produced = !__syncthreads_or(tid < ns && !mine_ok);
    const bool overflowed = __syncthreads_or(tid < ns && !mine_full);
    if (tid == 0 && (!produced || overflowed)) okf = 0;
    __syncthreads();
    // gather: E and R staged on chip, pending written out validated
    unsigned long long* eL = B.st_lt;
    unsigned int* eS = B.st_slot;
    unsigned long long* rL = B.st_lt + kSvcStage;
    unsigned int* rS = B.st_slot + kSvcStage;
    for (int g = tid; g < M; g += T) {
        int lo = 0, hi = ns;  // the CTA whose range holds g: off[c] <= g < off[c + 1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (off[mid] <= g) lo = mid;
            else hi = mid;
        }
        const size_t idx = ((size_t)par * P.raw_grid + lo) * kRawCap + (g - off[lo]);
        const unsigned int l = P.raw_list[idx];
        const unsigned long long x = P.raw_lt[idx];
        const unsigned int sl = P.raw_slot[idx];
        if (l < 2) {
            const int p = atomicAdd(&cntL[l], 1);
            if (p < kSvcStage) {
                (l ? rL : eL)[p] = x;
                (l ? rS : eS)[p] = sl;
            } else {
                okf = 0;
            }
        } else {
            const int p = atomicAdd(&cntL[2], 1);
            if (p < kPendCap) {
                const size_t o = (size_t)2 * kPendCap + p;
                P.pl_lt[o] = x;
                P.pl_slot[o] = sl;
                P.pl_agent[p] = P.raw_agent[idx];
                P.pl_ok[o] = __ldcg(P.lt + sl) == x ? 1 : 0;
            } else {
                okf = 0;
            }
        }
    }
    __syncthreads();
    if (tid == 0) P.dbg[blockIdx.x * 16 + 7] = gtimer();
    const int mE = min(cntL[0], kSvcStage), mR = min(cntL[1], kSvcStage);
    const bool bad = okf == 0;
    // two warp groups (named barriers 1 and 2): group 0 finalizes E, group 1 R, at once
    const int nw = (int)blockDim.x >> 5, w0 = (nw + 1) >> 1;
    const int grp = warp_id() < w0 ? 0 : 1;
    // group 0 selects with the CTA's SelectSmem, group 1 with one in the (idle) TMA ring
    SelectSmem& Sgr =
        grp == 0 ? Sel : *reinterpret_cast<SelectSmem*>(reinterpret_cast<unsigned char*>(B.st_lt) + kOffRing);
    const int gn = (grp == 0 ? w0 : nw - w0) * 32, gt = tid - (grp == 0 ? 0 : w0 * 32);
    const int m = grp ? mR : mE;
    const unsigned long long* vl = grp ? rL : eL;
    const unsigned int* vs = grp ? rS : eS;
    unsigned long long* tl = B.sd_lt + (grp ? kPreK + 2 : 0);  // selected, kPreK per group
    unsigned int* ts = B.sd_slot + (grp ? kPreK + 2 : 0);
    if (gt == 0) ng[grp] = 0;
    group_sync(1 + grp, gn);
    const unsigned long long v = m > kPreK ? group_kth(vl, m, kPreK, Sgr, gt, gn, 1 + grp) : kNoBound;
    for (int j = gt; j < m; j += gn) {
        const unsigned long long x = vl[j];
        if (m <= kPreK || x <= v) {
            const int p = atomicAdd(&ng[grp], 1);
            tl[p] = x;
            ts[p] = vs[j];
        }
    }
    group_sync(1 + grp, gn);
    const int n = ng[grp];  // min(m, kPreK) (distinct ticks)
    if (gt == 0) Sgr.acc_or = kNoBound;  // (free after the select) rank kPreK / 2 - 1
    group_sync(1 + grp, gn);
    const size_t base = (size_t)grp * kPendCap;
    for (int j = gt; j < n; j += gn) {
        const unsigned long long x = tl[j];
        const unsigned int sl = ts[j];
        const int r = count_below(tl, n, x);
        P.pl_lt[base + r] = x;
        P.pl_slot[base + r] = sl;
        P.pl_ok[base + r] = __ldcg(P.lt + sl) == x ? 1 : 0;  // validation: last_touch unchanged
        if (grp == 0 && r < kChunk + 2) P.pl_key[r] = __ldcg(P.key + sl);
        if (r == 0) Sgr.hmax = x;
        if (r == kPreK / 2 - 1) Sgr.acc_or = x;
    }
    group_sync(1 + grp, gn);
    if (gt == 0) {
        const unsigned long long Tl = m > kPreK ? v : hused[grp];
        P.pl_n[grp] = n;
        P.pl_T[grp] = Tl;
        // (a seq mismatch: nothing was read; the old threshold stays)
        if (produced)
            P.pre_hint[par * 3 + grp] = n == 0 ? kNoBound
                                        : bad ? Tl
                                        : n == kPreK ? next_hint_mid(Sgr.acc_or, Tl)
                                                     : next_hint(Sgr.hmax, Tl);
    }
    __syncthreads();
    if (tid == 0) {
        P.pl_n[2] = min(cntL[2], kPendCap);
        P.pl_T[2] = hused[0];  // pending shares E's acceptance threshold
        P.pl_n[3] = bad ? 0 : 1;
        if (bad) atomicAdd(reinterpret_cast<unsigned long long*>(&C->pre_badcnt), 1ull);
        __threadfence();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&C->svc_l_seq), "l"(a.seq) : "memory");
        P.dbg[blockIdx.x * 16 + 8] = gtimer();
    }
}

// Acceptance thresholds for the next prescan from a regular select's lists (CTA 0, thread 0):
// the keep oldest of E and R extrapolated to ~2 kPreK ranks. Agent-carrying slots are kept whole.
__device__ void hints_from_fin(const DevPool& P, int NL, int keep, int par) {
    const int E = P.e_max, Rl = NL - 1;
    const int lists[2] = {E, Rl};
    for (int q = 0; q < 2; ++q) {
        const int l = lists[q];
        const int kl = keep_of(l, NL, keep);
        const int n = P.fin_n[l];
        unsigned long long h = kNoBound;
        if (n == kl && n >= 2) {
            const unsigned long long v1 = P.fin_lt[(long long)l * (kChunk + 2)];
            const unsigned long long vk = P.fin_lt[(long long)l * (kChunk + 2) + n - 1];
            const unsigned long long span = vk - v1;
            const unsigned long long mult = (unsigned long long)((2 * kPreK + n - 1) / n);
            h = span > (kNoBound - v1) / (mult + 1) ? kNoBound : v1 + span * mult;
        }
        P.pre_hint[par * 3 + q] = h;
        P.pre_hint[(par ^ 1) * 3 + q] = h;  // (the next pipelined launch's prescan reads the other slot)
    }
    P.pre_hint[par * 3 + 2] = kNoBound;
    P.pre_hint[(par ^ 1) * 3 + 2] = kNoBound;
}

__device__ __forceinline__ bool tset_insert(unsigned int* t, unsigned int s) {
    unsigned int h = xhash(s);
    for (int c = 0; c < kTset; ++c) {
        const unsigned int old = atomicCAS(&t[h], kNoSlot, s);
        if (old == kNoSlot || old == s) return true;
        h = (h + 1) & (kTset - 1);
    }
    return false;
}

__device__ __forceinline__ bool tset_has(const unsigned int* t, unsigned int s) {
    unsigned int h = xhash(s);
    for (int c = 0; c < kTset; ++c) {
        const unsigned int k = t[h];
        if (k == s) return true;
        if (k == kNoSlot) return false;
        h = (h + 1) & (kTset - 1);
    }
    return false;
}

// The consumer of the previous launch's prescan (CTA 0, after phase 0): the list service's
// output (service_lists: sorted, validated against the pool as this launch found it) minus this
// launch's phase-0 changes (touched prefix = tset, unpinned = U, re-read in phase 0); writes
// chunk 0's E and R lists, E's keys and the other classes' non-empty flags straight into the
// replay view. False: unusable (the admission scans instead).
__device__ bool consume_svc(const DevPool& P, const AdmitArgs& a, EarlySmem& es, ReplaySmem& R, const ScanBufs& B,
                            ScanSmem& S, RedSmem& Red) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int NL = P.n_lists, E = P.e_max, Rl = NL - 1;
    if (tid == 0) {
        unsigned long long spins = 0;
        while (ld_acquire_u64(&C->svc_l_seq) != a.seq) {
            if (++spins > 4096) __nanosleep(64);
            if (spins > (1ull << 28)) trap_at(105);
        }
    }
    __syncthreads();
    // one round of (L2-resident) loads: the counts and bounds, and the first kPreK entries of E
    // and of R whatever their counts (the lists hold at most kPreK each; unused entries ignored)
    static_assert(2 * kPreK < kThreads, "one E or R entry per thread");
    if (tid < kPreK) {
        es.E_lt[tid] = __ldcg(P.pl_lt + tid);
        es.E_slot[tid] = __ldcg(P.pl_slot + tid);
        es.E_ok[tid] = __ldcg(P.pl_ok + tid);
        if (tid < kChunk + 2) es.E_key[tid] = __ldcg(P.pl_key + tid);
    } else if (tid < 2 * kPreK) {
        const int j = tid - kPreK;
        es.R_lt[j] = __ldcg(P.pl_lt + kPendCap + j);
        es.R_slot[j] = __ldcg(P.pl_slot + kPendCap + j);
        es.R_ok[j] = __ldcg(P.pl_ok + kPendCap + j);
    } else if (tid == 2 * kPreK) {
        es.nE = __ldcg(P.pl_n + 0);
        es.nR = __ldcg(P.pl_n + 1);
        es.nP = __ldcg(P.pl_n + 2);
        es.valid = __ldcg(P.pl_n + 3);
        es.TE = __ldcg(P.pl_T + 0);
        es.TR = __ldcg(P.pl_T + 1);
        es.TP = __ldcg(P.pl_T + 2);
    }
    __syncthreads();
    pstamp(P, 7);
    if (!es.valid) return false;
    const unsigned long long TEs = min(es.TE, es.TP), TR = es.TR, TP = es.TP;
    const int nE = es.nE, nR = es.nR, nP = es.nP;
    unsigned long long* xl = B.sd_lt;
    unsigned int* xs = B.sd_slot;
    unsigned char* ef = B.st_list;  // E flags [0, kPreK), R flags [kPreK, 2 kPreK)
    if (tid < kMaxLists) S.lcnt[tid] = 0;
    if (tid == 0) S.side_n = 0;
    __syncthreads();
    auto add_member = [&](unsigned long long x, unsigned int s, int c) {
        if (c == E) {
            if (x <= TEs) {
                const int p = atomicAdd(&S.side_n, 1);
                if (p < kSide) {
                    xl[p] = x;
                    xs[p] = s;
                }
            }
        } else {
            S.lcnt[c] = 1;
        }
    };
    const int nU = es.xn;
    for (int q = tid; q < nE + nR + nP + nU; q += T) {
        if (q < nE) {
            const unsigned int s = es.E_slot[q];
            ef[q] = (es.E_ok[q] && es.E_lt[q] <= TEs && !xset_has(S, s) && !tset_has(es.tset, s)) ? 1 : 0;
        } else if (q < nE + nR) {
            const int j = q - nE;
            ef[kPreK + j] = (es.R_ok[j] && !tset_has(es.tset, es.R_slot[j])) ? 1 : 0;
        } else if (q < nE + nR + nP) {  // agent-carrying unpinned: class from this launch's BFS
            const int j = q - nE - nR;
            const size_t o = (size_t)2 * kPendCap + j;
            const unsigned int s = __ldcg(P.pl_slot + o);
            if (__ldcg(P.pl_ok + o) && !xset_has(S, s) && !tset_has(es.tset, s))
                add_member(__ldcg(P.pl_lt + o), s, B.cls[__ldcg(P.pl_agent + j)]);
        } else {
            const int j = es.xl[q - nE - nR - nP];
            const unsigned int s = S.xset[j];
            if (!es.U_ok[j] || tset_has(es.tset, s)) continue;
            const unsigned int ag = es.U_agent[j];
            add_member(es.U_lt[j], s, ag == kNoAgent ? E : B.cls[ag]);
        }
    }
    __syncthreads();
    if (TP < kNoBound && tid < E) S.lcnt[tid] = 1;  // some agent-carrying members unseen: assume present
    const int nx = S.side_n;
    int fe = 0, fr = 0;
    {
        const int q = tid < kPreK ? tid : 0;
        const long long both = ((long long)(tid < nE ? ef[q] : 0) << 32) | (tid < nR ? ef[kPreK + q] : 0);
        long long incl = both;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane_id() >= o) incl += y;
        }
        if (lane_id() == 31) Red.v[warp_id()] = incl;
        __syncthreads();
        long long off = 0;
        for (int w = 0; w < warp_id(); ++w) off += Red.v[w];
        const long long excl = off + incl - both;
        fe = (int)(excl >> 32);
        fr = (int)(excl & 0xffffffffll);
        if (tid < nE) es.efx[tid] = fe;
        __syncthreads();
        if (tid == (int)blockDim.x - 1) Red.u[0] = (unsigned long long)(off + incl);
        __syncthreads();
    }
    const long long tot = (long long)Red.u[0];
    const int totE = (int)(tot >> 32), totR = (int)(tot & 0xffffffffll);
    if (tid == 0) es.efx[nE] = totE;
    __syncthreads();
    if (!(nx <= kSide && (totR > 0 || TR >= kNoBound))) return false;
    const int cap = kChunk + 1;
    if (tid < nR && ef[kPreK + tid] && fr < cap) {
        R.L_lt[Rl][fr] = es.R_lt[tid];
        R.L_slot[Rl][fr] = es.R_slot[tid];
    }
    if (tid < nE && ef[tid]) {
        const unsigned long long x = es.E_lt[tid];
        const int r = fe + count_below(xl, nx, x);
        if (r < cap) {
            R.L_lt[E][r] = x;
            R.L_slot[E][r] = es.E_slot[tid];
            R.E_key[r] = es.E_key[tid];
            R.E_key_ok[r] = tid < kChunk + 2 ? 1 : 0;
        }
    }
    for (int i = tid; i < nx; i += T) {
        const unsigned long long x = xl[i];
        int r = count_below(xl, nx, x);
        int lo2 = 0, hi2 = nE;
        while (lo2 < hi2) {
            const int mid = (lo2 + hi2) >> 1;
            if (es.E_lt[mid] < x) lo2 = mid + 1;
            else hi2 = mid;
        }
        r += es.efx[lo2];  // the surviving E entries before position lo2
        if (r < cap) {
            R.L_lt[E][r] = x;
            R.L_slot[E][r] = xs[i];
            R.E_key_ok[r] = 0;  // key loaded by the apply if it is a victim
        }
    }
    if (tid < NL) R.L_n[tid] = tid == E ? min(totE + nx, cap) : tid == Rl ? min(totR, cap) : S.lcnt[tid];
    if (tid == 0) R.lists_ready = 1;
    __syncthreads();
    return true;
}

// Debug (P.dbg_check, small pools): every true E member below the last listed E entry must be
// listed. Records misses (slot, lt, refs, agent, in U, touched, in the prescan list and its flag)
// at dbg[grid*16 + 16 ...].
__device__ void debug_check_e(const DevPool& P, const EarlySmem& es, const ReplaySmem& R, const ScanBufs& B,
                              const ScanSmem& S, const AdmitArgs& a) {
    const int E = P.e_max;
    const int n = R.L_n[E];
    if (n <= 0) return;
    const unsigned long long last = R.L_lt[E][n - 1];
    unsigned long long* out = P.dbg + gridDim.x * 16 + 16;
    for (long long s = threadIdx.x; s < P.cap; s += blockDim.x) {
        const unsigned long long x = __ldcg(P.lt + s);
        if (x == kFreeTick || x > last || __ldcg(P.refs + s) != 0u) continue;
        const unsigned int ag = __ldcg(P.agent + s);
        const int c = ag == kNoAgent ? E : B.cls[ag];
        if (c != E) continue;
        int lo = 0, hi = n;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (R.L_lt[E][mid] < x) lo = mid + 1;
            else hi = mid;
        }
        if (lo < n && R.L_lt[E][lo] == x) continue;
        int inpl = -1;
        for (int j = 0; j < es.nE; ++j)
            if (es.E_slot[j] == (unsigned int)s) inpl = j;
        const unsigned long long k = atomicAdd(out, 1ull);
        if (k < 8) {
            unsigned long long* r = out + 1 + k * 6;
            r[0] = (unsigned long long)s;
            r[1] = x;
            r[2] = ((unsigned long long)ag << 32) | (unsigned long long)xset_has(S, (unsigned int)s) << 1 |
                   (unsigned long long)tset_has(es.tset, (unsigned int)s);
            r[3] = (unsigned long long)(long long)inpl | (inpl >= 0 ? (unsigned long long)es.E_ok[inpl] << 40 : 0ull);
            r[4] = a.seq;
            r[5] = P.dbg_unpin ? P.dbg_unpin[s] : 0ull;
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------------ K5b: replay + apply

__device__ __forceinline__ unsigned int hslot(unsigned int s) { return (s * 2654435761u) >> 23; }  // 9 bits

// Exact replay of admit_pinned over prompt blocks [lo, hi) (engine.cpp:141-168). Each
// eviction is evict_one (engine.cpp:102-125): the argmin of (score, last_touch) over the class
// heads; oldest_live_touch (engine.cpp:90-100) = min(tick, resident-list head, earliest touch
// of this admission). One warp; lane l owns list l.
// List-independent part of the replay of chunk A.chunk (CTA 0, all threads): the chunk's
// prompt slots and their pins, free slots, the slot -> prompt index hash, pool counters.
// Depends only on phase 0 and earlier chunks, so a speculative pass runs it before the lists
// exist.
__device__ void replay_prologue(const DevPool& P, ReplaySmem& R, AdmSmem& A, RedSmem& Red,
                                unsigned long long seq) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    // the table service usually finished long ago: hand the queue counters back to CTA 0 now
    // (this round of loads), so the apply's queue_ready finds nothing to wait for
    if (tid == 0 && A.q_deleg && ld_acquire_u64(&C->svc_q_seq) == seq) {
        C->tq_erase = 0;
        C->tq_insert = 0;
        A.tq_e = 0;
        A.tq_i = 0;
        A.q_deleg = 0;
    }
    const int lo = A.chunk * kChunk;
    const int hi = min(A.admit_n, lo + kChunk);
    const int len = hi - lo;
    for (int j = tid; j < 512; j += T) {
        R.ph_key[j] = kNoSlot;
        R.vh_key[j] = kNoSlot;
    }
    const long long ftop = A.free_top;  // (CTA 0 keeps it: loaded at admission start, updated by every apply)
    int absent = 0, pre_unpinned = 0;
    for (int i = tid; i < len; i += T) {
        const unsigned int sl = P.p_slot[lo + i];
        const unsigned int r0 = P.p_refs0[lo + i];
        R.c_slot[i] = sl;
        R.c_refs0[i] = r0;
        R.touched[i] = 0;
        R.pevict[i] = 0;
        if (sl == kNoSlot) ++absent;
        else if (r0 == 0u) ++pre_unpinned;
    }
    for (int j = tid; j < kChunk + 2; j += T) R.rremoved[j] = 0;
    for (int j = tid; j < len && j < ftop; j += T) R.freeslots[j] = P.free_stack[ftop - 1 - j];
    if (tid == 0) {
        R.n_vict = 0;
        R.n_new_global = 0;
        R.n_reused = 0;
        R.n_ins = 0;
        R.lists_ready = 0;
        R.ftop = ftop;
        R.res0 = C->resident;
        R.pinned0 = A.pin_c;
    }
    const long long both = block_sum(((long long)absent << 32) | (long long)pre_unpinned, Red);
    // slot -> prompt index of this chunk's resident blocks
    for (int i = tid; i < len; i += T) {
        const unsigned int s = R.c_slot[i];
        if (s == kNoSlot) continue;
        unsigned int h = hslot(s);
        for (int n = 0; n < 512; ++n) {
            const unsigned int old = atomicCAS(&R.ph_key[h], kNoSlot, s);
            if (old == kNoSlot || old == s) {
                R.ph_val[h] = (short)i;
                break;
            }
            h = (h + 1) & 511u;
        }
    }
    if (tid == 0) {
        R.absent = (int)(both >> 32);
        R.pre_unpinned = (int)(both & 0xffffffffll);
    }
    __syncthreads();
}

// Exact replay of admit_pinned over prompt blocks [lo, hi) (engine.cpp:141-168) after
// replay_prologue. Each eviction is evict_one (engine.cpp:102-125): the argmin of
// (score, last_touch) over the class heads; oldest_live_touch (engine.cpp:90-100) = min(tick,
// resident-list head, earliest touch of this admission). One warp; lane l owns list l.
// Loads the final candidate lists (all, or only E and R) from the finalizers' output: counts
// into shared memory first, then every entry in one round.
__device__ void load_lists(const DevPool& P, ReplaySmem& R, int NL, bool scanned, bool only_er) {
    const int tid = threadIdx.x, T = blockDim.x;
    const int E = P.e_max, Rl = NL - 1;
    if (tid < NL) {
        const bool mine = !only_er || tid == E || tid == Rl;
        // a class list that is not final yet: 1 marks "non-empty" (all the bulk test needs)
        R.L_n[tid] = !scanned ? 0 : mine ? P.fin_n[tid] : (P.gcount[tid] > 0 ? 1 : 0);
    }
    __syncthreads();
    for (int q = tid; q < NL * (kChunk + 2); q += T) {
        const int l = q / (kChunk + 2), j = q - l * (kChunk + 2);
        if (only_er && l != E && l != Rl) continue;
        if (j < R.L_n[l]) {
            R.L_lt[l][j] = P.fin_lt[q];
            R.L_slot[l][j] = P.fin_slot[q];
        }
    }
    __syncthreads();
}

// CTA 0, all threads: the queue counters are CTA 0's again. In a pipelined launch CTA kSvcQ
// applies the previous admission's queue (service_queue); wait for it, then start the new queue.
__device__ void queue_ready(const DevPool& P, const AdmitArgs& a, AdmSmem& A) {
    if (!A.q_deleg) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        Ctrl* C = P.ctrl;
        unsigned long long spins = 0;
        while (ld_acquire_u64(&C->svc_q_seq) != a.seq) {
            if (++spins > 4096) __nanosleep(64);
            if (spins > (1ull << 28)) trap_at(106);
        }
        C->tq_erase = 0;
        C->tq_insert = 0;
        A.tq_e = 0;
        A.tq_i = 0;
        A.q_deleg = 0;
    }
    __syncthreads();
}

__device__ void fill_status(AdmitStatus* st, const DevPool& P, const AdmSmem& A, long long n_evicted,
                            long long resident, long long pinned, unsigned long long ev_total, long long tombstones);

// The early status record (fill_status) written by one warp: lane 0 the scalars, the lanes the
// phase timers and the pending warmups.
__device__ void warp_fill_status(AdmitStatus* st, const DevPool& P, const AdmSmem& A, long long n_evicted,
                                 long long resident, long long pinned, unsigned long long ev_total,
                                 long long tombstones) {
    Ctrl* C = P.ctrl;
    const int lane = lane_id();
    const int np = min(__ldcg(&C->n_pend), kMaxPending);
    if (lane == 0) {
        st->started = A.started;
        st->error = A.error;
        st->first_miss = A.first_miss;
        st->admit_n = A.admit_n;
        st->cached = A.cached;
        st->n_evicted = n_evicted;
        st->resident = resident;
        st->pinned = pinned;
        st->tick_after = A.tick;
        st->ev_total = ev_total;
        st->warm_issued = A.warm_issued;
        st->needed = A.needed;
        st->scans = A.scans;
        st->tombstones = tombstones;
        st->srv_t0 = A.srv_t0;
        st->n_pend = np;
    }
    if (lane < kPhases) st->phase_ns[lane] = A.ph[lane];
    for (int k = lane; k < np; k += 32) {
        st->pend_target[k] = __ldcg(&C->pend_target[k]);
        st->pend_tick[k] = __ldcg(&C->pend_tick[k]);
    }
}

// early: only lists E and R are final (CTA 0 finalized E, CTA 1 signalled R); the other
// lists are awaited only if the bulk test fails.
__device__ void replay_apply(const DevPool& P, const AdmitArgs& a, ReplaySmem& R, AdmSmem& A, int NL, bool scanned,
                             RedSmem& Red, bool early = false, bool pre = false) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int lo = A.chunk * kChunk;
    const int hi = min(A.admit_n, lo + kChunk);
    const int len = hi - lo;
    const int Rl = NL - 1;
    const long long ftop = R.ftop;
    early = early && scanned;
    dstamp(P, 0);

    // ---- the candidate lists
    if (!R.lists_ready) load_lists(P, R, NL, scanned, early);
    dstamp(P, 1);
    // Bulk replay (the common case, no serial loop): when the victims are the first n_ev
    // class-E candidates, all inside the dominance prefix (below) and none of them a prompt
    // block of this chunk, the sequential replay reduces to: the absent block of rank r takes a
    // free slot while the pool is below budget, else the next class-E candidate; every block is
    // touched once in prompt order (tick0 + 1 + i).
    //
    // Dominance: within an admission `now` only grows and oldest_live_touch never decreases,
    // so rho(lt) of a fixed block only shrinks (the exact ratio shrinks, rounding is monotone).
    // A class-E (survival 0, score = rho) entry whose rho at the replay-start context is below
    // min over the other non-empty classes of fl(w_pred*S_c) therefore beats every other class
    // head at every later eviction of this chunk (score_c >= fl(w_pred*S_c) > rho_E); rho grows
    // with lt along the sorted list, so those entries form a prefix [0, pdom).
    const int E = P.e_max;
    double dom_bound = __longlong_as_double(0x7ff0000000000000ll);  // +inf: no other class
    bool dom_ok = true;
    if (P.policy == 1) {
        if (!(P.w_pred > 0.0)) dom_ok = false;
        for (int c = 0; c < E; ++c)
            if (R.L_n[c] > 0) dom_bound = fmin(dom_bound, A.wsurv[c]);
    }
    const unsigned long long tick0 = A.tick;
    unsigned long long old0 = tick0;
    if (R.L_n[Rl] > 0 && R.L_lt[Rl][0] < old0) old0 = R.L_lt[Rl][0];
    if (A.first_touch < old0) old0 = A.first_touch;
    auto prompt_index = [&](unsigned int s) -> short {
        unsigned int h = hslot(s);
        for (int c = 0; c < 512; ++c) {
            const unsigned int k = R.ph_key[h];
            if (k == kNoSlot) return -1;
            if (k == s) return R.ph_val[h];
            h = (h + 1) & 511u;
        }
        return -1;
    };
    {
        const long long res0 = R.res0;
        const int absent = R.absent, pre_unpinned = R.pre_unpinned;
        const long long room = P.cap - res0;
        const int n_free = (int)min((long long)absent, room > 0 ? room : 0ll);
        const int n_ev = absent - n_free;
        int bad = n_ev > R.L_n[E] || (n_ev > 0 && !dom_ok);
        if (blockIdx.x == 0 && tid == 0) P.dbg[48 + 10] = clock64();
        // a needed victim that is one of this chunk's prompt blocks, or outside the prefix
        for (int j = tid; !bad && j < n_ev; j += T) bad |= prompt_index(R.L_slot[E][j]) >= 0;
        if (!bad && tid == 0 && n_ev > 0) bad = !(recency(R.L_lt[E][n_ev - 1], tick0, old0) < dom_bound);
        if (blockIdx.x == 0 && tid == 0) P.dbg[48 + 11] = clock64();
        const bool bulk = !__syncthreads_or(bad);
        dstamp(P, 2);
        if (bulk) {
            // exclusive rank of each absent block (len <= kChunk = 128: 4 warps)
            __shared__ int wsum[kChunk / 32];
            int rank = 0;
            if (tid < kChunk) {
                const bool ab = tid < len && R.c_slot[tid] == kNoSlot;
                const unsigned int ball = __ballot_sync(0xffffffffu, ab);
                if (lane_id() == 0) wsum[warp_id()] = __popc(ball);
                rank = __popc(ball & ((1u << lane_id()) - 1u));
            }
            __syncthreads();
            if (tid < len) {
                for (int w = 0; w < warp_id(); ++w) rank += wsum[w];
                const unsigned long long t = A.tick + 1 + (unsigned long long)tid;
                const unsigned int s = R.c_slot[tid];
                R.out_lt[tid] = t;
                if (s != kNoSlot) {
                    R.out_slot[tid] = s;
                    R.out_new[tid] = 0;
                } else {
                    R.out_slot[tid] = rank < n_free ? R.freeslots[rank] : R.L_slot[E][rank - n_free];
                    R.out_new[tid] = 1;
                }
            }
            for (int k = tid; k < n_ev; k += T) R.victims[k] = R.L_slot[E][k];
            __syncthreads();
            if (tid == 0) {
                if (len > 0 && A.first_touch == ~0ull) A.first_touch = A.tick + 1;
                A.tick += (unsigned long long)len;
                A.resident = res0 + absent - n_ev;
                A.pinned = R.pinned0 + pre_unpinned + absent;
                R.n_vict = n_ev;
                R.n_reused = n_ev;
                R.n_new_global = n_free;
                A.ph[11] += (unsigned long long)n_ev;
                A.ph[12] += (unsigned long long)n_ev;
                A.ph[14] += 1;  // bulk chunks
            }
        }
        if (tid == 0) R.bulk = bulk ? 1 : 0;
        __syncthreads();
    }
    if (!R.bulk && pre) {  // prescan lists feed only the bulk replay: nothing applied, scan instead
        if (tid == 0) A.need_full = 1;
        __syncthreads();
        return;
    }
    if (!R.bulk && early) {  // the serial replay needs every list: wait for the other finalizers
        if (tid == 0) {
            unsigned long long spins = 0;
            while (ld_acquire(&C->fin_done) < (unsigned int)A.fin_want) {
                if (++spins > 4096) __nanosleep(64);
                if (spins > (1ull << 27)) trap_at(107);
            }
            __threadfence();
        }
        __syncthreads();
        load_lists(P, R, NL, scanned, false);
    }
    if (!R.bulk) {
        // serial path: per list entry, the prompt index (a touch removes it) and the position in
        // the resident list (an eviction from a class list removes it there too); pdom in full
        const int nres = R.L_n[Rl];
        for (int l = 0; l < NL; ++l) {
            const int n = R.L_n[l];
            for (int j = tid; j < n; j += T) {
                const unsigned int s = R.L_slot[l][j];
                R.L_pidx[l][j] = prompt_index(s);
                short rp = -1;
                if (l == Rl) {
                    rp = (short)j;
                } else {
                    const unsigned long long x = R.L_lt[l][j];
                    int lo2 = 0, hi2 = nres;  // binary search by the unique last_touch
                    while (lo2 < hi2) {
                        const int mid = (lo2 + hi2) >> 1;
                        if (R.L_lt[Rl][mid] < x) lo2 = mid + 1;
                        else hi2 = mid;
                    }
                    if (lo2 < nres && R.L_lt[Rl][lo2] == x) rp = (short)lo2;
                }
                R.L_rpos[l][j] = rp;
            }
        }
        const int nE = R.L_n[E];
        long long first_fail = dom_ok ? nE : 0;
        for (int j = tid; dom_ok && j < nE; j += T) {
            const double rho = recency(R.L_lt[E][j], tick0, old0);
            if (!(rho < dom_bound)) first_fail = min(first_fail, (long long)j);
        }
        first_fail = block_min(first_fail, Red);
        if (tid == 0) R.pdom = (int)first_fail;
        __syncthreads();
    }
    stamp(A, 6);
    dstamp(P, 3);

    // ---- the sequential replay (warp 0)
    if (warp_id() == 0 && !R.bulk) {
        const int lane = lane_id();
        int cursor = 0;
        const int my_n = lane < NL ? R.L_n[lane] : 0;
        const double my_ws = lane < kMaxLists ? A.wsurv[lane] : 0.0;
        unsigned long long tick = A.tick;
        unsigned long long first_touch = A.first_touch;
        long long resident = R.res0;
        long long pinned = R.pinned0;
        int nv = 0, nre = 0, nglob = 0;
        int error = 0;
        const int E = P.e_max;      // agentless / unreachable class (survival 0)
        const int pdom = R.pdom;    // class-E heads below this index win outright
        long long fast = 0;
        for (int i = 0; i < len; ++i) {
            const unsigned int s = R.c_slot[i];
            if (s != kNoSlot && !R.pevict[i]) {  // resident: touch + pin
                ++tick;
                if (lane == 0) {
                    R.out_slot[i] = s;
                    R.out_lt[i] = tick;
                    R.out_new[i] = 0;
                    R.touched[i] = 1;
                }
                if (R.c_refs0[i] == 0u) ++pinned;
                if (first_touch == ~0ull) first_touch = tick;
                __syncwarp();
                continue;
            }
            while (resident >= P.cap) {
                // fast path: the class-E head is inside the dominated prefix (see pdom)
                if (lane == E) {
                    while (cursor < my_n) {
                        const short pi = R.L_pidx[E][cursor];
                        if (!(pi >= 0 && R.touched[pi])) break;
                        ++cursor;
                    }
                }
                const int ecur = __shfl_sync(0xffffffffu, cursor, E);
                if (ecur < pdom) {
                    if (lane == E) {
                        const short pi = R.L_pidx[E][cursor];
                        const short rp = R.L_rpos[E][cursor];
                        if (pi >= 0) R.pevict[pi] = 1;
                        if (rp >= 0) R.rremoved[rp] = 1;
                        R.victims[nv] = R.L_slot[E][cursor];
                        ++cursor;
                    }
                    ++nv;
                    --resident;
                    ++fast;
                    __syncwarp();
                    continue;
                }
                if (lane < NL) {  // skip entries touched (pinned) or evicted via another list
                    while (cursor < my_n) {
                        const short pi = R.L_pidx[lane][cursor];
                        const bool gone = (pi >= 0 && R.touched[pi]) || (lane == Rl && R.rremoved[cursor]);
                        if (!gone) break;
                        ++cursor;
                    }
                }
                const unsigned long long rhead =
                    __shfl_sync(0xffffffffu, (lane == Rl && cursor < my_n) ? R.L_lt[Rl][cursor] : ~0ull, Rl);
                unsigned long long old = tick;
                if (rhead < old) old = rhead;
                if (first_touch < old) old = first_touch;
                // (score, last_touch) as two 64-bit keys; non-negative doubles order like their bits
                unsigned long long sk = ~0ull, lk = ~0ull;
                if (lane < Rl && cursor < my_n) {
                    lk = R.L_lt[lane][cursor];
                    const double rho = recency(lk, tick, old);
                    sk = (unsigned long long)__double_as_longlong(P.policy == 0 ? rho : __dadd_rn(my_ws, rho));
                }
                const unsigned int m1 = __reduce_min_sync(0xffffffffu, (unsigned int)(sk >> 32));
                if (m1 == 0xffffffffu) {
                    error = 1;  // evict_one: all resident blocks are pinned
                    break;
                }
                bool c = (unsigned int)(sk >> 32) == m1;
                const unsigned int m2 = __reduce_min_sync(0xffffffffu, c ? (unsigned int)sk : 0xffffffffu);
                c = c && (unsigned int)sk == m2;
                unsigned int ball = __ballot_sync(0xffffffffu, c);
                if (__popc(ball) > 1) {  // equal scores: the older block wins (engine.cpp:111-114)
                    const unsigned int m3 = __reduce_min_sync(0xffffffffu, c ? (unsigned int)(lk >> 32) : 0xffffffffu);
                    c = c && (unsigned int)(lk >> 32) == m3;
                    const unsigned int m4 = __reduce_min_sync(0xffffffffu, c ? (unsigned int)lk : 0xffffffffu);
                    c = c && (unsigned int)lk == m4;
                    ball = __ballot_sync(0xffffffffu, c);
                }
                const int w = __ffs(ball) - 1;
                if (lane == w) {
                    const unsigned int v = R.L_slot[lane][cursor];
                    const short pi = R.L_pidx[lane][cursor];
                    const short rp = R.L_rpos[lane][cursor];
                    if (pi >= 0) R.pevict[pi] = 1;  // reached later in this chunk: absent then
                    if (rp >= 0) R.rremoved[rp] = 1;
                    R.victims[nv] = v;
                    ++cursor;
                }
                ++nv;
                --resident;
                __syncwarp();
            }
            if (error) break;
            // allocate: this chunk's victims first, then the free stack
            unsigned int ns;
            if (nre < nv) {
                ns = R.victims[nre++];
            } else {
                ns = R.freeslots[nglob++];
            }
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
            R.n_vict = nv;
            R.n_reused = nre;
            R.n_new_global = nglob;
            if (error) A.error = 1;
            A.ph[11] += (unsigned long long)fast;  // instrumentation: evictions on the fast path
            A.ph[12] += (unsigned long long)nv;
        }
    }
    __syncthreads();
    stamp(A, 7);
    const bool err = A.error != 0;
    const int nv = R.n_vict;
    // ---- apply: victims first (queue the erase, free slot), then inserts and touches
    queue_ready(P, a, A);
    const unsigned long long ev0 = A.n_ev_c;
    // victim keys first (a reused victim slot is rewritten below)
    for (int k = tid; k < nv; k += T) {
        const unsigned int v = R.victims[k];
        R.vkey[k] = (R.lists_ready && R.bulk && R.E_key_ok[k]) ? R.E_key[k] : P.key[v];
        unsigned int h = hslot(v);
        for (int c = 0; c < 512; ++c) {
            if (atomicCAS(&R.vh_key[h], kNoSlot, v) == kNoSlot) break;
            h = (h + 1) & 511u;
        }
    }
    __syncthreads();
    dstamp(P, 4);
    // The table updates are queued, erases and inserts, and applied by the next launch (its
    // CTA kSvcQ concurrently with its probe, or its phase 0): nothing reads the table for the rest
    // of this admission (later chunks re-resolve through the victim set), and a block this
    // admission inserted is pinned, so it is never among its own victims (the queue applies every
    // erase before every insert).
    const int q_e = A.tq_e, q_i = A.tq_i;
    // This chunk completes a plain admission served from a prescan: its status is final once the
    // victims are known, so the apply's idle warp publishes it (and the victims) to the host while
    // the other warps apply; the host schedules the next admission meanwhile.
    const bool early_st = pre && R.bulk && !err && hi >= A.admit_n && !(a.flags & kUnpinAfter) && a.status != nullptr;
    for (int k = tid; k < nv; k += T) {
        const unsigned long long kk = R.vkey[k];
        P.tq_key[q_e + k] = kk;
        P.evlog[(ev0 + k) % (unsigned long long)P.evlog_cap] = kk;  // ring; the host drains it
        if (!early_st && a.vict_host && A.n_ev_adm + k < a.vict_cap)
            a.vict_host[A.n_ev_adm + k] = kk;  // mapped host memory
        if (k >= R.n_reused) {  // victims[0, n_reused) are overwritten by new blocks below
            const unsigned int v = R.victims[k];
            P.lt[v] = kFreeTick;
            P.refs[v] = 0u;
            P.agent[v] = kNoAgent;
            P.pk[v] = kPkFreeWord;
        }
    }
    if (early_st && warp_id() == (T >> 5) - 1) {  // (the apply below leaves it idle: len <= kChunk)
        const int lane = lane_id();
        tstamp(P, a.seq, 3);
        warp_fill_status(a.status, P, A, A.n_ev_adm + nv, A.resident, A.pinned, ev0 + nv,
                         C->tombstones + (long long)(q_e + nv));
        if (a.vict_host)
            for (int k = lane; k < nv && A.n_ev_adm + k < a.vict_cap; k += 32) a.vict_host[A.n_ev_adm + k] = R.vkey[k];
        __threadfence_system();  // each lane's record words and victims before the flag
        __syncwarp();
        if (lane == 0) {
            *(volatile unsigned long long*)&a.status->done_seq = a.seq;
            A.st_done = 1;
            tstamp(P, a.seq, 4);
        }
    }
    // A serial chunk may evict a later prompt block and re-admit it into the victim's slot:
    // the victim's reset above must land before the new block's writes.
    if (!R.bulk) __syncthreads();
    const int done_len = err ? 0 : len;  // an erroring chunk is not applied
    for (int i = tid; i < done_len; i += T) {
        const unsigned int s = R.out_slot[i];
        if (R.out_new[i]) {
            const int gi = lo + i;
            P.key[s] = a.keys[gi];
            P.tokens[s] = a.counts[gi];
            const unsigned int ag = (a.agent != kNoAgent && gi < A.anchor) ? a.agent : kNoAgent;
            P.agent[s] = ag;
            P.lt[s] = R.out_lt[i];
            P.refs[s] = 1u;
            P.pk[s] = pk_make(R.out_lt[i], ag, true);
            const int q = q_i + atomicAdd(&R.n_ins, 1);
            P.tq_key[P.p_cap + q] = a.keys[gi];
            P.tq_slot[q] = s;
        } else {
            P.lt[s] = R.out_lt[i];
            atomicAdd(&P.refs[s], 1u);
            P.pk[s] = pk_make(R.out_lt[i], P.agent[s], true);
        }
        P.p_slot[lo + i] = s;
        if (a.pins_out) a.pins_out[lo + i] = s;  // final: later chunks only re-resolve positions >= hi
    }
    // blocks of later chunks evicted here are absent when reached
    if (nv > 0) {
        for (int j = hi + tid; j < A.admit_n; j += T) {
            const unsigned int s = P.p_slot[j];
            if (s == kNoSlot) continue;
            unsigned int h = hslot(s);
            for (int c = 0; c < 512; ++c) {
                const unsigned int k = R.vh_key[h];
                if (k == kNoSlot) break;
                if (k == s) {
                    P.p_slot[j] = kNoSlot;
                    break;
                }
                h = (h + 1) & 511u;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        long long top = ftop - R.n_new_global;
        for (int k = R.n_reused; k < nv; ++k) P.free_stack[top++] = R.victims[k];
        C->resident = A.resident;
        C->pinned = A.pinned;
        A.pin_c = A.pinned;
        C->free_top = top;
        A.free_top = top;
        C->n_ev = ev0 + nv;
        C->tq_erase = q_e + nv;
        C->tq_insert = q_i + R.n_ins;
        A.n_ev_c = ev0 + nv;
        A.tq_e = q_e + nv;
        A.tq_i = q_i + R.n_ins;
        A.n_ev_adm += nv;
    }
    __syncthreads();
    stamp(A, 8);
    dstamp(P, 5);
}

// On-chip overlay of the queued table updates (phase 0): key -> new slot, kSlotTomb (erased) or
// both (erased, then re-inserted). Open addressing over kOv entries in the (idle) TMA ring.
constexpr int kOv = 2048;
constexpr int kOvMax = kOv / 2;
// phase 0's early table finds: slots and keys of up to kFindMax prompt blocks, in the TMA ring
// after the overlay (below the early-validation view)
constexpr int kFindMax = 2048;
constexpr size_t kFindOff = 12ull * kOv;
// per prompt position: slot (the find, then the resolved slot), key, token count, pins before
static_assert(kFindOff + 20ull * kFindMax <= kEarlyOff, "early finds must stay below the early-validation view");
constexpr unsigned int kOvErase = 0x7FFFFFFFu;  // erased only (slots stay below 2^31 - 16)
constexpr unsigned int kOvBoth = 0x80000000u;   // slot | kOvBoth: erased, then re-inserted
constexpr unsigned int kOvSlot = ~kOvBoth;

__device__ __forceinline__ bool ov_both(unsigned int v) {
    return v != kSlotEmpty && v != kSlotClaim && (v & kOvBoth) != 0u;
}

// Adds an erase (slot = kOvErase) or an insert of key; order-free: a key seen as both becomes
// slot | kOvBoth whichever arrives first.
__device__ __forceinline__ void ov_put(unsigned long long* ovk, unsigned int* ovs, unsigned long long key,
                                       unsigned int val) {
    unsigned int h = (unsigned int)(mix64(key) >> 53) & (kOv - 1);
    for (int c = 0; c < kOv; ++c) {
        const unsigned int old = atomicCAS(&ovs[h], kSlotEmpty, kSlotClaim);
        if (old == kSlotEmpty) {
            ovk[h] = key;
            __threadfence_block();
            const unsigned int prev = atomicExch(&ovs[h], val);
            (void)prev;  // only a claimer writes an unclaimed entry
            return;
        }
        unsigned int cur = old;
        while (cur == kSlotClaim) cur = *(volatile unsigned int*)&ovs[h];  // a peer is publishing
        if (*(volatile unsigned long long*)&ovk[h] == key) {
            if (val == kOvErase) atomicOr(&ovs[h], kOvBoth);  // the insert's slot stays
            else atomicExch(&ovs[h], val | kOvBoth);
            return;
        }
        h = (h + 1) & (kOv - 1);
    }
}

__device__ __forceinline__ unsigned int ov_get(const unsigned long long* ovk, const unsigned int* ovs,
                                               unsigned long long key) {
    unsigned int h = (unsigned int)(mix64(key) >> 53) & (kOv - 1);
    for (int c = 0; c < kOv; ++c) {
        const unsigned int v = ovs[h];
        if (v == kSlotEmpty) return kSlotEmpty;
        if (ovk[h] == key) return v;
        h = (h + 1) & (kOv - 1);
    }
    return kSlotEmpty;
}

// Applies the block-table updates queued by the previous admission (all threads of one CTA):
// every erase, then every insert (a key erased and re-admitted in one admission is inserted
// after its erase; an inserted block is pinned, so no admission erases it again).
__device__ void apply_table_queue(const DevPool& P, RedSmem& Red) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int ne = C->tq_erase, ni = C->tq_insert;
    if (ne == 0 && ni == 0) return;
    for (int k = tid; k < ne; k += T) table_erase(P, P.tq_key[k]);
    __syncthreads();
    long long reused = 0;
    for (int i = tid; i < ni; i += T) reused += table_insert(P, P.tq_key[P.p_cap + i], P.tq_slot[i]);
    reused = block_sum(reused, Red);
    if (tid == 0) {
        C->tombstones += (long long)ne - reused;
        C->tq_erase = 0;
        C->tq_insert = 0;
    }
    __syncthreads();
}

__global__ void table_flush_kernel(DevPool P) {
    __shared__ RedSmem Red;
    apply_table_queue(P, Red);
}

cudaError_t launch_table_flush(const DevPool& P, cudaStream_t s) {
    table_flush_kernel<<<1, 512, 0, s>>>(P);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ the admission kernel

__device__ void fill_status(AdmitStatus* st, const DevPool& P, const AdmSmem& A, long long n_evicted,
                            long long resident, long long pinned, unsigned long long ev_total, long long tombstones) {
    Ctrl* C = P.ctrl;
    st->started = A.started;
    st->error = A.error;
    st->first_miss = A.first_miss;
    st->admit_n = A.admit_n;
    st->cached = A.cached;
    st->n_evicted = n_evicted;
    st->resident = resident;
    st->pinned = pinned;
    st->tick_after = A.tick;
    st->ev_total = ev_total;
    st->warm_issued = A.warm_issued;
    st->needed = A.needed;
    st->scans = A.scans;
    st->tombstones = tombstones;
    for (int k = 0; k < kPhases; ++k) st->phase_ns[k] = A.ph[k];
    st->srv_t0 = A.srv_t0;
    st->n_pend = C->n_pend;
    for (int k = 0; k < C->n_pend && k < kMaxPending; ++k) {
        st->pend_target[k] = C->pend_target[k];
        st->pend_tick[k] = C->pend_tick[k];
    }
}

__device__ void write_status(const DevPool& P, const AdmitArgs& a, const AdmSmem& A) {
    Ctrl* C = P.ctrl;
    // after queue_ready: nothing else changes either until the next launch applies the queue;
    // the queued erases leave tombstones then (an insert may reuse some): an upper bound, so the
    // host's rebuild decision is deterministic and conservative
    fill_status(a.status, P, A, A.n_ev_adm, C->resident, C->pinned, C->n_ev, C->tombstones + (long long)C->tq_erase);
}


// One admission (the body of admit_kernel; the device-resident engine kernel runs it in a loop).
// Every CTA of the cooperative grid calls it; a CTA returns when its part is done.
__device__ __forceinline__ void admit_body(const DevPool& P, const AdmitArgs& a, unsigned char* dsm, ScanSmem& S,
                                        SelectSmem& Sel, RedSmem& Red, AdmSmem& A) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int NL = P.n_lists;
    const ScanBufs B = scan_bufs(dsm);
    ReplaySmem& Rp = *reinterpret_cast<ReplaySmem*>(dsm + kOffRing);
    if (tid == 0) P.dbg[blockIdx.x * 16 + 9] = gtimer();  // kernel entry (instrumentation)
    progress(a.seq, 2);
    if (tid == 0 && blockIdx.x == 0) tstamp(P, a.seq, 1);
    const int par_prev = (int)((a.seq - 1ull) & 1ull), par_next = (int)(a.seq & 1ull);
    const bool pre_run = (a.flags & kPrescan) && gridDim.x > kStream0;
    // The host asks for the previous prescan's lists (kUsePrescan): the prescan CTAs start the
    // next stream at once; CTA 0 checks the lists are there and usable (else it scans as before).
    const bool pre_avail = pre_run && (a.flags & kUsePrescan);
    EarlySmem& es = *reinterpret_cast<EarlySmem*>(dsm + kOffRing + kEarlyOff);

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
            A.q_deleg = 0;
            A.st_done = 0;
            A.first_touch = ~0ull;
            A.tick = a.tick_base;
            A.free_top = C->free_top;  // (the replay prologue's free-stack reads need it: one round earlier)
            A.n_ev_c = C->n_ev;
            A.pin_c = C->pinned;
            A.tq_e = C->tq_erase;
            A.tq_i = C->tq_insert;
            for (int k = 0; k < kPhases; ++k) A.ph[k] = 0;
#pragma unroll
            for (int c = 0; c < kMaxLists; ++c) A.wsurv[c] = P.wsurv[c];  // constant indices
            A.tl = gtimer();
            C->done = 0;
            C->error = 0;
            es.ok = 0;
            {  // (thread 0 waits for this round of loads anyway)
                const long long wh = C->win_head, wsz = C->win_size;
                A.pf_head = wh;
                A.pf_size = wsz;
                // a pipelined launch: CTA kSvcB computes the dispatch's observe concurrently
                // (service_learner evaluates the same predicate on the same inputs)
                A.svc_b = pre_avail && gridDim.x > kSvcB && (a.flags & kDispatch) && P.policy == 1 && a.next >= 0 &&
                          wsz <= kBfsPre;
                A.pf_on = !A.svc_b && (a.flags & kDispatch) && P.policy != 0 && a.next >= 0 && C->cur_agent != a.next &&
                          wsz <= 2 * (long long)blockDim.x && wsz <= kBfsPre;
            }
            // a pipelined launch: the list service validates the previous prescan concurrently;
            // phase 0 tracks this launch's own changes (U, touched) for its consumer
            es.ok = pre_avail && unpin_total(a, true) <= kXsetMax ? 1 : 0;
            if (a.flags & kPollReset) {
                C->step_warmups = 0;
                C->n_pend = 0;
            }
        }
        __syncthreads();
        pstamp(P, 0);
        const int n = a.n;
        long long miss_min = n, need = 0;
        const int ne = A.tq_e, ni = A.tq_i;
        // a pipelined launch: CTA kSvcQ applies the queued table updates (service_queue)
        const bool deleg = pre_avail;
        if (tid == 0) A.q_deleg = deleg ? 1 : 0;
        // BFS inputs of observe(AgentDispatch), issued now so their round trips overlap the two
        // table rounds: the window pairs (here), their counts and row totals (round 2)
        const long long W_ = P.window, pf_head = A.pf_head, pf_size = A.pf_size;
        const bool pf = A.pf_on != 0;
        int pf_a[2] = {0, 0}, pf_b[2] = {0, 0};
        unsigned int pf_c[2] = {0u, 0u}, pf_t[2] = {0u, 0u};
        if (pf) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const long long j = tid + (long long)k * T;
                if (j < pf_size) {
                    const long long q = (pf_head + j) % W_;
                    pf_a[k] = P.win_a[q];
                    pf_b[k] = P.win_b[q];
                }
            }
        }
        auto pf_issue2 = [&]() {
            if (!pf) return;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const long long j = tid + (long long)k * T;
                if (j < pf_size) {
                    pf_c[k] = __ldcg(P.counts + (long long)pf_a[k] * P.a_cap + pf_b[k]);
                    pf_t[k] = __ldcg(P.totals + pf_a[k]);
                }
            }
        };
        if (ne + ni <= kOvMax) {
            // The previous admission's table updates run concurrently with this admission's probe:
            // the probe resolves the queued keys from an on-chip overlay (insert wins: a key erased
            // and re-admitted is re-inserted), and a table operation on one key never misleads a
            // find of another (finds skip claimed and erased entries, and an erased entry's key
            // is cleared first). In a pipelined launch CTA kSvcQ applies them (service_queue);
            // otherwise this CTA does, erase+insert of one key in order on one thread.
            unsigned long long* ovk = reinterpret_cast<unsigned long long*>(dsm + kOffRing);
            unsigned int* ovs = reinterpret_cast<unsigned int*>(dsm + kOffRing + 8 * kOv);
            for (int j = tid; j < kOv; j += T) ovs[j] = kSlotEmpty;
            const bool early = es.ok != 0;
            // the class table for the consumer, stored on chip after the first round (its loads
            // complete meanwhile instead of holding the barrier below)
            unsigned char cls_r[kMaxAgents / kThreads + 1];
            if (early) {
                for (int j = tid; j < kXset; j += T) S.xset[j] = kNoSlot;
                for (int j = tid; j < kTset; j += T) es.tset[j] = kNoSlot;
#pragma unroll
                for (int k = 0; k < kMaxAgents / kThreads + 1; ++k) {
                    const int x = tid + k * T;
                    cls_r[k] = x < a.n_agents ? __ldcg(P.cls + x) : (unsigned char)0;
                }
                if (tid == 0) es.xn = 0;
            }
            __syncthreads();
            // one round: the overlay of the queued keys, the deferred EngineSim::unpin calls of
            // completed requests (engine.cpp:170-180) and, feeding a prescan consumer, the set U
            // of unpinned slots (this launch's and the previous launch's)
            // The prompt's table finds run in this round too (their slots and keys kept on chip):
            // a find never depends on the overlay or the unpins (a queued key is resolved from the
            // overlay in the next round, and a find of any other key is exact while the queue is
            // applied, see above), so the next round only reads the pins.
            long long dec = 0;
            const int nu = unpin_total(a, false);
            const int nuv = early ? unpin_total(a, true) : nu;
            const int nf = n <= kFindMax ? n : 0;
            unsigned int* f_slot = reinterpret_cast<unsigned int*>(dsm + kOffRing + kFindOff);
            unsigned long long* f_key = reinterpret_cast<unsigned long long*>(dsm + kOffRing + kFindOff + 4 * kFindMax);
            int* f_cnt = reinterpret_cast<int*>(dsm + kOffRing + kFindOff + 12 * kFindMax);
            for (int q = tid; q < nf + nuv + ne + ni; q += T) {
                if (q < nf) {
                    f_cnt[q] = a.counts[q];  // (for the lookup: issued with the key, used much later)
                    const unsigned long long t0 = P.dbg_warps ? gtimer() : 0ull;
                    const unsigned long long key = a.keys[q];
                    f_key[q] = key;
                    const unsigned long long t1 = P.dbg_warps ? (key != 0ull ? gtimer() : 0ull) : 0ull;
                    f_slot[q] = table_find_line(P, key);
                    if (P.dbg_warps && (q & 31) == 0 && q < 96) {  // (instrumentation: lane 0 of warps 0-2)
                        const unsigned long long t2 = f_slot[q] != 0xFFFFFFFEu ? gtimer() : 0ull;
                        unsigned long long* o = P.dbg + (size_t)gridDim.x * 16 + 100 + (q >> 5) * 4;
                        o[0] = t0;
                        o[1] = t1;
                        o[2] = t2;
                        // the same find again (now an L2 hit): its time against the first one's
                        const unsigned int s2 = table_find_line(P, key);
                        o[3] = s2 != 0xFFFFFFFEu ? gtimer() : 0ull;
                    }
                } else if (q < nf + nuv) {
                    const int i = q - nf;
                    const unsigned int us = unpin_at(a, i);
                    if (us == kNoSlot) continue;
                    if (i < nu && atomicSub(&P.refs[us], 1u) == 1u) {
                        pk_unpinned(P, us);
                        ++dec;
                        if (P.dbg_unpin) P.dbg_unpin[us] = (a.seq << 8) | 1u;
                    }
                    if (early) {
                        const int pos = xset_insert_pos(S, us);
                        if (pos >= 0) es.xl[atomicAdd(&es.xn, 1)] = (unsigned short)pos;
                    }
                } else if (q < nf + nuv + ne) {
                    ov_put(ovk, ovs, P.tq_key[q - nf - nuv], kOvErase);
                } else {
                    const int k = q - nf - nuv - ne;
                    ov_put(ovk, ovs, P.tq_key[P.p_cap + k], P.tq_slot[k]);
                }
            }
            if (P.dbg_warps && lane_id() == 0) P.dbg[(size_t)gridDim.x * 16 + 48 + warp_id()] = gtimer();
            if (early) {
#pragma unroll
                for (int k = 0; k < kMaxAgents / kThreads + 1; ++k) {
                    const int x = tid + k * T;
                    if (x < a.n_agents) B.cls[x] = cls_r[k];
                }
            }
            dec = block_sum(dec, Red);  // (its barriers also publish the overlay and the U list)
            if (tid == 0) {
                A.pin_c -= dec;
                C->pinned = A.pin_c;  // (a store, not a read-modify-write round trip)
            }
            pstamp(P, 1);
            pf_issue2();
            long long reused = 0;
            const int nxs = early ? es.xn : 0;  // U: one entry per distinct unpinned slot
            const int nq = deleg ? 0 : ne + ni;  // queued table updates this CTA applies
            for (int q = tid; q < nq + n + nxs; q += T) {
                if (q < nq && q < ne) {
                    const unsigned long long key = P.tq_key[q];
                    if (ov_get(ovk, ovs, key) == kOvErase) table_erase(P, key);  // else its insert erases
                } else if (q < nq) {
                    const int k = q - ne;
                    const unsigned long long key = P.tq_key[P.p_cap + k];
                    if (ov_both(ov_get(ovk, ovs, key))) table_erase(P, key);
                    reused += table_insert(P, key, P.tq_slot[k]);
                } else if (q < nq + n) {
                    const int i = q - nq;
                    const unsigned long long key = nf ? f_key[i] : a.keys[i];
                    const unsigned int ov = ov_get(ovk, ovs, key);
                    const unsigned int s = ov == kSlotEmpty ? (nf ? f_slot[i] : table_find(P, key))
                                                            : ov == kOvErase ? kNoSlot : (ov & kOvSlot);
                    const unsigned int r0 = s == kNoSlot ? 0u : P.refs[s];
                    P.p_slot[i] = s;
                    P.p_refs0[i] = r0;
                    if (nf) f_slot[i] = s;  // (the lookup below reads the resolved slot on chip)
                    if (s == kNoSlot && i < miss_min) miss_min = i;
                    if (s == kNoSlot || r0 == 0u) ++need;
                } else {  // U re-read, after every unpin of this launch
                    const int j = es.xl[q - nq - n];
                    const unsigned int us = S.xset[j];
                    const unsigned long long x = __ldcg(P.lt + us);
                    es.U_lt[j] = x;
                    es.U_agent[j] = __ldcg(P.agent + us);
                    es.U_ok[j] = (x != kFreeTick && __ldcg(P.refs + us) == 0u) ? 1 : 0;
                }
            }
            if (P.dbg_warps && lane_id() == 0) P.dbg[(size_t)gridDim.x * 16 + 48 + 24 + warp_id()] = gtimer();
            reused = block_sum(reused, Red);
            if (tid == 0 && !deleg) {
                C->tombstones += (long long)ne - reused;
                C->tq_erase = 0;
                C->tq_insert = 0;
                A.tq_e = 0;
                A.tq_i = 0;
            }
            pstamp(P, 2);
        } else {  // too many queued keys for the overlay: the probe waits for the table
            if (tid == 0) es.ok = 0;  // (no consumer: the admission scans)
            if (deleg)
                queue_ready(P, a, A);
            else
                apply_table_queue(P, Red);  // the previous admission's erases / inserts
            if (tid == 0 && !deleg) {
                A.tq_e = 0;
                A.tq_i = 0;
            }
            pstamp(P, 1);
            pf_issue2();
            // deferred EngineSim::unpin calls of completed requests (engine.cpp:170-180), in order
            if (a.n_unpin_ranges > 0) {
                long long dec = 0;
                const int nu = unpin_total(a, false);
                for (int i = tid; i < nu; i += T) {
                    const unsigned int us = unpin_at(a, i);
                    if (us != kNoSlot && atomicSub(&P.refs[us], 1u) == 1u) {
                        pk_unpinned(P, us);
                        ++dec;
                        if (P.dbg_unpin) P.dbg_unpin[us] = (a.seq << 8) | 2u;
                    }
                }
                dec = block_sum(dec, Red);
                if (tid == 0) {
                A.pin_c -= dec;
                C->pinned = A.pin_c;  // (a store, not a read-modify-write round trip)
            }
                __syncthreads();
            }
            pstamp(P, 2);
            for (int i = tid; i < n; i += T) {
                const unsigned int s = table_find(P, a.keys[i]);
                const unsigned int r0 = s == kNoSlot ? 0u : P.refs[s];
                P.p_slot[i] = s;
                P.p_refs0[i] = r0;
                if (s == kNoSlot && i < miss_min) miss_min = i;
                if (s == kNoSlot || r0 == 0u) ++need;
            }
        }
        if (pf) {  // (the BFS view is free until observe_dispatch)
            BfsSmem& Bf = *reinterpret_cast<BfsSmem*>(dsm);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const long long j = tid + (long long)k * T;
                if (j < pf_size) {
                    Bf.wa[j] = (unsigned short)pf_a[k];
                    Bf.wb[j] = (unsigned short)pf_b[k];
                    Bf.pc[j] = pf_c[k];
                    Bf.pt[j] = pf_t[k];
                }
            }
            if (tid == 0) Bf.pf_size = (int)pf_size;
        }
        need = block_sum(need, Red);
        miss_min = block_min(miss_min, Red);
        if (tid == 0) A.needed = (int)need;
        if ((a.flags & kFeasible) && A.pin_c + need > P.cap) {
            if (tid == 0) A.started = 0;  // try_start_head: wait for in-flight pins to clear
        }
        __syncthreads();
        pstamp(P, 3);
        if (A.started) {
            if (a.flags & kDispatch) {
                if (tid == 0) A.tick = A.tick + 1;
                __syncthreads();
                // the learner service's observe is committed after the lookup (below): nothing
                // until the consumer reads the classes, so the service has that much longer
                if (!A.svc_b) observe_dispatch(P, a.prev, a.next, A.tick, a.n_agents, dsm, Red, A, B.cls, pf);
            }
            const unsigned long long dispatch_tick = A.tick;
            pstamp(P, 4);
            if (a.flags & kLookup) {
                const int f = (int)miss_min;
                long long cached = 0;
                const bool early = es.ok != 0 && f <= kTset / 2;
                // the resolved slots and token counts are on chip when phase 0 ran its early finds
                const bool onchip = ne + ni <= kOvMax && n <= kFindMax;
                const unsigned int* f_slot = reinterpret_cast<const unsigned int*>(dsm + kOffRing + kFindOff);
                const int* f_cnt = reinterpret_cast<const int*>(dsm + kOffRing + kFindOff + 12 * kFindMax);
                for (int i = tid; i < f; i += T) {
                    cached += onchip ? f_cnt[i] : a.counts[i];
                    const unsigned int ts = onchip ? f_slot[i] : P.p_slot[i];
                    P.lt[ts] = A.tick + 1 + (unsigned long long)i;  // EngineSim::touch
                    pk_touch(P, ts, A.tick + 1 + (unsigned long long)i);
                    if (a.touch_agent) a.touch_agent[i] = P.agent[ts];
                    if (early) tset_insert(es.tset, ts);
                }
                if (tid == 0 && !early) es.ok = 0;
                cached = block_sum(cached, Red);
                if (tid == 0) {
                    A.first_miss = f;
                    A.cached = cached;
                    A.tick += (unsigned long long)f;
                }
            }
            if (tid == 0) {
                int an = (a.flags & kAdmit) ? n : 0;
                const long long room = P.cap - A.pin_c;
                if (a.flags & kTruncate) an = (int)room;
                if (a.flags & kWarmupRoom) an = (int)min((long long)n, room);
                A.admit_n = an;
                A.anchor = a.anchor < 0 ? an : a.anchor;
            }
            if ((a.flags & kDispatch) && A.svc_b) commit_observe(P, a, dispatch_tick, A, B.cls);
        }
        __syncthreads();
        if (tid == 0) {  // phase 0 is complete: publish for the speculative scanners
            __threadfence();
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&C->p0_seq), "l"(a.seq) : "memory");
        }
        stamp(A, 0);
        pstamp(P, 5);
        if (tid == 0) tstamp(P, a.seq, 2);
    }
    if (tid == 0) {
        S.spec = 0;
        S.cls_ready = 1;
    }
    __syncthreads();

    // ---- pipelined launch: CTAs kStream0.. stream the pool for the NEXT admission while CTA 0
    // serves this one from the previous launch's prescan, which CTA kSvcL finalizes and validates
    // meanwhile (service_lists); CTA kSvcQ applies the previous admission's table updates
    bool run_loop = true;
    bool pending_rescan = false;  // CTA 0: the last pass must be redone (safe, no hints)
    if (pre_avail) {
        if (blockIdx.x != 0) {
            if (blockIdx.x == kSvcQ)
                service_queue(P, a, Red);
            else if (blockIdx.x == kSvcL)
                service_lists(P, a, B, Sel, Red, dsm, par_prev);
            else if (blockIdx.x == kSvcB) {
                if ((a.flags & kDispatch) && P.policy == 1 && a.next >= 0 && __ldcg(&C->win_size) <= kBfsPre)
                    service_learner(P, a, dsm, Red);
            }
            else {
                if (P.dbg_warps > 1) {  // experiment (CS_DEBUG_WARPS=us): start the stream later
                    const unsigned long long t = gtimer();
                    while (gtimer() - t < 1000ull * (unsigned long long)P.dbg_warps) __nanosleep(500);
                }
                prescan_pass(P, B, S, dsm, par_next, P.stream_generic != 0, a.seq);
            }
            // The verdict word is (seq << 2) | verdict. A later admission's verdict means this
            // one's was "done": a "join the command loop" verdict holds CTA 0 in this admission
            // until every CTA joined (the admission server lets CTA 0 run ahead otherwise).
            __shared__ int join;
            progress(a.seq, 4);
            if (tid == 0) {
                P.dbg[blockIdx.x * 16 + 4] = gtimer();
                unsigned long long spins = 0, w;
                while (((w = ld_acquire_u64(&C->verdict_w)) >> 2) < a.seq) {
                    if (++spins > 4096) __nanosleep(128);
                    if (spins > (1ull << 28)) trap_at(108);
                }
                join = (w >> 2) == a.seq && (w & 3ull) == 2ull ? 1 : 0;
                P.dbg[blockIdx.x * 16 + 5] = gtimer();
                if (blockIdx.x == kStream0) tstamp(P, a.seq, 6);
            }
            __syncthreads();
            run_loop = join != 0;
            progress(a.seq, run_loop ? 6 : 5);
            if (!run_loop) return;
        } else {
            if (tid == 0) {  // this launch's scoring pass is the prescan
                A.scans += 1;
                atomicAdd(reinterpret_cast<unsigned long long*>(&C->scans), 1ull);
                atomicAdd(reinterpret_cast<unsigned long long*>(&C->scanned_slots), (unsigned long long)P.cap);
                A.need_full = 0;
            }
            __syncthreads();
            bool need_loop = false;
            if (A.started && !A.error && A.admit_n > 0) {
                replay_prologue(P, Rp, A, Red, a.seq);
                stamp(A, 1);
                pstamp(P, 6);
                const bool need0 = C->resident + Rp.absent > P.cap;
                const bool ok = !need0 ? true : es.ok ? consume_svc(P, a, es, Rp, B, S, Red) : false;
                if (ok && need0 && es.ok && P.dbg_check) debug_check_e(P, es, Rp, B, S, a);
                stamp(A, 3);
                pstamp(P, 9);
                if (ok) replay_apply(P, a, Rp, A, NL, need0, Red, true, true);
                pstamp(P, 10);
                if (tid == 0) {
                    if (ok && !A.need_full) {
                        A.chunk = 1;
                        atomicAdd(reinterpret_cast<unsigned long long*>(&C->pre_used), 1ull);
                    } else {
                        atomicAdd(reinterpret_cast<unsigned long long*>(&C->pre_fallbacks), 1ull);
                    }
                }
                __syncthreads();
                stamp(A, 4);
                need_loop = A.chunk * kChunk < A.admit_n;
            }
            if (tid == 0) {
                const unsigned long long w = (a.seq << 2) | (need_loop ? 2ull : 1ull);
                __threadfence();
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&C->verdict_w), "l"(w) : "memory");
            }
            run_loop = need_loop;
        }
    }

    // ---- speculative first pass: every CTA but 0 starts scanning at once, concurrently with
    // phase 0. Slots phase 0 may change are left out and restaged by CTA 0 with their new
    // state; agent-carrying slots are classified once phase 0 has fixed the survival classes.
    if (!pre_avail && (a.flags & kSpeculate) && gridDim.x > 1) {
        const int keep0 = min(a.n, kChunk);
        int need_scan0 = 0;
        if (tid == 0) {
            S.spec = 1;
            S.cls_ready = blockIdx.x == 0 ? 1 : 0;
        }
        if (blockIdx.x == 0) build_xset(P, a, S);
        for (int x = tid; x < a.n_agents; x += T) B.cls[x] = blockIdx.x == 0 ? __ldcg(P.cls + x) : (unsigned char)kPend;
        if (blockIdx.x == 0) {
            const int hi0 = min(A.admit_n, kChunk);
            long long absent = 0;
            for (int j = tid; j < hi0; j += T) absent += P.p_slot[j] == kNoSlot ? 1 : 0;
            absent = block_sum(absent, Red);
            need_scan0 = C->resident + absent > P.cap ? 1 : 0;
            if (tid == 0) {
                A.scans += 1;
                atomicAdd(reinterpret_cast<unsigned long long*>(&C->scans), 1ull);
                atomicAdd(reinterpret_cast<unsigned long long*>(&C->scanned_slots), (unsigned long long)P.cap);
                C->keep = keep0;  // a rescan of this chunk keeps the same candidate count
            }
        }
        if (tid < NL) S.hinted[tid] = P.ghint[tid] < kNoBound ? 1 : 0;  // before any finalizer rewrites it
        const int slow = __syncthreads_or(tid < NL && !(P.ghint[tid] < kNoBound) && !P.gsmall[tid]);
        if (blockIdx.x == 0) replay_prologue(P, Rp, A, Red, a.seq);  // the lists are not needed for it
        stamp(A, 1);
        scan_pass(P, NL, keep0, B, S, Sel, dsm, !slow, a);
        grid_barrier(C);
        if (tid == 0) P.dbg[blockIdx.x * 16 + 4] = gtimer();
        stamp(A, 2);
        // list owners: CTA 0 selects class E (the one the bulk replay consumes), CTA 1 the
        // resident list, CTAs 2.. the other classes; CTA 0 waits only for the resident list
        const int Ev = P.e_max, Rv = NL - 1;
        int mine = 0;
        for (int l = 0; l < NL; ++l) {
            const int owner = (l == Ev ? 0 : l == Rv ? 1 : 2 + l) % (int)gridDim.x;
            if (owner != (int)blockIdx.x) continue;
            finalize_list(P, l, NL, keep0, B, Sel);
            ++mine;
            if (l == Rv && tid == 0) {
                __threadfence();
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&C->r_seq), "l"(a.seq) : "memory");
            }
        }
        if (tid == 0 && blockIdx.x < 2) P.dbg[16 + 10 + blockIdx.x] = gtimer();  // finalize ends
        if (blockIdx.x != 0) {
            if (tid == 0 && mine) {
                __threadfence();
                atomicAdd(&C->fin_done, (unsigned int)mine);
            }
        } else {
            // a hinted list that came up short (finalize_list's test, from the counts alone)
            const int short_hint = __syncthreads_or(tid < NL && S.hinted[tid] &&
                                                    *(volatile int*)(P.gcount + tid) < keep_of(tid, NL, keep0));
            if (tid == 0) {
                const unsigned long long tw = gtimer();
                unsigned long long spins = 0;
                while (ld_acquire_u64(&C->r_seq) != a.seq) {
                    if (++spins > 4096) __nanosleep(64);
                    if (spins > (1ull << 27)) trap_at(109);
                }
                __threadfence();
                A.ph[15] += gtimer() - tw;  // instrumentation: CTA 0 waiting for the resident list
            }
            if (tid == 0) A.fin_want = NL - mine;
            __syncthreads();
            stamp(A, 3);
            pending_rescan = short_hint || *(volatile int*)&C->rescan != 0;
            const bool stop = !A.started || A.error || A.admit_n <= 0;
            if (!pending_rescan && !stop) {
                replay_apply(P, a, Rp, A, NL, need_scan0 != 0, Red, true);
                if (tid == 0) A.chunk = 1;
                __syncthreads();
                stamp(A, 4);
            }
            // every finalizer of this pass is done before the command loop resets its state
            if (tid == 0) {
                unsigned long long spins = 0;
                while (ld_acquire(&C->fin_done) < (unsigned int)A.fin_want) {
                    if (++spins > 4096) __nanosleep(64);
                    if (spins > (1ull << 27)) trap_at(110);
                }
            }
            __syncthreads();
        }
        if (tid == 0) S.spec = 0;
        __syncthreads();
    }

    // ---- command loop. CTA 0 decides the next step (scan pass of a chunk, or done); every CTA
    // scans; CTAs 0..NL-1 select one list each; only CTA 0 consumes the lists, so it waits on
    // a counter instead of a grid barrier; CTA 0 replays. Per chunk: 2 grid barriers.
    const bool looped = run_loop;
    for (; run_loop;) {
        if (blockIdx.x == 0) {
            const bool stop = !A.started || A.error || A.chunk * kChunk >= A.admit_n;
            if (stop) {
                if (tid == 0) {
                    C->done = 1;
                    if (pre_run && !pre_avail) hints_from_fin(P, NL, C->keep, par_next);  // for the prescan below
                }
            } else if (pending_rescan) {
                // a hint was too tight (or the fast pass overflowed): same chunk, safe pass
                if (tid < NL) {
                    P.ghint[tid] = kNoBound;
                    P.gbound[tid] = kNoBound;
                    P.gcount[tid] = 0;
                    P.gmaxk[tid] = 0ull;
                }
                if (tid == 0) {
                    C->rescan = 0;
                    C->fin_done = 0u;
                    C->pass = 1;
                    C->fast = 0;
                    C->need_scan = 1;
                    C->rescans += 1;
                    A.ph[13] += 1;
                }
            } else {
                const int lo = A.chunk * kChunk, hi = min(A.admit_n, lo + kChunk);
                long long absent = 0;
                for (int j = lo + tid; j < hi; j += T) absent += P.p_slot[j] == kNoSlot ? 1 : 0;
                absent = block_sum(absent, Red);
                const int need_scan = C->resident + absent > P.cap ? 1 : 0;
                if (tid < NL && need_scan) {
                    P.gbound[tid] = kNoBound;
                    P.gcount[tid] = 0;
                    P.gmaxk[tid] = 0ull;
                }
                // warp-specialized pass only when every list has a hint or is known small
                const int slow = __syncthreads_or(tid < NL && !(P.ghint[tid] < kNoBound) && !P.gsmall[tid]);
                if (tid == 0) {
                    C->rescan = 0;
                    C->fin_done = 0u;
                    C->pass = 0;
                    C->fast = slow ? 0 : 1;
                    C->need_scan = need_scan;
                    C->keep = hi - lo;
                    if (need_scan) {
                        A.scans += 1;
                        atomicAdd(reinterpret_cast<unsigned long long*>(&C->scans), 1ull);
                        atomicAdd(reinterpret_cast<unsigned long long*>(&C->scanned_slots), (unsigned long long)P.cap);
                    }
                }
            }
        }
        grid_barrier(C);
        stamp(A, 1);
        if (*(volatile int*)&C->done) break;
        const int need_scan = *(volatile int*)&C->need_scan;
        const int keep = *(volatile int*)&C->keep;
        if (need_scan) {
            const int pass = *(volatile int*)&C->pass;
            for (int x = tid; x < a.n_agents; x += T) B.cls[x] = P.cls[x];
            __syncthreads();
            scan_pass(P, NL, keep, B, S, Sel, dsm, pass == 0 && *(volatile int*)&C->fast, a);
            if (blockIdx.x == 0 && tid == 0) {
                A.ph[9] += S.flush_ns;
                A.ph[10] += S.flushes;
            }
            grid_barrier(C);
            if (tid == 0) P.dbg[blockIdx.x * 16 + 4] = gtimer();
            stamp(A, 2);
            int mine = 0;
            for (int l = blockIdx.x; l < NL; l += gridDim.x) {
                finalize_list(P, l, NL, keep, B, Sel);
                ++mine;
            }
            if (blockIdx.x != 0) {
                if (tid == 0 && mine) {
                    __threadfence();
                    atomicAdd(&C->fin_done, (unsigned int)mine);
                }
            } else {
                if (tid == 0) {  // CTA 0 waits for the other lists' selects
                    const unsigned int want = (unsigned int)(NL - mine);
                    unsigned long long spins = 0;
                    while (ld_acquire(&C->fin_done) < want) {
                        if (++spins > 4096) __nanosleep(64);
                        if (spins > (1ull << 27)) trap_at(111);
                    }
                    __threadfence();
                }
                __syncthreads();
                stamp(A, 3);
                pending_rescan = pass == 0 && *(volatile int*)&C->rescan;
            }
        }
        if (blockIdx.x == 0 && !pending_rescan) {
            replay_prologue(P, Rp, A, Red, a.seq);
            replay_apply(P, a, Rp, A, NL, need_scan != 0, Red);
            if (tid == 0) A.chunk += 1;
            __syncthreads();
            stamp(A, 4);
        }
    }
    // Every CTA has read C->done before CTA 0 can reset the loop's control words: in the admission
    // server CTA 0 starts the next admission (its phase 0 resets them) without a grid barrier.
    if (looped) grid_barrier(C);

    // ---- no usable prescan came in: CTAs kStream0.. now prescan for the next admission
    if (pre_run && !pre_avail && blockIdx.x != 0) {
        if (blockIdx.x >= kStream0) prescan_pass(P, B, S, dsm, par_next, true, a.seq);
        return;
    }
    if (pre_run && !pre_avail && blockIdx.x == 0 && tid == 0) {
        A.scans += 1;
        atomicAdd(reinterpret_cast<unsigned long long*>(&C->scans), 1ull);
        atomicAdd(reinterpret_cast<unsigned long long*>(&C->scanned_slots), (unsigned long long)P.cap);
    }

    // ---- epilogue (CTA 0): EngineSim::admit unpins at once; pins out; status
    if (blockIdx.x == 0) {
        if (A.started && !A.error && (a.flags & kUnpinAfter)) {  // (pins_out was written by apply)
            long long dec = 0;
            for (int i = tid; i < A.admit_n; i += T) {
                const unsigned int s = P.p_slot[i];
                {
                    if (atomicSub(&P.refs[s], 1u) == 1u) {
                        pk_unpinned(P, s);
                        ++dec;
                        if (P.dbg_unpin) P.dbg_unpin[s] = (a.seq << 8) | 3u;
                    }
                }
            }
            dec = block_sum(dec, Red);
            if (tid == 0) {
                A.pin_c -= dec;
                C->pinned = A.pin_c;  // (a store, not a read-modify-write round trip)
            }
        }
        __syncthreads();
        queue_ready(P, a, A);  // (an admission that applied nothing: the counters are reset here)
        stamp(A, 5);
        pstamp(P, 11);
        if (tid == 0 && a.status && !A.st_done) {
            write_status(P, a, A);
            __threadfence_system();  // status and victims reach the host before the flag
            *(volatile unsigned long long*)&a.status->done_seq = a.seq;
        }
        pstamp(P, 12);
        // per-list scan state for the next launch (a speculative pass starts without a prep)
        if (tid < kMaxLists) {
            P.gbound[tid] = kNoBound;
            P.gcount[tid] = 0;
            P.gmaxk[tid] = 0ull;
        }
        if (tid == 0) {
            C->fin_done = 0u;
            C->rescan = 0;
        }
    }
}

__global__ void __launch_bounds__(kThreads + 32, 1) admit_kernel(DevPool P, AdmitArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ ScanSmem S;
    __shared__ SelectSmem Sel;
    __shared__ RedSmem Red;
    __shared__ AdmSmem A;
    if (threadIdx.x == 0) A.srv_t0 = 0;
    admit_body(P, a, dsm, S, Sel, Red, A);
}

// ------------------------------------------------------------------ hash-sharded pool

#include "cs_shard.cuh"

// ------------------------------------------------------------------ Belady baseline (policy 3)

#include "cs_belady.cuh"

// ------------------------------------------------------------------ device-resident scheduler

#include "cs_engine_dev.cuh"

// ------------------------------------------------------------------ admission server


// One persistent cooperative launch serves every admission the host scheduler posts: CTA 0 polls
// the host-mapped mailbox, relays the arguments (and, on the end-to-end path, copies the
// admission's prompt blocks from pinned host memory into device scratch), one grid barrier
// orders everything the previous admission wrote, and every CTA runs admit_body exactly as
// admit_kernel would. The host's scheduler loop is unchanged; what disappears per admission is
// the cooperative launch itself and the host's enqueue behind the previous kernel.
__global__ void __launch_bounds__(kThreads + 32, 1) server_kernel(DevPool P, SrvMailbox* mb, AdmitArgs* dargs,
                                                                  unsigned long long post0) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ ScanSmem S;
    __shared__ SelectSmem Sel;
    __shared__ RedSmem Red;
    __shared__ AdmSmem A;
    __shared__ AdmitArgs a;
    const int tid = threadIdx.x, T = blockDim.x;
    Ctrl* C = P.ctrl;
    for (unsigned long long post = post0;; ++post) {
        AdmitArgs* dslot = dargs + (post & 1ull);  // (double-buffered: never rewritten while read)
        if (blockIdx.x == 0) {
            // the host posts within microseconds while its scheduler loop runs (a process that
            // dies takes its context, and this kernel, with it). The first kArgWords threads poll
            // the tagged pairs: one round that sees every tag == post carries the arguments too.
            static_assert(kArgWords <= kThreads, "one tagged pair per polling thread");
            {
                unsigned long long spins = 0;
                for (;;) {
                    int mine = 1;
                    unsigned long long w = 0;
                    if (tid < kArgWords) {
                        unsigned long long t;
                        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];"
                                     : "=l"(t), "=l"(w)
                                     : "l"(&mb->pair[tid])
                                     : "memory");
                        mine = t == post ? 1 : 0;
                    }
                    if (__syncthreads_and(mine)) {
                        if (tid < kArgWords) {
                            reinterpret_cast<unsigned long long*>(&a)[tid] = w;
                            reinterpret_cast<unsigned long long*>(dslot)[tid] = w;
                        }
                        break;
                    }
                    if (++spins > 64) __nanosleep(100);
                }
            }
            __syncthreads();
            if (tid == 0) {
                A.srv_t0 = gtimer();
                tstamp(P, a.seq, 0);
            }
            if (a.stage_src != nullptr && !(a.flags & kSrvStop)) {  // host -> device prompt blocks
                const unsigned int* hs = reinterpret_cast<const unsigned int*>(a.stage_src);
                unsigned int* dk = reinterpret_cast<unsigned int*>(const_cast<unsigned long long*>(a.keys));
                for (int i = tid; i < 3 * a.n; i += T) dk[i] = __ldcv(hs + i);
            }
            // hand the admission to the other CTAs without waiting for them: they finished the
            // previous one among themselves (prescan_barrier below), and everything CTA 0 wrote
            // in it is ordered before this release
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&C->srv_go), "l"(post) : "memory");
            }
        } else {
            progress(post, 9);
            prescan_barrier(C);  // CTAs 1..: every one of them finished the previous admission
            progress(post, 10);
            if (tid == 0) {
                unsigned long long spins = 0;
                while (ld_acquire_u64(&C->srv_go) != post)
                    if (++spins > 64) __nanosleep(100);
            }
            __syncthreads();
            for (int i = tid; i < kArgWords; i += T)
                reinterpret_cast<unsigned long long*>(&a)[i] = __ldcg(reinterpret_cast<const unsigned long long*>(dslot) + i);
            __syncthreads();
        }
        if (a.flags & kSrvStop) {
            if (blockIdx.x == 0 && tid == 0 && a.status) {
                a.status->srv_t0 = A.srv_t0;
                __threadfence_system();
                *(volatile unsigned long long*)&a.status->done_seq = a.seq;
            }
            return;
        }
        admit_body(P, a, dsm, S, Sel, Red, A);
        __syncthreads();
        if (blockIdx.x == 0 && tid == 0) tstamp(P, a.seq, 5);
        fence_proxy_async_smem();  // this admission's generic shared-memory use before the next TMA writes
    }
}

cudaError_t launch_server(const DevPool& P, SrvMailbox* mb_dev, AdmitArgs* args_dev, unsigned long long first_post,
                          const LaunchCfg& lc, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(server_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lc.smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    DevPool p = P;
    SrvMailbox* m = mb_dev;
    AdmitArgs* d = args_dev;
    unsigned long long q = first_post;
    void* args[] = {&p, &m, &d, &q};
    return cudaLaunchCooperativeKernel((const void*)server_kernel, dim3(lc.grid), dim3(lc.threads), args, lc.smem, s);
}

// ------------------------------------------------------------------ host side

cudaError_t set_trap_word(unsigned long long* host_mapped, int progress_on) {
    const cudaError_t e = cudaMemcpyToSymbol(cs_trap_host, &host_mapped, sizeof(host_mapped));
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbol(cs_progress_on, &progress_on, sizeof(progress_on));
}

LaunchCfg admit_launch_config(const DevPool& P, int device, int want_grid) {
    LaunchCfg lc{0, 0, 0, 0};
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return lc;
    const size_t smem = kDynSmem;
    if (smem + sizeof(ScanSmem) + sizeof(SelectSmem) + sizeof(RedSmem) + sizeof(AdmSmem) > prop.sharedMemPerBlockOptin)
        return lc;
    if (cudaFuncSetAttribute(admit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return lc;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, admit_kernel, kThreads + 32, smem) != cudaSuccess ||
        occ < 1)
        return lc;
    int grid = prop.multiProcessorCount * occ;
    if (want_grid > 0 && want_grid < grid) grid = want_grid;
    lc.grid = grid;
    lc.threads = kThreads + 32;  // 16 consumer warps + 1 TMA producer warp
    lc.cap_per_list = 0;
    lc.smem = smem;
    return lc;
}

cudaError_t launch_admit(const DevPool& P, const AdmitArgs& a, const LaunchCfg& lc, int grid, cudaStream_t s) {
    DevPool p = P;
    AdmitArgs aa = a;
    void* args[] = {&p, &aa};
    if (grid <= 1) return cudaLaunchKernel((const void*)admit_kernel, dim3(1), dim3(lc.threads), args, lc.smem, s);
    return cudaLaunchCooperativeKernel((const void*)admit_kernel, dim3(grid), dim3(lc.threads), args, lc.smem, s);
}

}  // namespace csb
