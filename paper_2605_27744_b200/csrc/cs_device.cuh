// Device-side layout of the CacheSage block pool in HBM and the small helpers every kernel
// shares. See DESIGN.md §3 for the byte layout and the roofline each kernel is held to.
#pragma once

#include <cstddef>
#include <cstdint>

namespace csb {

// ---------------------------------------------------------------- constants

constexpr unsigned long long kFreeTick = ~0ull;  // last_touch of a free slot (never a real tick)
constexpr unsigned long long kNoBound = ~0ull - 1;  // "no threshold": every real tick passes, free slots do not
constexpr unsigned int kNoAgent = 0xFFFFFFFFu;   // Block::agent == nullopt (types.hpp:45)
constexpr unsigned int kNoSlot = 0xFFFFFFFFu;
constexpr unsigned int kSlotEmpty = 0xFFFFFFFFu;  // table entry never used
constexpr unsigned int kSlotTomb = 0xFFFFFFFEu;   // table entry erased
constexpr unsigned int kSlotClaim = 0xFFFFFFFDu;  // being written by an inserter

constexpr int kMaxLists = 24;        // survival classes (e_max + 1) + 1 resident-oldest list
constexpr int kChunk = 128;          // prompt blocks replayed per scan pass (candidates per class)
constexpr int kSlack = 128;          // staged candidates tolerated before a CTA trims
constexpr int kMaxAgents = 4096;     // dense A x A learner counts
constexpr int kMaxPending = 64;      // queued warmups between drains
constexpr int kPhases = 16;          // per-phase device timers reported with each admission

// hashing.hpp:13-14 + the identity seed of cachesage_policy.cpp:26
constexpr unsigned long long kHashSeed = 0x5ca9e5a6e0f1c3b7ull;
constexpr unsigned long long kRootParent = 0x9d2c5680f0a5b4d1ull;
constexpr unsigned long long kGolden = 0x9e3779b97f4a7c15ull;
constexpr unsigned long long kIdentitySalt = 0xa9e0c7d35b1f64e9ull;

// splitmix64 finalizer (hashing.hpp:17-22)
__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x += kGolden;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// ---------------------------------------------------------------- HBM layout

// One open-addressing entry of the block table: BlockKey -> slot. 16 B, one sector per probe.
struct __align__(16) TableEntry {
    unsigned long long key;
    unsigned int slot;  // kSlotEmpty / kSlotTomb / kSlotClaim or a pool slot
    unsigned int pad;
};

// Mutable scalars of the pool + learner. Lives in device memory; only kernels write it.
struct Ctrl {
    long long resident;      // |cache_|
    long long pinned;        // pinned_count_ (engine.hpp:177)
    long long free_top;      // entries on the free-slot stack
    long long tombstones;
    unsigned long long n_ev; // eviction log length
    long long scans;
    long long scanned_slots;
    unsigned long long rebuilds;
    long long win_head, win_size;
    unsigned long long recorded;  // TransitionLearner::recorded_ (transitions_recorded)
    int cur_agent;           // CacheSagePolicy::current_ (-1 = none)
    int reach_built;         // !reach_.empty()
    int step_warmups;
    int n_pend;
    int pend_target[kMaxPending];
    unsigned long long pend_tick[kMaxPending];
    // per-launch control of the cooperative admission kernel
    unsigned int bar_count;
    unsigned int bar_gen;
    int done;
    int need_scan;
    int keep;
    int chunk_lo, chunk_hi;
    int error;
    int rescan;        // a hinted list came up short: scan again without hints
    int fast;          // this chunk's first scan pass runs warp-specialized (no per-tile barrier)
    unsigned int fin_done;  // lists finalized in this pass (CTA 0 waits for all, no grid barrier)
    int pass;          // scan pass of the current chunk (1 = safe, no hints)
    long long rescans; // instrumentation
    unsigned long long p0_seq;  // AdmitArgs::seq of the launch whose phase 0 finished
    int tq_erase, tq_insert;    // block-table updates queued by the last admission (applied next)
    unsigned long long r_seq;   // AdmitArgs::seq once the resident-oldest list is final
    // prescan: the next admission's scoring pass, run by CTAs 1.. of this launch while CTA 0
    // serves this admission; double-buffered by launch-sequence parity
    unsigned int pbar_count, pbar_gen;  // barrier of the prescan CTAs
    // service CTAs of a pipelined launch -> CTA 0 (AdmitArgs::seq, release/acquire):
    unsigned long long svc_q_seq;       // CTA kSvcQ applied the previous admission's table queue
    unsigned long long svc_l_seq;       // CTA kSvcL published the validated prescan lists
    // CTA 0 -> prescan CTAs: (AdmitArgs::seq << 2) | verdict (1: done, 2: everyone joins the
    // command loop), one word so a reader never pairs one admission's seq with another's verdict
    unsigned long long verdict_w;
    long long pre_used, pre_fallbacks, pre_badcnt;  // instrumentation
    unsigned long long svc_b_seq;  // CTA kSvcB -> CTA 0: LearnSpec / spec_hop are this admission's
    unsigned long long srv_go;     // admission server: CTA 0 -> CTAs 1..: the arguments of this post
};

// prescan list lengths: E (agentless unpinned) and R (resident) keep the kPreK oldest; the
// agent-carrying unpinned slots (classified by the consumer, after its BFS) are kept whole
constexpr int kPreK = 192;  // >= kChunk + 1 list entries plus the front the previous admission evicts
constexpr int kPendCap = 4096;
// Roles in a pipelined launch (admit_kernel): CTA 0 serves this admission; CTA kSvcQ applies the
// previous admission's queued block-table updates; CTA kSvcL finalizes and validates the previous
// launch's prescan for CTA 0; CTAs kStream0.. stream the pool for the next admission.
// CTA kSvcB runs this admission's observe(AgentDispatch) speculatively (the learner service).
constexpr int kSvcQ = 1, kSvcL = 2, kSvcB = 3, kStream0 = 4;

// The learner service's result for CTA 0 (service_learner): observe(AgentDispatch{prev, next})
// computed on the learner state as this dispatch's record will leave it, committed by CTA 0 only
// if the request starts. The BFS hops go to DevPool::spec_hop.
// Every 16-byte word carries the admission's seq next to its payload, so CTA 0 reads the whole
// result in one round of 16-byte loads and knows it is this admission's (no flag round trip).
struct LearnSpec {
    unsigned long long seq0;
    int changed;              // CacheSagePolicy::current_ != next: the reachability was rebuilt
    int oa;
    unsigned long long seq1;
    int ob;                   // (oa, ob): the window pair the record pushes out of a full window
    int best_b;               // argmax_row(next) after the record (-1: no positive count)
    unsigned long long seq2;
    unsigned int best_c, total_next;
};
static_assert(sizeof(LearnSpec) == 48, "three tagged 16-byte words");
constexpr int kRawCap = 6144;  // raw prescan candidates per streaming CTA (its staging capacity)
// header of one streaming CTA's raw prescan output
struct RawHdr {
    unsigned long long seq;  // AdmitArgs::seq of the launch that wrote it
    int n;                   // staged candidates (every list, staging order)
    int bad;                 // staging overflowed: the prescan is unusable
};

// ---------------------------------------------------------------- hash-sharded pool
// A pool of budget N split over G GPUs: a block lives on shard owner(key) = (key >> 40) % G.
// Slots are named across shards by gslot = shard << kShardBits | local slot.
constexpr int kShardBits = 29;
constexpr unsigned int kShardMask = (1u << kShardBits) - 1u;
constexpr int kMaxShards = 8;
constexpr unsigned int kNewRemote = 0xFFFFFFFCu;  // new block inserted on another shard

__host__ __device__ __forceinline__ int shard_owner(unsigned long long key, int world) {
    return (int)((key >> 40) % (unsigned long long)world);
}

// exchange 1 (after the probe): per shard a header and, per prompt position, the owner's slot
struct ShardHdr {
    long long resident, pinned;
};
struct ShardPos {
    unsigned int gslot;  // kNoSlot: not owned here or not resident
    unsigned int refs0;
};
// exchange 2 (after each scan): per shard and list the shard's keep oldest candidates, sorted
struct ShardCand {
    unsigned long long lt, key;
    unsigned int gslot, pad;
};
struct ShardLists {
    int n[kMaxLists];
    ShardCand c[kMaxLists][kChunk + 1];
};
// bytes of one shard's list message with NL lists in use: the counts and the first NL lists
// (the exchange moves only those; receivers index shard r at r * this stride)
__host__ __device__ __forceinline__ size_t shard_lists_bytes(int NL) {
    return (offsetof(ShardLists, c) + (size_t)NL * (kChunk + 1) * sizeof(ShardCand) + 15) & ~(size_t)15;
}
// replicated admission state (identical on every shard), carried between the admission's kernels
struct ShardState {
    unsigned long long tick, first_touch;
    long long cached, res_g, pinned_g, n_ev_adm;
    int started, error, first_miss, admit_n, anchor, needed, warm_issued, chunk, need_scan, scans;
};

// ---------------------------------------------------------------- Belady (policy 3)
// BeladyPolicy (baselines.cpp:34-70): a block's score depends on the next request that
// references it, so the pool keeps per slot that request id (kNoRef: never again) and the key's
// index into a CSR of request ids per unique key, built once from the materialized requests.
constexpr unsigned int kNoRef = 0xFFFFFFFFu;
constexpr int kBelCand = 4096;   // candidates one selection pass hands to the replay
constexpr int kBelPasses = 16;   // 8-bit digits of the (score, last_touch) composite

struct BelCand {
    unsigned long long hi, lo;  // order-preserving score bits, last_touch
    unsigned int slot, pad;
};

struct BelCtl {
    unsigned long long hi_or, hi_and, lo_or, lo_and;  // over this pass's candidates
    unsigned long long m;                             // candidates (resident, unpinned)
    int n_cand;                                       // compacted
    int pos;                                          // next prompt block of the replay
    int more;                                         // 1: the replay needs another pass
    int started, error, first_miss, admit_n, anchor, needed, scans;
    long long cached, n_ev_adm;
    unsigned long long tick;                          // before admit_pinned's touches
    unsigned int hist[kBelPasses][256];
};

struct DevPool {
    long long cap;            // slots == EngineConfig::budget_blocks
    long long cap_scan;       // cap rounded up to 64: the SoA tail is padded with free slots
    int policy;               // 0 lru, 1 cachesage, 3 belady
    int e_max;
    int n_lists;              // e_max + 2 (classes 0..e_max, resident list last)
    int a_cap;
    double tau, w_pred, min_conf;
    double wsurv[kMaxLists];  // fl(w_pred * survival(c)) per class c <= e_max, host-computed (no FMA)
    unsigned long long min_row;
    int budget_per_step;
    long long window;
    unsigned long long tmask;

    // SoA pool (the exact state) + the packed scan word of every slot (pk_make): the scan
    // streams 8 B per slot instead of lt/agent/refs' 16 B
    unsigned long long* pk;
    unsigned long long* lt;
    unsigned int* agent;
    unsigned int* refs;
    unsigned long long* key;
    int* tokens;
    TableEntry* table;
    unsigned int* free_stack;
    unsigned long long* evlog;
    long long evlog_cap;

    // learner (dense over agent indices)
    unsigned int* counts;     // a_cap * a_cap
    unsigned int* totals;     // a_cap
    int* win_a;               // window ring
    int* win_b;
    unsigned char* hop;       // a_cap
    unsigned char* cls;       // a_cap: survival class used by the scan
    unsigned long long* agent_ids;

    // scan scratch
    unsigned long long* gbound;   // [kMaxLists] running upper bound of each list's keep-th value
    int* gcount;                  // [kMaxLists]
    unsigned long long* ghint;    // [kMaxLists] acceptance hint carried to the next scan (~0 = none)
    unsigned long long* gmaxk;    // [kMaxLists] max over CTAs of their local keep-th value
    unsigned int* grej;           // unused (kept for layout stability)
    unsigned char* gsmall;        // [kMaxLists] list had fewer than keep members in its last scan
    unsigned long long* gmin;     // [kMaxLists][grid] each CTA's smallest candidate per list (kNoBound: none)
    unsigned long long* gbuf_lt;  // [kMaxLists][gcap]
    unsigned int* gbuf_slot;
    long long gcap;
    unsigned long long* fin_lt;   // [kMaxLists][kChunk + 2]
    unsigned int* fin_slot;
    int* fin_n;

    unsigned long long* dbg;      // [grid * 8] per-CTA instrumentation timestamps
    int dbg_warps;                // CS_DEBUG_WARPS: CTA 0's per-warp phase-0 round ends (tools)

    // per-admission prompt scratch (grown by the host)
    unsigned int* p_slot;
    unsigned int* p_refs0;
    long long p_cap;
    // block-table updates of the last admission, applied at the start of the next launch
    // (erase keys at [0, p_cap), insert keys at [p_cap, 2 p_cap) with their slots)
    unsigned long long* tq_key;
    unsigned int* tq_slot;

    Ctrl* ctrl;
    LearnSpec* spec;        // the learner service's speculative observe (Ctrl::svc_b_seq)
    ulonglong2* spec_hop;     // [a_cap / 8]: {seq, 8 BFS hops} per 16-byte word

    // raw prescan output, per launch parity and streaming CTA: the CTA's staged candidates in
    // staging order ([2][raw_grid][kRawCap] lt / slot / list id / agent) and its header
    unsigned long long* raw_lt;
    unsigned int* raw_slot;
    unsigned char* raw_list;
    unsigned int* raw_agent;
    RawHdr* raw_hdr;  // [2][raw_grid]
    int raw_grid;
    // the list service's output for this launch's CTA 0: [list E, R, pending][kPendCap] (E and
    // R sorted, the first kPreK), validity against the pool at launch start, E keys, counts
    // pl_n[0..2] + usable flag pl_n[3], completeness thresholds pl_T[0..2]
    unsigned long long* pl_lt;
    unsigned int* pl_slot;
    unsigned int* pl_agent;
    unsigned char* pl_ok;
    unsigned long long* pl_key;
    int* pl_n;
    unsigned long long* pl_T;
    unsigned long long* pre_hint;  // [parity][3]: acceptance thresholds of the prescan of a launch of that parity
    int dbg_check;  // debug: brute-force check of the prescan consumer's list E (small pools)
    int stream_generic;  // stream the pool with L2 loads instead of TMA (the persistent engine kernel)
    unsigned long long* dbg_unpin;  // debug: per slot (admission seq << 8 | source) of its last unpin

    // hash-sharded mode (world > 1 or an explicit shard): this shard's rank, the shard count,
    // the GLOBAL budget, the exchange buffers and the replicated admission state
    int rank, world;
    long long gbudget;
    unsigned char* sh_send1;   // ShardHdr + ShardPos[p_cap]
    unsigned char* sh_recv1;   // world x the above
    ShardLists* sh_send2;
    ShardLists* sh_recv2;      // [world]
    ShardState* sh_state;
    unsigned int* sh_gslot;    // [p_cap] replicated prompt position -> gslot (kNoSlot: absent)
    unsigned int* sh_grefs0;   // [p_cap]

    // Belady (policy 3; cs_belady.cuh)
    unsigned int* bel_nu;             // [cap] next request id that references the slot's block
    unsigned int* bel_kid;            // [cap] unique-key index of the slot's block
    unsigned int* bel_kid_slot;       // [n_kids] slot holding that key (kNoSlot: not resident)
    const unsigned int* bel_ref;      // [n_flat] request ids per key, ascending (CSR)
    const long long* bel_ref_off;     // [n_kids + 1]
    const int* bel_depth;             // [n_kids] chain position of the key's first occurrence
    const unsigned int* bel_kid_of;   // [n_flat] key index of every request block
    unsigned long long* bel_hi;       // [cap] per-pass composite (score bits)
    unsigned long long* bel_lo;       // [cap] per-pass composite (last_touch)
    BelCand* bel_cand;                // [kBelCand]
    BelCtl* bel_ctl;
};

// ---------------------------------------------------------------- packed scan word
// bits 0..39 last_touch (kPkFree: free slot), 40..52 agent index (kPkNoAgent: none), 63 pinned
// (refs > 0). Ticks stay below 2^40 - 1 (the host checks), so the scan's decoded last_touch is
// the exact tick. Every writer of lt / agent / a refs 0 <-> 1 transition keeps it in step.
constexpr unsigned long long kPkLtMask = (1ull << 40) - 1ull;
constexpr unsigned long long kPkFree = kPkLtMask;
constexpr unsigned long long kPkNoAgent = 0x1FFFull;
constexpr unsigned long long kPkPin = 1ull << 63;
constexpr unsigned long long kPkFreeWord = kPkFree | (kPkNoAgent << 40);
constexpr unsigned long long kMaxTick = kPkLtMask - 1ull;

__host__ __device__ __forceinline__ unsigned long long pk_make(unsigned long long lt, unsigned int agent, bool pinned) {
    const unsigned long long l = lt == kFreeTick ? kPkFree : (lt & kPkLtMask);
    const unsigned long long a = agent == kNoAgent ? kPkNoAgent : (unsigned long long)(agent & 0x1FFFu);
    return l | (a << 40) | (pinned ? kPkPin : 0ull);
}

__host__ __device__ __forceinline__ void pk_decode(unsigned long long w, unsigned long long& lt, unsigned int& agent,
                                                   unsigned int& pinned) {
    const unsigned long long l = w & kPkLtMask;
    const unsigned long long a = (w >> 40) & kPkNoAgent;
    lt = l == kPkFree ? kFreeTick : l;
    agent = a == kPkNoAgent ? kNoAgent : (unsigned int)a;
    pinned = (unsigned int)(w >> 63);
}

#ifdef __CUDACC__
// A watchdog that fires (a wait that never ends, a corrupted table) records where before it
// traps: the site code and CTA go to host-mapped memory (cs_trap_word), which outlives the
// context the trap takes down, so the host can name the site in its error.
static __device__ unsigned long long* cs_trap_host;  // (per translation unit; set for cs_admit.cu)
static __device__ int cs_progress_on;  // CS_DEBUG_PROGRESS: per-CTA progress marks in cs_trap_host[1 + cta]
__device__ __forceinline__ void progress(unsigned long long seq, int stage) {
    if (cs_progress_on && threadIdx.x == 0)
        *(volatile unsigned long long*)(cs_trap_host + 1 + blockIdx.x) = (seq << 8) | (unsigned long long)stage;
}
static __device__ __noinline__ void trap_at(int code) {
    unsigned long long* w = cs_trap_host;
    if (w) {
        *(volatile unsigned long long*)w = ((unsigned long long)code << 32) | (unsigned long long)blockIdx.x;
        __threadfence_system();
    }
    __trap();
}

// ---------------------------------------------------------------- block table

__device__ __forceinline__ unsigned long long table_home(unsigned long long key, unsigned long long mask) {
    return mix64(key ^ 0x51afd7ed558ccd1dull) & mask;
}

// Slot of `key` or kNoSlot. Lookups never run concurrently with inserts/erases (phases are
// separated by barriers), so plain loads suffice. The table is kept at most half full of
// live + tombstoned entries (the host rebuilds it past that), so probes always hit an EMPTY
// entry; a probe that wraps the whole table is a corrupted table and traps instead of hanging.
__device__ __forceinline__ unsigned int table_find(const DevPool& P, unsigned long long key) {
    unsigned long long h = table_home(key, P.tmask);
    for (unsigned long long n = 0; n <= P.tmask; ++n) {
        const TableEntry e = P.table[h];
        if (e.slot == kSlotEmpty) return kNoSlot;
        if (e.slot < kSlotClaim && e.key == key) return e.slot;
        h = (h + 1) & P.tmask;
    }
    trap_at(201);
    return kNoSlot;
}

// The same answer with one round trip per 128-byte line instead of per entry, for the
// latency-critical probe of an admission (phase 0): all entries of the line from h on are loaded
// together (L2-coherent 16-byte loads, each an atomic {key, slot} pair) and scanned in probe
// order. Entries may change while they are read (the block-table queue is applied concurrently,
// csrc/cs_admit.cu phase 0); a find of a key the queue does not touch is exact under any
// interleaving (the key's entry precedes every EMPTY on its path and is never moved), and queued
// keys are resolved by the caller's overlay.
__device__ __forceinline__ unsigned int table_find_line(const DevPool& P, unsigned long long key) {
    unsigned long long h = table_home(key, P.tmask);
    for (unsigned long long n = 0; n <= P.tmask; n += 8) {
        const unsigned long long base = h & ~7ull;
        ulonglong2 e[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) e[k] = __ldcg(reinterpret_cast<const ulonglong2*>(P.table + base + k));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (base + k < h) continue;
            const unsigned int slot = (unsigned int)e[k].y;
            if (slot == kSlotEmpty) return kNoSlot;
            if (slot < kSlotClaim && e[k].x == key) return slot;
        }
        h = (base + 8) & P.tmask;
    }
    trap_at(202);
    return kNoSlot;
}

// Lock-free insert of a key known to be absent: claim the first EMPTY or TOMB entry on the
// probe path with a CAS on its slot word, then publish key and slot. Concurrent inserters
// (bulk restore) race only through the CAS. Returns 1 if a tombstone was reused.
__device__ __forceinline__ int table_insert(const DevPool& P, unsigned long long key, unsigned int slot) {
    unsigned long long h = table_home(key, P.tmask);
    for (unsigned long long n = 0; n <= 2 * P.tmask + 64; ++n) {
        unsigned int s = P.table[h].slot;
        if (s == kSlotEmpty || s == kSlotTomb) {
            unsigned int old = atomicCAS(&P.table[h].slot, s, kSlotClaim);
            if (old == s) {
                // Concurrent inserters only read slot words (a CLAIM entry is skipped). A find
                // racing this insert (phase 0) sees CLAIM, or the new slot with the old key
                // (cleared by the erase, never a probed key), or the new pair.
                P.table[h].key = key;
                __threadfence_block();  // the racing finds run in the same CTA (phase 0)
                atomicExch(&P.table[h].slot, slot);
                return s == kSlotTomb ? 1 : 0;
            }
            continue;  // lost the race for this entry: re-read it
        }
        h = (h + 1) & P.tmask;
    }
    trap_at(203);
    return 0;
}

__device__ __forceinline__ void table_erase(const DevPool& P, unsigned long long key) {
    unsigned long long h = table_home(key, P.tmask);
    for (unsigned long long n = 0; n <= P.tmask; ++n) {
        const TableEntry e = P.table[h];
        if (e.slot == kSlotEmpty) return;
        if (e.slot < kSlotClaim && e.key == key) {
            // clear the key first: a find of another key that races a later reuse of this entry
            // (phase 0 overlaps the previous admission's table updates with its probe) must
            // never pair the new slot with the erased key
            P.table[h].key = ~0ull;
            __threadfence_block();  // the racing finds run in the same CTA (phase 0)
            P.table[h].slot = kSlotTomb;
            return;
        }
        h = (h + 1) & P.tmask;
    }
    trap_at(204);
}

__device__ __forceinline__ void pk_unpinned(const DevPool& P, unsigned int s) { atomicAnd(P.pk + s, ~kPkPin); }

// a touch of a resident block (EngineSim::touch): last_touch changes, agent and pin bit do not
__device__ __forceinline__ void pk_touch(const DevPool& P, unsigned int s, unsigned long long lt) {
    P.pk[s] = (P.pk[s] & ~kPkLtMask) | (lt & kPkLtMask);
}

// ---------------------------------------------------------------- exact fp64 scoring

// recency_residual (runtime.cpp:23-32), no contraction.
__device__ __forceinline__ double recency(unsigned long long lt, unsigned long long now, unsigned long long old) {
    if (now <= old) return 1.0;
    if (lt <= old) return 0.0;  // offset 0 -> 0/span = +0.0 exactly (skips the fp64 divide)
    const double span = (double)(now - old);
    const double off = lt >= old ? (double)(lt - old) : 0.0;
    double r = __ddiv_rn(off, span);
    r = r < 0.0 ? 0.0 : r;
    r = r > 1.0 ? 1.0 : r;
    return r;
}

// ReachabilityState::survival (reachability.cpp:17-20) for a hop class.
__device__ __forceinline__ double survival_of_class(int c, int e_max) {
    const int capped = c < e_max ? c : e_max;
    return __dsub_rn(1.0, __ddiv_rn((double)capped, (double)e_max));
}

// CacheSagePolicy::score (cachesage_policy.cpp:79-85) / LruPolicy::score (baselines.cpp:12-14)
__device__ __forceinline__ double score_of(int policy, double w_pred, double surv, unsigned long long lt,
                                           unsigned long long now, unsigned long long old) {
    const double rho = recency(lt, now, old);
    if (policy == 0) return rho;
    return __dadd_rn(__dmul_rn(w_pred, surv), rho);
}

// ---------------------------------------------------------------- sync helpers

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Sense-reversing grid barrier for a cooperatively launched (co-resident) grid.
__device__ __forceinline__ void grid_barrier(Ctrl* c) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = ld_acquire(&c->bar_gen);
        __threadfence();
        if (atomicAdd(&c->bar_count, 1u) == gridDim.x - 1) {
            c->bar_count = 0;
            __threadfence();
            atomicAdd(&c->bar_gen, 1u);
        } else {
            // watchdog: a barrier that never opens (a CTA that cannot be co-resident, or a
            // CTA that died) traps after ~10 s instead of hanging the device
            unsigned long long spins = 0;
            while (ld_acquire(&c->bar_gen) == gen) {
                if (++spins > 4096) __nanosleep(64);  // hot spin first: barriers are short
                if (spins > (1ull << 27)) trap_at(205);
            }
        }
        __threadfence();
    }
    __syncthreads();
}
#endif  // __CUDACC__

}  // namespace csb
