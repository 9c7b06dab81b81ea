// cs_pool: device allocation, the admission driver, and the pool-level C ABI.
#include "cs_pool.hpp"

#include <atomic>
#include <chrono>

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <thread>

using csb::ck;
using csb::CsError;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return CS_OK;
    } catch (const CsError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return CS_ERR_INVALID_ARGUMENT;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return CS_ERR_LOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return CS_ERR_RUNTIME;
    }
}

template <class T>
T* dmalloc(size_t n, const char* what) {
    void* p = nullptr;
    ck(cudaMalloc(&p, sizeof(T) * (n ? n : 1)), what);
    return static_cast<T*>(p);
}
}  // namespace

extern "C" const char* cs_last_error(void) { return g_err.c_str(); }
extern "C" const char* cs_version(void) { return "cachesage_b200 0.1 (sm_100a)"; }

void cs_set_error(const std::string& m) { g_err = m; }

// the device watchdogs' trap word (host-mapped, one per process; see csb::trap_at)
static unsigned long long* g_trap_word = nullptr;
extern "C" uint64_t cs_debug_trap_word(void) { return g_trap_word ? *g_trap_word : 0; }

void cs_pool::create(const cs_pool_cfg& c, long long shard_slots, cs_comm* cm) {
    cfg = c;
    comm = cm;
    if (c.budget_blocks < 1) throw std::invalid_argument("EngineSim: budget, block size, and concurrency must be positive");
    if (c.e_max <= 0) throw std::invalid_argument("CacheSagePolicy: e_max must be positive");
    if (c.e_max > csb::kMaxLists - 2) throw CsError(CS_ERR_CAPACITY, "e_max > 22 is not supported by the device select");
    if (c.tau < 0.0 || c.tau > 1.0) throw std::invalid_argument("CacheSagePolicy: tau must be a probability");
    if (c.min_confidence < 0.0 || c.budget_per_step < 0) throw std::invalid_argument("CacheSagePolicy: invalid prefetch gate");
    if (c.window <= 0) throw std::invalid_argument("TransitionLearner: window capacity must be positive");
    if (c.agent_capacity < 1 || c.agent_capacity > csb::kMaxAgents)
        throw CsError(CS_ERR_CAPACITY, "agent_capacity must be in [1, 4096]");
    if (c.budget_blocks >= (int64_t)0x7FFFFFF0ll) throw CsError(CS_ERR_CAPACITY, "budget exceeds 31-bit slot ids");
    const int world = comm ? comm->world : 1;
    if (comm) {
        if (world < 1 || world > csb::kMaxShards) throw std::invalid_argument("sharded pool: 1 <= world <= 8");
        if (shard_slots <= 0) shard_slots = std::min<long long>(c.budget_blocks, c.budget_blocks * 5 / (4 * world) + 4096);
        if (shard_slots >= (long long)csb::kShardMask - 16)
            throw CsError(CS_ERR_CAPACITY, "shard exceeds 2^29 slots (global slot ids)");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw CsError(CS_ERR_CUDA, "no CUDA device: cachesage_b200 has no CPU fallback");
    device = c.device;
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreate(&ev0), "cudaEventCreate");
    ck(cudaEventCreate(&ev1), "cudaEventCreate");

    csb::DevPool& p = P;
    p.cap = comm ? shard_slots : c.budget_blocks;
    p.rank = comm ? comm->rank : 0;
    p.world = world;
    p.gbudget = c.budget_blocks;
    // TtlPolicy (baselines.cpp:22-28) picks the same victims as LruPolicy: last_touch_us never
    // decreases along last_touch (ticks and the simulated clock advance together), so the
    // blocks still inside the pin horizon (score 1e6 + rho) are the youngest, and the argmin of
    // (score, last_touch) over unpinned blocks is the oldest one under both scorers.
    if (c.policy < 0 || c.policy > 3)
        throw std::invalid_argument("policy must be 0 (lru), 1 (cachesage), 2 (ttl) or 3 (belady)");
    if (c.policy == 3 && comm) throw std::invalid_argument("belady: the hash-sharded pool runs lru / ttl / cachesage");
    p.policy = c.policy == 2 ? 0 : c.policy;
    p.e_max = c.e_max;
    p.n_lists = c.e_max + 2;
    p.a_cap = c.agent_capacity;
    p.tau = c.tau;
    p.w_pred = c.w_pred;
    p.min_conf = c.min_confidence;
    p.min_row = c.min_row_count;
    p.budget_per_step = c.budget_per_step;
    p.window = c.window;
    unsigned long long tcap = 1024;
    while (tcap < 4ull * (unsigned long long)p.cap) tcap <<= 1;  // live+tombstones <= tcap/2 + one admission
    p.tmask = tcap - 1;

    p.cap_scan = (p.cap + 63) & ~63ll;  // bulk copies move whole 16-B granules
    p.pk = dmalloc<unsigned long long>(p.cap_scan, "pk");
    p.lt = dmalloc<unsigned long long>(p.cap_scan, "lt");
    p.agent = dmalloc<unsigned int>(p.cap_scan, "agent");
    p.refs = dmalloc<unsigned int>(p.cap_scan, "refs");
    p.key = dmalloc<unsigned long long>(p.cap, "key");
    p.tokens = dmalloc<int>(p.cap, "tokens");
    p.table = dmalloc<csb::TableEntry>(tcap, "table");
    p.free_stack = dmalloc<unsigned int>(p.cap, "free_stack");
    p.evlog_cap = 1ll << 22;
    p.evlog = dmalloc<unsigned long long>(p.evlog_cap, "evlog");
    const size_t A = (size_t)p.a_cap;
    p.counts = dmalloc<unsigned int>(A * A, "counts");
    p.totals = dmalloc<unsigned int>(A, "totals");
    p.win_a = dmalloc<int>(p.window, "win_a");
    p.win_b = dmalloc<int>(p.window, "win_b");
    p.hop = dmalloc<unsigned char>(A, "hop");
    p.cls = dmalloc<unsigned char>(A, "cls");
    p.agent_ids = dmalloc<unsigned long long>(A, "agent_ids");
    ck(cudaMemsetAsync(p.counts, 0, sizeof(unsigned int) * A * A, stream), "memset");
    ck(cudaMemsetAsync(p.totals, 0, sizeof(unsigned int) * A, stream), "memset");
    p.ctrl = dmalloc<csb::Ctrl>(1, "ctrl");
    ck(cudaMemsetAsync(p.ctrl, 0, sizeof(csb::Ctrl), stream), "memset");
    p.gbound = dmalloc<unsigned long long>(csb::kMaxLists, "gbound");
    p.gcount = dmalloc<int>(csb::kMaxLists, "gcount");
    p.ghint = dmalloc<unsigned long long>(csb::kMaxLists, "ghint");
    p.gmaxk = dmalloc<unsigned long long>(csb::kMaxLists, "gmaxk");
    p.grej = dmalloc<unsigned int>(1, "grej");
    p.gsmall = dmalloc<unsigned char>(csb::kMaxLists, "gsmall");
    ck(cudaMemsetAsync(p.gsmall, 0, csb::kMaxLists, stream), "memset");
    ck(cudaMemsetAsync(p.ghint, 0xff, sizeof(unsigned long long) * csb::kMaxLists, stream), "memset");
    p.fin_lt = dmalloc<unsigned long long>((size_t)csb::kMaxLists * (csb::kChunk + 2), "fin_lt");
    p.fin_slot = dmalloc<unsigned int>((size_t)csb::kMaxLists * (csb::kChunk + 2), "fin_slot");
    p.fin_n = dmalloc<int>(csb::kMaxLists, "fin_n");
    p.p_cap = 0;
    p.p_slot = nullptr;
    p.p_refs0 = nullptr;
    p.tq_key = nullptr;
    p.tq_slot = nullptr;
    ensure_prompt_scratch(4096);

    if (const char* e = std::getenv("CS_SPECULATE")) speculate = std::atoi(e) != 0;  // A/B switch (tools)
    if (const char* e = std::getenv("CS_PRESCAN")) prescan = std::atoi(e) != 0;       // A/B switch (tools)
    // fl(w_pred * (1 - min(c, e_max) / e_max)) per survival class, as CacheSagePolicy::score and
    // ReachabilityState::survival compute it (reachability.cpp:17-20); host code builds with
    // -ffp-contract=off, so the product is the same IEEE double the device would form
    for (int cl = 0; cl < csb::kMaxLists; ++cl) {
        const int cap = cl < p.e_max ? cl : p.e_max;
        const double surv = 1.0 - (double)cap / (double)p.e_max;
        p.wsurv[cl] = p.w_pred * surv;
    }
    lc = csb::admit_launch_config(p, device, c.grid_ctas);
    if (lc.grid <= 0) throw CsError(CS_ERR_CUDA, "admit kernel: no launch configuration fits this device");
    p.gcap = (long long)lc.grid * (csb::kChunk + 1);
    p.gbuf_lt = dmalloc<unsigned long long>((size_t)csb::kMaxLists * p.gcap, "gbuf_lt");
    p.gbuf_slot = dmalloc<unsigned int>((size_t)csb::kMaxLists * p.gcap, "gbuf_slot");
    p.gmin = dmalloc<unsigned long long>((size_t)csb::kMaxLists * lc.grid, "gmin");
    // per-CTA rows + CTA-0 stamps + debug records + the admission server's trace ring (8 x 8)
    p.dbg = dmalloc<unsigned long long>((size_t)lc.grid * 16 + 256, "dbg");
    if (const char* e = std::getenv("CS_DEBUG_PRESCAN")) p.dbg_check = std::atoi(e);
    if (const char* e = std::getenv("CS_DEBUG_WARPS")) p.dbg_warps = std::atoi(e);
    if (p.dbg_check) {
        p.dbg_unpin = dmalloc<unsigned long long>(p.cap_scan, "dbg_unpin");
        ck(cudaMemset(p.dbg_unpin, 0, 8 * p.cap_scan), "memset");
    }
    p.raw_grid = lc.grid;
    {
        const size_t nraw = (size_t)2 * lc.grid * csb::kRawCap;
        p.raw_lt = dmalloc<unsigned long long>(nraw, "raw_lt");
        p.raw_slot = dmalloc<unsigned int>(nraw, "raw_slot");
        p.raw_list = dmalloc<unsigned char>(nraw, "raw_list");
        p.raw_agent = dmalloc<unsigned int>(nraw, "raw_agent");
        p.raw_hdr = dmalloc<csb::RawHdr>((size_t)2 * lc.grid, "raw_hdr");
        ck(cudaMemset(p.raw_hdr, 0, sizeof(csb::RawHdr) * 2 * lc.grid), "memset");  // seq 0: nothing written
    }
    p.pl_lt = dmalloc<unsigned long long>((size_t)3 * csb::kPendCap, "pl_lt");
    p.pl_slot = dmalloc<unsigned int>((size_t)3 * csb::kPendCap, "pl_slot");
    p.pl_agent = dmalloc<unsigned int>((size_t)csb::kPendCap, "pl_agent");
    p.pl_ok = dmalloc<unsigned char>((size_t)3 * csb::kPendCap, "pl_ok");
    p.pl_key = dmalloc<unsigned long long>((size_t)csb::kPreK, "pl_key");
    p.pl_n = dmalloc<int>(4, "pl_n");
    p.pl_T = dmalloc<unsigned long long>(3, "pl_T");
    p.pre_hint = dmalloc<unsigned long long>(6, "pre_hint");
    {
        const unsigned long long h[6] = {csb::kNoBound, csb::kNoBound, csb::kNoBound,
                                         csb::kNoBound, csb::kNoBound, csb::kNoBound};
        ck(cudaMemcpy(p.pre_hint, h, sizeof(h), cudaMemcpyHostToDevice), "pre_hint");
    }
    ck(cudaMemsetAsync(p.dbg, 0, sizeof(unsigned long long) * (lc.grid * 16 + 256), stream), "memset");

    if (comm) {
        p.sh_send2 = dmalloc<csb::ShardLists>(1, "sh_send2");
        p.sh_recv2 = dmalloc<csb::ShardLists>((size_t)world, "sh_recv2");
        p.sh_state = dmalloc<csb::ShardState>(1, "sh_state");
        ck(cudaMallocHost(reinterpret_cast<void**>(&hstate), sizeof(csb::ShardState)), "cudaMallocHost");
        ensure_prompt_scratch(8192);
    }
    if (p.policy == 3) {
        p.bel_nu = dmalloc<unsigned int>(p.cap, "bel_nu");
        p.bel_kid = dmalloc<unsigned int>(p.cap, "bel_kid");
        p.bel_hi = dmalloc<unsigned long long>(p.cap, "bel_hi");
        p.bel_lo = dmalloc<unsigned long long>(p.cap, "bel_lo");
        p.bel_cand = dmalloc<csb::BelCand>(csb::kBelCand, "bel_cand");
        p.bel_ctl = dmalloc<csb::BelCtl>(1, "bel_ctl");
        ck(cudaMemsetAsync(p.bel_ctl, 0, sizeof(csb::BelCtl), stream), "memset");
        blc = csb::belady_launch_config(p, device);
        if (blc.grid <= 0) throw CsError(CS_ERR_CUDA, "belady kernel: no launch configuration fits this device");
    }
    ck(cudaHostAlloc(reinterpret_cast<void**>(&st), sizeof(csb::AdmitStatus), cudaHostAllocMapped), "cudaHostAlloc");
    std::memset(st, 0, sizeof(*st));
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&st_dev), st, 0), "cudaHostGetDevicePointer");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&mb), sizeof(csb::SrvMailbox), cudaHostAllocMapped), "cudaHostAlloc");
    std::memset(mb, 0, sizeof(*mb));
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mb_dev), mb, 0), "cudaHostGetDevicePointer");
    d_srv_args = dmalloc<csb::AdmitArgs>(2, "server args");  // (double-buffered by post parity)
    {  // the device watchdogs' trap site (one per process, host-mapped)
        unsigned long long*& trap_word = g_trap_word;
        if (!trap_word) {
            ck(cudaHostAlloc(reinterpret_cast<void**>(&trap_word), 8 * 4096, cudaHostAllocMapped | cudaHostAllocPortable),
               "cudaHostAlloc(trap word)");
            std::memset(trap_word, 0, 8 * 4096);
            unsigned long long* dp = nullptr;
            ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), trap_word, 0), "cudaHostGetDevicePointer");
            const char* pe = std::getenv("CS_DEBUG_PROGRESS");
            ck(csb::set_trap_word(dp, pe ? std::atoi(pe) : 0), "set_trap_word");
        }
        trap_word_host = trap_word;
    }
    P.spec = dmalloc<csb::LearnSpec>(1, "learner service");
    P.spec_hop = dmalloc<ulonglong2>((P.a_cap + 7) / 8, "learner service hops");
    ck(cudaMemset(P.spec, 0, sizeof(csb::LearnSpec)), "memset");
    ck(cudaMemset(P.spec_hop, 0, sizeof(ulonglong2) * ((P.a_cap + 7) / 8)), "memset");
    if (const char* e = std::getenv("CS_SERVER")) server = std::atoi(e) != 0;
    if (const char* e = std::getenv("CS_SERVER_GENERIC")) server_generic = std::atoi(e) != 0;
    ck(csb::launch_init_pool(p, stream), "init_pool");
    sync();
}

void cs_pool::destroy() {
    try {
        server_stop();
    } catch (...) {
    }
    csb::DevPool& p = P;
    void* ptrs[] = {p.pk, p.lt, p.agent, p.refs, p.key, p.tokens, p.table, p.free_stack, p.evlog, p.counts, p.totals,
                    p.win_a, p.win_b, p.hop, p.cls, p.agent_ids, p.ctrl, p.gbound, p.gcount, p.fin_lt, p.fin_slot,
                    p.fin_n, p.p_slot, p.p_refs0, p.gbuf_lt, p.gbuf_slot, p.ghint, p.gmaxk, p.grej, p.dbg, p.gsmall, p.gmin, p.tq_key, p.tq_slot,
                    p.sh_send1, p.sh_recv1, p.sh_send2, p.sh_recv2, p.sh_state, p.sh_gslot, p.sh_grefs0,
                    p.pl_lt, p.pl_slot, p.pl_agent, p.pl_ok, p.pl_key, p.pl_n, p.pl_T, p.pre_hint,
                    p.raw_lt, p.raw_slot, p.raw_list, p.raw_agent, p.raw_hdr,
                    (void*)p.spec, (void*)p.spec_hop, p.bel_nu, p.bel_kid, p.bel_kid_slot, (void*)p.bel_ref, (void*)p.bel_ref_off, (void*)p.bel_depth,
                    (void*)p.bel_kid_of, p.bel_hi, p.bel_lo, p.bel_cand, p.bel_ctl};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    d_keys.release();
    d_counts.release();
    d_pins.release();
    d_aux.release();
    d_aux2.release();
    d_aux3.release();
    if (st) cudaFreeHost(st);
    if (mb) cudaFreeHost(mb);
    if (d_srv_args) cudaFree(d_srv_args);
    if (hstate) cudaFreeHost(hstate);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
}

void cs_pool::ensure_prompt_scratch(long long n) {
    if (n <= P.p_cap && (!comm || P.sh_gslot)) return;
    if (comm) {
        const long long c = std::max<long long>(n, P.p_cap * 2);
        for (void* q : {(void*)P.sh_send1, (void*)P.sh_recv1, (void*)P.sh_gslot, (void*)P.sh_grefs0})
            if (q) cudaFree(q);
        const size_t rec = sizeof(csb::ShardHdr) + sizeof(csb::ShardPos) * (size_t)c;
        P.sh_send1 = dmalloc<unsigned char>(rec, "sh_send1");
        P.sh_recv1 = dmalloc<unsigned char>(rec * (size_t)P.world, "sh_recv1");
        P.sh_gslot = dmalloc<unsigned int>(c, "sh_gslot");
        P.sh_grefs0 = dmalloc<unsigned int>(c, "sh_grefs0");
        if (n <= P.p_cap) return;
        n = c;
    }
    long long c = std::max<long long>(n, P.p_cap * 2);
    server_stop();  // (the scratch is the server's: never reallocated under it)
    if (P.p_slot) {
        ck(csb::launch_table_flush(P, stream), "table flush");  // the queue lives in this scratch
        ++launches;
        ck(cudaStreamSynchronize(stream), "sync");
        cudaFree(P.p_slot);
        cudaFree(P.p_refs0);
        cudaFree(P.tq_key);
        cudaFree(P.tq_slot);
    }
    P.p_slot = dmalloc<unsigned int>(c, "p_slot");
    P.p_refs0 = dmalloc<unsigned int>(c, "p_refs0");
    P.tq_key = dmalloc<unsigned long long>(2 * c, "tq_key");
    P.tq_slot = dmalloc<unsigned int>(c, "tq_slot");
    P.p_cap = c;
}

void cs_pool::flush_table() {
    ck(csb::launch_table_flush(P, stream), "table flush");
    ++launches;
}

std::vector<unsigned long long> cs_pool::allgather_u64(unsigned long long v) {
    if (!comm) return {v};
    std::vector<unsigned long long> out((size_t)P.world);
    ck(cudaMemcpyAsync(P.sh_send1, &v, 8, cudaMemcpyHostToDevice, stream), "H2D");
    comm->allgather(P.sh_send1, P.sh_recv1, 8, stream);
    ck(cudaMemcpyAsync(out.data(), P.sh_recv1, 8 * out.size(), cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
    return out;
}

void cs_pool::fetch_state() {
    ck(cudaMemcpyAsync(hstate, P.sh_state, sizeof(csb::ShardState), cudaMemcpyDeviceToHost, stream), "state D2H");
    sync();
}

// One admission of a sharded pool (cs_shard.cuh): probe -> allgather -> decide -> per chunk
// that can evict [scan -> allgather] -> replay. Every shard calls it with the same arguments.
const csb::AdmitStatus& cs_pool::admit_sharded(const csb::AdmitArgs& in) {
    try {
        return admit_sharded_once(in);
    } catch (...) {
        comm->abort();  // a shard that fails must not leave its peers waiting in an exchange
        throw;
    }
}

const csb::AdmitStatus& cs_pool::admit_sharded_once(const csb::AdmitArgs& in) {
    csb::AdmitArgs a = in;
    ensure_prompt_scratch(std::max(1, a.n));
    a.status = st_dev;
    a.n_agents = n_agents;
    if (poll_reset_pending) a.flags |= csb::kPollReset;
    if ((int)unpin_q.size() > csb::kMaxUnpinRanges) flush_unpins();
    a.n_unpin_ranges = 0;
    for (const auto& u : unpin_q) {
        a.unpin_ptr[a.n_unpin_ranges] = u.first;
        a.unpin_n[a.n_unpin_ranges] = u.second;
        ++a.n_unpin_ranges;
    }
    unpin_q.clear();
    unpin_q_slots = 0;
    a.seq = ++seq;
    st->started = -1;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing) {
        e0 = take_event();
        e1 = take_event();
        ck(cudaEventRecord(e0, stream), "cudaEventRecord");
    }
    // exchange 1 (probe -> decide) and, per chunk, exchange 2 (scan -> replay). World 1: nothing
    // to exchange (one front kernel). Peer transport: fused into the admission kernels. Other
    // transports: an allgather between the kernels.
    csb::ShardX x{};
    const bool fz = P.world > 1 && comm->fused(&x.t, &x.cap);
    const size_t rec1 = sizeof(csb::ShardHdr) + sizeof(csb::ShardPos) * (size_t)std::max(a.n, 0);
    if (fz && (rec1 > x.cap || csb::shard_lists_bytes(P.n_lists) > x.cap))
        throw CsError(CS_ERR_CAPACITY, "peer exchange: message exceeds the window capacity");
    if (P.world == 1 || fz) {
        if (fz) {
            x.fused = 1;
            x.seq = comm->fused_next();
            comm->fused_meet(stream);
        }
        ck(csb::launch_shard_front(P, a, x, stream), "shard front");
        ++launches;
        if (fz) comm->fused_end(stream);
    } else {
        ck(csb::launch_shard_probe(P, a, stream), "shard probe");
        comm->allgather(P.sh_send1, P.sh_recv1, rec1, stream);
        ck(csb::launch_shard_decide(P, a, stream), "shard decide");
        launches += 2;
    }
    // every possible chunk is enqueued without a host round trip: the kernels read the
    // replicated state (admit_n, need_scan) and no-op past the admission's end
    const int n_chunks = (std::max(a.n, 1) + csb::kChunk - 1) / csb::kChunk;
    for (int c = 0; c < n_chunks; ++c) {
        if (fz) x.seq = comm->fused_next();
        ck(csb::launch_shard_scan(P, a, c, x, lc, stream), "shard scan");
        if (fz) comm->fused_meet(stream);
        else if (P.world > 1) comm->allgather(P.sh_send2, P.sh_recv2, csb::shard_lists_bytes(P.n_lists), stream);
        ck(csb::launch_shard_replay(P, a, x, stream), "shard replay");
        if (fz) comm->fused_end(stream);
        launches += 2;
    }
    if (timing) ck(cudaEventRecord(e1, stream), "cudaEventRecord");
    // the replay (or decide, for an admission that does not start) publishes the status before
    // it applies the table updates: inside an engine loop the host schedules the next admission
    // meanwhile (stream order keeps every later device operation behind this one)
    wait_status(a.seq, "shard kernels");
    if (!early_status) ck(cudaStreamSynchronize(stream), "shard kernels");
    poll_reset_pending = false;
    if (timing) {
        t_pending.push_back({e0, e1, st->scans > 0});
        resolve_timing(false);
    }
    if (st->started < 0) throw CsError(CS_ERR_CUDA, "shard kernels did not report a status");
    resident = st->resident;
    pinned = st->pinned;
    ev_safe = ev_total;  // (this admission's own log entries may still be in flight: early status)
    ev_total = st->ev_total;
    pending_targets.assign(st->pend_target, st->pend_target + std::min(st->n_pend, csb::kMaxPending));
    pending_ticks.assign(st->pend_tick, st->pend_tick + std::min(st->n_pend, csb::kMaxPending));
    if (st->error == 2) throw CsError(CS_ERR_CAPACITY, "sharded pool: a shard ran out of slots (raise shard_slots)");
    if (st->error) throw std::runtime_error("evict_one: all resident blocks are pinned");
    // this shard holds at most P.cap live entries: rebuild before cap + tombstones pass half
    if ((unsigned long long)(P.cap + st->tombstones) > (P.tmask + 1) / 2) {
        ck(csb::launch_table_rebuild(P, stream), "table rebuild");  // subsumes the queued updates
        ++table_rebuilds;
        launches += 2;
    }
    return *st;
}

void cs_pool::belady_index(const unsigned long long* keys, long long n_flat, const std::vector<long long>& blk_off) {
    if (P.policy != 3) throw std::logic_error("belady_index: not a belady pool");
    const long long n_req = (long long)blk_off.size() - 1;
    const long long nf = std::max(1ll, n_flat);
    P.bel_ref = dmalloc<unsigned int>(nf, "bel_ref");
    P.bel_ref_off = dmalloc<long long>(nf + 1, "bel_ref_off");
    P.bel_depth = dmalloc<int>(nf, "bel_depth");
    P.bel_kid_of = dmalloc<unsigned int>(nf, "bel_kid_of");
    long long* d_off = dmalloc<long long>(blk_off.size(), "blk_off");
    ck(cudaMemcpyAsync(d_off, blk_off.data(), 8 * blk_off.size(), cudaMemcpyHostToDevice, stream), "H2D");
    bel_kids = csb::build_belady_index(keys, n_flat, d_off, n_req, const_cast<unsigned int*>(P.bel_ref),
                                       const_cast<long long*>(P.bel_ref_off), const_cast<int*>(P.bel_depth),
                                       const_cast<unsigned int*>(P.bel_kid_of), stream);
    cudaFree(d_off);
    if (bel_kids < 0) throw CsError(CS_ERR_CUDA, "belady: next-use index build failed");
    P.bel_kid_slot = dmalloc<unsigned int>(std::max(1ll, bel_kids), "bel_kid_slot");
    ck(cudaMemsetAsync(P.bel_kid_slot, 0xff, 4 * (size_t)std::max(1ll, bel_kids), stream), "memset");
    launches += 5;
    sync();
}

// One Belady admission launch (cs_belady.cuh); same contract as admit().
const csb::AdmitStatus& cs_pool::admit_belady(const csb::AdmitArgs& in, int n_for_grid) {
    if (bel_kids < 0 || !in.kids) throw std::invalid_argument("belady: the pool needs the request stream (cs_engine)");
    csb::AdmitArgs a = in;
    ensure_prompt_scratch(std::max(1, a.n));
    a.status = st_dev;
    a.n_agents = n_agents;
    const bool may_evict = (a.flags & csb::kAdmit) && resident + n_for_grid > P.cap;
    // one CTA per 4K slots: the selection passes are short, the grid barriers are not free
    const char* ge = std::getenv("CS_BELADY_CTAS");  // tests: force a grid (multi-CTA select on small pools)
    const int grid_env = ge ? std::atoi(ge) : 0;
    int grid = may_evict ? (int)std::max(1ll, std::min<long long>(blc.grid, (P.cap + 4095) / 4096)) : 1;
    if (may_evict && grid_env > 0) grid = std::min(grid_env, blc.grid);
    if ((int)unpin_q.size() > csb::kMaxUnpinRanges) flush_unpins();
    a.n_unpin_ranges = 0;
    for (const auto& u : unpin_q) {
        a.unpin_ptr[a.n_unpin_ranges] = u.first;
        a.unpin_n[a.n_unpin_ranges] = u.second;
        ++a.n_unpin_ranges;
    }
    unpin_q.clear();
    unpin_q_slots = 0;
    a.n_prev_ranges = 0;
    a.seq = ++seq;
    st->started = -1;
    if (timing) ck(cudaEventRecord(ev0, stream), "cudaEventRecord");
    ck(csb::launch_belady_admit(P, a, blc, grid, stream), "belady_admit_kernel launch");
    ++launches;
    if (timing) ck(cudaEventRecord(ev1, stream), "cudaEventRecord");
    vpref_done = 0;
    if (vpref && vpref_n > 0) {
        const unsigned long long cap = (unsigned long long)P.evlog_cap, off = ev_total % cap;
        const unsigned long long n1 = std::min<unsigned long long>((unsigned long long)vpref_n, cap - off);
        ck(cudaMemcpyAsync(vpref, P.evlog + off, 8 * n1, cudaMemcpyDeviceToHost, stream), "victims D2H");
        if (n1 < (unsigned long long)vpref_n)
            ck(cudaMemcpyAsync(vpref + n1, P.evlog, 8 * (vpref_n - n1), cudaMemcpyDeviceToHost, stream), "victims D2H");
        vpref_done = vpref_n;
    }
    vpref = nullptr;
    vpref_n = 0;
    ck(cudaStreamSynchronize(stream), "belady_admit_kernel");
    poll_reset_pending = false;
    if (timing) {
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, ev0, ev1), "cudaEventElapsedTime");
        admit_ms += ms;
        ++admit_launches;
        if (st->scans > 0) {
            scan_launch_ms += ms;
            ++scan_launches;
        }
    }
    if (st->started < 0) throw CsError(CS_ERR_CUDA, "belady kernel did not report a status");
    resident = st->resident;
    pinned = st->pinned;
    ev_safe = ev_total;  // (this admission's own log entries may still be in flight: early status)
    ev_total = st->ev_total;
    pending_targets.clear();
    pending_ticks.clear();
    if (st->error) throw std::runtime_error("evict_one: all resident blocks are pinned");
    if ((unsigned long long)(st->resident + st->tombstones) > (P.tmask + 1) / 2) {
        ck(csb::launch_table_rebuild(P, stream), "table rebuild");
        ++table_rebuilds;
        launches += 2;
    }
    return *st;
}

const csb::AdmitStatus& cs_pool::admit(const csb::AdmitArgs& in, int n_for_grid) {
    // the packed scan word keeps 40 bits of last_touch (cs_device.cuh)
    // (no wrap: a caller-supplied tick_base near 2^64 must not pass; a dispatch-only call writes
    // no last_touch, so any event tick is fine there)
    if (in.n > 0 && in.tick_base > csb::kMaxTick - (2ull * (unsigned long long)in.n + 16ull))
        throw CsError(CS_ERR_CAPACITY, "tick space exhausted (last_touch must stay below 2^40 - 1)");
    if (comm) return admit_sharded(in);
    if (P.policy == 3) return admit_belady(in, n_for_grid);
    csb::AdmitArgs a = in;
    ensure_prompt_scratch(std::max(1, a.n));
    a.status = st_dev;
    a.n_agents = n_agents;
    if (poll_reset_pending) a.flags |= csb::kPollReset;
    // No eviction is possible when every block could be inserted without reaching the budget:
    // one CTA then suffices (the grid barrier degenerates), saving the cooperative launch.
    const bool may_evict = (a.flags & csb::kAdmit) && resident + n_for_grid > P.cap;
    static const bool full_grid = [] {
        const char* e = std::getenv("CS_FULL_GRID");  // A/B switch (tools): every admission cooperative
        return e && std::atoi(e) != 0;
    }();
    const bool srv = uses_server();
    const int grid = (srv || may_evict || full_grid) ? lc.grid : 1;
    // queued unpins run first inside this launch (they fit the change set of a speculative pass)
    if ((int)unpin_q.size() > csb::kMaxUnpinRanges) flush_unpins();
    a.n_unpin_ranges = 0;
    for (const auto& u : unpin_q) {
        a.unpin_ptr[a.n_unpin_ranges] = u.first;
        a.unpin_n[a.n_unpin_ranges] = u.second;
        ++a.n_unpin_ranges;
    }
    const int xn = a.n + unpin_q_slots;
    const int cur_unpins = unpin_q_slots;
    unpin_q.clear();
    unpin_q_slots = 0;
    a.seq = ++seq;
    if (speculate && grid > 1 && xn <= csb::kXsetMax) a.flags |= csb::kSpeculate;
    if (prescan && grid > csb::kStream0) a.flags |= csb::kPrescan;
    a.n_prev_ranges = 0;
    if ((a.flags & csb::kPrescan) && pre_ok && cur_unpins + prev_slots <= csb::kXsetMax &&
        (int)prev_ranges.size() <= csb::kMaxUnpinRanges + 1) {
        a.flags |= csb::kUsePrescan;
        for (const auto& u : prev_ranges) {
            a.prev_ptr[a.n_prev_ranges] = u.first;
            a.prev_n[a.n_prev_ranges] = u.second;
            ++a.n_prev_ranges;
        }
    }
    pre_ok = false;
    st->started = -1;
    // the end-to-end path: CTA 0 writes this admission's victims (<= one per block) into the
    // caller's pinned buffer itself, before the status flag
    a.vict_host = nullptr;
    a.vict_cap = 0;
    if (vpref && vpref_n > 0) {
        unsigned long long* dp = nullptr;
        ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), vpref, 0), "cudaHostGetDevicePointer(victims)");
        a.vict_host = dp;
        a.vict_cap = vpref_n;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (srv) {
        // the server must run on the current pool arguments (scratch may have been reallocated)
        csb::DevPool want = P;
        want.stream_generic = server_generic ? 1 : 0;
        if (srv_running && std::memcmp(&want, &srv_P, sizeof(want)) != 0) server_stop();
        if (!srv_running) {
            srv_P = want;
            ck(csb::launch_server(srv_P, mb_dev, d_srv_args, srv_post + 1, lc, stream), "server_kernel launch");
            ++launches;
            ++server_launches;
            srv_running = true;
            srv_have_t0 = false;
        }
        if (srv_status_seen) {  // instrumentation: the host's part of the turnaround
            host_turnaround_ns += (unsigned long long)std::chrono::duration_cast<std::chrono::nanoseconds>(
                                      std::chrono::steady_clock::now() - srv_status_t).count();
            ++host_turnarounds;
        }
        server_post(a);
    } else {
        if (timing) {
            e0 = take_event();
            e1 = take_event();
            ck(cudaEventRecord(e0, stream), "cudaEventRecord");
        }
        ck(csb::launch_admit(P, a, lc, grid, stream), "admit_kernel launch");
        ++launches;
        if (timing) ck(cudaEventRecord(e1, stream), "cudaEventRecord");
    }
    // The status flag is set by CTA 0 while the prescan CTAs still stream the next admission's
    // pass: the host prepares and enqueues the next launch behind this one instead of waiting
    // for the kernel's end (stream order keeps every later device operation behind it).
    wait_status(a.seq, srv ? "server_kernel" : "admit_kernel");
    if (srv) {
        srv_status_t = std::chrono::steady_clock::now();
        srv_status_seen = true;
    }
    if (!early_status) ck(cudaStreamSynchronize(stream), "admit_kernel");
    vpref_done = (vpref && vpref_n > 0) ? (int)std::min<long long>(st->n_evicted, vpref_n) : 0;
    vpref = nullptr;
    vpref_n = 0;
    poll_reset_pending = false;
    if (timing && srv) {
        server_account(st->srv_t0);
        srv_last_scan = st->scans > 0;
    } else if (timing) {
        t_pending.push_back({e0, e1, st->scans > 0});
        resolve_timing(false);
    }
    if (st->started < 0) throw CsError(CS_ERR_CUDA, "admit kernel did not report a status");
    // the slots this launch unpinned, for the next launch's use of this launch's prescan
    prev_ranges.clear();
    prev_slots = 0;
    for (int r = 0; r < a.n_unpin_ranges; ++r) {
        prev_ranges.emplace_back(a.unpin_ptr[r], a.unpin_n[r]);
        prev_slots += a.unpin_n[r];
    }
    if ((a.flags & csb::kUnpinAfter) && a.pins_out && st->started && !st->error && st->admit_n > 0) {
        prev_ranges.emplace_back(a.pins_out, st->admit_n);
        prev_slots += st->admit_n;
    }
    pre_ok = (a.flags & csb::kPrescan) != 0 && !st->error;
    resident = st->resident;
    pinned = st->pinned;
    ev_safe = ev_total;  // (this admission's own log entries may still be in flight: early status)
    ev_total = st->ev_total;
    for (int k = 0; k < csb::kPhases; ++k) phase_ns[k] += st->phase_ns[k];
    pending_targets.assign(st->pend_target, st->pend_target + std::min(st->n_pend, csb::kMaxPending));
    pending_ticks.assign(st->pend_tick, st->pend_tick + std::min(st->n_pend, csb::kMaxPending));
    if (st->error) throw std::runtime_error("evict_one: all resident blocks are pinned");
    // erased entries become tombstones; rebuild before live + tombstones pass half the table
    if ((unsigned long long)(st->resident + st->tombstones) > (P.tmask + 1) / 2) {
        server_stop();
        ck(csb::launch_table_rebuild(P, stream), "table rebuild");
        ++table_rebuilds;
        launches += 2;
    }
    return *st;
}

void cs_pool::ck_trap(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    if (trap_word_host && *trap_word_host) {
        const unsigned long long w = *trap_word_host;
        m += " (device watchdog site " + std::to_string(w >> 32) + ", CTA " + std::to_string(w & 0xffffffffull) + ")";
        if (std::getenv("CS_DEBUG_PROGRESS")) {  // each CTA's last progress mark: (seq << 8) | stage
            m += " progress:";
            for (int c = 0; c < lc.grid; ++c) {
                const unsigned long long v = trap_word_host[1 + c];
                m += " " + std::to_string(c) + ":" + std::to_string(v >> 8) + "/" + std::to_string(v & 0xff);
            }
        }
    }
    throw CsError(CS_ERR_CUDA, m);
}

void cs_pool::server_post(const csb::AdmitArgs& a) {
    // every word, then its tag, in the same 16-byte pair (csb::SrvMailbox): a device load that
    // sees the new tag sees the new word
    const unsigned long long tag = ++srv_post;
    unsigned long long w[csb::kArgWords];
    std::memcpy(w, &a, sizeof(a));
    for (int i = 0; i < csb::kArgWords; ++i) {
        volatile csb::SrvMailbox::Pair* p = &mb->pair[i];
        p->word = w[i];
        std::atomic_signal_fence(std::memory_order_release);  // (compiler order: word, then tag)
        p->tag = tag;
    }
}

void cs_pool::server_account(unsigned long long t_next) {
    if (srv_have_t0 && t_next >= srv_last_t0) {
        const double ms = (double)(t_next - srv_last_t0) / 1e6;
        admit_ms += ms;
        ++admit_launches;
        if (srv_last_scan) {
            scan_launch_ms += ms;
            ++scan_launches;
        }
    }
    srv_last_t0 = t_next;
    srv_have_t0 = true;
}

void cs_pool::server_stop() {
    if (!srv_running) return;
    srv_running = false;
    // The stop takes the next sequence number without consuming it: the next admission reuses
    // it, so the prescan parity (AdmitArgs::seq & 1) of the last admission before the stop and
    // of the first one after it stay consecutive and the next admission can use that prescan.
    csb::AdmitArgs a{};
    a.flags = csb::kSrvStop;
    a.status = st_dev;
    a.seq = seq + 1;
    server_post(a);
    ck_trap(cudaStreamSynchronize(stream), "server_kernel");
    if (st->done_seq != a.seq) throw CsError(CS_ERR_CUDA, "server_kernel: no stop acknowledgement");
    srv_status_seen = false;
    st->done_seq = 0;  // (the next admission waits for this number again)
    if (timing) server_account(st->srv_t0);
    srv_have_t0 = false;
}

cudaEvent_t cs_pool::take_event() {
    if (!t_free.empty()) {
        cudaEvent_t e = t_free.back();
        t_free.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

void cs_pool::resolve_timing(bool wait) {
    size_t k = 0;
    for (; k < t_pending.size(); ++k) {
        const TimedLaunch& t = t_pending[k];
        if (wait) ck(cudaEventSynchronize(t.e1), "cudaEventSynchronize");
        else if (cudaEventQuery(t.e1) != cudaSuccess) break;
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, t.e0, t.e1), "cudaEventElapsedTime");
        admit_ms += ms;
        ++admit_launches;
        if (t.scan) {
            scan_launch_ms += ms;
            ++scan_launches;
        }
        t_free.push_back(t.e0);
        t_free.push_back(t.e1);
    }
    t_pending.erase(t_pending.begin(), t_pending.begin() + k);
}

void cs_pool::wait_status(unsigned long long seq, const char* what) {
    volatile unsigned long long* flag = &st->done_seq;
    for (unsigned long long spin = 0;; ++spin) {
        if (*flag == seq) return;
        if (spin >= 256) std::this_thread::yield();  // a long wait: let other host threads run
        if ((spin & 1023) == 1023) {
            const cudaError_t e = cudaStreamQuery(stream);
            if (e == cudaSuccess) {  // the kernel has ended: its flag write is visible by now
                if (*flag == seq) return;
                throw CsError(CS_ERR_CUDA, std::string(what) + ": no status from the kernel");
            }
            if (e != cudaErrorNotReady) ck_trap(e, what);
        }
    }
}

void cs_pool::defer_unpin(const unsigned int* dev_slots, int n) {
    if (n <= 0) return;
    if ((int)unpin_q.size() == csb::kMaxUnpinRanges) flush_unpins();
    unpin_q.emplace_back(dev_slots, n);
    unpin_q_slots += n;
}

void cs_pool::flush_unpins() {
    if (unpin_q.empty()) return;
    server_stop();
    pre_ok = false;  // unpins outside an admission launch: no prescan reuse
    for (const auto& u : unpin_q) {
        ck(csb::launch_unpin(P, u.first, u.second, stream), "unpin");
        ++launches;
    }
    unpin_q.clear();
    unpin_q_slots = 0;
}

void cs_pool::copy_victims(unsigned long long from, unsigned long long to, unsigned long long* out) {
    const unsigned long long cap = (unsigned long long)P.evlog_cap;
    if (to - from > cap) throw CsError(CS_ERR_CAPACITY, "eviction log overrun before it was drained");
    unsigned long long i = from;
    while (i < to) {
        const unsigned long long off = i % cap;
        const unsigned long long n = std::min(to - i, cap - off);
        ck(cudaMemcpy(out + (i - from), P.evlog + off, n * 8, cudaMemcpyDeviceToHost), "evlog D2H");
        i += n;
    }
}

// ---------------------------------------------------------------------- C ABI (pool level)

extern "C" {

void cs_pool_cfg_default(cs_pool_cfg* c) {
    c->budget_blocks = 120;
    c->policy = 1;
    c->e_max = 8;
    c->tau = 0.01;
    c->w_pred = 1.0;
    c->window = 1024;
    c->min_confidence = 0.5;
    c->min_row_count = 5;
    c->budget_per_step = 1;
    c->agent_capacity = 1024;
    c->device = 0;
    c->grid_ctas = 0;
}

int cs_pool_create(const cs_pool_cfg* cfg, cs_pool_t* out) {
    return guard([&] {
        if (!cfg || !out) throw std::invalid_argument("cs_pool_create: null argument");
        auto* p = new cs_pool();
        try {
            p->create(*cfg);
        } catch (...) {
            p->destroy();
            delete p;
            throw;
        }
        *out = p;
    });
}

int cs_pool_create_sharded(const cs_pool_cfg* cfg, int64_t shard_slots, cs_comm_t comm, cs_pool_t* out) {
    return guard([&] {
        if (!cfg || !out || !comm) throw std::invalid_argument("cs_pool_create_sharded: null argument");
        auto* p = new cs_pool();
        try {
            p->create(*cfg, shard_slots, comm);
        } catch (...) {
            p->destroy();
            delete p;
            throw;
        }
        *out = p;
    });
}

int cs_pool_destroy(cs_pool_t pool) {
    return guard([&] {
        if (!pool) return;
        pool->destroy();
        delete pool;
    });
}

int cs_register_agents(cs_pool_t pool, const uint64_t* ids, int n, int* first) {
    return guard([&] {
        if (!pool || (n > 0 && !ids)) throw std::invalid_argument("cs_register_agents: null argument");
        if (pool->n_agents + n > pool->P.a_cap) throw CsError(CS_ERR_CAPACITY, "agent capacity exceeded");
        if (first) *first = pool->n_agents;
        if (n <= 0) return;
        ck(cudaMemcpyAsync(pool->P.agent_ids + pool->n_agents, ids, sizeof(uint64_t) * n, cudaMemcpyHostToDevice,
                           pool->stream),
           "agent ids H2D");
        pool->agent_ids.insert(pool->agent_ids.end(), ids, ids + n);
        pool->n_agents += n;
        pool->sync();
    });
}

int64_t cs_blocks_for(const int64_t* tok_off, int n, int bs, int64_t* blk_off) {
    if (bs <= 0 || n < 0) return -1;
    int64_t acc = 0;
    for (int i = 0; i < n; ++i) {
        if (blk_off) blk_off[i] = acc;
        const int64_t len = tok_off[i + 1] - tok_off[i];
        acc += (len + bs - 1) / bs;
    }
    if (blk_off) blk_off[n] = acc;
    return acc;
}

int cs_hash_prompts(cs_pool_t pool, const uint32_t* tokens, const int64_t* tok_off, int n, int bs, int skip, int take,
                    const int64_t* blk_off, uint64_t* keys_out, int32_t* counts_out, uint64_t* agents_out) {
    return guard([&] {
        if (!pool || !tok_off || !blk_off || n < 0) throw std::invalid_argument("cs_hash_prompts: null argument");
        if (bs <= 0) throw std::invalid_argument("block_keys_for: block_size must be positive");
        if (skip < 0 || take < 1) throw std::invalid_argument("derive_agent_identity: skip >= 0 and take >= 1 required");
        if (n == 0) return;
        const int64_t ntok = tok_off[n] - tok_off[0];
        const int64_t nblk = blk_off[n];
        for (int i = 0; i < n; ++i)
            if (tok_off[i + 1] <= tok_off[i]) throw std::invalid_argument("chain_hash: token sequence must be nonempty");
        cudaStream_t s = pool->stream;
        csb::DevBuf tok, off, boff, k, c, ag, err;
        tok.ensure(sizeof(uint32_t) * (ntok + 4));
        off.ensure(sizeof(int64_t) * (n + 1));
        boff.ensure(sizeof(int64_t) * (n + 1));
        k.ensure(sizeof(uint64_t) * nblk);
        c.ensure(sizeof(int32_t) * nblk);
        ag.ensure(sizeof(uint64_t) * n);
        err.ensure(sizeof(int));
        std::vector<int64_t> rel(n + 1);
        for (int i = 0; i <= n; ++i) rel[i] = tok_off[i] - tok_off[0];
        ck(cudaMemcpyAsync(tok.p, tokens + tok_off[0], sizeof(uint32_t) * ntok, cudaMemcpyHostToDevice, s), "H2D");
        ck(cudaMemcpyAsync(off.p, rel.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s), "H2D");
        ck(cudaMemcpyAsync(boff.p, blk_off, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s), "H2D");
        ck(cudaMemsetAsync(err.p, 0, sizeof(int), s), "memset");
        ck(csb::launch_hash_prompts(tok.as<unsigned int>(), off.as<long long>(), n, bs, skip, take,
                                    boff.as<long long>(), k.as<unsigned long long>(), c.as<int>(),
                                    ag.as<unsigned long long>(), err.as<int>(), s),
           "hash_prompts");
        if (keys_out) ck(cudaMemcpyAsync(keys_out, k.p, sizeof(uint64_t) * nblk, cudaMemcpyDeviceToHost, s), "D2H");
        if (counts_out) ck(cudaMemcpyAsync(counts_out, c.p, sizeof(int32_t) * nblk, cudaMemcpyDeviceToHost, s), "D2H");
        if (agents_out) ck(cudaMemcpyAsync(agents_out, ag.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s), "D2H");
        int herr = 0;
        ck(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
        pool->sync();
        tok.release();
        off.release();
        boff.release();
        k.release();
        c.release();
        ag.release();
        err.release();
        if (herr) throw std::invalid_argument("chain_hash: token sequence must be nonempty");
    });
}

static void need_device() {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw CsError(CS_ERR_CUDA, "no CUDA device: cachesage_b200 has no CPU fallback");
}

int cs_chain_hash(const uint64_t* parents, const uint8_t* has_parent, const uint32_t* tokens, const int64_t* tok_off,
                  int n, uint64_t* out) {
    return guard([&] {
        if (n < 0 || (n > 0 && (!tokens || !tok_off || !out))) throw std::invalid_argument("cs_chain_hash: null argument");
        for (int i = 0; i < n; ++i)
            if (tok_off[i + 1] <= tok_off[i]) throw std::invalid_argument("chain_hash: token sequence must be nonempty");
        if (n == 0) return;
        need_device();
        const int64_t ntok = tok_off[n] - tok_off[0];
        csb::DevBuf tk, off, par, hp, o;
        tk.ensure(4 * (size_t)ntok);
        off.ensure(8 * (size_t)(n + 1));
        o.ensure(8 * (size_t)n);
        std::vector<int64_t> rel(n + 1);
        for (int i = 0; i <= n; ++i) rel[i] = tok_off[i] - tok_off[0];
        ck(cudaMemcpy(tk.p, tokens + tok_off[0], 4 * (size_t)ntok, cudaMemcpyHostToDevice), "H2D");
        ck(cudaMemcpy(off.p, rel.data(), 8 * (size_t)(n + 1), cudaMemcpyHostToDevice), "H2D");
        if (parents && has_parent) {
            par.ensure(8 * (size_t)n);
            hp.ensure((size_t)n);
            ck(cudaMemcpy(par.p, parents, 8 * (size_t)n, cudaMemcpyHostToDevice), "H2D");
            ck(cudaMemcpy(hp.p, has_parent, (size_t)n, cudaMemcpyHostToDevice), "H2D");
        }
        ck(csb::launch_chain_hash(par.as<unsigned long long>(), hp.as<unsigned char>(), tk.as<unsigned int>(),
                                  off.as<long long>(), n, o.as<unsigned long long>(), 0),
           "chain_hash");
        ck(cudaMemcpy(out, o.p, 8 * (size_t)n, cudaMemcpyDeviceToHost), "D2H");
    });
}

int cs_derive_agent_identity(const uint64_t* keys, const int64_t* key_off, int n, int skip, int take, uint64_t* out) {
    return guard([&] {
        if (n < 0 || (n > 0 && (!key_off || !out))) throw std::invalid_argument("cs_derive_agent_identity: null argument");
        if (skip < 0 || take < 1) throw std::invalid_argument("derive_agent_identity: skip >= 0 and take >= 1 required");
        if (n == 0) return;
        need_device();
        const int64_t nk = key_off[n] - key_off[0];
        csb::DevBuf k, off, o;
        k.ensure(8 * (size_t)std::max<int64_t>(nk, 1));
        off.ensure(8 * (size_t)(n + 1));
        o.ensure(8 * (size_t)n);
        std::vector<int64_t> rel(n + 1);
        for (int i = 0; i <= n; ++i) rel[i] = key_off[i] - key_off[0];
        if (nk > 0) ck(cudaMemcpy(k.p, keys + key_off[0], 8 * (size_t)nk, cudaMemcpyHostToDevice), "H2D");
        ck(cudaMemcpy(off.p, rel.data(), 8 * (size_t)(n + 1), cudaMemcpyHostToDevice), "H2D");
        ck(csb::launch_identity(k.as<unsigned long long>(), off.as<long long>(), n, skip, take,
                                o.as<unsigned long long>(), 0),
           "derive_agent_identity");
        ck(cudaMemcpy(out, o.p, 8 * (size_t)n, cudaMemcpyDeviceToHost), "D2H");
    });
}

static void stage_prompt(cs_pool_t pool, const uint64_t* keys, const int32_t* counts, int n) {
    pool->d_keys.ensure(sizeof(uint64_t) * std::max(n, 1));
    pool->d_counts.ensure(sizeof(int32_t) * std::max(n, 1));
    pool->d_pins.ensure(sizeof(uint32_t) * std::max(n, 1));
    if (n > 0) {
        ck(cudaMemcpyAsync(pool->d_keys.p, keys, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, pool->stream), "H2D");
        if (counts)
            ck(cudaMemcpyAsync(pool->d_counts.p, counts, sizeof(int32_t) * n, cudaMemcpyHostToDevice, pool->stream),
               "H2D");
        else
            ck(cudaMemsetAsync(pool->d_counts.p, 0, sizeof(int32_t) * n, pool->stream), "memset");
    }
}

int cs_lookup(cs_pool_t pool, const uint64_t* keys, const int32_t* counts, int n, uint64_t tick_base,
              int64_t* cached, int* first_miss) {
    return guard([&] {
        if (!pool || n < 0 || (n > 0 && (!keys || !counts))) throw std::invalid_argument("cs_lookup: null argument");
        stage_prompt(pool, keys, counts, n);
        csb::AdmitArgs a{};
        a.keys = pool->d_keys.as<unsigned long long>();
        a.counts = pool->d_counts.as<int>();
        a.n = n;
        a.flags = csb::kLookup;
        a.prev = -1;
        a.next = -1;
        a.agent = CS_NO_AGENT;
        a.anchor = 0;
        a.tick_base = tick_base;
        const auto& st = pool->admit(a, 0);
        if (cached) *cached = st.cached;
        if (first_miss) *first_miss = st.first_miss;
    });
}

int cs_probe_needed(cs_pool_t pool, const uint64_t* keys, int n, int* needed) {
    return guard([&] {
        if (!pool || n < 0 || (n > 0 && !keys) || !needed) throw std::invalid_argument("cs_probe_needed: null argument");
        pool->flush_unpins();
        pool->flush_table();
        stage_prompt(pool, keys, nullptr, n);
        pool->d_aux.ensure(sizeof(int));
        ck(csb::launch_probe(pool->P, pool->d_keys.as<unsigned long long>(), n, pool->d_aux.as<int>(), pool->stream),
           "probe");
        ck(cudaMemcpyAsync(needed, pool->d_aux.p, sizeof(int), cudaMemcpyDeviceToHost, pool->stream), "D2H");
        pool->sync();
    });
}

int cs_observe_dispatch(cs_pool_t pool, int prev, int next, uint64_t tick, int* warmup_target) {
    return guard([&] {
        if (!pool || next < 0 || next >= pool->n_agents || prev >= pool->n_agents)
            throw std::invalid_argument("cs_observe_dispatch: agent index out of range");
        pool->check_tick(tick);  // Runtime::dispatch_event (runtime.cpp:59-64)
        csb::AdmitArgs a{};
        a.keys = nullptr;
        a.counts = nullptr;
        a.n = 0;
        a.flags = csb::kDispatch;
        a.prev = prev;
        a.next = next;
        a.agent = CS_NO_AGENT;
        a.tick_base = tick - 1;  // the kernel assigns tick_base + 1 to the dispatch
        const auto& st = pool->admit(a, 0);
        pool->note_dispatch(prev, next);
        if (warmup_target) *warmup_target = st.warm_issued;
    });
}

int cs_admit_pinned(cs_pool_t pool, const uint64_t* keys, const int32_t* counts, int n, uint32_t agent,
                    int anchor_blocks, uint64_t tick_base, uint64_t* evicted, int64_t cap, int64_t* n_evicted,
                    uint32_t* pins) {
    return guard([&] {
        if (!pool || n < 0 || (n > 0 && (!keys || !counts))) throw std::invalid_argument("cs_admit_pinned: null argument");
        if (agent != CS_NO_AGENT && (int)agent >= pool->n_agents)
            throw std::invalid_argument("cs_admit_pinned: unregistered agent index");
        stage_prompt(pool, keys, counts, n);
        csb::AdmitArgs a{};
        a.keys = pool->d_keys.as<unsigned long long>();
        a.counts = pool->d_counts.as<int>();
        a.n = n;
        a.flags = csb::kAdmit;
        a.prev = -1;
        a.next = -1;
        a.agent = agent;
        a.anchor = anchor_blocks;
        a.tick_base = tick_base;
        a.pins_out = pool->d_pins.as<unsigned int>();
        const unsigned long long ev_before = pool->ev_total;
        const auto& st = pool->admit(a, n);
        const long long ne = (long long)(st.ev_total - ev_before);
        if (n_evicted) *n_evicted = ne;
        if (evicted && cap > 0 && ne > 0) {
            std::vector<unsigned long long> v(ne);
            pool->copy_victims(ev_before, st.ev_total, v.data());
            std::memcpy(evicted, v.data(), sizeof(uint64_t) * std::min<long long>(ne, cap));
        }
        if (pins && n > 0)
            ck(cudaMemcpy(pins, pool->d_pins.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost), "pins D2H");
    });
}

int cs_unpin_slots(cs_pool_t pool, const uint32_t* slots, int n) {
    return guard([&] {
        if (!pool || n < 0 || (n > 0 && !slots)) throw std::invalid_argument("cs_unpin_slots: null argument");
        pool->sync();  // (an engine's last admission may still be finishing its prescan)
        pool->flush_unpins();
        pool->pre_ok = false;
        pool->d_aux.ensure(sizeof(uint32_t) * std::max(n, 1));
        ck(cudaMemcpyAsync(pool->d_aux.p, slots, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, pool->stream), "H2D");
        ck(csb::launch_unpin(pool->P, pool->d_aux.as<unsigned int>(), n, pool->stream), "unpin");
        pool->sync();
        csb::Ctrl c;
        ck(cudaMemcpy(&c, pool->P.ctrl, sizeof(c), cudaMemcpyDeviceToHost), "ctrl D2H");
        pool->pinned = c.pinned;
    });
}

int cs_restore(cs_pool_t pool, const uint64_t* keys, const uint64_t* lt, const uint32_t* agents, const uint32_t* refs,
               int64_t n) {
    return guard([&] {
        if (!pool || n < 0 || (n > 0 && (!keys || !lt))) throw std::invalid_argument("cs_restore: null argument");
        for (int64_t i = 0; i < n; ++i)
            if (lt[i] >= csb::kMaxTick) throw std::invalid_argument("cs_restore: last_touch must stay below 2^40 - 1");
        pool->flush_unpins();
        pool->flush_table();
        pool->pre_ok = false;
        // a shard keeps the snapshot blocks it owns (the caller may pass the whole snapshot)
        std::vector<uint64_t> fk, fl;
        std::vector<uint32_t> fa, fr;
        if (pool->comm && pool->P.world > 1) {
            for (int64_t i = 0; i < n; ++i) {
                if (csb::shard_owner(keys[i], pool->P.world) != pool->P.rank) continue;
                fk.push_back(keys[i]);
                fl.push_back(lt[i]);
                if (agents) fa.push_back(agents[i]);
                if (refs) fr.push_back(refs[i]);
            }
            n = (int64_t)fk.size();
            keys = fk.data();
            lt = fl.data();
            if (agents) agents = fa.data();
            if (refs) refs = fr.data();
            csb::Ctrl c0;
            ck(cudaMemcpy(&c0, pool->P.ctrl, sizeof(c0), cudaMemcpyDeviceToHost), "ctrl D2H");
            pool->resident = c0.resident;
        }
        if (pool->resident + n > pool->P.cap) throw std::invalid_argument("cs_restore: snapshot exceeds the budget");
        if (n == 0) return;
        cudaStream_t s = pool->stream;
        csb::DevBuf k, l, ag, rf;
        k.ensure(8 * n);
        l.ensure(8 * n);
        ck(cudaMemcpyAsync(k.p, keys, 8 * n, cudaMemcpyHostToDevice, s), "H2D");
        ck(cudaMemcpyAsync(l.p, lt, 8 * n, cudaMemcpyHostToDevice, s), "H2D");
        if (agents) {
            ag.ensure(4 * n);
            ck(cudaMemcpyAsync(ag.p, agents, 4 * n, cudaMemcpyHostToDevice, s), "H2D");
        }
        if (refs) {
            rf.ensure(4 * n);
            ck(cudaMemcpyAsync(rf.p, refs, 4 * n, cudaMemcpyHostToDevice, s), "H2D");
        }
        ck(csb::launch_restore(pool->P, k.as<unsigned long long>(), l.as<unsigned long long>(),
                               agents ? ag.as<unsigned int>() : nullptr, refs ? rf.as<unsigned int>() : nullptr, n, s),
           "restore");
        pool->sync();
        k.release();
        l.release();
        ag.release();
        rf.release();
        csb::Ctrl c;
        ck(cudaMemcpy(&c, pool->P.ctrl, sizeof(c), cudaMemcpyDeviceToHost), "ctrl D2H");
        pool->resident = c.resident;
        pool->pinned = c.pinned;
    });
}

int cs_score_snapshot(cs_pool_t pool, uint64_t now_tick, uint64_t* keys, double* scores, int64_t cap, int64_t* n) {
    return guard([&] {
        if (!pool) throw std::invalid_argument("cs_score_snapshot: null pool");
        pool->sync();  // (an engine's last admission may still be finishing its prescan)
        pool->flush_unpins();
        const long long N = pool->P.cap;
        csb::DevBuf k, s, cnt, scr;
        k.ensure(8 * N);
        s.ensure(8 * N);
        cnt.ensure(8);
        scr.ensure(8);
        ck(csb::launch_scores(pool->P, now_tick, k.as<unsigned long long>(), s.as<double>(), cnt.as<long long>(),
                              scr.as<unsigned long long>(), pool->stream),
           "scores");
        long long m = 0;
        ck(cudaMemcpyAsync(&m, cnt.p, 8, cudaMemcpyDeviceToHost, pool->stream), "D2H");
        pool->sync();
        if (n) *n = m;
        const long long c = std::min<long long>(m, cap);
        if (c > 0 && keys) ck(cudaMemcpy(keys, k.p, 8 * c, cudaMemcpyDeviceToHost), "D2H");
        if (c > 0 && scores) ck(cudaMemcpy(scores, s.p, 8 * c, cudaMemcpyDeviceToHost), "D2H");
    });
}

int cs_set_hops(cs_pool_t pool, const uint8_t* hops, int n) {
    return guard([&] {
        if (!pool || (n > 0 && !hops) || n < 0 || n > pool->P.a_cap) throw std::invalid_argument("cs_set_hops: bad argument");
        pool->flush_unpins();
        pool->sync();
        // ReachabilityState as rebuild_reachability would leave it (reachability.cpp:39-81): the
        // survival class of an agent is its hop count, capped at e_max (reachability.cpp:12-20)
        std::vector<unsigned char> h(std::max(n, 1)), c(std::max(n, 1));
        for (int i = 0; i < n; ++i) {
            h[i] = hops[i];
            c[i] = (unsigned char)std::min<int>(hops[i], pool->P.e_max);
        }
        if (n > 0) {
            ck(cudaMemcpyAsync(pool->P.hop, h.data(), n, cudaMemcpyHostToDevice, pool->stream), "hop H2D");
            ck(cudaMemcpyAsync(pool->P.cls, c.data(), n, cudaMemcpyHostToDevice, pool->stream), "cls H2D");
        }
        const int one = 1;
        ck(cudaMemcpyAsync(reinterpret_cast<char*>(pool->P.ctrl) + offsetof(csb::Ctrl, reach_built), &one, sizeof(int),
                           cudaMemcpyHostToDevice, pool->stream),
           "reach_built H2D");
        pool->pre_ok = false;  // classes changed out of band: no prescan reuse
        pool->reach_known = (size_t)n;
        pool->sync();
    });
}

int cs_hops(cs_pool_t pool, int* hops, int n) {
    return guard([&] {
        if (!pool || !hops || n < 0 || n > pool->P.a_cap) throw std::invalid_argument("cs_hops: bad argument");
        pool->sync();  // (an engine's last admission may still be finishing its prescan)
        csb::Ctrl c;
        ck(cudaMemcpy(&c, pool->P.ctrl, sizeof(c), cudaMemcpyDeviceToHost), "ctrl D2H");
        std::vector<unsigned char> h(std::max(n, 1));
        if (n > 0) ck(cudaMemcpy(h.data(), pool->P.hop, n, cudaMemcpyDeviceToHost), "hop D2H");
        for (int i = 0; i < n; ++i) hops[i] = c.reach_built ? (int)h[i] : -1;
    });
}

int cs_poll_actions(cs_pool_t pool, int* targets, uint64_t* ticks, int cap, int* n) {
    return guard([&] {
        if (!pool || !n) throw std::invalid_argument("cs_poll_actions: null argument");
        pool->sync();  // (an engine's last admission may still be finishing its prescan)
        const int m = (int)pool->pending_targets.size();
        for (int i = 0; i < m && i < cap; ++i) {
            if (targets) targets[i] = pool->pending_targets[i];
            if (ticks) ticks[i] = pool->pending_ticks[i];
        }
        *n = m;
        pool->pending_targets.clear();
        pool->pending_ticks.clear();
        pool->poll_reset_pending = true;
    });
}

/* Instrumentation: per-CTA timestamps of the last scan (grid x 8 u64, globaltimer ns). */
int cs_pool_check(cs_pool_t pool, int64_t* out4) {
    return guard([&] {
        if (!pool || !out4) throw std::invalid_argument("cs_pool_check: null argument");
        pool->flush_unpins();
        pool->flush_table();
        pool->sync();
        unsigned long long* d = nullptr;
        ck(cudaMalloc(&d, 32), "cudaMalloc");
        ck(cudaMemset(d, 0, 32), "memset");
        unsigned long long h[4] = {0, 0, 0, 0};
        cudaError_t e = csb::launch_check_pool(pool->P, d, pool->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(pool->stream);
        if (e == cudaSuccess) e = cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        cudaFree(d);
        ck(e, "check_pool_kernel");
        csb::Ctrl c;
        ck(cudaMemcpy(&c, pool->P.ctrl, sizeof(c), cudaMemcpyDeviceToHost), "ctrl D2H");
        out4[0] = (int64_t)h[0];
        out4[1] = (int64_t)h[1] - c.resident;  // 0 when the count matches the pool's scalar
        out4[2] = (int64_t)h[2] - c.pinned;
        out4[3] = (int64_t)h[3];
    });
}

int cs_pool_debug(cs_pool_t pool, uint64_t* out, int cap, int* grid) {
    return guard([&] {
        if (!pool || !out) throw std::invalid_argument("cs_pool_debug: null argument");
        pool->sync();
        const int n = std::min(cap, pool->lc.grid * 16 + 256);
        ck(cudaMemcpy(out, pool->P.dbg, 8 * (size_t)n, cudaMemcpyDeviceToHost), "dbg D2H");
        if (grid) *grid = pool->lc.grid;
    });
}

int cs_pool_get_stats(cs_pool_t pool, cs_pool_stats* out) {
    return guard([&] {
        if (!pool || !out) throw std::invalid_argument("cs_pool_get_stats: null argument");
        pool->flush_unpins();
        pool->sync();
        csb::Ctrl c;
        ck(cudaMemcpy(&c, pool->P.ctrl, sizeof(c), cudaMemcpyDeviceToHost), "ctrl D2H");
        out->resident = c.resident;
        out->pinned = c.pinned;
        out->evictions = (int64_t)c.n_ev;
        out->tombstones = c.tombstones;
        out->scans = c.scans;
        out->scanned_slots = c.scanned_slots;
        out->rebuilds = c.rebuilds;
        out->n_agents = pool->n_agents;
        for (int k = 0; k < csb::kPhases; ++k) out->phase_ns[k] = pool->phase_ns[k];
        out->prescan_used = c.pre_used;
        out->prescan_fallbacks = c.pre_fallbacks;
        out->prescan_unusable = c.pre_badcnt;
        out->server_launches = pool->server_launches;
        out->host_turnarounds = pool->host_turnarounds;
        out->host_turnaround_ns = pool->host_turnaround_ns;
    });
}

}  // extern "C"
