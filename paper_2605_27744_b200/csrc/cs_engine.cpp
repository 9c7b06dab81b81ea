// cs_engine: the EngineSim-equivalent host scheduler over a device pool, plus the (widened)
// trace generator. The scheduler is host C++ by design ("scheduler = caller,
// kept on the host"); every pool / policy decision it needs is one admission launch.
//
// Reference behaviour restated (paths relative to /root/reference/proj):
//   generate_trace                 workload.cpp:156-182 (draws :131-153)
//   materialize_requests           engine.cpp:8-35      -> K1 hash_turns on the device
//   build_warmup_catalog           engine.cpp:37-54     -> K1 hash_turns (warmup descriptors)
//   load / step / done             engine.cpp:240-255, 372-392
//   arrive / activate_sessions     engine.cpp:262-276
//   start_request / try_start_head engine.cpp:278-351   -> one admit_kernel launch
//   complete_earliest              engine.cpp:353-370   -> unpin_kernel
//   drain_and_run_warmups          engine.cpp:197-238   -> admit_kernel (lookup + room + unpin)
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <deque>
#include <map>
#include <random>
#include <unordered_map>
#include <vector>

#include "cs_engine_state.h"
#include "cs_output.hpp"
#include "cs_pool.hpp"

using csb::ck;
using csb::CsError;

void cs_set_error(const std::string& m);  // cs_pool.cpp

namespace {

template <class F>
int eguard(F&& f) {
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

struct Spec {
    int n_agents;
    std::vector<int> anchor;
    std::vector<double> trans;
    int supervisor;
    int turns_min, turns_max, sessions, task_tokens, history_growth, decode_tokens, template_tokens;
    int concurrency, budget_blocks;
    uint64_t seed;
    uint32_t anchor_stride;
    int pos_bits;
    std::vector<double> start_dist;  // supervisor == -2: per-session start draw
};

Spec to_spec(const cs_workload_spec* s) {
    if (!s || s->n_agents < 1 || !s->anchor_tokens || !s->transition)
        throw std::invalid_argument("workload: no agents");
    Spec o;
    o.n_agents = s->n_agents;
    o.anchor.assign(s->anchor_tokens, s->anchor_tokens + s->n_agents);
    o.trans.assign(s->transition, s->transition + (size_t)s->n_agents * s->n_agents);
    o.supervisor = s->supervisor;
    o.turns_min = s->turns_min;
    o.turns_max = s->turns_max;
    o.sessions = s->sessions;
    o.task_tokens = s->task_tokens;
    o.history_growth = s->history_growth;
    o.decode_tokens = s->decode_tokens;
    o.template_tokens = s->template_tokens;
    o.concurrency = s->concurrency;
    o.budget_blocks = s->budget_blocks;
    o.seed = s->seed;
    o.anchor_stride = s->anchor_stride ? s->anchor_stride : 0x00010000u;
    o.pos_bits = s->hist_pos_bits ? s->hist_pos_bits : 20;
    if (s->supervisor == -2) {
        if (!s->start_dist) throw std::invalid_argument("workload: supervisor -2 needs start_dist");
        o.start_dist.assign(s->start_dist, s->start_dist + s->n_agents);
    }
    // WorkloadSpec::validate (workload.cpp:60-123), with the token-id limits of the chosen scheme
    for (int i = 0; i < o.n_agents; ++i) {
        double sum = 0.0;
        for (int j = 0; j < o.n_agents; ++j) {
            const double p = o.trans[(size_t)i * o.n_agents + j];
            if (p < 0.0) throw std::invalid_argument("workload: negative transition probability");
            sum += p;
        }
        if (std::abs(sum - 1.0) > 1e-9) throw std::invalid_argument("workload: transition row does not sum to 1");
        if (o.anchor[i] < 1 || (uint32_t)o.anchor[i] >= o.anchor_stride)
            throw std::invalid_argument("workload: anchor_tokens out of range");
    }
    if ((uint64_t)o.n_agents * o.anchor_stride > 0x01000000ull)
        throw std::invalid_argument("workload: too many agents for the anchor token stride");
    if (o.supervisor >= o.n_agents || o.supervisor < -2) throw std::invalid_argument("workload: supervisor index out of range");
    if (o.turns_min < 1 || o.turns_max < o.turns_min) throw std::invalid_argument("workload: bad turns_per_session range");
    if (o.sessions < 1 || (uint64_t)o.sessions > (1ull << (31 - o.pos_bits)))
        throw std::invalid_argument("workload: sessions out of range");
    if (o.task_tokens < 0 || o.history_growth < 0 || o.decode_tokens < 1 || o.template_tokens < 0)
        throw std::invalid_argument("workload: negative size parameter");
    const long long max_hist = (long long)o.task_tokens + (long long)(o.turns_max - 1) * o.history_growth;
    if (max_hist > (1ll << o.pos_bits) - 1) throw std::invalid_argument("workload: history exceeds token id space");
    return o;
}

// Turn = (session, turn_index, agent, anchor, history, prompt, decode)
struct Turn {
    int64_t v[7];
};

// generate_trace (workload.cpp:156-182): one std::mt19937_64 per session seeded from the spec
// seed; uniform turn count by modulo; categorical walk by cumulative sum over positive entries.
int categorical(std::mt19937_64& rng, const double* row, int n) {
    const double u = (double)(rng() >> 11) * 0x1.0p-53;
    double acc = 0.0;
    int last = 0;
    for (int i = 0; i < n; ++i) {
        if (row[i] <= 0.0) continue;
        last = i;
        acc += row[i];
        if (u < acc) return i;
    }
    return last;  // u fell into the rounding gap below 1.0
}

std::vector<Turn> generate(const Spec& s) {
    std::vector<Turn> out;
    const int start = s.supervisor >= 0 ? s.supervisor : 0;
    for (int sess = 0; sess < s.sessions; ++sess) {
        std::mt19937_64 rng(csb::mix64(s.seed ^ csb::mix64(0x5e5510ull + (uint64_t)sess)));
        const int turns = s.turns_min + (int)(rng() % (uint64_t)(s.turns_max - s.turns_min + 1));
        int agent = start;
        if (!s.start_dist.empty()) agent = categorical(rng, s.start_dist.data(), s.n_agents);
        for (int t = 0; t < turns; ++t) {
            if (t > 0) agent = categorical(rng, s.trans.data() + (size_t)agent * s.n_agents, s.n_agents);
            Turn x;
            x.v[0] = sess;
            x.v[1] = t;
            x.v[2] = agent;
            x.v[3] = s.anchor[agent];
            x.v[4] = (int64_t)s.task_tokens + (int64_t)t * s.history_growth;
            x.v[5] = s.template_tokens + x.v[3] + x.v[4];
            x.v[6] = s.decode_tokens;
            out.push_back(x);
        }
    }
    return out;
}

}  // namespace

struct cs_engine {
    cs_engine_cfg cfg{};
    Spec spec;
    cs_pool* pool = nullptr;
    int budget = 0, conc = 0, bs = 16;

    struct Req {
        int session, turn_index;
        int agent;  // dense index
        int64_t blk_off;
        int nb;
        int anchor_blocks;
        int64_t prompt_tokens;
        int decode;
        int spec_agent;  // workload agent (its label in turns.csv)
    };
    std::vector<Req> reqs;
    struct Cat {
        int agent;
        int64_t blk_off;
        int nb;
        int64_t prompt_tokens;
    };
    std::unordered_map<int, Cat> catalog;  // by agent index
    csb::DevBuf d_keys, d_counts, d_pins, d_cat_pins;
    // host_inputs: prompt blocks in pinned host memory, staged per admission
    uint64_t* h_keys = nullptr;
    int* h_counts = nullptr;
    // host_inputs: per request one pinned blob [keys (8 nb) | counts (4 nb)] at byte 12 * blk_off,
    // so an admission's inputs are ONE H2D copy; victims land in h_vict (pinned) by a D2H copy
    // queued right behind the admission kernel (one stream sync for the whole admission)
    unsigned char* h_blob = nullptr;
    unsigned long long* h_vict = nullptr;
    int h_vict_cap = 0;
    csb::DevBuf d_stage_keys, d_stage_keys2, d_stage_counts;
    bool stage_flip = false;
    int64_t h2d_bytes = 0, d2h_bytes = 0;
    void stage(csb::AdmitArgs& a, int64_t blk_off, int nb);
    void fetch_victims(unsigned long long before);

    // scheduler (EngineSim::Scheduler, engine.hpp:158-168)
    std::map<int, std::vector<int64_t>> by_session;
    std::deque<int> pending_sessions;
    std::unordered_map<int, size_t> session_pos;
    std::vector<double> arrival_us;
    std::deque<int64_t> ready;
    struct Flight {
        double end_us;
        uint64_t seq;
        int64_t req;
        int npins;
        int64_t cached;
        double start_us;
    };
    std::vector<Flight> in_flight;
    uint64_t flight_seq = 0;
    int active_sessions = 0;
    bool loaded = false;

    uint64_t tick = 0;
    // Belady: BeladyPolicy::cursor_ (highest arrived request id) and its value at the last launch
    unsigned long long bel_cursor = 0, bel_cursor_dev = 0;
    std::vector<long long> bel_off;  // request block offsets (n_req + 1)
    void belady_args(csb::AdmitArgs& a, int64_t blk_off) {
        if (pool->P.policy != 3) return;
        a.kids = pool->bel_kid_of() + blk_off;
        a.cursor = bel_cursor;
        a.adv_lo = bel_off[bel_cursor_dev + 1 < bel_off.size() ? bel_cursor_dev + 1 : bel_off.size() - 1];
        a.adv_hi = bel_off[bel_cursor + 1 < bel_off.size() ? bel_cursor + 1 : bel_off.size() - 1];
        if (a.adv_hi < a.adv_lo) a.adv_hi = a.adv_lo;
    }
    double sim_now = 0.0;
    int last_dispatched = -1;

    // outputs
    std::vector<int64_t> t_cached, t_prompt;
    std::vector<double> t_start, t_end;
    std::vector<char> t_done;
    std::vector<unsigned long long> evictions;
    unsigned long long ev_drained = 0;
    std::vector<int64_t> w_step;
    std::vector<uint64_t> w_target, w_tick;
    int64_t completed = 0, truncated = 0, warm_exec = 0, warm_drop = 0, steps = 0, admissions = 0;
    int64_t warm_uncached = 0;     // EngineSim::warmup_uncached_tokens_ (engine.cpp:223)
    double warm_time_us = 0.0;     // EngineSim::warmup_time_us_ (engine.cpp:224-227)
    // recorded event stream (events.jsonl): EngineSim::events_ (engine.cpp:72-88)
    bool rec_events = false;
    std::vector<csb::EventRec> events;
    csb::DevBuf d_touch;
    std::vector<unsigned int> h_touch;
    std::vector<unsigned long long> h_tkeys;
    void ev_push(uint64_t tick_, uint8_t kind, uint64_t a, uint64_t b, bool has_a = true, bool has_b = true) {
        csb::EventRec e{};
        e.tick = tick_;
        e.kind = kind;
        e.a = a;
        e.b = b;
        e.has_a = has_a;
        e.has_b = has_b;
        events.push_back(e);
    }
    // BlockTouch events of a lookup that touched the first f prompt blocks from tick t0 + 1 on
    void ev_touches(const csb::AdmitArgs& a, int f, uint64_t t0) {
        if (!rec_events || f <= 0) return;
        h_touch.resize(f);
        h_tkeys.resize(f);
        ck(cudaMemcpy(h_touch.data(), a.touch_agent, 4 * (size_t)f, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(h_tkeys.data(), a.keys, 8 * (size_t)f, cudaMemcpyDeviceToHost), "D2H");
        for (int i = 0; i < f; ++i) {
            const unsigned int ag = h_touch[i];
            const bool has = ag != csb::kNoAgent;
            ev_push(t0 + 1 + (uint64_t)i, csb::EventRec::kBlockTouch, h_tkeys[i], has ? pool->agent_ids[ag] : 0, true, has);
        }
    }
    void ev_prepare(csb::AdmitArgs& a, int nb) {
        if (!rec_events) return;
        if (4 * (size_t)std::max(nb, 1) > d_touch.n) pool->server_stop();  // (never while it runs)
        d_touch.ensure(4 * (size_t)std::max(nb, 1));
        a.touch_agent = d_touch.as<unsigned int>();
    }
    int64_t tot_prompt = 0, tot_cached = 0;

    static bool later(const Flight& a, const Flight& b) {
        return a.end_us > b.end_us || (a.end_us == b.end_us && a.seq > b.seq);
    }

    void build(const cs_engine_cfg& c, const cs_workload_spec* ws, long long shard_slots = 0, cs_comm* comm = nullptr,
               const int64_t* turns7 = nullptr, int64_t n_turns = -1);
    int64_t warm_prompt = 0;  // EngineSim::warmup_prompt_tokens_ (engine.cpp:222)
    // device-resident scheduler (cs_engine_dev.cuh): whole steps in one persistent launch
    bool dev = false;
    csb::EngState hs{};  // authoritative between launches
    csb::DevBuf d_state, d_reqs, d_soff, d_sreqs, d_spos, d_cat, d_tc, d_tp, d_ts, d_te, d_td, d_ta, d_ws, d_wt,
        d_wk, d_args, d_cmd;
    long long w_cap = 0;
    void dev_setup();
    void dev_run(long long stop_at, long long max_steps);
    void dev_pull_outputs();
    long long max_nb = 1;
    // admissions per persistent launch: the eviction log (drained between launches) must not wrap
    long long dev_chunk() const { return std::max(1ll, (long long)pool->P.evlog_cap / (2 * std::max(1ll, max_nb))); }
    void drain_evictions(bool force);
    bool done() const {
        if (dev) return hs.n_flight == 0 && hs.ready_n == 0 && hs.next_session >= hs.n_sessions;
        return loaded && in_flight.empty() && ready.empty() && pending_sessions.empty();
    }
    void arrive(int64_t idx);
    void activate_sessions();
    bool try_start_head();
    void complete_earliest();
    void drain_and_run_warmups();
    void execute_warmup(int target);
    void step();
};

void cs_engine::build(const cs_engine_cfg& c, const cs_workload_spec* ws, long long shard_slots, cs_comm* comm,
                      const int64_t* turns7, int64_t n_turns) {
    cfg = c;
    spec = to_spec(ws);
    bs = c.block_size;
    if (bs < 1) throw std::invalid_argument("EngineSim: budget, block size, and concurrency must be positive");
    if (c.skip < 0 || c.take < 1) throw std::invalid_argument("CacheSagePolicy: invalid identity window");
    budget = c.pool.budget_blocks > 0 ? (int)c.pool.budget_blocks : spec.budget_blocks;
    conc = c.concurrency > 0 ? c.concurrency : spec.concurrency;
    if (budget < 1 || conc < 1) throw std::invalid_argument("EngineSim: budget, block size, and concurrency must be positive");
    // CostModel validation (engine.cpp:60-63)
    if (!(c.prefill_per_token_us > 0.0) || !(c.prefill_base_us > 0.0) || !(c.decode_per_token_us > 0.0))
        throw std::invalid_argument("EngineSim: cost model parameters must be positive");

    // the spec's generated trace, or an explicit one (a trace read back from JSONL, run_sim)
    std::vector<Turn> turns;
    if (turns7) {
        turns.resize(n_turns);
        for (int64_t i = 0; i < n_turns; ++i) {
            std::memcpy(turns[i].v, turns7 + 7 * i, sizeof(turns[i].v));
            if (turns[i].v[2] < 0 || turns[i].v[2] >= spec.n_agents)
                throw std::invalid_argument("trace: agent index out of range");
            if (turns[i].v[5] <= 0) throw std::invalid_argument("trace: prompt must be non-empty");
        }
    } else {
        turns = generate(spec);
    }
    const int64_t nt = (int64_t)turns.size();
    // materialize_requests on the device: K1 over synthesised token ids
    std::vector<csb::TurnDesc> desc(nt + spec.n_agents);
    int64_t off = 0;
    for (int64_t i = 0; i < nt; ++i) {
        const Turn& t = turns[i];
        csb::TurnDesc& d = desc[i];
        d.session = (int)t.v[0];
        d.agent = (int)t.v[2];
        d.anchor_tokens = (int)t.v[3];
        d.history_tokens = (int)t.v[4];
        d.template_tokens = spec.template_tokens;
        d.warmup = 0;
        d.blk_off = off;
        off += (t.v[5] + bs - 1) / bs;
    }
    const int64_t req_blocks = off;
    for (int a = 0; a < spec.n_agents; ++a) {  // build_warmup_catalog: template + anchor + 1 token
        csb::TurnDesc& d = desc[nt + a];
        d.session = 0;
        d.agent = a;
        d.anchor_tokens = spec.anchor[a];
        d.history_tokens = 0;
        d.template_tokens = spec.template_tokens;
        d.warmup = 1;
        d.blk_off = off;
        off += (spec.template_tokens + spec.anchor[a] + 1 + bs - 1) / bs;
    }
    const int64_t total_blocks = off;
    cs_pool_cfg pc = c.pool;
    pc.budget_blocks = budget;
    pool = new cs_pool();
    try {
        pool->create(pc, shard_slots, comm);  // selects the device; every allocation below lands on it
    } catch (...) {
        pool->destroy();
        delete pool;
        pool = nullptr;
        throw;
    }
    pool->timing = c.timing != 0;
    // the scheduler needs only the status of an admission: it enqueues the next one while the
    // previous launch's prescan CTAs (sharded: the replay's table updates) finish
    // (cs_pool::wait_status)
    pool->early_status = true;
    d_keys.ensure(8 * total_blocks);
    d_counts.ensure(4 * total_blocks);
    d_pins.ensure(4 * total_blocks);
    csb::DevBuf d_desc, d_agents;
    d_desc.ensure(sizeof(csb::TurnDesc) * desc.size());
    d_agents.ensure(8 * desc.size());
    cudaStream_t s = pool->stream;
    ck(cudaMemcpyAsync(d_desc.p, desc.data(), sizeof(csb::TurnDesc) * desc.size(), cudaMemcpyHostToDevice, s), "H2D");
    ck(csb::launch_hash_turns(d_desc.as<csb::TurnDesc>(), (int)desc.size(), bs, c.skip, c.take, spec.anchor_stride,
                              spec.pos_bits, d_keys.as<unsigned long long>(), d_counts.as<int>(),
                              d_agents.as<unsigned long long>(), s),
       "hash_turns");
    std::vector<uint64_t> ids(desc.size());
    ck(cudaMemcpyAsync(ids.data(), d_agents.p, 8 * desc.size(), cudaMemcpyDeviceToHost, s), "D2H");
    pool->sync();
    d_desc.release();
    d_agents.release();

    // dense agent indices in first-seen order (requests, then catalog)
    std::unordered_map<uint64_t, int> index;
    std::vector<uint64_t> order;
    auto idx_of = [&](uint64_t id) {
        auto it = index.find(id);
        if (it != index.end()) return it->second;
        const int k = (int)order.size();
        index.emplace(id, k);
        order.push_back(id);
        return k;
    };
    reqs.resize(nt);
    for (int64_t i = 0; i < nt; ++i) {
        const Turn& t = turns[i];
        Req& r = reqs[i];
        r.session = (int)t.v[0];
        r.turn_index = (int)t.v[1];
        r.agent = idx_of(ids[i]);
        r.blk_off = desc[i].blk_off;
        r.nb = (int)((t.v[5] + bs - 1) / bs);
        r.anchor_blocks = (int)((spec.template_tokens + t.v[3]) / bs);
        r.prompt_tokens = t.v[5];
        r.decode = (int)t.v[6];
        r.spec_agent = (int)t.v[2];
    }
    for (int a = 0; a < spec.n_agents; ++a) {
        const int k = idx_of(ids[nt + a]);
        if (catalog.count(k)) continue;  // catalog.emplace keeps the first
        Cat ct;
        ct.agent = k;
        ct.blk_off = desc[nt + a].blk_off;
        ct.nb = (int)((spec.template_tokens + spec.anchor[a] + 1 + bs - 1) / bs);
        ct.prompt_tokens = spec.template_tokens + spec.anchor[a] + 1;
        catalog.emplace(k, ct);
    }
    if ((int)order.size() > pool->P.a_cap)
        throw CsError(CS_ERR_CAPACITY, "distinct agent identities exceed agent_capacity");
    ck(cudaMemcpyAsync(pool->P.agent_ids, order.data(), 8 * order.size(), cudaMemcpyHostToDevice, s), "H2D");
    pool->agent_ids = order;
    pool->n_agents = (int)order.size();
    pool->sync();
    if (pool->P.policy == 3) {
        // BeladyPolicy(requests) (baselines.cpp:34-46): the next-use index over the request blocks
        std::vector<long long> offs(nt + 1);
        for (int64_t i = 0; i < nt; ++i) offs[i] = desc[i].blk_off;
        offs[nt] = req_blocks;
        pool->belady_index(d_keys.as<unsigned long long>(), req_blocks, offs);
        bel_off = std::move(offs);
    }
    if (c.host_inputs) {
        // the end-to-end path: prompt blocks live on the host and cross PCIe per admission
        ck(cudaMallocHost(reinterpret_cast<void**>(&h_keys), 8 * total_blocks), "cudaMallocHost");
        ck(cudaMallocHost(reinterpret_cast<void**>(&h_counts), 4 * total_blocks), "cudaMallocHost");
        ck(cudaMemcpy(h_keys, d_keys.p, 8 * total_blocks, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(h_counts, d_counts.p, 4 * total_blocks, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMallocHost(reinterpret_cast<void**>(&h_blob), 12 * std::max<int64_t>(total_blocks, 1)), "cudaMallocHost");
        int max_nb = 1;
        auto pack = [&](int64_t off, int nb) {
            std::memcpy(h_blob + 12 * off, h_keys + off, 8 * (size_t)nb);
            std::memcpy(h_blob + 12 * off + 8 * (size_t)nb, h_counts + off, 4 * (size_t)nb);
            max_nb = std::max(max_nb, nb);
        };
        for (int64_t i = 0; i < nt; ++i) pack(desc[i].blk_off, (int)((turns[i].v[5] + bs - 1) / bs));
        for (int ag = 0; ag < spec.n_agents; ++ag)
            pack(desc[nt + ag].blk_off, (int)((spec.template_tokens + spec.anchor[ag] + 1 + bs - 1) / bs));
        h_vict_cap = max_nb;
        ck(cudaMallocHost(reinterpret_cast<void**>(&h_vict), 8 * (size_t)h_vict_cap), "cudaMallocHost");
        d_stage_keys.ensure(12 * (size_t)max_nb);  // sized once: no allocation inside the engine loop
        d_stage_keys2.ensure(12 * (size_t)max_nb);
        pool->ensure_prompt_scratch(max_nb);
        d_keys.release();
        d_counts.release();
    }

    {  // size the per-admission scratch once for the largest prompt: nothing is (re)allocated
       // inside the engine loop (cudaMalloc / cudaFree synchronize the whole device, which would
       // deadlock shards sharing one GPU whose exchanges wait on each other on the device)
        long long mx = 1;
        for (int64_t i = 0; i < nt; ++i) mx = std::max<long long>(mx, (turns[i].v[5] + bs - 1) / bs);
        for (const auto& kv : catalog) mx = std::max<long long>(mx, kv.second.nb);
        pool->ensure_prompt_scratch(mx);
    }

    // load (engine.cpp:240-255)
    for (int64_t i = 0; i < nt; ++i) by_session[reqs[i].session].push_back(i);
    for (const auto& kv : by_session) pending_sessions.push_back(kv.first);
    arrival_us.assign(nt, 0.0);
    t_cached.assign(nt, 0);
    t_prompt.assign(nt, 0);
    t_start.assign(nt, 0.0);
    t_end.assign(nt, 0.0);
    t_done.assign(nt, 0);
    loaded = true;
    dev_setup();
}

void cs_engine::dev_setup() {
    const char* env = std::getenv("CS_DEVICE_SCHED");  // tools: overrides the config either way
    const char* env2 = std::getenv("CS_USE_PRESCAN");  // A/B switch (tools): prescans run, never consumed
    const bool want = env ? std::atoi(env) != 0 : cfg.device_scheduler != 0;
    // (the Belady baseline runs on the host scheduler: its admissions are a different kernel)
    if (!want || cfg.host_inputs || pool->comm || conc > csb::kMaxConc || pool->P.policy == 3) return;
    const int64_t nt = (int64_t)reqs.size();
    // sessions in ascending id order (the std::map order of the host scheduler)
    std::vector<int> soff(1, 0), sreqs;
    std::unordered_map<int, int> slot;
    for (const auto& kv : by_session) {
        slot[kv.first] = (int)soff.size() - 1;
        for (int64_t r : kv.second) sreqs.push_back((int)r);
        soff.push_back((int)sreqs.size());
    }
    std::vector<csb::EngReq> er(std::max<int64_t>(nt, 1));
    int max_nb = 1;
    for (int64_t i = 0; i < nt; ++i) {
        const Req& r = reqs[i];
        csb::EngReq& q = er[i];
        q.blk_off = r.blk_off;
        q.prompt_tokens = r.prompt_tokens;
        q.session = slot[r.session];
        q.agent = r.agent;
        q.nb = r.nb;
        q.anchor_blocks = r.anchor_blocks;
        q.decode = r.decode;
        q.pad = 0;
        max_nb = std::max(max_nb, r.nb);
    }
    std::vector<csb::EngCat> cat(pool->P.a_cap);
    for (auto& c : cat) c = csb::EngCat{0, 0, 0, 0};
    for (const auto& kv : catalog) {
        cat[kv.first] = csb::EngCat{kv.second.blk_off, kv.second.prompt_tokens, kv.second.nb, 0};
        max_nb = std::max(max_nb, kv.second.nb);
    }
    pool->ensure_prompt_scratch(max_nb);
    this->max_nb = max_nb;
    const int bps = std::max(1, pool->cfg.budget_per_step);
    w_cap = (2 * nt + 64) * bps;
    auto up = [&](csb::DevBuf& b, const void* src, size_t bytes) {
        b.ensure(std::max<size_t>(bytes, 8));
        if (bytes) ck(cudaMemcpy(b.p, src, bytes, cudaMemcpyHostToDevice), "H2D");
    };
    up(d_reqs, er.data(), sizeof(csb::EngReq) * er.size());
    up(d_soff, soff.data(), 4 * soff.size());
    up(d_sreqs, sreqs.data(), 4 * std::max<size_t>(sreqs.size(), 1));
    d_spos.ensure(4 * std::max<size_t>(soff.size(), 1));
    up(d_cat, cat.data(), sizeof(csb::EngCat) * cat.size());
    d_tc.ensure(8 * std::max<int64_t>(nt, 1));
    d_tp.ensure(8 * std::max<int64_t>(nt, 1));
    d_ts.ensure(8 * std::max<int64_t>(nt, 1));
    d_te.ensure(8 * std::max<int64_t>(nt, 1));
    d_td.ensure(std::max<int64_t>(nt, 1));
    d_ta.ensure(8 * std::max<int64_t>(nt, 1));
    ck(cudaMemset(d_td.p, 0, std::max<int64_t>(nt, 1)), "memset");
    d_ws.ensure(8 * w_cap);
    d_wt.ensure(8 * w_cap);
    d_wk.ensure(8 * w_cap);
    d_args.ensure(sizeof(csb::AdmitArgs));
    ck(cudaMemset(d_args.p, 0, sizeof(csb::AdmitArgs)), "memset");  // fields eng_issue never sets stay null
    d_cmd.ensure(8);
    d_state.ensure(sizeof(csb::EngState));
    std::memset(&hs, 0, sizeof(hs));
    hs.conc = conc;
    hs.budget = budget;
    hs.cost_base = cfg.prefill_base_us;
    hs.cost_tok = cfg.prefill_per_token_us;
    hs.cost_dec = cfg.decode_per_token_us;
    hs.prefetch = cfg.prefetch ? 1 : 0;
    hs.speculate = pool->speculate ? 1 : 0;
    hs.prescan = pool->prescan ? 1 : 0;
    hs.use_prescan = (env2 && std::atoi(env2) == 0) ? 0 : 1;
    hs.n_sessions = (int)soff.size() - 1;
    hs.last_dispatched = -1;
    hs.phase = 0;
    dev = true;
    pool->mirror_ok = false;  // arrivals and dispatches happen on the device from here on
}

void cs_engine::dev_run(long long stop_at, long long max_steps) {
    pool->flush_unpins();  // (host-queued unpins: none while the device schedules)
    hs.tick = tick;
    hs.seq = pool->seq;
    hs.pre_ok = pool->pre_ok ? 1 : 0;
    hs.poll_reset_pending = pool->poll_reset_pending ? 1 : 0;
    ck(cudaMemcpyAsync(d_state.p, &hs, sizeof(hs), cudaMemcpyHostToDevice, pool->stream), "H2D");
    csb::EngDev E{};
    E.st = d_state.as<csb::EngState>();
    E.reqs = d_reqs.as<csb::EngReq>();
    E.sess_off = d_soff.as<int>();
    E.sess_reqs = d_sreqs.as<int>();
    E.session_pos = d_spos.as<int>();
    E.cat = d_cat.as<csb::EngCat>();
    E.keys = d_keys.as<unsigned long long>();
    E.counts = d_counts.as<int>();
    E.pins = d_pins.as<unsigned int>();
    E.agent_ids = pool->P.agent_ids;
    E.t_cached = d_tc.as<long long>();
    E.t_prompt = d_tp.as<long long>();
    E.t_start = d_ts.as<double>();
    E.t_end = d_te.as<double>();
    E.t_done = d_td.as<unsigned char>();
    E.t_arrival = d_ta.as<double>();
    E.w_step = d_ws.as<long long>();
    E.w_target = d_wt.as<unsigned long long>();
    E.w_tick = d_wk.as<unsigned long long>();
    E.w_cap = w_cap;
    E.args = d_args.as<csb::AdmitArgs>();
    E.cmd = d_cmd.as<int>();
    csb::Ctrl c0;
    ck(cudaMemcpyAsync(&c0, pool->P.ctrl, sizeof(c0), cudaMemcpyDeviceToHost, pool->stream), "ctrl D2H");
    if (pool->timing) ck(cudaEventRecord(pool->ev0, pool->stream), "cudaEventRecord");
    ck(csb::launch_engine(pool->P, E, stop_at, max_steps, pool->n_agents, pool->lc, pool->stream), "engine_kernel");
    ++pool->launches;
    if (pool->timing) ck(cudaEventRecord(pool->ev1, pool->stream), "cudaEventRecord");
    ck(cudaMemcpyAsync(&hs, d_state.p, sizeof(hs), cudaMemcpyDeviceToHost, pool->stream), "D2H");
    csb::Ctrl c;
    ck(cudaMemcpyAsync(&c, pool->P.ctrl, sizeof(c), cudaMemcpyDeviceToHost, pool->stream), "ctrl D2H");
    pool->sync();
    if (pool->timing) {
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, pool->ev0, pool->ev1), "cudaEventElapsedTime");
        pool->admit_ms += ms;
        const long long sc = c.scans - c0.scans;
        if (sc > 0) {  // one persistent launch covers many scoring passes: timed per pass
            pool->scan_launch_ms += ms;
            pool->scan_launches += sc;
        }
        pool->admit_launches += hs.admissions - admissions;
    }
    tick = hs.tick;
    sim_now = hs.sim_now;
    admissions = hs.admissions;
    steps = hs.steps;
    completed = hs.completed;
    truncated = hs.truncated;
    warm_exec = hs.warm_exec;
    warm_drop = hs.warm_drop;
    tot_prompt = hs.tot_prompt;
    tot_cached = hs.tot_cached;
    pool->seq = hs.seq;
    pool->pre_ok = hs.pre_ok != 0;
    pool->poll_reset_pending = hs.poll_reset_pending != 0;
    pool->resident = c.resident;
    pool->pinned = c.pinned;
    pool->ev_total = c.n_ev;
    if (hs.error == 1) throw std::runtime_error("scheduler stalled with an idle engine");
    if (hs.error == 2) throw std::runtime_error("evict_one: all resident blocks are pinned");
    if (hs.error == 3) throw CsError(CS_ERR_CAPACITY, "device scheduler: warmup output capacity exceeded");
    if (hs.error) throw std::runtime_error("device scheduler error");
    drain_evictions(false);
}

void cs_engine::dev_pull_outputs() {
    const int64_t nt = (int64_t)reqs.size();
    if (nt > 0) {
        ck(cudaMemcpy(t_cached.data(), d_tc.p, 8 * nt, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(t_prompt.data(), d_tp.p, 8 * nt, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(t_start.data(), d_ts.p, 8 * nt, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(t_end.data(), d_te.p, 8 * nt, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(t_done.data(), d_td.p, nt, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(arrival_us.data(), d_ta.p, 8 * nt, cudaMemcpyDeviceToHost), "D2H");
    }
    const long long nw = hs.n_warm;
    w_step.resize(nw);
    w_target.resize(nw);
    w_tick.resize(nw);
    if (nw > 0) {
        ck(cudaMemcpy(w_step.data(), d_ws.p, 8 * nw, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(w_target.data(), d_wt.p, 8 * nw, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(w_tick.data(), d_wk.p, 8 * nw, cudaMemcpyDeviceToHost), "D2H");
    }
}

void cs_engine::drain_evictions(bool force) {
    // a forced drain follows a sync (every entry is in the log); inside the engine loop the last
    // admission's entries may still be being written (its status goes out before its apply)
    if (force) pool->sync();
    const unsigned long long tot = force ? pool->ev_total : pool->ev_safe;
    if (tot <= ev_drained) return;
    if (!force && tot - ev_drained < (unsigned long long)pool->P.evlog_cap / 2) return;
    const size_t base = evictions.size();
    evictions.resize(base + (tot - ev_drained));
    pool->copy_victims(ev_drained, tot, evictions.data() + base);
    ev_drained = tot;
}

void cs_engine::stage(csb::AdmitArgs& a, int64_t blk_off, int nb) {
    if (!cfg.host_inputs) {
        a.keys = d_keys.as<unsigned long long>() + blk_off;
        a.counts = d_counts.as<int>() + blk_off;
        return;
    }
    // the admission server may copy the next admission's blocks while this one is still being
    // applied (its look-ahead fetch): consecutive admissions alternate between two buffers
    const bool srv = pool->uses_server();
    csb::DevBuf& buf = (srv && (stage_flip = !stage_flip)) ? d_stage_keys2 : d_stage_keys;
    if (12 * (size_t)std::max(nb, 1) > buf.n) pool->server_stop();  // (never while it runs)
    buf.ensure(12 * (size_t)std::max(nb, 1));
    if (srv) {  // the admission server's CTA 0 reads them from pinned host memory
        unsigned char* dp = nullptr;
        ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), h_blob, 0), "cudaHostGetDevicePointer(prompts)");
        a.stage_src = dp + 12 * blk_off;
    } else {
        ck(cudaMemcpyAsync(buf.p, h_blob + 12 * blk_off, 12 * (size_t)nb, cudaMemcpyHostToDevice, pool->stream),
           "H2D");
    }
    h2d_bytes += 12 * (int64_t)nb;
    a.keys = buf.as<unsigned long long>();
    a.counts = reinterpret_cast<int*>(buf.as<unsigned char>() + 8 * (size_t)nb);
    // the victims (at most one per prompt block) come back behind the kernel, same stream
    pool->vpref = h_vict;
    pool->vpref_n = nb;
}

// host_inputs: the admission's result (victim keys) is read back immediately
void cs_engine::fetch_victims(unsigned long long before) {
    if (!cfg.host_inputs) {
        drain_evictions(false);
        return;
    }
    const unsigned long long tot = pool->ev_total;
    if (tot > ev_drained) {
        const size_t base = evictions.size();
        const unsigned long long n = tot - ev_drained;
        evictions.resize(base + n);
        if (ev_drained == before && n <= (unsigned long long)pool->vpref_done) {
            std::memcpy(evictions.data() + base, h_vict, 8 * n);
        } else {  // (not this admission's window alone: read the log, once it is all written)
            pool->sync();
            pool->copy_victims(ev_drained, tot, evictions.data() + base);
            d2h_bytes += 8 * (int64_t)n;
        }
        ev_drained = tot;
    }
    pool->vpref_done = 0;
    d2h_bytes += (int64_t)sizeof(csb::AdmitStatus);  // the mapped status record
}

void cs_engine::arrive(int64_t idx) {
    arrival_us[idx] = sim_now;
    ++tick;  // emit(RequestArrival): note_agent only (no decision depends on alphabet order)
    if (pool->P.policy == 1) pool->note_agent(reqs[idx].agent);  // for serialize_state's alphabet
    if ((unsigned long long)idx > bel_cursor) bel_cursor = (unsigned long long)idx;  // BeladyPolicy::observe
    pool->bel_cursor = bel_cursor;
    if (rec_events) ev_push(tick, csb::EventRec::kRequestArrival, (uint64_t)idx, pool->agent_ids[reqs[idx].agent]);
    ready.push_back(idx);
}

void cs_engine::activate_sessions() {
    while (active_sessions < conc && !pending_sessions.empty()) {
        const int sid = pending_sessions.front();
        pending_sessions.pop_front();
        ++active_sessions;
        session_pos[sid] = 0;
        arrive(by_session[sid][0]);
    }
}

bool cs_engine::try_start_head() {
    if (ready.empty() || in_flight.size() >= (size_t)conc) return false;
    const int64_t idx = ready.front();
    const Req& r = reqs[idx];
    const bool oversized = r.nb > budget;
    if (oversized && !in_flight.empty()) return false;  // oversized prompts run solo
    csb::AdmitArgs a{};
    stage(a, r.blk_off, r.nb);
    a.n = r.nb;
    a.flags = csb::kDispatch | csb::kAdmit | (oversized ? csb::kTruncate : (csb::kFeasible | csb::kLookup));
    a.prev = last_dispatched;
    a.next = r.agent;
    a.agent = (unsigned int)r.agent;
    a.anchor = r.anchor_blocks;
    a.tick_base = tick;
    a.pins_out = d_pins.as<unsigned int>() + r.blk_off;
    belady_args(a, r.blk_off);
    ev_prepare(a, r.nb);
    const unsigned long long ev_before = pool->ev_total;
    const csb::AdmitStatus& st = pool->admit(a, r.nb);
    bel_cursor_dev = bel_cursor;
    if (rec_events && st.started) {
        ev_push(tick + 1, csb::EventRec::kAgentDispatch, last_dispatched >= 0 ? pool->agent_ids[last_dispatched] : 0,
                pool->agent_ids[r.agent], last_dispatched >= 0, true);
        if (!oversized) ev_touches(a, st.first_miss, tick + 1);
    }
    d2h_bytes += 8 * (int64_t)pool->vpref_done;  // the victim window copied behind the kernel
    ++admissions;
    if (cfg.host_inputs) d2h_bytes += (int64_t)sizeof(csb::AdmitStatus);
    if (!st.started) return false;  // wait for in-flight pins to clear
    ready.pop_front();
    pool->note_dispatch(last_dispatched, r.agent);
    last_dispatched = r.agent;
    tick = st.tick_after;
    if (oversized) ++truncated;
    Flight f;
    f.seq = flight_seq++;
    f.req = idx;
    f.npins = st.admit_n;
    f.cached = oversized ? 0 : st.cached;
    f.start_us = sim_now;
    // engine.cpp:302-305: ttft = base + per_token * uncached; end = now + ttft + decode * tokens
    const double ttft = cfg.prefill_base_us + cfg.prefill_per_token_us * (double)(r.prompt_tokens - f.cached);
    f.end_us = sim_now + ttft + cfg.decode_per_token_us * r.decode;
    in_flight.push_back(f);
    std::push_heap(in_flight.begin(), in_flight.end(), later);
    fetch_victims(ev_before);
    return true;
}

void cs_engine::complete_earliest() {
    std::pop_heap(in_flight.begin(), in_flight.end(), later);
    Flight f = in_flight.back();
    in_flight.pop_back();
    sim_now = f.end_us;
    ++tick;  // emit(TurnComplete)
    if (rec_events) ev_push(tick, csb::EventRec::kTurnComplete, (uint64_t)f.req, 0);
    const Req& r = reqs[f.req];
    pool->defer_unpin(d_pins.as<unsigned int>() + r.blk_off, f.npins);  // runs inside the next admission launch
    const int sid = r.session;
    auto& list = by_session[sid];
    if (++session_pos[sid] < list.size()) {
        arrive(list[session_pos[sid]]);
    } else {
        --active_sessions;
    }
    t_cached[f.req] = f.cached;
    t_prompt[f.req] = r.prompt_tokens;
    t_start[f.req] = f.start_us;
    t_end[f.req] = f.end_us;
    t_done[f.req] = 1;
    tot_prompt += r.prompt_tokens;
    tot_cached += f.cached;
    ++completed;
}

void cs_engine::execute_warmup(int target) {
    auto it = catalog.find(target);
    if (it == catalog.end()) {
        ++warm_drop;
        return;
    }
    const Cat& c = it->second;
    csb::AdmitArgs a{};
    stage(a, c.blk_off, c.nb);
    a.n = c.nb;
    a.flags = csb::kLookup | csb::kAdmit | csb::kWarmupRoom | csb::kUnpinAfter;
    a.prev = -1;
    a.next = -1;
    a.agent = (unsigned int)c.agent;
    a.anchor = -1;
    a.tick_base = tick;
    a.pins_out = d_pins.as<unsigned int>() + c.blk_off;
    ev_prepare(a, c.nb);
    const unsigned long long ev_before = pool->ev_total;
    const csb::AdmitStatus& st = pool->admit(a, c.nb);
    d2h_bytes += 8 * (int64_t)pool->vpref_done;
    ++admissions;
    ev_touches(a, st.first_miss, tick);
    tick = st.tick_after;
    ++warm_exec;
    warm_prompt += c.prompt_tokens;
    // engine.cpp:223-227
    warm_uncached += c.prompt_tokens - st.cached;
    warm_time_us += cfg.prefill_base_us + cfg.prefill_per_token_us * (double)(c.prompt_tokens - st.cached) +
                    cfg.decode_per_token_us * 1;
    fetch_victims(ev_before);
}

void cs_engine::drain_and_run_warmups() {
    // Runtime::drain_side_effects -> poll_actions (cachesage_policy.cpp:125-130)
    std::vector<int> fx = pool->pending_targets;
    for (size_t k = 0; k < fx.size(); ++k) {
        w_step.push_back(steps);
        w_target.push_back(pool->agent_ids[fx[k]]);
        w_tick.push_back(pool->pending_ticks[k]);
    }
    pool->pending_targets.clear();
    pool->pending_ticks.clear();
    pool->poll_reset_pending = true;
    if (!cfg.prefetch) return;
    for (int t : fx) execute_warmup(t);
}

void cs_engine::step() {
    if (done()) return;
    activate_sessions();
    bool progressed = false;
    while (try_start_head()) progressed = true;
    if (!progressed) {
        if (!in_flight.empty()) {
            complete_earliest();
        } else if (!ready.empty()) {
            throw std::runtime_error("scheduler stalled with an idle engine");
        }
    }
    drain_and_run_warmups();
    ++steps;
}

// ---------------------------------------------------------------------- C ABI (engine level)

extern "C" {

int64_t cs_generate_trace(const cs_workload_spec* ws, int64_t* turns7, int64_t cap) {
    try {
        const std::vector<Turn> t = generate(to_spec(ws));
        for (int64_t i = 0; i < (int64_t)t.size() && i < cap && turns7; ++i)
            std::memcpy(turns7 + 7 * i, t[i].v, sizeof(t[i].v));
        return (int64_t)t.size();
    } catch (const std::exception& e) {
        cs_set_error(e.what());
        return CS_ERR_INVALID_ARGUMENT;
    }
}

void cs_engine_cfg_default(cs_engine_cfg* c) {
    cs_pool_cfg_default(&c->pool);
    c->pool.budget_blocks = 0;
    c->concurrency = 0;
    c->block_size = 16;
    c->prefetch = 1;
    c->skip = 4;
    c->take = 4;
    c->timing = 0;
    c->host_inputs = 0;
    c->device_scheduler = 0;
    c->prefill_per_token_us = 50.0;  // CostModel defaults (engine.hpp:22-26)
    c->prefill_base_us = 1000.0;
    c->decode_per_token_us = 20000.0;
}

int cs_engine_create(const cs_engine_cfg* cfg, const cs_workload_spec* spec, cs_engine_t* out) {
    return eguard([&] {
        if (!cfg || !spec || !out) throw std::invalid_argument("cs_engine_create: null argument");
        auto* e = new cs_engine();
        try {
            e->build(*cfg, spec);
        } catch (...) {
            if (e->pool) {
                e->pool->destroy();
                delete e->pool;
            }
            delete e;
            throw;
        }
        *out = e;
    });
}

int cs_engine_create_from_turns(const cs_engine_cfg* cfg, const cs_workload_spec* spec, const int64_t* turns7,
                                int64_t n_turns, cs_engine_t* out) {
    return eguard([&] {
        if (!cfg || !spec || !out || n_turns < 0 || (n_turns > 0 && !turns7))
            throw std::invalid_argument("cs_engine_create_from_turns: null argument");
        auto* e = new cs_engine();
        try {
            e->build(*cfg, spec, 0, nullptr, turns7, n_turns);
        } catch (...) {
            if (e->pool) {
                e->pool->destroy();
                delete e->pool;
            }
            delete e;
            throw;
        }
        *out = e;
    });
}

int cs_engine_turn_arrivals(cs_engine_t e, double* arrival_us, int64_t cap) {
    return eguard([&] {
        if (!e) throw std::invalid_argument("cs_engine_turn_arrivals: null engine");
        if (e->dev) e->dev_pull_outputs();
        const int64_t n = std::min<int64_t>(cap, (int64_t)e->reqs.size());
        for (int64_t i = 0; i < n && arrival_us; ++i) arrival_us[i] = e->arrival_us[i];
    });
}

int cs_engine_create_sharded(const cs_engine_cfg* cfg, const cs_workload_spec* spec, int64_t shard_slots,
                             cs_comm_t comm, cs_engine_t* out) {
    return eguard([&] {
        if (!cfg || !spec || !out || !comm) throw std::invalid_argument("cs_engine_create_sharded: null argument");
        auto* e = new cs_engine();
        try {
            e->build(*cfg, spec, shard_slots, comm);
        } catch (...) {
            if (e->pool) {
                e->pool->destroy();
                delete e->pool;
            }
            delete e;
            throw;
        }
        *out = e;
    });
}

int cs_engine_destroy(cs_engine_t e) {
    return eguard([&] {
        if (!e) return;
        e->d_keys.release();
        e->d_counts.release();
        e->d_pins.release();
        e->d_stage_keys.release();
        e->d_stage_keys2.release();
        e->d_stage_counts.release();
        if (e->h_keys) cudaFreeHost(e->h_keys);
        if (e->h_blob) cudaFreeHost(e->h_blob);
        if (e->h_vict) cudaFreeHost(e->h_vict);
        if (e->h_counts) cudaFreeHost(e->h_counts);
        if (e->pool) {
            e->pool->destroy();
            delete e->pool;
        }
        delete e;
    });
}

namespace {
// Engine loops leave no admission server running behind them (csb::server_kernel): the next
// pool or engine call may need the stream.
struct ServerScope {
    cs_pool* pool;
    ~ServerScope() {
        try {
            pool->server_stop();
        } catch (...) {  // (the loop's own error, if any, is the one reported)
        }
    }
};
}  // namespace

int cs_engine_step(cs_engine_t e, int* done) {
    return eguard([&] {
        if (!e) throw std::invalid_argument("cs_engine_step: null engine");
        ServerScope scope{e->pool};
        if (e->dev) {
            if (!e->done()) e->dev_run(LLONG_MAX, 1);
        } else {
            e->step();
        }
        if (done) *done = e->done() ? 1 : 0;
    });
}

int cs_engine_run(cs_engine_t e) {
    return eguard([&] {
        if (!e) throw std::invalid_argument("cs_engine_run: null engine");
        ServerScope scope{e->pool};
        if (e->dev) {
            while (!e->done()) e->dev_run(e->admissions + e->dev_chunk(), LLONG_MAX);
        } else {
            while (!e->done()) e->step();
        }
        e->pool->flush_unpins();
        e->drain_evictions(true);
    });
}

int cs_engine_run_for(cs_engine_t e, int64_t max_adm, int* done) {
    return eguard([&] {
        if (!e) throw std::invalid_argument("cs_engine_run_for: null engine");
        ServerScope scope{e->pool};
        const int64_t stop = e->admissions + max_adm;
        if (e->dev) {
            while (!e->done() && e->admissions < stop) e->dev_run(std::min<int64_t>(stop, e->admissions + e->dev_chunk()), LLONG_MAX);
        } else {
            while (!e->done() && e->admissions < stop) e->step();
        }
        if (done) *done = e->done() ? 1 : 0;
    });
}

int cs_engine_result_get(cs_engine_t e, cs_engine_result* o) {
    return eguard([&] {
        if (!e || !o) throw std::invalid_argument("cs_engine_result_get: null argument");
        e->drain_evictions(true);
        std::memset(o, 0, sizeof(*o));
        o->turns = (int64_t)e->reqs.size();
        o->completed = e->completed;
        o->total_prompt_tokens = e->tot_prompt;
        o->total_cached_tokens = e->tot_cached;
        o->hit_rate = e->tot_prompt > 0 ? (double)e->tot_cached / (double)e->tot_prompt : 0.0;
        o->evictions = (int64_t)e->evictions.size();
        o->truncated = e->truncated;
        o->warmups_executed = e->warm_exec;
        o->warmups_dropped = e->warm_drop;
        o->warmups_issued = e->dev ? (int64_t)e->hs.n_warm : (int64_t)e->w_target.size();
        o->sim_us = e->sim_now;
        o->steps = e->steps;
        o->admissions = e->admissions;
        cs_pool_stats ps;
        if (cs_pool_get_stats(e->pool, &ps) != CS_OK) throw std::runtime_error(cs_last_error());
        o->scans = ps.scans;
        o->scanned_slots = ps.scanned_slots;
        o->tick = e->tick;
        o->scan_ms = e->pool->scan_launch_ms;
        o->admit_ms = e->pool->admit_ms;
        o->scan_launches = e->pool->scan_launches;
        o->h2d_bytes = e->h2d_bytes;
        o->d2h_bytes = e->d2h_bytes;
        o->gpu_launches = e->pool->launches;
        o->warmup_prompt_tokens = e->dev ? e->hs.warm_prompt : e->warm_prompt;
    });
}

int cs_engine_run_timed(cs_engine_t e, int64_t max_adm, double* device_ms, int* done) {
    return eguard([&] {
        if (!e) throw std::invalid_argument("cs_engine_run_timed: null engine");
        cudaEvent_t a, b;
        ck(cudaEventCreate(&a), "cudaEventCreate");
        ck(cudaEventCreate(&b), "cudaEventCreate");
        e->pool->sync();
        ck(cudaEventRecord(a, e->pool->stream), "cudaEventRecord");
        const int64_t stop = e->admissions + max_adm;
        {
            ServerScope scope{e->pool};
            if (e->dev) {
                while (!e->done() && e->admissions < stop)
                    e->dev_run(std::min<int64_t>(stop, e->admissions + e->dev_chunk()), LLONG_MAX);
            } else {
                while (!e->done() && e->admissions < stop) e->step();
            }
            e->pool->server_stop();  // (inside the timed region: the server's exit is part of it)
        }
        ck(cudaEventRecord(b, e->pool->stream), "cudaEventRecord");
        ck(cudaEventSynchronize(b), "cudaEventSynchronize");
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (device_ms) *device_ms = ms;
        if (done) *done = e->done() ? 1 : 0;
    });
}

int cs_engine_restore(cs_engine_t e, const uint64_t* keys, const uint64_t* lt, const uint32_t* agents,
                      const uint32_t* refs, int64_t n) {
    return eguard([&] {
        if (!e) throw std::invalid_argument("cs_engine_restore: null engine");
        if (e->admissions > 0) throw std::logic_error("cs_engine_restore: restore before the first step");
        uint64_t mx = 0;
        for (int64_t i = 0; i < n; ++i) {
            mx = std::max<uint64_t>(mx, lt[i]);
            if (agents && agents[i] != CS_NO_AGENT && (int)agents[i] >= e->pool->n_agents)
                throw std::invalid_argument("cs_engine_restore: agent index out of range");
        }
        const int rc = cs_restore(e->pool, keys, lt, agents, refs, n);
        if (rc != CS_OK) throw CsError(rc, cs_last_error());
        if (e->pool->comm) {  // sharded: the engine clock and the residency are global
            long long res = 0;
            csb::Ctrl c;
            ck(cudaMemcpy(&c, e->pool->P.ctrl, sizeof(c), cudaMemcpyDeviceToHost), "ctrl D2H");
            for (unsigned long long v : e->pool->allgather_u64((unsigned long long)c.resident)) res += (long long)v;
            if (res > e->pool->P.gbudget) throw std::invalid_argument("cs_restore: snapshot exceeds the budget");
            for (unsigned long long v : e->pool->allgather_u64(mx)) mx = std::max<uint64_t>(mx, v);
            e->pool->resident = res;
        }
        e->tick = std::max<uint64_t>(e->tick, mx);
    });
}

int cs_engine_agents(cs_engine_t e, uint64_t* ids, int cap) {
    if (!e) return CS_ERR_INVALID_ARGUMENT;
    const int n = (int)e->pool->agent_ids.size();
    for (int i = 0; i < n && i < cap && ids; ++i) ids[i] = e->pool->agent_ids[i];
    return n;
}

int cs_engine_turns(cs_engine_t e, int64_t* cached, int64_t* prompt, double* start_us, double* end_us, int64_t cap) {
    return eguard([&] {
        if (!e) throw std::invalid_argument("cs_engine_turns: null engine");
        if (e->dev) e->dev_pull_outputs();
        const int64_t n = std::min<int64_t>(cap, (int64_t)e->reqs.size());
        for (int64_t i = 0; i < n; ++i) {
            if (cached) cached[i] = e->t_cached[i];
            if (prompt) prompt[i] = e->t_prompt[i];
            if (start_us) start_us[i] = e->t_start[i];
            if (end_us) end_us[i] = e->t_end[i];
        }
    });
}

int cs_engine_record_events(cs_engine_t e, int on) {
    return eguard([&] {
        if (!e) throw std::invalid_argument("cs_engine_record_events: null engine");
        if (on && (e->dev || e->pool->comm))
            throw std::invalid_argument("events: recorded by the host scheduler on one pool (no device scheduler, no shards)");
        if (on && (e->admissions > 0 || e->steps > 0)) throw std::logic_error("events: enable before the first step");
        e->rec_events = on != 0;
    });
}

int cs_engine_write_outputs(cs_engine_t e, const char* dir, const char* workload, const char* policy, uint64_t seed,
                            const char* const* labels, int n_labels, int write_events) {
    return eguard([&] {
        if (!e || !dir || !workload || !policy) throw std::invalid_argument("cs_engine_write_outputs: null argument");
        if (e->dev) e->dev_pull_outputs();
        if (!e->done()) throw std::logic_error("cs_engine_write_outputs: the run is not finished");
        if (write_events && !e->rec_events) throw std::logic_error("events were not recorded (cs_engine_record_events)");
        e->drain_evictions(true);
        csb::CellOut c;
        c.workload = workload;
        c.policy = policy;
        c.seed = seed;
        for (int i = 0; i < n_labels; ++i) c.labels.emplace_back(labels && labels[i] ? labels[i] : "");
        c.budget_blocks = e->budget;
        c.block_size = e->bs;
        c.concurrency = e->conc;
        c.prefetch = e->cfg.prefetch != 0;
        c.prefill_per_token_us = e->cfg.prefill_per_token_us;
        c.prefill_base_us = e->cfg.prefill_base_us;
        c.decode_per_token_us = e->cfg.decode_per_token_us;
        const cs_pool_cfg& pc = e->cfg.pool;
        c.skip = e->cfg.skip;
        c.take = e->cfg.take;
        c.tau = pc.tau;
        c.e_max = pc.e_max;
        c.w_pred = pc.w_pred;
        c.window = (uint64_t)pc.window;
        c.min_confidence = pc.min_confidence;
        c.min_row_count = (uint64_t)pc.min_row_count;
        c.budget_per_step = pc.budget_per_step;
        c.ttl_pin_horizon_us = 5000000.0;  // TtlConfig default (baselines.hpp:25)
        const int64_t nt = (int64_t)e->reqs.size();
        c.turns.reserve(nt);
        for (int64_t i = 0; i < nt; ++i) {
            if (!e->t_done[i]) continue;
            const auto& r = e->reqs[i];
            csb::TurnRec t{};
            t.turn_id = (uint64_t)i;
            t.session = r.session;
            t.turn_index = r.turn_index;
            t.agent = e->pool->agent_ids[r.agent];
            t.label = r.spec_agent;
            t.prompt_tokens = (long)e->t_prompt[i];
            t.cached_tokens = (long)e->t_cached[i];
            t.ttft_us = e->cfg.prefill_base_us +
                        e->cfg.prefill_per_token_us * (double)(r.prompt_tokens - e->t_cached[i]);  // engine.cpp:302-304
            t.arrival_us = e->arrival_us[i];
            t.start_us = e->t_start[i];
            t.end_us = e->t_end[i];
            t.latency_us = t.end_us - t.arrival_us;
            c.turns.push_back(t);
        }
        c.sim_duration_us = e->sim_now;
        c.evictions = e->evictions.size();
        c.truncated = (uint64_t)e->truncated;
        c.warmups_executed = (uint64_t)e->warm_exec;
        c.warmups_dropped = (uint64_t)e->warm_drop;
        c.warmup_prompt_tokens = (long)e->warm_prompt;
        c.warmup_uncached_tokens = (long)e->warm_uncached;
        c.warmup_time_us = e->warm_time_us;
        c.events = write_events ? &e->events : nullptr;
        csb::write_cell(c, dir);
    });
}

int64_t cs_engine_evictions(cs_engine_t e, uint64_t* keys, int64_t cap) {
    if (!e) return CS_ERR_INVALID_ARGUMENT;
    try {
        e->drain_evictions(true);
    } catch (const std::exception& ex) {
        cs_set_error(ex.what());
        return CS_ERR_CUDA;
    }
    const int64_t n = (int64_t)e->evictions.size();
    if (keys) std::memcpy(keys, e->evictions.data(), 8 * std::min(n, cap));
    return n;
}

int64_t cs_engine_warmups(cs_engine_t e, int64_t* step, uint64_t* target, uint64_t* tick, int64_t cap) {
    if (!e) return CS_ERR_INVALID_ARGUMENT;
    if (e->dev) {
        try {
            e->dev_pull_outputs();
        } catch (const std::exception& ex) {
            cs_set_error(ex.what());
            return CS_ERR_CUDA;
        }
    }
    const int64_t n = (int64_t)e->w_target.size();
    for (int64_t i = 0; i < n && i < cap; ++i) {
        if (step) step[i] = e->w_step[i];
        if (target) target[i] = e->w_target[i];
        if (tick) tick[i] = e->w_tick[i];
    }
    return n;
}

cs_pool_t cs_engine_pool(cs_engine_t e) { return e ? e->pool : nullptr; }

}  // extern "C"
