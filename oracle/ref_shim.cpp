// TEST INFRASTRUCTURE ONLY — never linked into, loaded by, or called from the product path.
//
// extern "C" shim over the UNMODIFIED reference sources (compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libcachesage_ref.so).
// It lets the Python tests and bench.py's reference arm drive the reference's own
// EngineSim + CacheSagePolicy through plain C types:
//   - ref_chain_hash / ref_block_keys / ref_identity   -> hashing.cpp:26-51, cachesage_policy.cpp:9-31
//   - ref_preset_spec / ref_generate                   -> presets.cpp:37-130, workload.cpp:156-182
//   - ref_run                                          -> the run_cell wiring of experiment.cpp:355-379,
//                                                         with a recording Policy decorator around the
//                                                         policy so drained warmups are logged per step
//   - ref_policy_trace                                 -> CacheSagePolicy::observe/score/poll_actions
//   - ref_evict_bench                                  -> EngineSim::admit / evict_one timing at pool N
// Nothing here re-implements reference logic; it only marshals arguments.

#include <algorithm>
#include <chrono>
#include <sstream>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "cachesage/baselines.hpp"
#include "cachesage/cachesage_policy.hpp"
#include "cachesage/engine.hpp"
#include "cachesage/experiment.hpp"
#include "cachesage/hashing.hpp"
#include "cachesage/reachability.hpp"
#include "cachesage/runtime.hpp"
#include "cachesage/survival_oracle.hpp"
#include "cachesage/workload.hpp"
#include "ref_shim.h"

using namespace cachesage;

namespace {

thread_local std::string g_err;
thread_local std::string g_state;  // the last ref_run's final Policy::serialize_state().dump()

struct RecordingPolicy : Policy {
    std::shared_ptr<Policy> inner;
    long step = 0;
    std::vector<long> w_step;
    std::vector<std::uint64_t> w_target;
    std::vector<std::uint64_t> w_tick;

    const char* name() const override { return inner->name(); }
    void observe(const Event& e) override { inner->observe(e); }
    double score(const Block& b, const ScoreContext& c) const override { return inner->score(b, c); }
    Forecast predict(int h) const override { return inner->predict(h); }
    std::vector<SideEffect> poll_actions() override {
        std::vector<SideEffect> out = inner->poll_actions();
        for (const SideEffect& s : out) {
            w_step.push_back(step);
            w_target.push_back(s.target.value);
            w_tick.push_back(s.issued_tick);
        }
        ++step;
        return out;
    }
    json serialize_state() const override { return inner->serialize_state(); }
};

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

}  // namespace

extern "C" {



const char* ref_last_error(void) { return g_err.c_str(); }
const char* ref_last_state(void) { return g_state.c_str(); }

unsigned long long ref_chain_hash(int has_parent, unsigned long long parent, const std::uint32_t* tokens,
                                  size_t n) {
    try {
        std::optional<std::uint64_t> p;
        if (has_parent) p = parent;
        return chain_hash(p, std::span<const TokenId>(tokens, n)).value;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 0;
    }
}

long ref_block_keys(const std::uint32_t* tokens, size_t n, int block_size, unsigned long long* keys,
                    int* counts) {
    try {
        auto b = block_keys_for(std::span<const TokenId>(tokens, n), block_size);
        for (size_t i = 0; i < b.size(); ++i) {
            keys[i] = b[i].key.value;
            counts[i] = b[i].token_count;
        }
        return static_cast<long>(b.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_identity(const unsigned long long* keys, size_t n, int skip, int take, unsigned long long* out) {
    try {
        std::vector<BlockKey> k(n);
        for (size_t i = 0; i < n; ++i) k[i].value = keys[i];
        *out = derive_agent_identity(k, IdentityConfig{skip, take}).value;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

static WorkloadSpec to_spec(const ref_spec* s) {
    WorkloadSpec spec;
    spec.name = "custom";
    for (int i = 0; i < s->n_agents; ++i) {
        spec.agents.push_back({"agent-" + std::to_string(i), s->anchor_tokens[i]});
    }
    spec.transition.assign(s->n_agents, std::vector<double>(s->n_agents, 0.0));
    for (int i = 0; i < s->n_agents; ++i)
        for (int j = 0; j < s->n_agents; ++j) spec.transition[i][j] = s->transition[i * s->n_agents + j];
    if (s->supervisor >= 0) spec.supervisor = s->supervisor;
    spec.turns_min = s->turns_min;
    spec.turns_max = s->turns_max;
    spec.sessions = s->sessions;
    spec.task_tokens = s->task_tokens;
    spec.history_growth = s->history_growth;
    spec.decode_tokens = s->decode_tokens;
    spec.template_tokens = s->template_tokens;
    spec.concurrency = s->concurrency;
    spec.budget_blocks = s->budget_blocks;
    spec.seed = s->seed;
    return spec;
}

// Fills `out` from a named preset. Arrays point at storage owned by the shim (valid until the
// next call on this thread).
int ref_preset_spec(const char* name, ref_spec* out) {
    static thread_local std::vector<int> anchors;
    static thread_local std::vector<double> trans;
    try {
        WorkloadSpec spec = preset_by_name(name);
        const int n = static_cast<int>(spec.agents.size());
        anchors.assign(n, 0);
        trans.assign(n * n, 0.0);
        for (int i = 0; i < n; ++i) {
            anchors[i] = spec.agents[i].anchor_tokens;
            for (int j = 0; j < n; ++j) trans[i * n + j] = spec.transition[i][j];
        }
        out->n_agents = n;
        out->anchor_tokens = anchors.data();
        out->transition = trans.data();
        out->supervisor = spec.supervisor ? *spec.supervisor : -1;
        out->turns_min = spec.turns_min;
        out->turns_max = spec.turns_max;
        out->sessions = spec.sessions;
        out->task_tokens = spec.task_tokens;
        out->history_growth = spec.history_growth;
        out->decode_tokens = spec.decode_tokens;
        out->template_tokens = spec.template_tokens;
        out->concurrency = spec.concurrency;
        out->budget_blocks = spec.budget_blocks;
        out->seed = spec.seed;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Generates the trace; writes up to `cap` turns as (session, turn_index, agent, anchor, history,
// prompt, decode) int64 7-tuples. Returns the turn count or -1.
long ref_generate(const ref_spec* s, long long* turns7, long cap) {
    try {
        const Trace trace = generate_trace(to_spec(s));
        const long n = static_cast<long>(trace.turns.size());
        for (long i = 0; i < n && i < cap; ++i) {
            const Turn& t = trace.turns[i];
            long long* o = turns7 + 7 * i;
            o[0] = t.session_id;
            o[1] = t.turn_index;
            o[2] = t.agent;
            o[3] = t.anchor_tokens;
            o[4] = t.history_tokens;
            o[5] = t.prompt_tokens;
            o[6] = t.decode_tokens;
        }
        return n;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Prompt tokens of turn `idx` of the generated trace (Trace::turn_tokens, workload.cpp:125-140).
long ref_turn_tokens(const ref_spec* s, long idx, std::uint32_t* out, long cap) {
    try {
        const Trace trace = generate_trace(to_spec(s));
        const auto tok = trace.turn_tokens(trace.turns.at(idx));
        for (long i = 0; i < static_cast<long>(tok.size()) && i < cap; ++i) out[i] = tok[i];
        return static_cast<long>(tok.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

static CacheSageConfig to_cs_cfg(const ref_run_cfg* c) {
    CacheSageConfig cs;
    cs.identity = IdentityConfig{c->skip, c->take};
    cs.tau = c->tau;
    cs.e_max = c->e_max;
    cs.w_pred = c->w_pred;
    cs.window = static_cast<std::size_t>(c->window);
    cs.gate.min_confidence = c->min_confidence;
    cs.gate.min_row_count = c->min_row_count;
    cs.gate.budget_per_step = c->budget_per_step;
    return cs;
}

}  // extern "C"

WorkloadSpec ref_to_spec(const ref_spec* s) { return to_spec(s); }

// ref_run with the scoring policy supplied by `make` (nullptr: the reference's own, by
// c->policy): the unmodified EngineSim / Runtime drive whatever Policy it returns. Used by
// adapter_check.cpp to run the reference engine over the B200 drop-in policy.
int ref_run_with(const ref_spec* s, const ref_run_cfg* c, ref_run_out* out,
                 std::shared_ptr<Policy> (*make)(const CacheSageConfig&, void*), void* ctx) {
    try {
        const Trace trace = generate_trace(to_spec(s));
        EngineConfig ec;
        ec.budget_blocks = c->budget_blocks > 0 ? c->budget_blocks : trace.spec.budget_blocks;
        ec.concurrency = c->concurrency > 0 ? c->concurrency : trace.spec.concurrency;
        ec.block_size = c->block_size;
        ec.identity = IdentityConfig{c->skip, c->take};
        ec.prefetch_enabled = c->prefetch != 0;
        if (c->prefill_base_us != 0.0) ec.cost.prefill_base_us = c->prefill_base_us;
        if (c->prefill_per_token_us != 0.0) ec.cost.prefill_per_token_us = c->prefill_per_token_us;
        if (c->decode_per_token_us != 0.0) ec.cost.decode_per_token_us = c->decode_per_token_us;
        const auto requests = materialize_requests(trace, ec.block_size, ec.identity);
        auto rec = std::make_shared<RecordingPolicy>();
        if (make) {
            rec->inner = make(to_cs_cfg(c), ctx);
        } else if (c->policy == 0) {
            rec->inner = std::make_shared<LruPolicy>();
        } else if (c->policy == 2) {
            rec->inner = std::make_shared<TtlPolicy>();
        } else if (c->policy == 3) {
            rec->inner = std::make_shared<BeladyPolicy>(requests);
        } else {
            rec->inner = std::make_shared<CacheSagePolicy>(to_cs_cfg(c));
        }
        Runtime runtime;
        runtime.register_policy(rec);
        EngineSim engine(ec, runtime);
        engine.set_warmup_catalog(build_warmup_catalog(trace, ec.block_size, ec.identity));
        engine.load(requests);
        long steps = 0;
        while (!engine.done()) {
            engine.step();
            ++steps;
        }
        RunResult r = engine.finalize();
        g_state = rec->inner->serialize_state().dump();
        std::vector<long> cached, prompt;
        std::vector<double> st, en;
        for (const TurnMetrics& t : r.turns) {
            cached.push_back(t.cached_tokens);
            prompt.push_back(t.prompt_tokens);
            st.push_back(t.start_us);
            en.push_back(t.end_us);
        }
        std::vector<unsigned long long> ev;
        for (BlockKey k : r.evictions) ev.push_back(k.value);
        out->n_turns = static_cast<long>(r.turns.size());
        out->cached_tokens = dup(cached);
        out->prompt_tokens = dup(prompt);
        out->start_us = dup(st);
        out->end_us = dup(en);
        out->n_evictions = static_cast<long>(ev.size());
        out->evictions = dup(ev);
        out->n_warmups = static_cast<long>(rec->w_step.size());
        out->warmup_step = dup(rec->w_step);
        std::vector<unsigned long long> wt(rec->w_target.begin(), rec->w_target.end());
        std::vector<unsigned long long> wk(rec->w_tick.begin(), rec->w_tick.end());
        out->warmup_target = dup(wt);
        out->warmup_tick = dup(wk);
        out->hit_rate = r.aggregate.hit_rate;
        out->truncated = static_cast<long>(r.aggregate.truncated_admissions);
        out->warmups_executed = static_cast<long>(r.aggregate.warmups_executed);
        out->warmups_dropped = static_cast<long>(r.aggregate.warmups_dropped);
        out->sim_us = r.aggregate.sim_duration_us;
        out->n_steps = steps;
        out->events = static_cast<long>(r.events.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

extern "C" {

int ref_run(const ref_spec* s, const ref_run_cfg* c, ref_run_out* out) { return ref_run_with(s, c, out, nullptr, nullptr); }

void ref_free_run(ref_run_out* o) {
    std::free(o->cached_tokens);
    std::free(o->prompt_tokens);
    std::free(o->start_us);
    std::free(o->end_us);
    std::free(o->evictions);
    std::free(o->warmup_step);
    std::free(o->warmup_target);
    std::free(o->warmup_tick);
    std::memset(o, 0, sizeof(*o));
}

// Drives a CacheSagePolicy with a dispatch stream and reports what the per-step hot path reads.
// events: n triples (has_prev, prev, next) of AgentDispatch; a drain (poll_actions) happens
// after every event whose index is in drain_mask (nonzero). Per event i: rebuilt[i] (0/1),
// warm_target[i] (0 when no warmup issued at that event). At the end: hops[] and survival[] for
// `query` agents, row_total[] for `query` agents, plus scores for the given blocks.
int ref_policy_trace(const ref_run_cfg* c, long n, const int* has_prev, const unsigned long long* prev,
                     const unsigned long long* next, const unsigned char* drain_mask, int* rebuilt,
                     unsigned long long* warm_target, long nq, const unsigned long long* query,
                     int* hops, double* survival, unsigned long long* row_total, long nb,
                     const unsigned long long* b_key, const int* b_has_agent,
                     const unsigned long long* b_agent, const unsigned long long* b_touch,
                     unsigned long long now_tick, unsigned long long oldest, double* scores,
                     unsigned long long* state_bytes) {
    try {
        CacheSagePolicy pol(to_cs_cfg(c));
        Tick tick = 0;
        for (long i = 0; i < n; ++i) {
            const std::uint64_t before = pol.rebuild_count();
            std::optional<AgentId> p;
            if (has_prev[i]) p = AgentId{prev[i]};
            pol.observe(Event{++tick, AgentDispatch{p, AgentId{next[i]}}});
            rebuilt[i] = pol.rebuild_count() != before ? 1 : 0;
            warm_target[i] = 0;
            if (drain_mask[i]) {
                auto fx = pol.poll_actions();
                if (!fx.empty()) warm_target[i] = fx.back().target.value;
            }
        }
        for (long q = 0; q < nq; ++q) {
            hops[q] = pol.reachability().empty() ? -1 : pol.reachability().hop(AgentId{query[q]});
            survival[q] = pol.reachability().empty() ? 0.0 : pol.reachability().survival(AgentId{query[q]});
            row_total[q] = pol.learner().row_total(AgentId{query[q]});
        }
        const ScoreContext ctx{now_tick, oldest, 0.0};
        for (long b = 0; b < nb; ++b) {
            Block blk;
            blk.key = BlockKey{b_key[b]};
            if (b_has_agent[b]) blk.agent = AgentId{b_agent[b]};
            blk.last_touch = b_touch[b];
            scores[b] = pol.score(blk, ctx);
        }
        *state_bytes = pol.state_bytes();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Drives the reference Runtime + a policy (policy: 0 lru, 1 cachesage, 2 ttl) with a general
// event stream (types.hpp:51-82): kind[i] 0 BlockTouch, 1 RequestArrival, 2 AgentDispatch,
// 3 ToolReturn, 4 TurnComplete; agent[i] = the arrival/tool/dispatch-next AgentId, prev[i] with
// has_prev[i] for dispatches, request[i]. After event i with drain[i]: drain_side_effects. After
// event i with ckpt[i]: a checkpoint object {"i", "state": serialize_state().dump(),
// "predict": predict(1) as [[hex id, p] ...] ranked (p desc, id asc), "next": {hex a:
// predict_next(a) ranked} for every learner agent, "drained": [[hex target, tick] ...]}.
// Writes the JSON array of checkpoints into out; returns its length, or -1 (message in
// ref_last_error; *fail_at = the event index that threw).
long ref_policy_events(const ref_run_cfg* c, long n, const int* kind, const unsigned long long* tick,
                       const unsigned long long* agent, const int* has_prev, const unsigned long long* prev,
                       const unsigned long long* request, const unsigned char* drain, const unsigned char* ckpt,
                       char* out, long cap, long* fail_at) {
    *fail_at = -1;
    try {
        std::shared_ptr<Policy> pol;
        std::shared_ptr<CacheSagePolicy> cs;
        if (c->policy == 0) {
            pol = std::make_shared<LruPolicy>();
        } else if (c->policy == 2) {
            pol = std::make_shared<TtlPolicy>();
        } else {
            cs = std::make_shared<CacheSagePolicy>(to_cs_cfg(c));
            pol = cs;
        }
        Runtime rt;
        rt.register_policy(pol);
        auto ranked = [](const Forecast& f) {
            std::vector<std::pair<AgentId, double>> v(f.distribution.begin(), f.distribution.end());
            std::sort(v.begin(), v.end(), [](const auto& x, const auto& y) {
                return x.second > y.second || (x.second == y.second && x.first < y.first);
            });
            json a = json::array();
            for (const auto& [id, p] : v) a.push_back(json::array({to_hex(id.value), p}));
            return a;
        };
        json cps = json::array();
        json drained = json::array();
        for (long i = 0; i < n; ++i) {
            Event e;
            e.tick = tick[i];
            switch (kind[i]) {
                case 0: e.payload = BlockTouch{BlockKey{request[i]}, AgentId{agent[i]}}; break;
                case 1: e.payload = RequestArrival{request[i], AgentId{agent[i]}}; break;
                case 2: {
                    std::optional<AgentId> p;
                    if (has_prev[i]) p = AgentId{prev[i]};
                    e.payload = AgentDispatch{p, AgentId{agent[i]}};
                    break;
                }
                case 3: e.payload = ToolReturn{AgentId{agent[i]}}; break;
                default: e.payload = TurnComplete{request[i]}; break;
            }
            *fail_at = i;
            rt.dispatch_event(e);
            *fail_at = -1;
            if (drain[i])
                for (const SideEffect& fx : rt.drain_side_effects())
                    drained.push_back(json::array({to_hex(fx.target.value), fx.issued_tick}));
            if (ckpt[i]) {
                json next = json::object();
                if (cs)
                    for (AgentId a : cs->learner().agents()) next[to_hex(a.value)] = ranked(cs->predict_next(a, 1));
                cps.push_back(json{{"i", i},
                                   {"state", pol->serialize_state().dump()},
                                   {"predict", ranked(rt.consult_forecast(1))},
                                   {"next", std::move(next)},
                                   {"drained", drained}});
                drained = json::array();
            }
        }
        const std::string d = cps.dump();
        if ((long)d.size() < cap) std::memcpy(out, d.c_str(), d.size() + 1);
        return (long)d.size();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

double ref_exact_survival(unsigned long long target, int k, long n, const unsigned long long* a,
                          const unsigned long long* b, unsigned long long current) {
    try {
        TransitionLearner l;
        for (long i = 0; i < n; ++i) l.record(AgentId{a[i]}, AgentId{b[i]});
        return oracle::exact_survival_prob(AgentId{target}, k, l, AgentId{current});
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// CPU reference timing at pool size N (SURVEY.md §8d "CPU reference timing"): fills a
// reference EngineSim (budget N) through EngineSim::admit with one-block prompts; the first
// `n_agent_blocks` blocks carry one of `n_agents` agent identities (anchor region), the rest are
// agentless, then the policy sees `n_agents` dispatches so reachability is built. Then times
// `k` further one-block admissions, each of which triggers exactly one evict_one (two O(N)
// passes). Returns seconds per eviction; fill seconds in *fill_s.
double ref_evict_bench(long N, int n_agents, long n_agent_blocks, long k_warm, long k, int cachesage,
                       double* fill_s, unsigned long long* last_victim) {
    try {
        using clk = std::chrono::steady_clock;
        Runtime rt;
        std::shared_ptr<Policy> pol;
        if (cachesage) pol = std::make_shared<CacheSagePolicy>();
        else pol = std::make_shared<LruPolicy>();
        rt.register_policy(pol);
        EngineConfig ec;
        ec.budget_blocks = static_cast<int>(N);
        EngineSim eng(ec, rt);
        std::vector<AgentId> agents;
        for (int a = 0; a < n_agents; ++a) agents.push_back(AgentId{mix64(0xa6e47ULL + a)});
        Tick t = 0;
        for (int a = 0; a < n_agents; ++a) {
            std::optional<AgentId> p;
            if (a) p = agents[a - 1];
            rt.dispatch_event(Event{++t, AgentDispatch{p, agents[a]}});
        }
        const auto f0 = clk::now();
        std::vector<PromptBlock> one(1);
        for (long i = 0; i < N; ++i) {
            one[0].key = BlockKey{mix64(0xf111ULL + static_cast<std::uint64_t>(i))};
            one[0].token_count = 16;
            std::optional<AgentId> ag;
            if (i < n_agent_blocks && n_agents > 0) ag = agents[i % n_agents];
            eng.admit(one, ag, ag ? 1 : 0);
        }
        *fill_s = std::chrono::duration<double>(clk::now() - f0).count();
        for (long i = 0; i < k_warm; ++i) {
            one[0].key = BlockKey{mix64(0xd111ULL + static_cast<std::uint64_t>(i))};
            eng.admit(one, std::nullopt, 0);
        }
        const auto e0 = clk::now();
        for (long i = 0; i < k; ++i) {
            one[0].key = BlockKey{mix64(0xe111ULL + static_cast<std::uint64_t>(i))};
            eng.admit(one, std::nullopt, 0);
        }
        const double s = std::chrono::duration<double>(clk::now() - e0).count();
        *last_victim = eng.eviction_log().empty() ? 0 : eng.eviction_log().back().value;
        return k > 0 ? s / static_cast<double>(k) : 0.0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// The reference TransitionLearner after recording n pairs with window W, as the device learner
// exposes it (cs_learner_*): the alphabet (first-seen order, <= cap), P(a,b) over it, row
// totals, state_bytes, argmax_row per row, rebuild_reachability hops from `current`, and
// exact_survival_prob(agent, k, current) per agent (k < 0: skipped). Returns the alphabet size.
long ref_learner_eval(long n, const unsigned long long* a, const unsigned long long* b, long window, long cap,
                      unsigned long long current, double tau, int e_max, int k, unsigned long long* agents,
                      double* prob, unsigned long long* totals, unsigned long long* state_bytes,
                      unsigned long long* amax_id, double* amax_p, int* amax_found, int* hops, double* surv) {
    try {
        TransitionLearner l((std::size_t)window);
        for (long i = 0; i < n; ++i) l.record(AgentId{a[i]}, AgentId{b[i]});
        const auto& al = l.agents();
        const long A = (long)al.size();
        if (A > cap) return -2;
        for (long i = 0; i < A; ++i) {
            agents[i] = al[i].value;
            totals[i] = l.row_total(al[i]);
            for (long j = 0; j < A; ++j) prob[i * A + j] = l.prob(al[i], al[j]);
            const auto am = l.argmax_row(al[i]);
            amax_found[i] = am ? 1 : 0;
            amax_id[i] = am ? am->first.value : 0ull;
            amax_p[i] = am ? am->second : 0.0;
        }
        *state_bytes = l.state_bytes();
        const ReachabilityState r = rebuild_reachability(l, AgentId{current}, tau, e_max);
        for (long i = 0; i < A; ++i) hops[i] = r.hop(al[i]);
        if (k >= 0)
            for (long i = 0; i < A; ++i) surv[i] = oracle::exact_survival_prob(al[i], k, l, AgentId{current});
        return A;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// The reference's Python surface (py_module.cpp:134-183): generate_trace(preset, sessions, seed)
// -> Trace.to_jsonl(), and run_sim(read_trace_jsonl(text), policy, budget, concurrency,
// block_size, prefetch) -> its metrics. Marshalling only.
long ref_preset_trace_jsonl(const char* preset, int sessions, long long seed, char* buf, long cap) {
    try {
        WorkloadSpec spec = preset_by_name(preset);
        if (sessions > 0) spec.sessions = sessions;
        if (seed >= 0) spec.seed = (std::uint64_t)seed;
        std::ostringstream out;
        write_trace_jsonl(generate_trace(spec), out);
        const std::string t = out.str();
        if (buf && cap > 0) std::memcpy(buf, t.data(), std::min<long>(cap, (long)t.size()));
        return (long)t.size();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// out: hit_rate, mean_ttft_ms, mean_latency_ms, throughput_turns_per_s, sim_duration_ms, turns,
// total_prompt_tokens, total_cached_tokens, evictions, truncated_admissions, warmups_executed,
// warmup_prompt_tokens (metrics_to_py order, py_module.cpp:48-63)
int ref_run_sim_jsonl(const char* jsonl, const char* policy, int budget, int concurrency, int block_size, int prefetch,
                      double* out) {
    try {
        std::istringstream in(jsonl);
        const Trace trace = read_trace_jsonl(in);
        RunConfig config;
        config.policies = {policy};
        if (budget > 0) config.budget_blocks = budget;
        if (concurrency > 0) config.concurrency = concurrency;
        config.block_size = block_size;
        config.prefetch = prefetch != 0;
        const RunResult r = run_cell(trace, policy, config);
        const RunMetrics& m = r.aggregate;
        const double v[12] = {m.hit_rate, m.mean_ttft_us / 1000.0, m.mean_latency_us / 1000.0,
                              m.throughput_turns_per_s, m.sim_duration_us / 1000.0, (double)m.turns,
                              (double)m.total_prompt_tokens, (double)m.total_cached_tokens, (double)m.evictions,
                              (double)m.truncated_admissions, (double)m.warmups_executed,
                              (double)m.warmup_prompt_tokens};
        std::memcpy(out, v, sizeof(v));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// The reference's experiment driver over a config text (experiment.cpp:238-330 parse, :380-495
// run_experiment): writes <out.dir>/<workload>/<policy>/{metrics.json,turns.csv,events.jsonl}
// and summary.json. Marshalling only.
int ref_run_experiment_text(const char* config_text) {
    try {
        RunConfig config = parse_run_config_text(config_text, "<config>");
        config.force = true;
        std::ostringstream summary;
        run_experiment(config, summary);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
