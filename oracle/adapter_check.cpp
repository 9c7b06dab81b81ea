// TEST INFRASTRUCTURE ONLY. Compiles the reference-side drop-in (include/cachesage_b200_policy.hpp)
// against the reference's own headers and drives the UNMODIFIED reference engine through it:
//
//   adapter_run        run_cell's loop (ref_shim.cpp ref_run_with) with B200Policy registered in
//                      the reference Runtime: every observe / predict / poll_actions /
//                      serialize_state goes to the GPU pool; the reference EngineSim calls
//                      B200Policy::score per block in its own evict_one.
//   adapter_lockstep   the reference EngineSim (with the reference CacheSagePolicy) and
//                      B200BatchEvictor side by side over one request stream: same dispatches,
//                      lookups and admissions; the evictor's victims (one device launch per
//                      admission) must equal the reference evict_one loop's, admission by
//                      admission.
//
// Built by `make -C oracle adapter` into oracle/_ref/ (needs /root/reference to build; travels
// to the GPU box with the snapshot like the rest of oracle/_ref).
#include <cstring>
#include <string>
#include <vector>

#include "cachesage/cachesage_policy.hpp"
#include "cachesage/engine.hpp"
#include "cachesage/runtime.hpp"
#include "cachesage/workload.hpp"
#include "cachesage_b200_policy.hpp"
#include "ref_shim.h"

using namespace cachesage;

namespace {

thread_local std::string g_err;
thread_local std::string g_state;

struct Ctx {
    int device;
};

std::shared_ptr<Policy> make_b200(const CacheSageConfig& cfg, void* ctx) {
    return std::make_shared<cachesage_b200::B200Policy>(cfg, 1024, static_cast<Ctx*>(ctx)->device);
}

}  // namespace

extern "C" {

const char* adapter_last_error(void) { return g_err.c_str(); }
const char* adapter_last_state(void) { return g_state.c_str(); }

int adapter_run(const ref_spec* s, const ref_run_cfg* c, ref_run_out* out, int device) {
    Ctx ctx{device};
    const int rc = ref_run_with(s, c, out, make_b200, &ctx);
    if (rc != 0) {
        g_err = "adapter_run failed (see ref_last_error)";
        return rc;
    }
    return 0;
}

// Lockstep over the first max_req requests of the spec's trace, one request at a time: dispatch
// (both runtimes), lookup (both), admit (reference EngineSim::admit = admit_pinned + unpin;
// B200BatchEvictor::select_victims + unpin). Writes per admission the victim count, and returns
// the number of admissions compared; -1 on an error, -2 - i at the first mismatching admission i.
long adapter_lockstep(const ref_spec* s, const ref_run_cfg* c, long max_req, int device, long* n_victims,
                      unsigned long long* victims, long victims_cap, long* cached_out) {
    try {
        const Trace trace = generate_trace(ref_to_spec(s));
        EngineConfig ec;
        ec.budget_blocks = c->budget_blocks > 0 ? c->budget_blocks : trace.spec.budget_blocks;
        ec.block_size = c->block_size;
        ec.identity = IdentityConfig{c->skip, c->take};
        const auto requests = materialize_requests(trace, ec.block_size, ec.identity);
        CacheSageConfig cs;
        cs.identity = ec.identity;
        cs.tau = c->tau;
        cs.e_max = c->e_max;
        cs.w_pred = c->w_pred;
        cs.window = static_cast<std::size_t>(c->window);
        cs.gate.min_confidence = c->min_confidence;
        cs.gate.min_row_count = c->min_row_count;
        cs.gate.budget_per_step = c->budget_per_step;
        Runtime rt;
        rt.register_policy(std::make_shared<CacheSagePolicy>(cs));
        EngineSim ref(ec, rt);

        auto pool = std::make_shared<cachesage_b200::B200Pool>(cs, ec.budget_blocks, 1, 1024, device);
        cachesage_b200::B200BatchEvictor ev(pool);
        std::optional<AgentId> prev;
        long done = 0, vpos = 0;
        std::vector<BlockKey> vb;
        for (const Request& r : requests) {
            if (done >= max_req) break;
            if (r.prompt_blocks.size() > static_cast<std::size_t>(ec.budget_blocks)) continue;
            // AgentDispatch into both runtimes at the reference engine's clock
            const Tick t = ref.now_tick() + 1;
            rt.dispatch_event(Event{t, AgentDispatch{prev, r.agent}});
            cs_event e{};
            e.tick = t;
            e.kind = CS_EV_AGENT_DISPATCH;
            e.agent = pool->index(r.agent);
            e.prev = prev ? pool->index(*prev) : -1;
            cachesage_b200::cs_check(cs_dispatch_event(pool->handle(), &e, nullptr));
            (void)rt.drain_side_effects();
            int n = 0;
            cachesage_b200::cs_check(cs_poll_actions(pool->handle(), nullptr, nullptr, 0, &n));
            prev = r.agent;
            // lookup, then the admission
            const Tick tl = ref.now_tick();
            const LookupResult lr = ref.lookup(r.prompt_blocks);
            const LookupResult lg = ev.lookup(r.prompt_blocks, tl);
            if (lr.cached_tokens != lg.cached_tokens || lr.first_miss_index != lg.first_miss_index) return -2 - done;
            const Tick ta = ref.now_tick();
            const std::size_t before = ref.eviction_log().size();
            ref.admit(r.prompt_blocks, r.agent, r.anchor_block_count);
            const std::size_t nr = ref.eviction_log().size() - before;
            cachesage_b200::AdmissionView v;
            v.blocks = r.prompt_blocks.data();
            v.n = r.prompt_blocks.size();
            v.agent = r.agent;
            v.anchor_block_count = r.anchor_block_count;
            v.tick_base = ta;
            vb.assign(v.n + 1, BlockKey{});
            const std::size_t ng = ev.select_victims(v, vb.size(), vb.data());
            std::vector<BlockKey> pins;
            for (const auto& b : r.prompt_blocks) pins.push_back(b.key);
            ev.unpin(pins);
            if (nr != ng) return -2 - done;
            for (std::size_t j = 0; j < nr; ++j) {
                if (ref.eviction_log()[before + j] != vb[j]) return -2 - done;
                if (vpos < victims_cap) victims[vpos] = vb[j].value;
                ++vpos;
            }
            n_victims[done] = static_cast<long>(nr);
            cached_out[done] = lr.cached_tokens;
            ++done;
        }
        return done;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// A B200Policy's serialize_state() after adapter-driven events equals CacheSagePolicy's: both
// policies observe the same stream (kind / tick / agent / prev / request as ref_policy_events).
int adapter_state_after(const ref_run_cfg* c, long n, const int* kind, const unsigned long long* tick,
                        const unsigned long long* agent, const int* has_prev, const unsigned long long* prev,
                        const unsigned long long* request, int device, int* same) {
    try {
        CacheSageConfig cs;
        cs.tau = c->tau;
        cs.e_max = c->e_max;
        cs.w_pred = c->w_pred;
        cs.window = static_cast<std::size_t>(c->window);
        cs.gate.min_confidence = c->min_confidence;
        cs.gate.min_row_count = c->min_row_count;
        cs.gate.budget_per_step = c->budget_per_step;
        CacheSagePolicy ref(cs);
        cachesage_b200::B200Policy gpu(cs, 1024, device);
        *same = 1;
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
            ref.observe(e);
            gpu.observe(e);
            // score() of a block of every known agent, at a context both policies see
            const ScoreContext ctx{tick[i] + 10, tick[i] / 2, 0.0};
            for (AgentId a : ref.learner().agents()) {
                Block b;
                b.agent = a;
                b.last_touch = tick[i] / 2 + (a.value & 7);
                if (ref.score(b, ctx) != gpu.score(b, ctx)) *same = 0;
            }
            if ((i & 15) == 15) {
                if (ref.poll_actions().size() != gpu.poll_actions().size()) *same = 0;
                const Forecast fr = ref.predict(1), fg = gpu.predict(1);
                if (fr.distribution != fg.distribution) *same = 0;
            }
        }
        g_state = gpu.serialize_state().dump();
        if (g_state != ref.serialize_state().dump()) *same = 0;
        if (gpu.state_bytes() != ref.state_bytes()) *same = 0;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
