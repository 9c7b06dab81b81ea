// The rest of the reference's Policy / Runtime surface over a device pool (paths relative to
// /root/reference/proj):
//   cs_dispatch_event     Runtime::dispatch_event (runtime.cpp:59-69) -> CacheSagePolicy::observe
//                         for every Event kind (types.hpp:51-82, cachesage_policy.cpp:50-77)
//   cs_unpin              EngineSim::unpin by BlockKey (engine.cpp:170-180)
//   cs_predict            CacheSagePolicy::predict / predict_next (cachesage_policy.cpp:87-107),
//                         ranked for prefetch on the device (forecast_kernel)
//   cs_serialize_state    CacheSagePolicy::serialize_state (cachesage_policy.cpp:139-153) and the
//                         baselines' (baselines.cpp:16, 30-32, 72-74), byte-identical dump()
//   cs_policy_state_bytes CacheSagePolicy::state_bytes (cachesage_policy.cpp:133-138)
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "cs_pool.hpp"
#include "json.hpp"

using csb::ck;
using csb::CsError;

void cs_set_error(const std::string& m);  // cs_pool.cpp

namespace {

using json = nlohmann::ordered_json;  // json_alias.hpp:8

template <class F>
int sguard(F&& f) {
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

std::string to_hex(uint64_t v) {  // hashing.cpp:8-12
    char buf[19];
    std::snprintf(buf, sizeof(buf), "0x%016llx", static_cast<unsigned long long>(v));
    return buf;
}

const char* policy_name(int policy) {  // name() of each Policy (baselines.hpp, cachesage_policy.hpp:52)
    switch (policy) {
        case 0: return "lru";
        case 2: return "ttl";
        case 3: return "belady";
        default: return "cachesage";
    }
}

// The learner and reachability state as the reference holds it, read back from the device.
struct PolicyState {
    csb::Ctrl c{};
    int n = 0;                          // registered agents (dense indices)
    std::vector<unsigned int> counts;   // n x n
    std::vector<unsigned int> totals;   // n
    std::vector<int> wa, wb;            // window, oldest first
    std::vector<unsigned char> hop;     // n
    long long nonzero = 0, rows = 0;
};

PolicyState read_state(cs_pool_t pool) {
    PolicyState s;
    pool->sync();  // (an engine's last admission may still be finishing its prescan)
    ck(cudaMemcpy(&s.c, pool->P.ctrl, sizeof(s.c), cudaMemcpyDeviceToHost), "ctrl D2H");
    const int n = s.n = pool->n_agents;
    const int A = pool->P.a_cap;
    s.counts.assign((size_t)n * n, 0u);
    s.totals.assign(n, 0u);
    s.hop.assign(n, 0);
    if (n > 0) {
        ck(cudaMemcpy2D(s.counts.data(), sizeof(unsigned int) * n, pool->P.counts, sizeof(unsigned int) * A,
                        sizeof(unsigned int) * n, n, cudaMemcpyDeviceToHost),
           "counts D2H");
        ck(cudaMemcpy(s.totals.data(), pool->P.totals, sizeof(unsigned int) * n, cudaMemcpyDeviceToHost), "totals D2H");
        ck(cudaMemcpy(s.hop.data(), pool->P.hop, n, cudaMemcpyDeviceToHost), "hop D2H");
    }
    const long long W = pool->P.window, head = s.c.win_head, size = s.c.win_size;
    std::vector<int> ra(W), rb(W);
    if (size > 0) {
        ck(cudaMemcpy(ra.data(), pool->P.win_a, sizeof(int) * W, cudaMemcpyDeviceToHost), "window D2H");
        ck(cudaMemcpy(rb.data(), pool->P.win_b, sizeof(int) * W, cudaMemcpyDeviceToHost), "window D2H");
    }
    for (long long j = 0; j < size; ++j) {
        s.wa.push_back(ra[(head + j) % W]);
        s.wb.push_back(rb[(head + j) % W]);
    }
    for (int a = 0; a < n; ++a) {
        bool any = false;
        for (int b = 0; b < n; ++b)
            if (s.counts[(size_t)a * n + b]) {
                ++s.nonzero;
                any = true;
            }
        if (any) ++s.rows;
    }
    return s;
}

// TransitionLearner::state_bytes (transition_learner.cpp:98-106) + the policy's own
// (cachesage_policy.cpp:133-138): u8 hop per agent of the last rebuild, 8 B anchor id.
unsigned long long policy_bytes(cs_pool_t pool, const PolicyState& s) {
    unsigned long long b = 0;
    b += (unsigned long long)s.wa.size() * 4;
    b += (unsigned long long)s.nonzero * 12;
    b += (unsigned long long)s.rows * 10;  // row_totals_ holds exactly the rows with a count
    b += (unsigned long long)pool->alphabet.size() * 8;
    b += 8;
    b += s.c.reach_built ? (unsigned long long)pool->reach_known : 0ull;
    b += 8;
    return b;
}

json serialize(cs_pool_t pool) {
    const int policy = pool->cfg.policy;  // (P.policy runs ttl as lru: cs_pool.cpp)
    if (!pool->mirror_ok)
        throw std::invalid_argument("serialize_state: not available under the device-resident scheduler");
    if (policy == 0) return json{{"policy", "lru"}};  // baselines.cpp:16
    if (policy == 2) return json{{"policy", "ttl"}, {"pin_horizon_us", 5000000.0}};  // baselines.cpp:30-32
    if (policy == 3) return json{{"policy", "belady"}, {"cursor", pool->bel_cursor}};  // baselines.cpp:72-74
    const PolicyState s = read_state(pool);
    const std::vector<uint64_t>& id = pool->agent_ids;
    auto by_id = [&](int x, int y) { return id[x] < id[y]; };
    // TransitionLearner::to_json (transition_learner.cpp:108-147): rows and columns by AgentId
    std::vector<int> order(s.n);
    for (int i = 0; i < s.n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), by_id);
    json rows = json::object();
    for (int a : order) {
        json row = json::object();
        bool any = false;
        for (int b : order) {
            const unsigned int c = s.counts[(size_t)a * s.n + b];
            if (!c) continue;
            row[to_hex(id[b])] = (unsigned long long)c;
            any = true;
        }
        if (any) rows[to_hex(id[a])] = std::move(row);
    }
    json window = json::array();
    for (size_t j = 0; j < s.wa.size(); ++j) window.push_back({to_hex(id[s.wa[j]]), to_hex(id[s.wb[j]])});
    json alphabet = json::array();
    for (int a : pool->alphabet) alphabet.push_back(to_hex(id[a]));
    json learner{{"window_capacity", (unsigned long long)pool->P.window},
                 {"transitions_recorded", s.c.recorded},
                 {"alphabet", std::move(alphabet)},
                 {"rows", std::move(rows)},
                 {"window", std::move(window)}};
    // ReachabilityState::to_json (reachability.cpp:22-37): every agent known at the rebuild
    json reach = nullptr;
    if (s.c.reach_built) {
        std::vector<int> known(pool->alphabet.begin(), pool->alphabet.begin() + std::min(pool->reach_known,
                                                                                          pool->alphabet.size()));
        std::sort(known.begin(), known.end(), by_id);
        json hops = json::object();
        for (int a : known) hops[to_hex(id[a])] = (int)s.hop[a];
        reach = json{{"tau", pool->P.tau},
                     {"e_max", pool->P.e_max},
                     {"anchor", to_hex(s.c.cur_agent >= 0 ? id[s.c.cur_agent] : 0ull)},
                     {"hops", std::move(hops)}};
    }
    json pending = json::array();
    for (size_t k = 0; k < pool->pending_targets.size(); ++k)
        pending.push_back({{"kind", "warmup"},
                           {"target", to_hex(id[pool->pending_targets[k]])},
                           {"issued_tick", pool->pending_ticks[k]}});
    return json{{"policy", policy_name(policy)},
                {"current", s.c.cur_agent >= 0 ? json(to_hex(id[s.c.cur_agent])) : json(nullptr)},
                {"learner", std::move(learner)},
                {"reachability", std::move(reach)},
                {"pending_warmups", std::move(pending)},
                {"rebuilds", s.c.rebuilds},
                {"state_bytes", policy_bytes(pool, s)}};
}

void check_agent(cs_pool_t pool, int a, const char* what) {
    if (a < 0 || a >= pool->n_agents) throw std::invalid_argument(std::string(what) + ": agent index out of range");
}

}  // namespace

void cs_pool::note_agent(int a) {
    if (a < 0) return;
    if ((int)noted.size() <= a) noted.resize(a + 1, 0);
    if (noted[a]) return;
    noted[a] = 1;
    alphabet.push_back(a);
}

void cs_pool::note_dispatch(int prev, int next) {
    if (P.policy != 1) return;  // the baselines' observe ignores dispatches (baselines.cpp:10, 20)
    note_agent(next);
    if (prev >= 0) {  // TransitionLearner::record notes both (transition_learner.cpp:22-24)
        note_agent(prev);
        note_agent(next);
    }
    if (host_cur != next) reach_known = alphabet.size();  // rebuild_reachability: all known agents
    host_cur = next;
}

void cs_pool::check_tick(unsigned long long tick) {
    if (has_last_tick && tick < last_tick)
        throw std::runtime_error("dispatch_event: tick regression (" + std::to_string(tick) + " after " +
                                 std::to_string(last_tick) + ")");
    has_last_tick = true;
    last_tick = tick;
}

extern "C" {

int cs_dispatch_event(cs_pool_t pool, const cs_event* ev, int* warmup_target) {
    return sguard([&] {
        if (!pool || !ev) throw std::invalid_argument("cs_dispatch_event: null argument");
        if (warmup_target) *warmup_target = -1;
        switch (ev->kind) {
            case CS_EV_BLOCK_TOUCH:
            case CS_EV_TURN_COMPLETE:
                pool->check_tick(ev->tick);  // observe ignores them (cachesage_policy.cpp:53-55, 75)
                break;
            case CS_EV_REQUEST_ARRIVAL:
            case CS_EV_TOOL_RETURN:
                check_agent(pool, ev->agent, "cs_dispatch_event");
                pool->check_tick(ev->tick);
                if (pool->P.policy == 1) pool->note_agent(ev->agent);  // note_agent (:56, :74)
                if (pool->P.policy == 3 && ev->kind == CS_EV_REQUEST_ARRIVAL)
                    pool->bel_cursor = std::max<unsigned long long>(pool->bel_cursor, ev->request);  // baselines.cpp:48-52
                break;
            case CS_EV_AGENT_DISPATCH: {
                const int rc = cs_observe_dispatch(pool, ev->prev, ev->agent, ev->tick, warmup_target);
                if (rc != CS_OK) throw CsError(rc, cs_last_error());
                break;
            }
            default:
                throw std::invalid_argument("cs_dispatch_event: unknown event kind");
        }
    });
}

int cs_unpin(cs_pool_t pool, const uint64_t* keys, int n) {
    return sguard([&] {
        if (!pool || n < 0 || (n > 0 && !keys)) throw std::invalid_argument("cs_unpin: null argument");
        if (n == 0) return;
        pool->sync();
        pool->flush_unpins();
        pool->flush_table();
        pool->pre_ok = false;
        cudaStream_t s = pool->stream;
        csb::DevBuf k, sl, bad;
        k.ensure(8 * (size_t)n);
        sl.ensure(4 * (size_t)n);
        bad.ensure(sizeof(int));
        ck(cudaMemcpyAsync(k.p, keys, 8 * (size_t)n, cudaMemcpyHostToDevice, s), "H2D");
        ck(cudaMemcpyAsync(bad.p, &n, sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
        ck(csb::launch_unpin_find(pool->P, k.as<unsigned long long>(), n, sl.as<unsigned int>(), bad.as<int>(), s),
           "unpin_find");
        int first_bad = n;
        ck(cudaMemcpyAsync(&first_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
        pool->sync();
        // engine.cpp:171-179: the keys before the first vanished one are unpinned, then it throws
        if (first_bad > 0) ck(csb::launch_unpin(pool->P, sl.as<unsigned int>(), first_bad, s), "unpin");
        pool->sync();
        csb::Ctrl c;
        ck(cudaMemcpy(&c, pool->P.ctrl, sizeof(c), cudaMemcpyDeviceToHost), "ctrl D2H");
        pool->pinned = c.pinned;
        if (first_bad < n) throw std::logic_error("unpin: block vanished while referenced");
    });
}

int cs_predict(cs_pool_t pool, int horizon, int current, uint64_t* ids, double* probs, int* idx, int cap, int* n) {
    return sguard([&] {
        if (!pool || !n || cap < 0) throw std::invalid_argument("cs_predict: null argument");
        (void)horizon;  // Forecast::horizon is carried, not used (cachesage_policy.cpp:94-107)
        *n = 0;
        if (pool->P.policy != 1) return;  // the baselines forecast nothing (baselines.hpp)
        pool->sync();
        if (current < 0) {  // predict(): rooted at the policy's current agent (cachesage_policy.cpp:87-92)
            csb::Ctrl c;
            ck(cudaMemcpy(&c, pool->P.ctrl, sizeof(c), cudaMemcpyDeviceToHost), "ctrl D2H");
            current = c.cur_agent;
            if (current < 0) return;
        }
        check_agent(pool, current, "cs_predict");
        const int na = pool->n_agents;
        csb::DevBuf oi, op, on;
        oi.ensure(sizeof(int) * std::max(na, 1));
        op.ensure(sizeof(double) * std::max(na, 1));
        on.ensure(sizeof(int));
        ck(csb::launch_forecast(pool->P, current, na, oi.as<int>(), op.as<double>(), on.as<int>(), pool->stream),
           "forecast");
        ++pool->launches;
        int m = 0;
        ck(cudaMemcpyAsync(&m, on.p, sizeof(int), cudaMemcpyDeviceToHost, pool->stream), "D2H");
        pool->sync();
        *n = m;
        const int c = std::min(m, cap);
        if (c <= 0) return;
        std::vector<int> hi(c);
        ck(cudaMemcpy(hi.data(), oi.p, sizeof(int) * c, cudaMemcpyDeviceToHost), "D2H");
        if (probs) ck(cudaMemcpy(probs, op.p, sizeof(double) * c, cudaMemcpyDeviceToHost), "D2H");
        for (int k = 0; k < c; ++k) {
            if (ids) ids[k] = pool->agent_ids[hi[k]];
            if (idx) idx[k] = hi[k];
        }
    });
}

int cs_serialize_state(cs_pool_t pool, char* buf, size_t cap, size_t* len) {
    return sguard([&] {
        if (!pool || !len) throw std::invalid_argument("cs_serialize_state: null argument");
        const std::string d = serialize(pool).dump();
        *len = d.size();
        if (buf && cap > 0) {
            const size_t c = std::min(cap - 1, d.size());
            std::memcpy(buf, d.data(), c);
            buf[c] = '\0';
        }
    });
}

int cs_policy_state_bytes(cs_pool_t pool, uint64_t* bytes) {
    return sguard([&] {
        if (!pool || !bytes) throw std::invalid_argument("cs_policy_state_bytes: null argument");
        if (pool->P.policy != 1) throw std::invalid_argument("cs_policy_state_bytes: only the cachesage policy has it");
        *bytes = policy_bytes(pool, read_state(pool));
    });
}

}  // extern "C"
