// cachesage_b200_policy.hpp — the reference-side drop-in (header only): what a maintainer of
// the reference (/root/reference/proj) adds to route its per-step policy hot path through
// libcachesage_b200.so. Compiled against the reference's own headers (cachesage/*.hpp) and the
// C ABI (cachesage_b200.h); no torch, no CUDA types.
//
//   B200Policy        a cachesage::Policy (runtime.hpp:48-61) whose learner, reachability BFS,
//                     prefetch gate, forecast and state live on the GPU pool; register it with
//                     cachesage::Runtime::register_policy exactly like CacheSagePolicy.
//   BatchEvictor      the batched eviction hook SURVEY.md §8b specifies (the per-block virtual
//                     score() cannot be served by a GPU per call), and B200BatchEvictor, which
//                     runs EngineSim::admit_pinned's whole evict_one loop (engine.cpp:102-168)
//                     as one device launch over the same pool.
//
// Errors map back to the reference's exception types (cs_check). Single-writer, like a
// reference Policy.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "cachesage/cachesage_policy.hpp"
#include "cachesage/engine.hpp"
#include "cachesage/hashing.hpp"
#include "cachesage/runtime.hpp"
#include "cachesage/types.hpp"
#include "cachesage_b200.h"

namespace cachesage_b200 {

// C ABI status -> the reference's exception type (SURVEY.md §8b "Errors").
inline void cs_check(int rc) {
    if (rc >= 0) return;
    const std::string m = cs_last_error();
    switch (rc) {
        case CS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case CS_ERR_LOGIC: throw std::logic_error(m);
        default: throw std::runtime_error(m);  // RUNTIME, CUDA, CAPACITY
    }
}

// Owns one device pool (blocks + learner) and the AgentId <-> dense index map the C ABI uses.
class B200Pool {
public:
    B200Pool(const cachesage::CacheSageConfig& cfg, int budget_blocks, int policy = 1, int agent_capacity = 1024,
             int device = 0) {
        cs_pool_cfg pc;
        cs_pool_cfg_default(&pc);
        pc.budget_blocks = budget_blocks;
        pc.policy = policy;
        pc.e_max = cfg.e_max;
        pc.tau = cfg.tau;
        pc.w_pred = cfg.w_pred;
        pc.window = static_cast<int64_t>(cfg.window);
        pc.min_confidence = cfg.gate.min_confidence;
        pc.min_row_count = cfg.gate.min_row_count;
        pc.budget_per_step = cfg.gate.budget_per_step;
        pc.agent_capacity = agent_capacity;
        pc.device = device;
        cs_check(cs_pool_create(&pc, &pool_));
    }
    ~B200Pool() {
        if (pool_) cs_pool_destroy(pool_);
    }
    B200Pool(const B200Pool&) = delete;
    B200Pool& operator=(const B200Pool&) = delete;

    cs_pool_t handle() const { return pool_; }
    // Dense index of an agent, registered on first sight.
    int index(cachesage::AgentId a) {
        const auto it = index_.find(a.value);
        if (it != index_.end()) return it->second;
        int first = 0;
        cs_check(cs_register_agents(pool_, &a.value, 1, &first));
        index_.emplace(a.value, first);
        ids_.push_back(a.value);
        return first;
    }
    int find(cachesage::AgentId a) const {
        const auto it = index_.find(a.value);
        return it == index_.end() ? -1 : it->second;
    }
    cachesage::AgentId id(int index) const { return cachesage::AgentId{ids_.at(index)}; }
    int agents() const { return static_cast<int>(ids_.size()); }

private:
    cs_pool_t pool_ = nullptr;
    std::unordered_map<std::uint64_t, int> index_;
    std::vector<std::uint64_t> ids_;
};

// CacheSagePolicy (cachesage_policy.hpp:48-85) with its state on the GPU. observe() forwards
// every Event (cs_dispatch_event); score() is the per-block host mirror the reference's
// evict_one consults (w_pred * survival + recency_residual, cachesage_policy.cpp:79-85, with the
// hops the device BFS produced); predict / poll_actions / serialize_state read the device.
class B200Policy : public cachesage::Policy {
public:
    explicit B200Policy(cachesage::CacheSageConfig cfg = {}, int agent_capacity = 1024, int device = 0,
                        int pool_budget = 64)
        : cfg_(cfg), pool_(std::make_shared<B200Pool>(cfg, pool_budget, 1, agent_capacity, device)) {
        if (cfg_.identity.skip < 0 || cfg_.identity.take < 1)
            throw std::invalid_argument("CacheSagePolicy: invalid identity window");
        if (cfg_.tau < 0.0 || cfg_.tau > 1.0) throw std::invalid_argument("CacheSagePolicy: tau must be a probability");
        if (cfg_.e_max <= 0) throw std::invalid_argument("CacheSagePolicy: e_max must be positive");
        if (cfg_.gate.min_confidence < 0.0 || cfg_.gate.budget_per_step < 0)
            throw std::invalid_argument("CacheSagePolicy: invalid prefetch gate");
    }

    const char* name() const override { return "cachesage"; }

    void observe(const cachesage::Event& event) override {
        cs_event ev{};
        ev.tick = event.tick;
        ev.prev = -1;
        bool dispatch = false;
        std::visit(cachesage::overloaded{
                       [&](const cachesage::BlockTouch&) { ev.kind = CS_EV_BLOCK_TOUCH; },
                       [&](const cachesage::RequestArrival& a) {
                           ev.kind = CS_EV_REQUEST_ARRIVAL;
                           ev.agent = pool_->index(a.agent);
                           ev.request = a.request;
                       },
                       [&](const cachesage::AgentDispatch& d) {
                           ev.kind = CS_EV_AGENT_DISPATCH;
                           ev.agent = pool_->index(d.next);
                           if (d.prev) ev.prev = pool_->index(*d.prev);
                           dispatch = true;
                       },
                       [&](const cachesage::ToolReturn& t) {
                           ev.kind = CS_EV_TOOL_RETURN;
                           ev.agent = pool_->index(t.agent);
                       },
                       [&](const cachesage::TurnComplete& c) {
                           ev.kind = CS_EV_TURN_COMPLETE;
                           ev.request = c.request;
                       },
                   },
                   event.payload);
        int warm = -1;
        cs_check(cs_dispatch_event(pool_->handle(), &ev, &warm));
        if (dispatch && ev.agent != current_) {  // the device rebuilt the reachability classes
            current_ = ev.agent;
            hops_.assign(pool_->agents(), cfg_.e_max);
            cs_check(cs_hops(pool_->handle(), hops_.data(), static_cast<int>(hops_.size())));
        }
    }

    double score(const cachesage::Block& block, const cachesage::ScoreContext& ctx) const override {
        double survival = 0.0;
        if (block.agent && current_ >= 0) {  // reach_ is non-empty after the first dispatch
            const int i = pool_->find(*block.agent);
            const int h = (i >= 0 && i < static_cast<int>(hops_.size()) && hops_[i] >= 0) ? hops_[i] : cfg_.e_max;
            const int capped = std::min(h, cfg_.e_max);  // ReachabilityState::survival, reachability.cpp:17-20
            survival = 1.0 - static_cast<double>(capped) / static_cast<double>(cfg_.e_max);
        }
        return cfg_.w_pred * survival + cachesage::recency_residual(block, ctx);
    }

    cachesage::Forecast predict(int horizon) const override { return forecast(-1, horizon); }

    cachesage::Forecast predict_next(cachesage::AgentId current, int horizon = 1) const {
        const int i = pool_->find(current);
        if (i < 0) return cachesage::Forecast{horizon, {}};
        return forecast(i, horizon);
    }

    std::vector<cachesage::SideEffect> poll_actions() override {
        std::vector<int> t(64);
        std::vector<uint64_t> k(64);
        int n = 0;
        cs_check(cs_poll_actions(pool_->handle(), t.data(), k.data(), static_cast<int>(t.size()), &n));
        std::vector<cachesage::SideEffect> out;
        for (int j = 0; j < n && j < static_cast<int>(t.size()); ++j)
            out.push_back(cachesage::SideEffect{cachesage::SideEffect::Kind::Warmup, pool_->id(t[j]), k[j]});
        return out;
    }

    cachesage::json serialize_state() const override {
        size_t len = 0;
        cs_check(cs_serialize_state(pool_->handle(), nullptr, 0, &len));
        std::string buf(len + 1, '\0');
        cs_check(cs_serialize_state(pool_->handle(), buf.data(), buf.size(), &len));
        buf.resize(len);
        return cachesage::json::parse(buf);
    }

    std::size_t state_bytes() const {
        uint64_t b = 0;
        cs_check(cs_policy_state_bytes(pool_->handle(), &b));
        return static_cast<std::size_t>(b);
    }

    const std::shared_ptr<B200Pool>& pool() const { return pool_; }

private:
    cachesage::Forecast forecast(int current, int horizon) const {
        cachesage::Forecast f;
        f.horizon = horizon;
        const int cap = std::max(pool_->agents(), 1);
        std::vector<uint64_t> ids(cap);
        std::vector<double> p(cap);
        int n = 0;
        cs_check(cs_predict(pool_->handle(), horizon, current, ids.data(), p.data(), nullptr, cap, &n));
        for (int j = 0; j < n && j < cap; ++j) f.distribution[cachesage::AgentId{ids[j]}] = p[j];
        return f;
    }

    cachesage::CacheSageConfig cfg_;
    std::shared_ptr<B200Pool> pool_;
    int current_ = -1;
    std::vector<int> hops_;
};

// ---------------------------------------------------------------- the batched eviction hook

// One admission as EngineSim::admit_pinned sees it (engine.cpp:141-168): the prompt's blocks,
// the request's agent and anchor count, and the engine clock before the first touch.
struct AdmissionView {
    const cachesage::PromptBlock* blocks = nullptr;
    std::size_t n = 0;
    std::optional<cachesage::AgentId> agent;
    int anchor_block_count = 0;
    cachesage::Tick tick_base = 0;
};

// an engine that finds this interface on its policy (dynamic_cast) hands it the
// whole admission instead of calling evict_one per missing block.
struct BatchEvictor {
    virtual ~BatchEvictor() = default;
    // Makes every block resident and pinned (touching block i at tick_base + 1 + i) and returns
    // the victims in evict_one order; at most k_max are written to out.
    virtual std::size_t select_victims(const AdmissionView& view, std::size_t k_max, cachesage::BlockKey* out) = 0;
};

// The GPU pool as a BatchEvictor: the exact victims of the reference's sequential loop from one
// launch, plus the pool-side lookup / unpin the same engine calls.
class B200BatchEvictor : public BatchEvictor {
public:
    explicit B200BatchEvictor(std::shared_ptr<B200Pool> pool) : pool_(std::move(pool)) {}

    std::size_t select_victims(const AdmissionView& v, std::size_t k_max, cachesage::BlockKey* out) override {
        stage(v.blocks, v.n);
        const uint32_t agent = v.agent ? static_cast<uint32_t>(pool_->index(*v.agent)) : CS_NO_AGENT;
        std::vector<uint64_t> ev(std::max<std::size_t>(v.n, 1));
        int64_t ne = 0;
        cs_check(cs_admit_pinned(pool_->handle(), keys_.data(), counts_.data(), static_cast<int>(v.n), agent,
                                 v.anchor_block_count, v.tick_base, ev.data(), static_cast<int64_t>(ev.size()), &ne,
                                 nullptr));
        const std::size_t m = std::min<std::size_t>(static_cast<std::size_t>(ne), k_max);
        for (std::size_t j = 0; j < m; ++j) out[j] = cachesage::BlockKey{ev[j]};
        return static_cast<std::size_t>(ne);
    }

    // EngineSim::lookup (engine.cpp:127-139) on the pool.
    cachesage::LookupResult lookup(const std::vector<cachesage::PromptBlock>& blocks, cachesage::Tick tick_base) {
        stage(blocks.data(), blocks.size());
        int64_t cached = 0;
        int fm = 0;
        cs_check(cs_lookup(pool_->handle(), keys_.data(), counts_.data(), static_cast<int>(blocks.size()), tick_base,
                           &cached, &fm));
        return cachesage::LookupResult{static_cast<long>(cached), static_cast<std::size_t>(fm)};
    }

    // EngineSim::unpin (engine.cpp:170-180).
    void unpin(const std::vector<cachesage::BlockKey>& keys) {
        std::vector<uint64_t> k(keys.size());
        for (std::size_t j = 0; j < keys.size(); ++j) k[j] = keys[j].value;
        cs_check(cs_unpin(pool_->handle(), k.data(), static_cast<int>(k.size())));
    }

private:
    void stage(const cachesage::PromptBlock* b, std::size_t n) {
        keys_.resize(std::max<std::size_t>(n, 1));
        counts_.resize(std::max<std::size_t>(n, 1));
        for (std::size_t j = 0; j < n; ++j) {
            keys_[j] = b[j].key.value;
            counts_[j] = b[j].token_count;
        }
    }
    std::shared_ptr<B200Pool> pool_;
    std::vector<uint64_t> keys_;
    std::vector<int32_t> counts_;
};

}  // namespace cachesage_b200
