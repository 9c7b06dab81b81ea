// Per-cell output writers of the reference's experiment driver (experiment.cpp:94-183, 424-440,
// paths relative to /root/reference/proj): metrics.json, turns.csv, events.jsonl, filled from an
// engine run. Formatting goes through nlohmann::json (the reference's own serializer), so the
// files are byte-identical for identical runs.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace csb {

// EngineSim::events_ (engine.cpp:72-88): one entry per emitted event
struct EventRec {
    enum Kind : uint8_t { kBlockTouch = 0, kRequestArrival = 1, kAgentDispatch = 2, kTurnComplete = 4 };
    uint64_t tick;
    uint64_t a, b;  // touch: key, agent | arrival: request, agent | dispatch: prev, next | complete: request
    uint8_t kind;
    uint8_t has_a, has_b;  // optional AgentId present (touch agent: has_b; dispatch prev: has_a)
};

struct TurnRec {  // TurnMetrics (metrics.hpp:12-25)
    uint64_t turn_id;
    int session, turn_index;
    uint64_t agent;
    int label;  // workload agent index
    long prompt_tokens, cached_tokens;
    double ttft_us, latency_us, arrival_us, start_us, end_us;
};

struct CellOut {
    std::string workload, policy;
    uint64_t seed;
    std::vector<std::string> labels;
    // EngineConfig as run_experiment re-derives it (experiment.cpp:419-424)
    int budget_blocks, block_size, concurrency;
    bool prefetch;
    double prefill_per_token_us, prefill_base_us, decode_per_token_us;
    // CacheSageConfig (policy_config_json, experiment.cpp:74-92)
    int skip, take, e_max, budget_per_step;
    double tau, w_pred, min_confidence;
    uint64_t window, min_row_count;
    double ttl_pin_horizon_us;
    // RunResult (engine.cpp:394-413)
    std::vector<TurnRec> turns;  // sorted by turn_id
    double sim_duration_us;
    uint64_t evictions, truncated, warmups_executed, warmups_dropped;
    long warmup_prompt_tokens, warmup_uncached_tokens;
    double warmup_time_us;
    const std::vector<EventRec>* events;  // null: no events.jsonl
};

// Writes <dir>/metrics.json, <dir>/turns.csv and (events != null) <dir>/events.jsonl.
void write_cell(const CellOut& c, const std::string& dir);

}  // namespace csb
