// TEST INFRASTRUCTURE ONLY: the C structs of the reference shim (ref_shim.cpp), shared with
// adapter_check.cpp. Marshalling only; the semantics are the reference's.
#pragma once

#include <cstdint>
#include <memory>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ref_spec {
    int n_agents;
    const int* anchor_tokens;   // [n_agents]
    const double* transition;   // [n_agents * n_agents], row-major
    int supervisor;             // -1 = none
    int turns_min, turns_max, sessions, task_tokens, history_growth, decode_tokens;
    int template_tokens, concurrency, budget_blocks;
    unsigned long long seed;
} ref_spec;

typedef struct ref_run_cfg {
    int policy;  // 0 = lru, 1 = cachesage, 2 = ttl, 3 = belady
    int budget_blocks;  // <= 0: the spec's pairing
    int concurrency;    // <= 0: the spec's pairing
    int block_size;
    int prefetch;
    int skip, take;
    double tau;
    int e_max;
    double w_pred;
    long window;
    double min_confidence;
    unsigned long long min_row_count;
    int budget_per_step;
    // CostModel (engine.hpp:22-26); 0 keeps the reference default
    double prefill_base_us, prefill_per_token_us, decode_per_token_us;
} ref_run_cfg;

typedef struct ref_run_out {
    long n_turns;
    long* cached_tokens;   // by turn id
    long* prompt_tokens;
    double* start_us;
    double* end_us;
    long n_evictions;
    unsigned long long* evictions;
    long n_warmups;  // drained side effects (executed or dropped)
    long* warmup_step;
    unsigned long long* warmup_target;
    unsigned long long* warmup_tick;
    double hit_rate;
    long truncated;
    long warmups_executed;
    long warmups_dropped;
    double sim_us;
    long n_steps;
    long events;
} ref_run_out;

#ifdef __cplusplus
}

namespace cachesage {
class Policy;
struct CacheSageConfig;
struct WorkloadSpec;
}  // namespace cachesage

// the shim's ref_spec -> WorkloadSpec conversion
cachesage::WorkloadSpec ref_to_spec(const ref_spec* s);

// ref_run with the scoring policy from `make` (nullptr: the reference's own by c->policy).
int ref_run_with(const ref_spec* s, const ref_run_cfg* c, ref_run_out* out,
                 std::shared_ptr<cachesage::Policy> (*make)(const cachesage::CacheSageConfig&, void*), void* ctx);
#endif
