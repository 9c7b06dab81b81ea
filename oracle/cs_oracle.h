/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the CacheSage per-step hot path.
 *
 * A plain-C restatement of the reference algorithm (each function cites the reference
 * file:line it follows, paths relative to /root/reference/proj). Only tests/, the
 * __graft_entry__.smoke() checker and bench.py's cpu_baseline / reference legs may load it.
 * The product (paper_2605_27744_b200) never links, loads or calls it.
 *
 * Parity PINNED: tests/test_oracle_golden.py checks this oracle against (a) the goldens of
 * SURVEY.md Appendix A.1/A.2, (b) the JSON fixtures in tests/golden produced by the UNMODIFIED reference
 * (oracle/_ref, tests/golden/make_golden.py), and (c) oracle/_ref itself on random specs.
 */
#ifndef CS_ORACLE_H
#define CS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* WorkloadSpec (workload.hpp:21-42). Token scheme knobs widen the generator:
 * anchor_stride = 0x10000 and hist_pos_bits = 20 reproduce the reference exactly. */
typedef struct cso_spec {
    int n_agents;
    const int* anchor_tokens;
    const double* transition; /* n_agents x n_agents row-major */
    int supervisor;           /* -1 = none (start agent 0) */
    int turns_min, turns_max, sessions, task_tokens, history_growth, decode_tokens;
    int template_tokens, concurrency, budget_blocks;
    uint64_t seed;
    uint32_t anchor_stride;   /* 0 -> 0x10000 */
    int hist_pos_bits;        /* 0 -> 20 */
    const double* start_dist; /* used when supervisor == -2 */
} cso_spec;

/* RunConfig subset + CacheSageConfig (experiment.hpp:28-44, cachesage_policy.hpp:17-43). */
typedef struct cso_cfg {
    int policy; /* 0 = lru, 1 = cachesage, 2 = ttl, 3 = belady (cso_run only) */
    int budget_blocks, concurrency, block_size, prefetch;
    int skip, take;
    double tau;
    int e_max;
    double w_pred;
    long window;
    double min_confidence;
    uint64_t min_row_count;
    int budget_per_step;
    /* 1: the indexed evict_one (per-agent heaps of unpinned blocks by last_touch + a heap of all
     * resident blocks), exact by the class-head lemma; 0: the reference's O(N) argmin. Belady
     * always uses the O(N) argmin (its score is not monotone in last_touch). */
    int fast_evict;
    /* CostModel (engine.hpp:20-24, experiment.cpp:272-279); 0 = the reference defaults
     * 1000 / 50 / 20000 us. */
    double prefill_base_us, prefill_per_token_us, decode_per_token_us;
} cso_cfg;

typedef struct cso_run_out {
    long n_turns;
    long* cached_tokens;
    long* prompt_tokens;
    double* start_us;
    double* end_us;
    long n_evictions;
    uint64_t* evictions;
    long n_warmups;
    long* warmup_step;
    uint64_t* warmup_target;
    uint64_t* warmup_tick;
    double hit_rate;
    long truncated, warmups_executed, warmups_dropped;
    double sim_us;
    long n_steps;
    long n_admissions; /* start_request + executed warmups */
    uint8_t* completed; /* per turn: 1 once complete_earliest retired it */
} cso_run_out;

uint64_t cso_mix64(uint64_t x);
/* returns 0 and sets *err = 1 on empty input */
uint64_t cso_chain_hash(int has_parent, uint64_t parent, const uint32_t* tokens, size_t n, int* err);
long cso_block_keys(const uint32_t* tokens, size_t n, int block_size, uint64_t* keys, int32_t* counts);
int cso_identity(const uint64_t* keys, size_t n, int skip, int take, uint64_t* out);

/* generator: turns7 = (session, turn_index, agent, anchor, history, prompt, decode) */
long cso_generate(const cso_spec* spec, int64_t* turns7, long cap);
long cso_turn_tokens(const cso_spec* spec, const int64_t* turn7, uint32_t* out, long cap);

int cso_run(const cso_spec* spec, const cso_cfg* cfg, cso_run_out* out);

/* A resident-pool snapshot installed before the first scheduler step (as cs_engine_restore):
 * agents are 64-bit AgentIds (has_agent = 0: none); the engine clock becomes max(last_touch). */
typedef struct cso_snapshot {
    long n;
    const uint64_t* keys;
    const uint64_t* last_touch;
    const int32_t* has_agent;
    const uint64_t* agents;
    const int32_t* refs; /* NULL: all unpinned */
} cso_snapshot;

/* cso_run from an optional snapshot, stopping after max_steps scheduler steps (< 0: run to the
 * end). out->n_turns counts every request; turns not completed keep cached/end = 0 and are
 * flagged by out->completed[i] = 0. */
int cso_run_ex(const cso_spec* spec, const cso_cfg* cfg, const cso_snapshot* snap, long max_steps,
               cso_run_out* out);
void cso_free_run(cso_run_out* out);

/* Engine-level primitives (EngineSim public surface + the start_request hot path). */
typedef struct cso_engine cso_engine;
cso_engine* cso_engine_new(const cso_cfg* cfg, long agent_cap);
void cso_engine_free(cso_engine* e);
/* EngineSim::lookup (engine.cpp:127-139) */
long cso_engine_lookup(cso_engine* e, const uint64_t* keys, const int32_t* counts, long n, long* first_miss);
/* AgentDispatch emitted through the engine clock (engine.cpp:280-281) */
int cso_engine_dispatch(cso_engine* e, uint64_t agent);
/* EngineSim::admit_pinned (engine.cpp:141-168); returns 0, or -1 when all blocks are pinned */
int cso_engine_admit_pinned(cso_engine* e, const uint64_t* keys, const int32_t* counts, long n,
                            int has_agent, uint64_t agent, int anchor_blocks);
int cso_engine_unpin(cso_engine* e, const uint64_t* keys, long n);
/* Pool snapshot restore: inserts resident blocks with explicit state (no eviction, no tick). */
int cso_engine_restore(cso_engine* e, const uint64_t* keys, const uint64_t* last_touch,
                       const int32_t* has_agent, const uint64_t* agents, const int32_t* refs, long n,
                       uint64_t tick);
long cso_engine_evictions(const cso_engine* e, uint64_t* out, long cap);
uint64_t cso_engine_tick(const cso_engine* e);
long cso_engine_resident(const cso_engine* e);
long cso_engine_pinned(const cso_engine* e);
/* poll_actions: drained warmup targets (issue order) */
long cso_engine_poll(cso_engine* e, uint64_t* targets, uint64_t* ticks, long cap);
/* ReachabilityState::hop for the listed agents (-1 before the first rebuild) */
int cso_engine_hops(const cso_engine* e, const uint64_t* agents, long n, int* hops);
/* CacheSagePolicy::score of every resident block at the engine's current context; rows are
 * (key, score) for resident blocks, in unspecified order. Returns count. */
long cso_engine_scores(const cso_engine* e, uint64_t* keys, double* scores, long cap);

#ifdef __cplusplus
}
#endif
#endif
