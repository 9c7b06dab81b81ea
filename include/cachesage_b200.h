/* cachesage_b200 — C ABI of the B200-native CacheSage per-step cache-policy hot path.
 *
 * The reference (/root/reference/proj, single-threaded C++20) runs the per-step loop
 *   observe -> score -> select -> act
 * inside EngineSim + CacheSagePolicy. This library keeps that behaviour bit-exact while the
 * block pool, the block table, the transition learner, the reachability classes, the scoring
 * scan and the k-victim select all live in HBM and run as sm_100a kernels. Plain pointers and
 * sizes only; no torch types. Every call returns 0 on success or a negative cs_status; the
 * message is in cs_last_error(). Handles are single-writer (SURVEY.md §8b "Threading").
 *
 * Each entry point names the reference interface it replaces (paths relative to
 * /root/reference/proj). INTEGRATION.md shows the binding a reference maintainer would add.
 */
#ifndef CACHESAGE_B200_H
#define CACHESAGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum cs_status {
    CS_OK = 0,
    CS_ERR_INVALID_ARGUMENT = -1, /* reference: std::invalid_argument */
    CS_ERR_RUNTIME = -2,          /* reference: std::runtime_error (all pinned, stall, tick regression) */
    CS_ERR_LOGIC = -3,            /* reference: std::logic_error (budget / vanished block) */
    CS_ERR_CUDA = -4,             /* CUDA failure or no device: there is NO CPU fallback */
    CS_ERR_CAPACITY = -5          /* a fixed device capacity (agents, prompt length) exceeded */
} cs_status;

typedef struct cs_pool* cs_pool_t;
typedef struct cs_engine* cs_engine_t;

#define CS_NO_AGENT 0xFFFFFFFFu

/* Policy and pool configuration: EngineConfig (engine.hpp:29-36) + CacheSageConfig
 * (cachesage_policy.hpp:36-43). policy: 0 = lru (baselines.cpp:12-14), 1 = cachesage,
 * 2 = ttl (baselines.cpp:22-28, default pin horizon: the same victims as lru, see cs_pool.cpp;
 * cs_score_snapshot reports the recency part only), 3 = belady (baselines.cpp:34-70: needs the
 * request stream, so only engines run it — cs_engine_create*; admissions on a bare pool fail
 * with CS_ERR_INVALID_ARGUMENT; not with a hash-sharded pool). */
typedef struct cs_pool_cfg {
    int64_t budget_blocks; /* pool slots N (EngineConfig::budget_blocks) */
    int policy;
    int e_max;         /* ReachabilityState::e_max, <= 22 */
    double tau;        /* edge threshold */
    double w_pred;     /* score = w_pred * survival + recency */
    int64_t window;    /* TransitionLearner window W */
    double min_confidence;
    uint64_t min_row_count;
    int budget_per_step;
    int agent_capacity; /* max distinct agents (dense A x A counts), <= 4096 */
    int device;         /* CUDA device ordinal */
    int grid_ctas;      /* 0 = one CTA per SM (cooperative scan grid) */
} cs_pool_cfg;

void cs_pool_cfg_default(cs_pool_cfg* cfg);

/* Creates the device pool: SoA slots (last_touch u64, agent u32, refs u32, key u64), the
 * open-addressing block table, the learner and the scan scratch.
 * Replaces: EngineSim::cache_ / pinned_count_ (engine.hpp:176-177), the CacheSagePolicy
 * constructor (cachesage_policy.cpp:33-48) and TransitionLearner (transition_learner.hpp:19). */
int cs_pool_create(const cs_pool_cfg* cfg, cs_pool_t* out);
int cs_pool_destroy(cs_pool_t pool);

/* Declares agent identities in dense-index order (index = position). The learner's alphabet
 * (TransitionLearner::note_agent, transition_learner.cpp:16-20); argmax ties break on these
 * 64-bit ids (transition_learner.cpp:89). Appends; returns the first new index in *first. */
int cs_register_agents(cs_pool_t pool, const uint64_t* agent_ids, int n, int* first);

/* K1: chained block hashing + agent identity for n prompts (host buffers in and out).
 * tokens: all prompts concatenated; tok_off[n+1] prefix offsets; blk_off[n+1] must equal the
 * prefix sums of ceil(len/block_size) (cs_blocks_for computes it). Replaces block_keys_for
 * (hashing.cpp:37-51), chain_hash (hashing.cpp:26-35), derive_agent_identity
 * (cachesage_policy.cpp:9-31). Empty prompts are invalid_argument (chain_hash :27-29). */
int cs_hash_prompts(cs_pool_t pool, const uint32_t* tokens, const int64_t* tok_off, int n_prompts,
                    int block_size, int skip, int take, const int64_t* blk_off, uint64_t* keys_out,
                    int32_t* counts_out, uint64_t* agent_ids_out);
int64_t cs_blocks_for(const int64_t* tok_off, int n_prompts, int block_size, int64_t* blk_off);

/* chain_hash (hashing.cpp:26-35) of n token spans (tok_off[n+1]); has_parent[i] != 0 chains
 * from parents[i], else from the root (both may be NULL). The reference's Python chain_hash. */
int cs_chain_hash(const uint64_t* parents, const uint8_t* has_parent, const uint32_t* tokens, const int64_t* tok_off,
                  int n, uint64_t* out);
/* derive_agent_identity (cachesage_policy.cpp:9-31) of n block-key lists (key_off[n+1]). */
int cs_derive_agent_identity(const uint64_t* keys, const int64_t* key_off, int n, int skip, int take, uint64_t* out);

/* K2: EngineSim::lookup (engine.cpp:127-139): longest resident prefix; each hit is touched
 * with ticks tick_base+1, tick_base+2, ... The caller's clock advances by *first_miss. */
int cs_lookup(cs_pool_t pool, const uint64_t* keys, const int32_t* counts, int n, uint64_t tick_base,
              int64_t* cached_tokens, int* first_miss);

/* K2: the try_start_head feasibility probe (engine.cpp:337-346): number of prompt blocks that
 * are not resident or not pinned. */
int cs_probe_needed(cs_pool_t pool, const uint64_t* keys, int n, int* needed);

/* K3+K3b+K6: CacheSagePolicy::observe(AgentDispatch) (cachesage_policy.cpp:57-72): learner
 * record (transition_learner.cpp:22-51), reachability rebuild on agent change
 * (reachability.cpp:39-81), prefetch gate (cachesage_policy.cpp:109-123). prev < 0 = none.
 * *warmup_target = agent index of an issued warmup or -1. */
int cs_observe_dispatch(cs_pool_t pool, int prev, int next, uint64_t tick, int* warmup_target);

/* K4+K5: EngineSim::admit_pinned (engine.cpp:141-168) with the full eviction semantics of
 * evict_one (engine.cpp:102-125) + CacheSagePolicy::score (cachesage_policy.cpp:79-85):
 * makes all n blocks resident and pinned, touching block i at tick_base+1+i; new blocks carry
 * agent `agent` iff i < anchor_blocks. Victim keys in eviction order -> evicted (cap entries),
 * count -> *n_evicted; pinned slot per block -> pins (may be NULL).
 * CS_ERR_RUNTIME = "evict_one: all resident blocks are pinned". */
int cs_admit_pinned(cs_pool_t pool, const uint64_t* keys, const int32_t* counts, int n, uint32_t agent,
                    int anchor_blocks, uint64_t tick_base, uint64_t* evicted, int64_t cap,
                    int64_t* n_evicted, uint32_t* pins);

/* EngineSim::unpin (engine.cpp:170-180): one pin released per key, in order (flight.pins are
 * the BlockKeys admit_pinned returned, engine.hpp:144-152). A key that is not resident (or holds
 * no pin) is CS_ERR_LOGIC "unpin: block vanished while referenced" after the keys before it were
 * unpinned, as the reference throws mid-loop. */
int cs_unpin(cs_pool_t pool, const uint64_t* keys, int n);
/* The same by pinned slot (as cs_admit_pinned returns them): no table probe. */
int cs_unpin_slots(cs_pool_t pool, const uint32_t* slots, int n);

/* Event kinds of the observe stream (types.hpp:51-82). */
typedef enum cs_event_kind {
    CS_EV_BLOCK_TOUCH = 0,     /* BlockTouch{key, agent}: ignored by every policy's observe */
    CS_EV_REQUEST_ARRIVAL = 1, /* RequestArrival{request, agent}: note_agent; Belady's cursor */
    CS_EV_AGENT_DISPATCH = 2,  /* AgentDispatch{prev, next}: the full observe (cs_observe_dispatch) */
    CS_EV_TOOL_RETURN = 3,     /* ToolReturn{agent}: note_agent */
    CS_EV_TURN_COMPLETE = 4    /* TurnComplete{request}: ignored */
} cs_event_kind;

typedef struct cs_event {
    uint64_t tick;    /* Event::tick: nondecreasing over the stream */
    int kind;         /* cs_event_kind */
    int agent;        /* arrival / tool-return agent, dispatch `next` (dense agent index) */
    int prev;         /* dispatch `prev` (-1 = std::nullopt) */
    uint64_t request; /* arrival / turn-complete RequestId */
} cs_event;

/* Runtime::dispatch_event (runtime.cpp:59-69) -> Policy::observe (cachesage_policy.cpp:50-77):
 * CS_ERR_RUNTIME "dispatch_event: tick regression" when ev->tick is below the last event's tick
 * (equal ticks allowed). *warmup_target = agent index of a warmup this dispatch issued, or -1. */
int cs_dispatch_event(cs_pool_t pool, const cs_event* ev, int* warmup_target);

/* CacheSagePolicy::predict(horizon) (current < 0: the policy's current agent) and
 * predict_next(current, horizon) (cachesage_policy.cpp:87-107): the full MLE row, count / row
 * total in fp64. The entries come ranked for prefetch: descending probability, ties to the
 * smaller AgentId (argmax_row's order, transition_learner.cpp:79-96), so entry 0 is the
 * warmup candidate maybe_prefetch gates. ids / probs / idx (dense agent index) may be NULL;
 * *n = the row's support (an empty Forecast: 0). Baseline policies forecast nothing. */
int cs_predict(cs_pool_t pool, int horizon, int current, uint64_t* ids, double* probs, int* idx, int cap, int* n);

/* Policy::serialize_state().dump() (cachesage_policy.cpp:139-153; baselines.cpp:16, 30-32,
 * 72-74): the documented JSON shape, byte-identical to the reference's for the same observe
 * stream. *len = bytes (without the NUL); buf gets min(cap - 1, len) bytes + NUL (may be NULL). */
int cs_serialize_state(cs_pool_t pool, char* buf, size_t cap, size_t* len);
/* CacheSagePolicy::state_bytes (cachesage_policy.cpp:133-138). */
int cs_policy_state_bytes(cs_pool_t pool, uint64_t* bytes);

/* Pool snapshot restore (stress inputs): resident blocks with explicit
 * last_touch / agent index (CS_NO_AGENT = none) / refs. Keys must be new and distinct. */
int cs_restore(cs_pool_t pool, const uint64_t* keys, const uint64_t* last_touch, const uint32_t* agents,
               const uint32_t* refs, int64_t n);

/* CacheSagePolicy::score (cachesage_policy.cpp:79-85) of every resident block at context
 * (now_tick, oldest_live_touch over the pool): rows (key, score), *n = resident count. */
int cs_score_snapshot(cs_pool_t pool, uint64_t now_tick, uint64_t* keys, double* scores, int64_t cap,
                      int64_t* n);

/* ReachabilityState::hop per agent index (-1 before the first rebuild). */
int cs_hops(cs_pool_t pool, int* hops, int n);
/* Installs reachability hops computed elsewhere (e.g. cs_learner_rebuild, or an external
 * learner): hop per agent index, survival class min(hop, e_max) (reachability.cpp:12-20); the
 * pool scores with them until its own observe rebuilds. SURVEY §8b cs_set_hops. */
int cs_set_hops(cs_pool_t pool, const uint8_t* hops, int n);

/* CacheSagePolicy::poll_actions (cachesage_policy.cpp:125-130): drains queued warmups
 * (agent indices, issue ticks) and resets the per-step budget. */
int cs_poll_actions(cs_pool_t pool, int* targets, uint64_t* ticks, int cap, int* n);

typedef struct cs_pool_stats {
    int64_t resident, pinned, evictions, tombstones, scans, scanned_slots;
    uint64_t rebuilds;
    int n_agents;
    /* device time per admission-kernel phase summed over launches (globaltimer ns, CTA 0):
     * probe/observe/lookup, prep+barrier, scan+barrier, select+barrier, replay+apply, epilogue */
    uint64_t phase_ns[16];
    /* admissions whose chunk 0 used the previous launch's prescan / fell back to a scan;
     * prescans that overflowed (unusable) */
    int64_t prescan_used, prescan_fallbacks, prescan_unusable;
    /* admission server: launches, and the host's turnaround (status seen -> next admission
     * posted) summed over the admissions that followed another one in the same launch */
    int64_t server_launches, host_turnarounds;
    uint64_t host_turnaround_ns;
} cs_pool_stats;
int cs_pool_get_stats(cs_pool_t pool, cs_pool_stats* out);
/* Instrumentation: per-CTA scan timestamps of the last admission (grid x 8 u64). */
int cs_pool_debug(cs_pool_t pool, uint64_t* out, int cap, int* grid);
/* Pool invariants (tests): out[0] = slots whose packed scan word disagrees with the exact
 * last_touch / agent / pin state, out[1] = resident slots minus the pool's resident count,
 * out[2] = pinned slots minus its pinned count, out[3] = resident slots the block table does not
 * map back. All zero on a consistent pool. */
int cs_pool_check(cs_pool_t pool, int64_t* out4);

/* ------------------------------------------------------------------ engine (EngineSim) */

/* WorkloadSpec (workload.hpp:21-42); anchor_stride / hist_pos_bits widen the token scheme
 * (0 = the reference's 0x10000 / 20). supervisor = -2 with start_dist (n_agents weights) draws
 * each session's start agent (widened generator: mixed multi-generator traces). */
typedef struct cs_workload_spec {
    int n_agents;
    const int* anchor_tokens;
    const double* transition;
    int supervisor;
    int turns_min, turns_max, sessions, task_tokens, history_growth, decode_tokens;
    int template_tokens, concurrency, budget_blocks;
    uint64_t seed;
    uint32_t anchor_stride;
    int hist_pos_bits;
    const double* start_dist;
} cs_workload_spec;

/* Generates the trace (generate_trace, workload.cpp:156-182) on the host: turns7 rows
 * (session, turn_index, agent, anchor_tokens, history_tokens, prompt_tokens, decode_tokens).
 * Returns the turn count (pass cap 0 to size). */
int64_t cs_generate_trace(const cs_workload_spec* spec, int64_t* turns7, int64_t cap);

typedef struct cs_engine_cfg {
    cs_pool_cfg pool; /* pool.budget_blocks <= 0: the spec's pairing */
    int concurrency;  /* <= 0: the spec's pairing */
    int block_size;
    int prefetch;     /* EngineConfig::prefetch_enabled */
    int skip, take;   /* IdentityConfig */
    int timing;       /* record CUDA events around each admission launch */
    int host_inputs;  /* 1: prompt blocks live in pinned host memory and are copied H2D per
                         admission, victims copied D2H per admission (the end-to-end path) */
    int device_scheduler; /* 1: EXPERIMENTAL device-resident scheduler: whole
                             EngineSim steps in one persistent launch; see DESIGN.md §4 */
    /* CostModel (engine.hpp:22-26; experiment.cpp:270-280 reads it from the cell config): ttft =
     * prefill_base_us + prefill_per_token_us * uncached tokens, decode = decode_per_token_us per
     * token. They set completion order, hence unpin order, hence the victims. All must be > 0
     * (engine.cpp:60-63); cs_engine_cfg_default sets 50 / 1000 / 20000. */
    double prefill_per_token_us, prefill_base_us, decode_per_token_us;
} cs_engine_cfg;

void cs_engine_cfg_default(cs_engine_cfg* cfg);

/* EngineSim (engine.hpp:90-208) with the pool on the device: run_cell wiring
 * (experiment.cpp:355-379) = materialize_requests (engine.cpp:8-35, hashed on the GPU by K1),
 * build_warmup_catalog (:37-54), load, step until done. */
int cs_engine_create(const cs_engine_cfg* cfg, const cs_workload_spec* spec, cs_engine_t* out);
int cs_engine_destroy(cs_engine_t e);
int cs_engine_step(cs_engine_t e, int* done); /* EngineSim::step (engine.cpp:372-392) */
int cs_engine_run(cs_engine_t e);             /* step until done */
/* Runs at most max_admissions more admissions (whole steps), for bounded timing windows. */
int cs_engine_run_for(cs_engine_t e, int64_t max_admissions, int* done);
/* Same, bracketed by CUDA events on the engine's stream: *device_ms = elapsed device time. */
int cs_engine_run_timed(cs_engine_t e, int64_t max_admissions, double* device_ms, int* done);
/* Restores a pool snapshot into the engine (cs_restore) and advances the engine clock past
 * the snapshot's last_touch values. Agent indices refer to the engine's agent order
 * (cs_engine_agents). */
int cs_engine_restore(cs_engine_t e, const uint64_t* keys, const uint64_t* last_touch, const uint32_t* agents,
                      const uint32_t* refs, int64_t n);
/* The engine's dense agent index -> AgentId table; returns the count. */
int cs_engine_agents(cs_engine_t e, uint64_t* ids, int cap);

typedef struct cs_engine_result {
    int64_t turns, completed;
    double hit_rate;
    int64_t total_prompt_tokens, total_cached_tokens;
    int64_t evictions, truncated, warmups_executed, warmups_dropped, warmups_issued;
    double sim_us;
    int64_t steps, admissions, scans, scanned_slots;
    uint64_t tick;
    double scan_ms, admit_ms; /* CUDA-event time of scan passes / whole admissions (timing=1) */
    int64_t scan_launches;    /* admission launches that ran at least one scan pass */
    int64_t h2d_bytes, d2h_bytes; /* host<->device bytes moved by admissions (host_inputs=1) */
    int64_t gpu_launches;         /* kernels launched by the engine so far */
    int64_t warmup_prompt_tokens; /* EngineSim::warmup_prompt_tokens_ (engine.cpp:222) */
} cs_engine_result;
int cs_engine_result_get(cs_engine_t e, cs_engine_result* out);
/* An engine over an explicit trace (turns7 rows as cs_generate_trace writes them, e.g. a trace
 * read back from JSONL, trace_io.cpp:87-136); the spec supplies agents, template, budget and
 * concurrency. run_cell (experiment.cpp:355-379) for a given Trace. */
int cs_engine_create_from_turns(const cs_engine_cfg* cfg, const cs_workload_spec* spec, const int64_t* turns7,
                                int64_t n_turns, cs_engine_t* out);
/* per-turn arrival time (simulated us), TurnMetrics::arrival_us (engine.cpp:316) */
int cs_engine_turn_arrivals(cs_engine_t e, double* arrival_us, int64_t cap);
/* per-turn (by turn id) cached/prompt tokens and start/end simulated us; any may be NULL */
int cs_engine_turns(cs_engine_t e, int64_t* cached, int64_t* prompt, double* start_us, double* end_us,
                    int64_t cap);
int64_t cs_engine_evictions(cs_engine_t e, uint64_t* keys, int64_t cap);
/* drained warmups: step index, target agent id, issued tick */
int64_t cs_engine_warmups(cs_engine_t e, int64_t* step, uint64_t* target, uint64_t* tick, int64_t cap);
cs_pool_t cs_engine_pool(cs_engine_t e);

/* Output writers: run_experiment's per-cell files (experiment.cpp:94-183,
 * 424-440), byte-identical to the reference's for the same cell:
 *   <dir>/metrics.json  metrics_to_json(...).dump(2)
 *   <dir>/turns.csv     write_turns_csv
 *   <dir>/events.jsonl  write_events_jsonl (write_events = 1; needs cs_engine_record_events)
 * workload / policy / seed / labels are the cell's names as run_experiment reports them (the
 * workload display name, the policy name, the trace seed, the workload's agent labels in spec
 * order). The run must be finished. */
int cs_engine_record_events(cs_engine_t e, int on); /* before the first step; host scheduler only */
int cs_engine_write_outputs(cs_engine_t e, const char* dir, const char* workload, const char* policy, uint64_t seed,
                            const char* const* labels, int n_labels, int write_events);

/* ------------------------------------------------------------------ standalone learner
 *
 * The reference's TransitionLearner (transition_learner.hpp:19-60; Python binding
 * py_module.cpp:103-123) on the device: dense counts over agent indices in first-seen order,
 * the window as an index-pair ring. record = K3 (warp-aggregated atomics), rebuild = K3b,
 * argmax = K6, and the horizon-k survival oracle (a21). */
typedef struct cs_learner* cs_learner_t;
int cs_learner_create(int64_t window, int agent_capacity, int device, cs_learner_t* out);
int cs_learner_destroy(cs_learner_t learner);
/* TransitionLearner::record (transition_learner.cpp:22-51) for n pairs, in order. */
int cs_learner_record(cs_learner_t learner, const uint64_t* prev, const uint64_t* next, int64_t n);
/* TransitionLearner::prob / row_total (transition_learner.cpp:53-71). */
int cs_learner_prob(cs_learner_t learner, uint64_t a, uint64_t b, double* p);
int cs_learner_row_total(cs_learner_t learner, uint64_t a, uint64_t* total);
/* TransitionLearner::agents (first-seen order); returns the count. */
int cs_learner_agents(cs_learner_t learner, uint64_t* ids, int cap);
/* TransitionLearner::state_bytes (transition_learner.cpp:98-106). */
int cs_learner_state_bytes(cs_learner_t learner, uint64_t* bytes);
/* rebuild_reachability (reachability.cpp:39-81): hop of every known agent (agents() order). */
int cs_learner_rebuild(cs_learner_t learner, uint64_t current, double tau, int e_max, int* hops, int cap);
/* TransitionLearner::argmax_row (transition_learner.cpp:79-96); *found = 0 for an unseen row. */
int cs_learner_argmax(cs_learner_t learner, uint64_t a, uint64_t* best, double* p, int* found);
/* oracle::exact_survival_prob (survival_oracle.cpp:9-62): P(the walk from current visits
 * target within k steps), same fp64 operation order. Alphabet <= 64, 0 <= k <= 32. */
int cs_exact_survival_prob(cs_learner_t learner, uint64_t target, int k, uint64_t current, double* out);

/* ------------------------------------------------------------------ hash-sharded pool
 *
 * one pool of GLOBAL budget N split over G <= 8 GPUs, block key k on shard
 * (k >> 40) % G. Each shard scans and k-selects its own slots; per admission the shards
 * exchange (allgather) their probe results and, per chunk that can evict, their per-class
 * candidate lists, and every shard then runs the same exact evict_one replay. Every shard
 * returns the decisions one pool of budget N makes: the same hits, victims (in order) and
 * warmups. The reference has no sharding; the replay is EngineSim::admit_pinned /
 * evict_one (engine.cpp:102-168) over the union of the shard candidates. */
typedef struct cs_comm* cs_comm_t;

/* Host allgather for the callback transport: recv[r * bytes .. ) = rank r's send. 0 = ok. */
typedef int (*cs_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes_per_rank);

/* world handles for world shards driven by world threads of this process (device-to-device
 * copies between the shards' buffers; the shards may share one device). */
int cs_comm_local_group(int world, cs_comm_t* comms_out);
/* Exchange through host memory and a caller-supplied allgather (e.g. torch.distributed). */
int cs_comm_callback(int rank, int world, cs_allgather_fn fn, void* ctx, cs_comm_t* out);
/* NCCL (ncclAllGather over NVLink / NVSwitch), one process per GPU. Rank 0 creates the id and
 * the caller broadcasts its 128 bytes; libnccl.so.2 is loaded at run time (CS_NCCL_LIB). */
int cs_nccl_unique_id(uint8_t* id128);
int cs_comm_nccl(const uint8_t* id128, int rank, int world, int device, cs_comm_t* out);
/* Peer memory (the fused exchange): a sharded engine's admission kernels store each shard's
 * contribution straight into every peer's window over NVLink / NVSwitch and wait on the peers'
 * flags themselves (no exchange kernel, no NCCL, no host round trip; CS_PEER_UNFUSED=1 exchanges
 * between kernels instead). cap: the largest exchange in bytes per rank (the shard lists in use
 * are <= 74,400 B; 262,144 fits prompts of up to 32,766 blocks).
 *   cs_comm_peer_group   world shards of this process (devices[r], NULL = all on device 0);
 *                        peer access is enabled between distinct devices.
 *   cs_comm_peer_create  one shard per process: returns this rank's 128-byte handle (CUDA IPC
 *                        handles of its window and flags); the caller allgathers the handles
 *                        (rank order) and passes all world * 128 bytes to cs_comm_peer_connect. */
int cs_comm_peer_group(int world, const int* devices, size_t cap, cs_comm_t* comms_out);
int cs_comm_peer_create(int rank, int world, int device, size_t cap, uint8_t* handle128_out, cs_comm_t* out);
int cs_comm_peer_connect(cs_comm_t comm, const uint8_t* handles);
/* One exchange from host buffers (tests, diagnostics): recv[r * bytes ..) = rank r's send. */
int cs_comm_allgather_host(cs_comm_t comm, const void* send, void* recv, size_t bytes);
int cs_comm_destroy(cs_comm_t comm);
/* The shard that owns a block key. */
int cs_shard_owner(uint64_t key, int world);

/* A shard of a sharded pool: cfg->budget_blocks is the GLOBAL budget N; shard_slots the
 * shard's physical slot count (0 = 1.25 N / world + 4096). The comm is borrowed. */
int cs_pool_create_sharded(const cs_pool_cfg* cfg, int64_t shard_slots, cs_comm_t comm, cs_pool_t* out);
/* The EngineSim of one shard: every shard runs the same trace and scheduler; cs_engine_restore
 * keeps only the snapshot blocks this shard owns. */
int cs_engine_create_sharded(const cs_engine_cfg* cfg, const cs_workload_spec* spec, int64_t shard_slots,
                             cs_comm_t comm, cs_engine_t* out);

const char* cs_last_error(void);
/* Diagnostics: the last device watchdog that fired, (site << 32) | CTA, or 0. */
uint64_t cs_debug_trap_word(void);
const char* cs_version(void);

#ifdef __cplusplus
}
#endif
#endif
