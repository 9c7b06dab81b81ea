// Host/device layout of the device-resident scheduler (cs_engine_dev.cuh): the trace, the
// catalog and the scheduler state the engine uploads once and the persistent kernel advances.
#pragma once

#include "cs_launch.h"

namespace csb {

constexpr int kMaxConc = 32;  // scheduler concurrency handled on device (host path above it)

struct EngReq {
    long long blk_off, prompt_tokens;
    int session, agent, nb, anchor_blocks, decode, pad;
};
struct EngCat {  // build_warmup_catalog entry by agent index (nb == 0: none)
    long long blk_off, prompt_tokens;
    int nb, pad;
};
struct EngFlight {
    double end_us, start_us;
    unsigned long long seq;
    long long req, cached;
    int npins, pad;
};

// The scheduler state (EngineSim::Scheduler, engine.hpp:158-168, and the engine's counters);
// lives in device memory between launches and in CTA 0's shared memory during one.
struct EngState {
    int conc, budget, prefetch, speculate, prescan, use_prescan, n_sessions;
    double cost_base, cost_tok, cost_dec;  // CostModel (engine.hpp:22-26)
    int active_sessions, next_session;
    int ready_head, ready_n;
    int ready[kMaxConc + 1];
    int n_flight;
    EngFlight flight[kMaxConc];
    unsigned long long flight_seq, tick, seq;
    double sim_now;
    int last_dispatched;
    long long completed, truncated, warm_exec, warm_drop, steps, admissions, tot_prompt, tot_cached, n_warm,
        warm_prompt;
    int poll_reset_pending;
    // the pool driver's bookkeeping (cs_pool::admit): deferred unpins, prescan reuse
    int n_unpin, unpin_slots;
    const unsigned int* unpin_ptr[kMaxUnpinRanges];
    int unpin_n[kMaxUnpinRanges];
    int n_prev, prev_slots, pre_ok;
    const unsigned int* prev_ptr[kMaxUnpinRanges + 1];
    int prev_n[kMaxUnpinRanges + 1];
    int error;  // 1 stall, 2 all pinned, 3 a warmup output overflow
    long long table_rebuilds;
    // coroutine position of the step in progress
    int phase, progressed, warm_i, n_fx, cur_req, cur_kind;
    int fx[kMaxPending];
    unsigned long long fx_tick[kMaxPending];
};

struct EngDev {
    EngState* st;
    const EngReq* reqs;
    const int* sess_off;   // sessions in ascending id order (std::map order), CSR of their turns
    const int* sess_reqs;
    int* session_pos;
    const EngCat* cat;
    const unsigned long long* keys;
    const int* counts;
    unsigned int* pins;
    const unsigned long long* agent_ids;
    long long* t_cached;
    long long* t_prompt;
    double* t_start;
    double* t_end;
    unsigned char* t_done;
    double* t_arrival;
    long long* w_step;
    unsigned long long* w_target;
    unsigned long long* w_tick;
    long long w_cap;
    AdmitArgs* args;  // the admission every CTA runs next
    int* cmd;         // 0 admit, 1 stop, 2 table rebuild
};


cudaError_t launch_engine(const DevPool& P, const EngDev& E, long long stop_at, long long max_steps, int n_agents,
                          const LaunchCfg& lc, cudaStream_t s);

}  // namespace csb
