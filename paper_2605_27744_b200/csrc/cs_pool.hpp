// Host-side owner of one device block pool (the cs_pool_t handle) and the admission driver.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cachesage_b200.h"
#include "cs_comm.hpp"
#include "cs_launch.h"

namespace csb {

struct CsError : std::runtime_error {
    int code;
    CsError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CsError(CS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    void ensure(size_t bytes) {
        if (bytes <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        ck(cudaMalloc(&p, bytes < 256 ? 256 : bytes), "cudaMalloc(scratch)");
        n = bytes < 256 ? 256 : bytes;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct AdmitResult {
    AdmitStatus st;
    std::vector<unsigned long long> victims;  // filled only when requested
};

}  // namespace csb

struct cs_pool {
    cs_pool_cfg cfg{};
    int device = 0;
    csb::DevPool P{};
    cudaStream_t stream = nullptr;
    csb::LaunchCfg lc{};
    csb::AdmitStatus* st = nullptr;      // host-mapped status
    csb::AdmitStatus* st_dev = nullptr;
    int n_agents = 0;
    std::vector<uint64_t> agent_ids;
    bool poll_reset_pending = false;
    long long resident = 0, pinned = 0;  // mirrors of the last status
    unsigned long long ev_total = 0;     // evictions logged so far
    unsigned long long ev_safe = 0;      // ... of which surely in the log (all but the last admission's)
    std::vector<int> pending_targets;
    std::vector<unsigned long long> pending_ticks;
    // Host mirror of what the reference keeps outside the counts (cs_state.cpp):
    // Runtime::last_tick_ (runtime.cpp:59-64), TransitionLearner::alphabet_ in note_agent order
    // (transition_learner.cpp:16-20), |ReachabilityState::hops| of the last rebuild
    // (reachability.cpp:48-51: every agent known then), BeladyPolicy::cursor_.
    bool has_last_tick = false;
    unsigned long long last_tick = 0;
    std::vector<int> alphabet;
    std::vector<unsigned char> noted;
    size_t reach_known = 0;
    int host_cur = -1;
    unsigned long long bel_cursor = 0;
    bool mirror_ok = true;  // false once a device-resident scheduler observes events on the device
    void note_agent(int a);
    // AgentDispatch{prev, next} as CacheSagePolicy::observe notes it (cachesage_policy.cpp:57-66)
    void note_dispatch(int prev, int next);
    // Runtime::dispatch_event's tick check (runtime.cpp:59-64): CS_ERR_RUNTIME on a regression
    void check_tick(unsigned long long tick);
    // scratch
    csb::DevBuf d_keys, d_counts, d_pins, d_aux, d_aux2, d_aux3;
    // timing (CUDA events around each admission launch)
    bool timing = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // per-admission timing without a sync: event pairs resolved once they complete
    struct TimedLaunch {
        cudaEvent_t e0, e1;
        bool scan;
    };
    std::vector<TimedLaunch> t_pending;
    std::vector<cudaEvent_t> t_free;
    cudaEvent_t take_event();
    void resolve_timing(bool wait);
    // waits for this launch's status (AdmitStatus::done_seq), not for the kernel's end
    void wait_status(unsigned long long seq, const char* what);
    // engine loop only: admit() returns at the status flag, not at the kernel's end (every
    // public pool entry point syncs first)
    bool early_status = false;
    double admit_ms = 0.0, scan_launch_ms = 0.0;
    long long admit_launches = 0, scan_launches = 0, scans_total = 0, table_rebuilds = 0;
    long long launches = 0;  // every kernel this handle launched (the bench's gpu_launches)
    unsigned long long phase_ns[csb::kPhases] = {};
    unsigned long long seq = 0;  // admission launch sequence (AdmitArgs::seq)
    bool speculate = true;       // overlap the first scan pass with phase 0 when it can evict
    // prescan: every cooperative launch streams the pool for the NEXT admission (kPrescan); the
    // next launch may use those lists (kUsePrescan) unless the pool changed out of band since
    bool prescan = true;
    // the next admission's victims land here (pinned) by a D2H copy queued behind the kernel:
    // vpref_n log entries from the pre-admission log end; vpref_done = entries copied
    unsigned long long* vpref = nullptr;
    int vpref_n = 0, vpref_done = 0;
    bool pre_ok = false;
    std::vector<std::pair<const unsigned int*, int>> prev_ranges;  // slots the last launch unpinned
    int prev_slots = 0;
    // deferred EngineSim::unpin calls (device slot lists), folded into the next admission launch
    std::vector<std::pair<const unsigned int*, int>> unpin_q;
    int unpin_q_slots = 0;

    // hash-sharded mode: this pool is one shard; comm is borrowed
    cs_comm* comm = nullptr;
    csb::ShardState* hstate = nullptr;  // pinned host copy of the replicated admission state

    // Belady (policy 3): launch shape and the next-use index over the request stream
    csb::LaunchCfg blc{};
    long long bel_kids = -1;  // unique keys of the installed index (-1: none)
    // Builds the index from the request blocks keys[0, n_flat) (device) with request offsets
    // blk_off[0, n_req] (host); kid_of() then gives every request block's key index.
    void belady_index(const unsigned long long* keys, long long n_flat, const std::vector<long long>& blk_off);
    const unsigned int* bel_kid_of() const { return P.bel_kid_of; }
    const csb::AdmitStatus& admit_belady(const csb::AdmitArgs& args_in, int n_for_grid);

    // shard_slots > 0 or comm: one shard of a pool of global budget c.budget_blocks
    void create(const cs_pool_cfg& c, long long shard_slots = 0, cs_comm* comm = nullptr);
    const csb::AdmitStatus& admit_sharded(const csb::AdmitArgs& args_in);
    const csb::AdmitStatus& admit_sharded_once(const csb::AdmitArgs& args_in);
    void fetch_state();
    // every shard's value of v (sharded pools; {v} otherwise)
    std::vector<unsigned long long> allgather_u64(unsigned long long v);
    void destroy();
    void ensure_prompt_scratch(long long n);
    // Runs one admission launch and waits for it. grid_hint: 0 = decide (1 CTA when no eviction
    // is possible, else the cooperative grid).
    const csb::AdmitStatus& admit(const csb::AdmitArgs& args_in, int n_for_grid);
    void copy_victims(unsigned long long from, unsigned long long to, unsigned long long* host_out);
    // Queues an unpin of device-resident slots; it runs at the start of the next admission
    // launch (or in flush_unpins, before any other pool operation reads pins).
    void defer_unpin(const unsigned int* dev_slots, int n);
    void flush_unpins();
    // Applies queued block-table updates (admissions defer them to the next launch's phase 0).
    void flush_table();
    void sync() {
        server_stop();  // (the admission server occupies the stream until it is told to stop)
        csb::ck(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
        resolve_timing(true);
    }

    // Admission server (csb::server_kernel): inside an engine loop (early_status) every admission
    // is posted to ONE persistent cooperative launch through a host-mapped mailbox instead of
    // launching admit_kernel. Anything else that needs the stream stops it first (sync(),
    // flush_unpins, the table rebuild); the next admission starts it again.
    bool server = true;           // use the server where it applies (A/B switch: CS_SERVER=0)
    bool server_generic = false;  // stream the pool with L2 loads instead of TMA in the server
    bool srv_running = false;
    csb::SrvMailbox* mb = nullptr;      // pinned, mapped
    csb::SrvMailbox* mb_dev = nullptr;
    csb::AdmitArgs* d_srv_args = nullptr;
    csb::DevPool srv_P{};
    long long server_launches = 0;
    unsigned long long srv_post = 0;  // mailbox posts so far (admissions and stops)
    long long host_turnarounds = 0;   // instrumentation: status seen -> next post, on the host
    unsigned long long host_turnaround_ns = 0;
    bool srv_status_seen = false;
    std::chrono::steady_clock::time_point srv_status_t;
    // per-admission device time from the server's pickup stamps: admission k's time is the
    // interval to admission k+1's pickup (the host's turnaround included)
    bool srv_have_t0 = false, srv_last_scan = false;
    unsigned long long srv_last_t0 = 0;
    bool uses_server() const { return server && early_status && !comm && P.policy != 3 && lc.grid > csb::kStream0; }
    void server_post(const csb::AdmitArgs& a);
    void server_start();
    void server_stop();
    void server_account(unsigned long long t_next);
    unsigned long long* trap_word_host = nullptr;  // the device watchdogs' last trap site
    void ck_trap(cudaError_t e, const char* what);   // ck() that names a watchdog's site
};
