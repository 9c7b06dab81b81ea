// Host-visible launch surface of the sm_100a kernels (implemented in cs_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "cs_device.cuh"

namespace csb {

enum AdmitFlags : int {
    kDispatch = 1,     // emit AgentDispatch{prev, next} through the policy first
    kLookup = 2,       // EngineSim::lookup over all n blocks before admitting
    kFeasible = 4,     // try_start_head feasibility probe; not started when it fails
    kTruncate = 8,     // oversized prompt: admit budget - pinned blocks, no lookup
    kWarmupRoom = 16,  // execute_warmup: admit min(n, budget - pinned) blocks
    kUnpinAfter = 32,  // EngineSim::admit: unpin immediately
    kPollReset = 64,   // a poll_actions drain happened before this call
    kAdmit = 128,      // run admit_pinned at all (lookup-only / observe-only calls clear it)
    kSpeculate = 256,  // scan chunk 0 concurrently with phase 0 (cooperative grid only)
    kPrescan = 512,    // CTAs 1.. run the NEXT admission's scoring pass in this launch
    kUsePrescan = 1024, // chunk 0 may use the lists the previous launch's prescan produced
    kSrvStop = 2048     // admission server (server_kernel): the host's stop command, no admission
};

constexpr int kMaxUnpinRanges = 8;  // deferred EngineSim::unpin calls folded into one launch
constexpr int kXset = 1024;         // slots phase 0 may change (prompt + unpinned), hashed per CTA
constexpr int kXsetMax = kXset / 2; // speculation only below half load

struct AdmitStatus {
    int started;
    int error;
    int first_miss;
    int admit_n;
    long long cached;
    long long n_evicted;
    long long resident;
    long long pinned;
    unsigned long long tick_after;
    unsigned long long ev_total;
    int n_pend;
    int warm_issued;
    int scans;
    int needed;
    long long tombstones;
    // CTA-0 view of the phase boundaries (%globaltimer ns), summed over chunks:
    // [0] phase 0 (probe/dispatch/lookup)  [1] prep + barrier  [2] scan + barrier
    // [3] finalize + barrier  [4] replay + apply  [5] epilogue
    // [6] replay setup [7] replay loop [8] apply [9] scan flushes (CTA 0) [10] flush count
    unsigned long long phase_ns[kPhases];
    int pend_target[kMaxPending];
    unsigned long long pend_tick[kMaxPending];
    // AdmitArgs::seq once every field above (and AdmitArgs::vict_host) is written: CTA 0 sets
    // it behind a system-scope fence, so the host continues while the prescan CTAs finish
    unsigned long long done_seq;
    // admission server: %globaltimer when CTA 0 picked this admission (or the stop) up
    unsigned long long srv_t0;
};

struct AdmitArgs {
    const unsigned long long* keys;
    const int* counts;
    int n;
    int flags;
    int prev, next;
    unsigned int agent;
    int anchor;  // < 0: all admitted blocks carry the agent
    unsigned long long tick_base;
    int n_agents;
    unsigned int* pins_out;
    AdmitStatus* status;  // host-mapped
    unsigned long long seq;  // launch sequence number (phase-0 completion flag)
    // EngineSim::unpin (engine.cpp:170-180) of completed requests, applied first in phase 0
    const unsigned int* unpin_ptr[kMaxUnpinRanges];
    int unpin_n[kMaxUnpinRanges];
    int n_unpin_ranges;
    // slots the PREVIOUS launch unpinned (its deferred unpins and, after a warmup, its own
    // pins): with this launch's unpins, the only slots whose membership of a list can grow
    // between the previous launch's prescan and this launch (kUsePrescan)
    const unsigned int* prev_ptr[kMaxUnpinRanges + 1];
    int prev_n[kMaxUnpinRanges + 1];
    int n_prev_ranges;
    // Belady (policy 3): the prompt blocks' key indices, BeladyPolicy::cursor_ (the highest
    // request id arrived so far) and the request blocks [adv_lo, adv_hi) whose next use the
    // cursor passed since the previous admission launch
    const unsigned int* kids;
    unsigned long long cursor;
    long long adv_lo, adv_hi;
    // recorded runs (events.jsonl): per looked-up prompt position < first_miss, the touched
    // block's agent index (BlockTouch{key, agent}, engine.cpp:79-88); null: not recorded
    unsigned int* touch_agent;
    // the end-to-end path: this admission's victim keys, written by CTA 0 straight into pinned
    // host memory (mapped) before done_seq; at most vict_cap
    unsigned long long* vict_host;
    int vict_cap;
    // the end-to-end path of the admission server: this admission's [keys (8 n) | counts (4 n)]
    // in pinned host memory; CTA 0 copies them into keys/counts (device) before phase 0
    const unsigned char* stage_src;
};

// The admission server's mailbox (server_kernel): pinned, host-mapped memory the host writes
// and CTA 0 polls. Every 8-byte word of the arguments travels in a 16-byte pair with the post
// number it belongs to: the host writes the word, then its tag (one cache line, x86 stores stay
// in order); CTA 0 reads all pairs in one round of 16-byte loads (each one atomic over PCIe)
// and accepts when every tag equals the post it waits for, so one PCIe round trip both detects
// the post and delivers the arguments. Posts count admissions and stop commands alike.
constexpr int kArgWords = (int)(sizeof(AdmitArgs) / 8);
static_assert(sizeof(AdmitArgs) % 8 == 0, "AdmitArgs travels as 64-bit words");
struct SrvMailbox {
    struct Pair {
        unsigned long long tag, word;
    } pair[kArgWords];
};

struct LaunchCfg {
    int grid;
    int threads;
    int cap_per_list;
    size_t smem;
};

// Picks threads / candidate capacity / dynamic smem for the pool's list count, sets the
// kernel attribute, and returns the co-resident grid. Throws nothing; returns grid 0 on error.
LaunchCfg admit_launch_config(const DevPool& P, int device, int want_grid);
cudaError_t launch_admit(const DevPool& P, const AdmitArgs& a, const LaunchCfg& lc, int grid,
                         cudaStream_t s);
// The admission server: ONE persistent cooperative launch that runs admit_body for every
// admission the host posts in the mailbox (posts first_post, first_post + 1, ...) until a
// kSrvStop post. args_dev (device) relays each admission's arguments from CTA 0 to the other CTAs.
// Where a device watchdog records its site before it traps (host-mapped u64; see trap_at).
cudaError_t set_trap_word(unsigned long long* host_mapped, int progress_on);
cudaError_t launch_server(const DevPool& P, SrvMailbox* mb_dev, AdmitArgs* args_dev, unsigned long long first_post,
                          const LaunchCfg& lc, cudaStream_t s);

// Belady admission (cs_belady.cuh): one cooperative launch per admission.
LaunchCfg belady_launch_config(const DevPool& P, int device);
cudaError_t launch_belady_admit(const DevPool& P, const AdmitArgs& a, const LaunchCfg& lc, int grid, cudaStream_t s);
// Next-use index over the materialized requests (cs_belady.cu): keys[0, n_flat) are the request
// blocks, blk_off[0, n_req] their offsets. Fills ref/ref_off/depth/kid_of (device buffers the
// caller sized n_flat, n_flat + 1, n_flat, n_flat) and returns the unique-key count.
long long build_belady_index(const unsigned long long* keys, long long n_flat, const long long* blk_off, long long n_req,
                             unsigned int* ref, long long* ref_off, int* depth, unsigned int* kid_of, cudaStream_t s);

// Hash-sharded admission (cs_shard.cuh): probe -> exchange 1 -> decide -> per chunk
// [scan -> exchange 2] -> replay.
struct ShardX;
cudaError_t launch_shard_probe(const DevPool& P, const AdmitArgs& a, cudaStream_t s);
cudaError_t launch_shard_decide(const DevPool& P, const AdmitArgs& a, cudaStream_t s);
// probe + (fused) exchange 1 + decide in one kernel: world 1, or the peer transport
cudaError_t launch_shard_front(const DevPool& P, const AdmitArgs& a, const ShardX& x, cudaStream_t s);
cudaError_t launch_shard_scan(const DevPool& P, const AdmitArgs& a, int chunk, const ShardX& x, const LaunchCfg& lc,
                              cudaStream_t s);
cudaError_t launch_shard_replay(const DevPool& P, const AdmitArgs& a, const ShardX& x, cudaStream_t s);

cudaError_t launch_init_pool(const DevPool& P, cudaStream_t s);
cudaError_t launch_hash_prompts(const unsigned int* tokens, const long long* tok_off, int n, int bs, int skip,
                                int take, const long long* blk_off, unsigned long long* keys, int* counts,
                                unsigned long long* agents, int* err, cudaStream_t s);
// Token-free K1 for generated traces: token ids synthesised from (session, agent, lengths).
struct TurnDesc {
    int session, agent, anchor_tokens, history_tokens;
    int template_tokens, warmup;  // warmup: template + anchor + kWarmupUserToken
    long long blk_off;
};
cudaError_t launch_hash_turns(const TurnDesc* turns, int n, int bs, int skip, int take, unsigned int anchor_stride,
                              int hist_pos_bits, unsigned long long* keys, int* counts, unsigned long long* agents,
                              cudaStream_t s);
cudaError_t launch_chain_hash(const unsigned long long* parents, const unsigned char* has_parent,
                              const unsigned int* tok, const long long* tok_off, int n, unsigned long long* out,
                              cudaStream_t s);
cudaError_t launch_identity(const unsigned long long* keys, const long long* key_off, int n, int skip, int take,
                            unsigned long long* out, cudaStream_t s);
cudaError_t launch_unpin(const DevPool& P, const unsigned int* slots, int n, cudaStream_t s);
cudaError_t launch_restore(const DevPool& P, const unsigned long long* keys, const unsigned long long* lt,
                           const unsigned int* agents, const unsigned int* refs, long long n, cudaStream_t s);
cudaError_t launch_probe(const DevPool& P, const unsigned long long* keys, int n, int* needed, cudaStream_t s);
// EngineSim::unpin by key, step 1 (slot per key; *first_bad = first missing/unpinned index)
cudaError_t launch_unpin_find(const DevPool& P, const unsigned long long* keys, int n, unsigned int* slots,
                              int* first_bad, cudaStream_t s);
// CacheSagePolicy::predict_next: the MLE row of cur, ranked (count desc, AgentId asc)
cudaError_t launch_forecast(const DevPool& P, int cur, int n_agents, int* out_idx, double* out_p, int* out_n,
                            cudaStream_t s);
cudaError_t launch_scores(const DevPool& P, unsigned long long now, unsigned long long* keys, double* scores,
                          long long* n_out, unsigned long long* scratch, cudaStream_t s);
cudaError_t launch_table_rebuild(const DevPool& P, cudaStream_t s);
// The peer-memory shard exchange (cs_comm.cpp PeerComm): every rank pushes its bytes into every
// peer's window over NVLink / NVSwitch (or the same device's memory), raises a flag in that
// peer's memory, then gathers the peers' contributions from its own window into drecv.
constexpr int kPeerParts = 8;  // CTAs (message parts) per peer in one exchange
struct PeerTable {
    unsigned char* win[kMaxShards];          // each rank's window, as addressable from this device
    unsigned long long* flags[kMaxShards];   // each rank's flags (one word per source rank x part)
};
cudaError_t launch_peer_allgather(const void* dsend, void* drecv, size_t bytes, const PeerTable& t, int rank,
                                  int world, unsigned long long seq, size_t cap, cudaStream_t s);
// The fused exchange of a sharded admission (peer transport): the admission kernels themselves
// store their message into the peers' windows and wait on the peers' flags (exchange 1 inside
// shard_front_kernel, exchange 2 from shard_scan_kernel's CTA 0 to shard_replay_kernel).
// fused 0: the exchange is an allgather between kernels, or nothing at world 1.
struct ShardX {
    PeerTable t;
    unsigned long long seq;  // this exchange's number (window parity seq & 1, flag value)
    size_t cap;              // window bytes per source rank
    int fused;
};
cudaError_t launch_check_pool(const DevPool& P, unsigned long long* out, cudaStream_t s);  // out[4], zeroed
// Applies the block-table updates the last admission queued (before any other table user).
cudaError_t launch_table_flush(const DevPool& P, cudaStream_t s);

}  // namespace csb
