// Small sm_100a kernels around the admission kernel (cs_admit.cu):
//   K1  hash_prompts / hash_turns  chain_hash + block_keys_for + derive_agent_identity
//                                  (hashing.cpp:26-51, cachesage_policy.cpp:9-31)
//   K2  probe / restore / table rebuild, unpin (engine.cpp:170-180), score snapshot
//       (cachesage_policy.cpp:79-85 over the whole pool)
// Paths relative to /root/reference/proj.
#include <cuda_runtime.h>

#include <algorithm>

#include "cs_block.cuh"
#include "cs_launch.h"

namespace csb {

// ------------------------------------------------------------------ small kernels

__global__ void init_pool_kernel(DevPool P) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long s = i; s < P.cap; s += stride) {
        P.key[s] = 0ull;
        P.tokens[s] = 0;
        P.free_stack[s] = (unsigned int)(P.cap - 1 - s);  // pops hand out slot 0 first
    }
    for (long long s = i; s < P.cap_scan; s += stride) {  // pad slots stay free forever
        P.lt[s] = kFreeTick;
        P.agent[s] = kNoAgent;
        P.refs[s] = 0u;
        P.pk[s] = kPkFreeWord;
    }
    for (long long e = i; e <= (long long)P.tmask; e += stride) {
        P.table[e].key = 0ull;
        P.table[e].slot = kSlotEmpty;
        P.table[e].pad = 0u;
    }
    for (long long x = i; x < P.a_cap; x += stride) {
        P.cls[x] = (unsigned char)P.e_max;
        P.hop[x] = (unsigned char)P.e_max;
    }
    if (i < kMaxLists) {  // per-list scan state; every admission launch resets it for the next
        P.gbound[i] = kNoBound;
        P.gcount[i] = 0;
        P.gmaxk[i] = 0ull;
    }
    if (i == 0) {
        Ctrl* C = P.ctrl;
        C->resident = 0;
        C->pinned = 0;
        C->free_top = P.cap;
        C->tombstones = 0;
        C->n_ev = 0;
        C->scans = 0;
        C->scanned_slots = 0;
        C->rebuilds = 0;
        C->win_head = 0;
        C->win_size = 0;
        C->recorded = 0;
        C->cur_agent = -1;
        C->reach_built = 0;
        C->step_warmups = 0;
        C->n_pend = 0;
        C->bar_count = 0;
        C->bar_gen = 0;
        C->done = 0;
        C->fin_done = 0u;
        C->rescan = 0;
        C->p0_seq = 0ull;
        C->tq_erase = 0;
        C->tq_insert = 0;
        C->svc_b_seq = 0ull;
    }
}

struct HashCursor {
    unsigned long long h, parent;
    long long pos, len, blk, bo;
    int in_blk, bs, has_parent;
    unsigned long long* keys;
    int* counts;
    __device__ __forceinline__ void start() {
        h = mix64(kHashSeed ^ kRootParent);
        in_blk = 0;
        blk = 0;
        pos = 0;
    }
    // chain_hash absorbs one token; a full (or final) block emits its key (hashing.cpp:26-51)
    __device__ __forceinline__ void eat(unsigned int t) {
        h = mix64(h ^ ((unsigned long long)t + kGolden));
        ++in_blk;
        ++pos;
        if (in_blk == bs || pos == len) {
            keys[bo + blk] = h;
            counts[bo + blk] = in_blk;
            ++blk;
            in_blk = 0;
            h = mix64(kHashSeed ^ h);
        }
    }
};

// derive_agent_identity (cachesage_policy.cpp:9-31) over this prompt's freshly written keys
__device__ __forceinline__ unsigned long long identity_of(const unsigned long long* k, long long nb, int skip,
                                                           int take) {
    long long lo = 0, hi = nb;
    if (nb >= (long long)skip + take) {
        lo = skip;
        hi = (long long)skip + take;
    } else if (nb > skip) {
        lo = skip;
    }
    unsigned long long h = mix64(kHashSeed ^ kIdentitySalt);
    for (long long j = lo; j < hi; ++j) h = mix64(h ^ k[j]);
    return h;
}

// chain_hash (hashing.cpp:26-35) of one token span per thread, from an explicit parent key or
// the root (the reference's Python chain_hash(parent, tokens), py_module.cpp:82-88)
__global__ void chain_hash_kernel(const unsigned long long* parents, const unsigned char* has_parent,
                                  const unsigned int* tok, const long long* tok_off, int n, unsigned long long* out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const bool hp = has_parent && has_parent[p];
    unsigned long long h = mix64(kHashSeed ^ (hp ? parents[p] : kRootParent));
    for (long long i = tok_off[p]; i < tok_off[p + 1]; ++i) h = mix64(h ^ ((unsigned long long)tok[i] + kGolden));
    out[p] = h;
}

// derive_agent_identity (cachesage_policy.cpp:9-31) of one block-key list per thread
__global__ void identity_kernel(const unsigned long long* keys, const long long* key_off, int n, int skip, int take,
                                unsigned long long* out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    out[p] = identity_of(keys + key_off[p], key_off[p + 1] - key_off[p], skip, take);
}

// K1 over explicit token streams: one thread per prompt (the chain is sequential within a
// prompt), tokens read as 128-bit vectors once 16-B aligned.
__global__ void hash_prompts_kernel(const unsigned int* __restrict__ tok, const long long* __restrict__ tok_off, int n,
                                    int bs, int skip, int take, const long long* __restrict__ blk_off,
                                    unsigned long long* keys, int* counts, unsigned long long* agents, int* err) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const long long off = tok_off[p];
    HashCursor c;
    c.len = tok_off[p + 1] - off;
    c.bs = bs;
    c.bo = blk_off[p];
    c.keys = keys;
    c.counts = counts;
    if (c.len <= 0) {
        atomicExch(err, 1);  // chain_hash: token sequence must be nonempty
        return;
    }
    c.start();
    const unsigned int* t = tok + off;
    long long i = 0;
    while (i < c.len && (reinterpret_cast<uintptr_t>(t + i) & 15u)) c.eat(t[i++]);
    for (; i + 4 <= c.len; i += 4) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(t + i));
        c.eat(q.x);
        c.eat(q.y);
        c.eat(q.z);
        c.eat(q.w);
    }
    while (i < c.len) c.eat(t[i++]);
    if (agents) agents[p] = identity_of(keys + c.bo, c.blk, skip, take);
}

// K1 for generated traces: token ids synthesised in registers from the turn descriptor
// (Trace::turn_tokens / warmup_tokens, workload.cpp:125-154), so no token stream crosses HBM.
__global__ void hash_turns_kernel(const TurnDesc* __restrict__ turns, int n, int bs, int skip, int take,
                                  unsigned int stride, int pos_bits, unsigned long long* keys, int* counts,
                                  unsigned long long* agents) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const TurnDesc d = turns[p];
    HashCursor c;
    c.len = (long long)d.template_tokens + d.anchor_tokens + (d.warmup ? 1 : d.history_tokens);
    c.bs = bs;
    c.bo = d.blk_off;
    c.keys = keys;
    c.counts = counts;
    c.start();
    for (int j = 0; j < d.template_tokens; ++j) c.eat(0x00100000u + (unsigned int)j);
    const unsigned int ab = 0x01000000u + (unsigned int)d.agent * stride;
    for (int j = 0; j < d.anchor_tokens; ++j) c.eat(ab + (unsigned int)j);
    if (d.warmup) {
        c.eat(0x02000000u);
    } else {
        const unsigned int hb = 0x80000000u | ((unsigned int)d.session << pos_bits);
        for (int q = 0; q < d.history_tokens; ++q) c.eat(hb | (unsigned int)q);
    }
    if (agents) agents[p] = identity_of(keys + c.bo, c.blk, skip, take);
}

__global__ void unpin_kernel(DevPool P, const unsigned int* slots, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int dec = 0;
    if (i < n && slots[i] != kNoSlot) {  // kNoSlot: a position another shard owns
        if (atomicSub(&P.refs[slots[i]], 1u) == 1u) {
            dec = 1;
            pk_unpinned(P, slots[i]);
        }
    }
    dec = __reduce_add_sync(0xffffffffu, dec);
    if (lane_id() == 0 && dec) atomicAdd(reinterpret_cast<unsigned long long*>(&P.ctrl->pinned),
                                         (unsigned long long)(-(long long)dec));
}

__global__ void restore_kernel(DevPool P, const unsigned long long* keys, const unsigned long long* lt,
                               const unsigned int* agents, const unsigned int* refs, long long n,
                               unsigned long long* acc /* [pinned, reused] */) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long top = P.ctrl->free_top;
    const unsigned int s = P.free_stack[top - 1 - i];
    P.key[s] = keys[i];
    P.lt[s] = lt[i];
    P.agent[s] = agents ? agents[i] : kNoAgent;
    const unsigned int r = refs ? refs[i] : 0u;
    P.refs[s] = r;
    P.pk[s] = pk_make(lt[i], agents ? agents[i] : kNoAgent, r != 0u);
    P.tokens[s] = 16;
    const int reused = table_insert(P, keys[i], s);
    if (r) atomicAdd(acc, 1ull);
    if (reused) atomicAdd(acc + 1, 1ull);
}

__global__ void restore_finish_kernel(DevPool P, long long n, const unsigned long long* acc) {
    Ctrl* C = P.ctrl;
    C->free_top -= n;
    C->resident += n;
    C->pinned += (long long)acc[0];
    C->tombstones -= (long long)acc[1];
}

__global__ void probe_kernel(DevPool P, const unsigned long long* keys, int n, int* needed) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int c = 0;
    if (i < n) {
        const unsigned int s = table_find(P, keys[i]);
        c = (s == kNoSlot || P.refs[s] == 0u) ? 1 : 0;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane_id() == 0 && c) atomicAdd(needed, c);
}

// EngineSim::unpin by key (engine.cpp:170-180), step 1: the slot of every key. The reference
// throws "unpin: block vanished while referenced" at the first key that is not resident, after
// unpinning the keys before it; *first_bad is the smallest such index (n: none). A resident key
// with no pin left (the reference would drive refs negative) is reported the same way.
__global__ void unpin_find_kernel(DevPool P, const unsigned long long* keys, int n, unsigned int* slots,
                                  int* first_bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned int s = table_find(P, keys[i]);
    slots[i] = s;
    if (s == kNoSlot || P.refs[s] == 0u) atomicMin(first_bad, i);
}

// CacheSagePolicy::predict_next (cachesage_policy.cpp:94-107): the full MLE row of `cur`,
// count / row_total in fp64, ranked for prefetch (the warmup candidates of maybe_prefetch,
// :109-123): descending count, ties to the smaller 64-bit AgentId exactly as argmax_row breaks
// them (transition_learner.cpp:79-96), so entry 0 is the argmax. One CTA; the row (A <= 4096
// u32 counts) is read once and its non-zero cells ranked in shared memory.
__global__ void __launch_bounds__(1024) forecast_kernel(DevPool P, int cur, int n_agents, int* out_idx,
                                                       double* out_p, int* out_n) {
    __shared__ int nz;
    __shared__ int z_idx[kMaxAgents];
    __shared__ unsigned int z_cnt[kMaxAgents];
    const int tid = threadIdx.x, T = blockDim.x;
    if (tid == 0) nz = 0;
    __syncthreads();
    const unsigned int* row = P.counts + (long long)cur * P.a_cap;
    for (int b = tid; b < n_agents; b += T) {
        const unsigned int c = row[b];
        if (c) {
            const int k = atomicAdd(&nz, 1);
            z_idx[k] = b;
            z_cnt[k] = c;
        }
    }
    __syncthreads();
    const int m = nz;
    const double total = (double)P.totals[cur];
    for (int k = tid; k < m; k += T) {
        const unsigned int c = z_cnt[k];
        const unsigned long long id = P.agent_ids[z_idx[k]];
        int rank = 0;
        for (int j = 0; j < m; ++j) {
            const unsigned int cj = z_cnt[j];
            rank += (cj > c || (cj == c && P.agent_ids[z_idx[j]] < id)) ? 1 : 0;
        }
        out_idx[rank] = z_idx[k];
        out_p[rank] = __ddiv_rn((double)c, total);
    }
    if (tid == 0) *out_n = m;
}

__global__ void min_lt_kernel(DevPool P, unsigned long long* out) {
    unsigned long long m = ~0ull;
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < P.cap;
         s += (long long)gridDim.x * blockDim.x) {
        const unsigned long long x = P.lt[s];
        if (x < m) m = x;
    }
    for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane_id() == 0) atomicMin(out, m);
}

__global__ void scores_kernel(DevPool P, unsigned long long now, const unsigned long long* minlt,
                              unsigned long long* keys, double* scores, long long* n_out) {
    const unsigned long long old = min(now, *minlt);
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < P.cap;
         s += (long long)gridDim.x * blockDim.x) {
        const unsigned long long x = P.lt[s];
        if (x == kFreeTick) continue;
        const unsigned int a = P.agent[s];
        const int c = (a == kNoAgent) ? P.e_max : (int)P.cls[a];
        const double sc = score_of(P.policy, P.w_pred, survival_of_class(c, P.e_max), x, now, old);
        const long long o = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(n_out), 1ull);
        keys[o] = P.key[s];
        scores[o] = sc;
    }
}

__global__ void table_clear_kernel(DevPool P) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e <= (long long)P.tmask;
         e += (long long)gridDim.x * blockDim.x) {
        P.table[e].slot = kSlotEmpty;
        P.table[e].key = 0ull;
    }
}

__global__ void table_fill_kernel(DevPool P) {
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < P.cap;
         s += (long long)gridDim.x * blockDim.x) {
        if (P.lt[s] != kFreeTick) table_insert(P, P.key[s], (unsigned int)s);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.ctrl->tombstones = 0;
        P.ctrl->tq_erase = 0;  // the SoA is the truth: queued table updates are subsumed
        P.ctrl->tq_insert = 0;
    }
}

// ------------------------------------------------------------------ host launchers

cudaError_t launch_init_pool(const DevPool& P, cudaStream_t s) {
    init_pool_kernel<<<1184, 256, 0, s>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_hash_prompts(const unsigned int* tokens, const long long* tok_off, int n, int bs, int skip,
                                int take, const long long* blk_off, unsigned long long* keys, int* counts,
                                unsigned long long* agents, int* err, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    hash_prompts_kernel<<<(n + 127) / 128, 128, 0, s>>>(tokens, tok_off, n, bs, skip, take, blk_off, keys, counts,
                                                         agents, err);
    return cudaGetLastError();
}

cudaError_t launch_hash_turns(const TurnDesc* turns, int n, int bs, int skip, int take, unsigned int anchor_stride,
                              int hist_pos_bits, unsigned long long* keys, int* counts, unsigned long long* agents,
                              cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    hash_turns_kernel<<<(n + 127) / 128, 128, 0, s>>>(turns, n, bs, skip, take, anchor_stride, hist_pos_bits, keys,
                                                       counts, agents);
    return cudaGetLastError();
}

cudaError_t launch_unpin(const DevPool& P, const unsigned int* slots, int n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    unpin_kernel<<<(n + 255) / 256, 256, 0, s>>>(P, slots, n);
    return cudaGetLastError();
}

cudaError_t launch_restore(const DevPool& P, const unsigned long long* keys, const unsigned long long* lt,
                           const unsigned int* agents, const unsigned int* refs, long long n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    unsigned long long* acc = nullptr;
    cudaError_t e = cudaMallocAsync(&acc, 16, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(acc, 0, 16, s);
    restore_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, keys, lt, agents, refs, n, acc);
    restore_finish_kernel<<<1, 1, 0, s>>>(P, n, acc);
    cudaFreeAsync(acc, s);
    return cudaGetLastError();
}

cudaError_t launch_chain_hash(const unsigned long long* parents, const unsigned char* has_parent,
                              const unsigned int* tok, const long long* tok_off, int n, unsigned long long* out,
                              cudaStream_t s) {
    if (n > 0) chain_hash_kernel<<<(n + 127) / 128, 128, 0, s>>>(parents, has_parent, tok, tok_off, n, out);
    return cudaGetLastError();
}

cudaError_t launch_identity(const unsigned long long* keys, const long long* key_off, int n, int skip, int take,
                            unsigned long long* out, cudaStream_t s) {
    if (n > 0) identity_kernel<<<(n + 127) / 128, 128, 0, s>>>(keys, key_off, n, skip, take, out);
    return cudaGetLastError();
}

cudaError_t launch_unpin_find(const DevPool& P, const unsigned long long* keys, int n, unsigned int* slots,
                              int* first_bad, cudaStream_t s) {
    if (n > 0) unpin_find_kernel<<<(n + 255) / 256, 256, 0, s>>>(P, keys, n, slots, first_bad);
    return cudaGetLastError();
}

cudaError_t launch_forecast(const DevPool& P, int cur, int n_agents, int* out_idx, double* out_p, int* out_n,
                            cudaStream_t s) {
    forecast_kernel<<<1, 1024, 0, s>>>(P, cur, n_agents, out_idx, out_p, out_n);
    return cudaGetLastError();
}

cudaError_t launch_probe(const DevPool& P, const unsigned long long* keys, int n, int* needed, cudaStream_t s) {
    cudaMemsetAsync(needed, 0, sizeof(int), s);
    if (n > 0) probe_kernel<<<(n + 255) / 256, 256, 0, s>>>(P, keys, n, needed);
    return cudaGetLastError();
}

cudaError_t launch_scores(const DevPool& P, unsigned long long now, unsigned long long* keys, double* scores,
                          long long* n_out, unsigned long long* scratch, cudaStream_t s) {
    cudaMemsetAsync(scratch, 0xff, 8, s);
    cudaMemsetAsync(n_out, 0, 8, s);
    min_lt_kernel<<<592, 256, 0, s>>>(P, scratch);
    scores_kernel<<<592, 256, 0, s>>>(P, now, scratch, keys, scores, n_out);
    return cudaGetLastError();
}

// Pool invariants (debug / tests): out[0] = slots whose packed scan word disagrees with
// lt / agent / refs, out[1] = resident slots, out[2] = pinned slots, out[3] = resident slots the
// block table does not map back to themselves.
__global__ void check_pool_kernel(DevPool P, unsigned long long* out) {
    unsigned long long bad = 0, res = 0, pin = 0, tab = 0;
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < P.cap_scan;
         s += (long long)gridDim.x * blockDim.x) {
        const unsigned long long lt = P.lt[s];
        const unsigned int r = P.refs[s];
        const unsigned long long want = lt == kFreeTick ? kPkFreeWord : pk_make(lt, P.agent[s], r != 0u);
        bad += P.pk[s] != want;
        if (lt != kFreeTick) {
            ++res;
            pin += r != 0u;
            tab += table_find(P, P.key[s]) != (unsigned int)s;
        }
    }
    atomicAdd(out + 0, bad);
    atomicAdd(out + 1, res);
    atomicAdd(out + 2, pin);
    atomicAdd(out + 3, tab);
}

cudaError_t launch_check_pool(const DevPool& P, unsigned long long* out, cudaStream_t s) {
    check_pool_kernel<<<592, 256, 0, s>>>(P, out);
    return cudaGetLastError();
}

// ---- the peer-memory allgather (PeerTable). kPeerParts CTAs per rank p of the group, each
// owning one contiguous part of the message: push this rank's part into p's window slot
// [seq & 1][rank], release p's flag for (this rank, part) (system scope: the window is on
// another GPU), then wait for p's flag for (p, part) in this rank's own flags and copy p's part
// to drecv + p * bytes. Windows are double-buffered by exchange parity: a rank can start
// exchange k + 2 only after every peer finished exchange k + 1, so after every peer read slot
// k & 1 (all ranks run the same sequence of exchanges). Parts split the copy over SMs (one CTA
// moved a 31 KB list exchange at ~1 GB/s: latency-bound) and need no cross-CTA counting.
// (128 threads, few registers: a CTA of it fits beside a cooperative scan CTA on one SM, so
// shards that share a GPU in the tests never starve each other's cooperative launches)
__global__ void __launch_bounds__(128) peer_allgather_kernel(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                                      size_t bytes, PeerTable t, int rank, unsigned long long seq, size_t cap) {
    const int p = blockIdx.x / kPeerParts, part = blockIdx.x % kPeerParts;
    const int tid = threadIdx.x, T = blockDim.x;
    const int world = gridDim.x / kPeerParts;
    const size_t slot = (size_t)(seq & 1ull) * (size_t)world * cap;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | bytes | cap) & 15u) == 0;
    // this CTA's part: 16-byte granules when aligned, else bytes
    const size_t units = vec ? bytes / 16 : bytes;
    const size_t per = (units + kPeerParts - 1) / kPeerParts;
    const size_t u0 = min(units, (size_t)part * per), u1 = min(units, u0 + per);
    {
        unsigned char* d = t.win[p] + slot + (size_t)rank * cap;
        if (vec) {
            const uint4* s4 = reinterpret_cast<const uint4*>(src);
            uint4* d4 = reinterpret_cast<uint4*>(d);
            for (size_t i = u0 + tid; i < u1; i += T) d4[i] = s4[i];
        } else {
            for (size_t i = u0 + tid; i < u1; i += T) d[i] = src[i];
        }
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(t.flags[p] + rank * kPeerParts + part), "l"(seq)
                     : "memory");
        const unsigned long long* mine = t.flags[rank] + p * kPeerParts + part;
        unsigned long long spins = 0, v;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
            if (v == ~0ull) trap_at(402);  // the peer aborted its admission (PeerComm::abort)
            if (v >= seq) break;
            if (++spins > 64) __nanosleep(100);
            if (spins > (1ull << 27)) trap_at(401);
        }
    }
    __syncthreads();
    {
        const unsigned char* w = t.win[rank] + slot + (size_t)p * cap;
        unsigned char* d = dst + (size_t)p * bytes;
        if (vec) {
            const uint4* w4 = reinterpret_cast<const uint4*>(w);
            uint4* d4 = reinterpret_cast<uint4*>(d);
            for (size_t i = u0 + tid; i < u1; i += T) d4[i] = __ldcg(w4 + i);
        } else {
            for (size_t i = u0 + tid; i < u1; i += T) d[i] = __ldcg(w + i);
        }
    }
}

cudaError_t launch_peer_allgather(const void* dsend, void* drecv, size_t bytes, const PeerTable& t, int rank,
                                  int world, unsigned long long seq, size_t cap, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {  // keep the SM's carve-out at max shared memory: never evicts a scan CTA's layout
        cudaFuncSetAttribute(peer_allgather_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        attr = true;
    }
    peer_allgather_kernel<<<world * kPeerParts, 128, 0, s>>>(static_cast<const unsigned char*>(dsend),
                                                             static_cast<unsigned char*>(drecv), bytes, t, rank, seq,
                                                             cap);
    return cudaGetLastError();
}

cudaError_t launch_table_rebuild(const DevPool& P, cudaStream_t s) {
    table_clear_kernel<<<1184, 256, 0, s>>>(P);
    table_fill_kernel<<<1184, 256, 0, s>>>(P);
    return cudaGetLastError();
}

}  // namespace csb
