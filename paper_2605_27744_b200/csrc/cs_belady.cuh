// The Belady baseline (policy 3) on the same pool: BeladyPolicy (baselines.cpp:34-70, paths
// relative to /root/reference/proj) under EngineSim::admit_pinned / evict_one
// (engine.cpp:102-168). Included at the end of cs_admit.cu (shares its table / unpin helpers).
//
// A block's Belady score is 1 / (1 + next_use - cursor) - 1e-10 * depth (0 when its key is never
// referenced again), so it does not decompose into a few survival classes the way the CacheSage
// score does: the admission selects instead the kBelCand smallest (score, last_touch) composites
// over the unpinned resident slots with a grid-wide radix select, and replays admit_pinned over
// them in order. One cooperative launch per admission:
//
//   all CTAs  cursor advance: the resident blocks of the requests that arrived since the last
//             launch get their next use past the new cursor (BeladyPolicy::observe, :48-52)
//   CTA 0     phase 0: queued table updates, deferred unpins, try_start_head probe
//             (engine.cpp:337-346), lookup touches (:127-139), admit_pinned over the resident
//             prefix (no eviction can happen before the first miss)
//   per pass  all CTAs: composites of every slot, then 8-bit radix digits (one grid barrier
//             each) down to the kBelCand-th smallest, then compaction of the candidates
//             CTA 0:    sorts them and replays admit_pinned: a candidate pinned since the pass
//             is skipped; when the candidates run out before the admission ends, another pass
//             runs over the pool as it is then (the unpinned set only shrinks during an
//             admission, so the smallest candidates of a pass stay the argmin until consumed)
//
// Exactness: last_touch is unique per resident block, so (score, last_touch) is a total order and
// evict_one's tie break on the key (engine.cpp:111-114) never decides; the fp64 score is formed
// with the reference's operations in its order (no contraction).

constexpr int kBelThreads = 512;
constexpr size_t kBelSmem = (size_t)kBelCand * (8 + 8 + 4);

// IEEE order of doubles as unsigned order (no NaN arises)
__device__ __forceinline__ unsigned long long bel_ord(double s) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(s);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// std::upper_bound over the key's request ids (baselines.cpp:60): the first id > c, kNoRef if none
__device__ __forceinline__ unsigned int bel_next(const DevPool& P, unsigned int kid, unsigned long long c) {
    long long lo = P.bel_ref_off[kid], hi = P.bel_ref_off[kid + 1];
    const long long end = hi;
    while (lo < hi) {
        const long long m = (lo + hi) >> 1;
        if ((unsigned long long)P.bel_ref[m] <= c) lo = m + 1;
        else hi = m;
    }
    return lo < end ? P.bel_ref[lo] : kNoRef;
}

// BeladyPolicy::score (baselines.cpp:54-70)
__device__ __forceinline__ double bel_score(unsigned int nu, int depth, unsigned long long cursor) {
    if (nu == kNoRef) return 0.0;  // never referenced again
    const double d = (double)((unsigned long long)nu - cursor);
    return __dsub_rn(__ddiv_rn(1.0, __dadd_rn(1.0, d)), __dmul_rn(1e-10, (double)depth));
}

struct BelSmem {
    RedSmem red;
    unsigned int hist[256];
    unsigned long long prefix;
    int k;
};

__device__ __forceinline__ void bel_reset_pass(BelCtl* B, int tid, int T) {
    if (tid == 0) {
        B->hi_or = 0ull;
        B->hi_and = ~0ull;
        B->lo_or = 0ull;
        B->lo_and = ~0ull;
        B->m = 0ull;
        B->n_cand = 0;
    }
    for (int j = tid; j < kBelPasses * 256; j += T) (&B->hist[0][0])[j] = 0u;
}

// One 8-bit digit of the grid-wide select: histogram of the digit at `shift` over the entries
// still matching (word & mask) == prefix (and, for the last_touch word, score == hT), then every
// CTA picks the same bucket from the global histogram.
__device__ void bel_digit(const DevPool& P, BelSmem& S, int pass, bool lo_word, unsigned long long hT, int shift,
                          unsigned long long mask, unsigned long long& prefix, int& k, long long i0, long long i1) {
    BelCtl* B = P.bel_ctl;
    const int tid = threadIdx.x, T = blockDim.x;
    for (int b = tid; b < 256; b += T) S.hist[b] = 0u;
    __syncthreads();
    for (long long i = i0 + tid; i < i1; i += T) {
        const unsigned long long hi = __ldcg(P.bel_hi + i);
        if (hi == ~0ull) continue;
        unsigned long long w = hi;
        if (lo_word) {
            if (hi != hT) continue;
            w = __ldcg(P.bel_lo + i);
        }
        if ((w & mask) == prefix) atomicAdd(&S.hist[(w >> shift) & 255ull], 1u);
    }
    __syncthreads();
    for (int b = tid; b < 256; b += T)
        if (S.hist[b]) atomicAdd(&B->hist[pass][b], S.hist[b]);
    grid_barrier(P.ctrl);
    if (tid < 32) {
        unsigned int c[8], sum = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            c[q] = __ldcg(&B->hist[pass][tid * 8 + q]);
            sum += c[q];
        }
        unsigned int inc = sum;
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned int t = __shfl_up_sync(0xffffffffu, inc, d);
            if (tid >= d) inc += t;
        }
        const unsigned int exc = inc - sum;
        if (exc < (unsigned)k && (unsigned)k <= inc) {
            unsigned int cum = exc;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (cum + c[q] >= (unsigned)k) {
                    S.prefix = prefix | ((unsigned long long)(tid * 8 + q) << shift);
                    S.k = k - (int)cum;
                    break;
                }
                cum += c[q];
            }
        }
    }
    __syncthreads();
    prefix = S.prefix;
    k = S.k;
    __syncthreads();
}

// k-th smallest over the words that differ in `diff`: all digits from the highest differing one
__device__ void bel_select_word(const DevPool& P, BelSmem& S, int& pass, bool lo_word, unsigned long long hT,
                                unsigned long long w_and, unsigned long long diff, unsigned long long& out, int& k,
                                long long i0, long long i1) {
    if (diff == 0ull) {
        out = w_and;
        return;
    }
    const int hb = 63 - __clzll((long long)diff);
    int shift = (hb / 8) * 8;
    unsigned long long mask = (shift + 8 >= 64) ? 0ull : ~((1ull << (shift + 8)) - 1ull);
    unsigned long long prefix = w_and & mask;
    for (;;) {
        bel_digit(P, S, pass++, lo_word, hT, shift, mask, prefix, k, i0, i1);
        mask |= 255ull << shift;
        if (shift == 0) break;
        shift -= 8;
    }
    out = prefix;
}

// One selection pass over the pool (all CTAs): B->n_cand candidates in P.bel_cand, unsorted.
__device__ void bel_pass(const DevPool& P, const AdmitArgs& a, BelSmem& S) {
    BelCtl* B = P.bel_ctl;
    const int tid = threadIdx.x, T = blockDim.x;
    const long long per = (P.cap + gridDim.x - 1) / gridDim.x;
    const long long i0 = (long long)blockIdx.x * per, i1 = min(P.cap, i0 + per);
    unsigned long long hor = 0ull, hand = ~0ull, lor = 0ull, land = ~0ull, m = 0ull;
    for (long long i = i0 + tid; i < i1; i += T) {
        const unsigned long long lt = __ldcg(P.lt + i);
        const unsigned int r = __ldcg(P.refs + i);
        unsigned long long hi = ~0ull, lo = ~0ull;
        if (lt != kFreeTick && r == 0u) {  // evict_one skips pinned blocks (engine.cpp:108-110)
            const unsigned int nu = __ldcg(P.bel_nu + i);
            const int depth = nu == kNoRef ? 0 : P.bel_depth[__ldcg(P.bel_kid + i)];
            hi = bel_ord(bel_score(nu, depth, a.cursor));
            lo = lt;
            hor |= hi;
            hand &= hi;
            lor |= lo;
            land &= lo;
            ++m;
        }
        P.bel_hi[i] = hi;
        P.bel_lo[i] = lo;
    }
    for (int o = 16; o; o >>= 1) {
        hor |= __shfl_xor_sync(0xffffffffu, hor, o);
        hand &= __shfl_xor_sync(0xffffffffu, hand, o);
        lor |= __shfl_xor_sync(0xffffffffu, lor, o);
        land &= __shfl_xor_sync(0xffffffffu, land, o);
        m += __shfl_xor_sync(0xffffffffu, m, o);
    }
    if ((tid & 31) == 0 && m) {
        atomicOr(&B->hi_or, hor);
        atomicAnd(&B->hi_and, hand);
        atomicOr(&B->lo_or, lor);
        atomicAnd(&B->lo_and, land);
        atomicAdd(&B->m, m);
    }
    grid_barrier(P.ctrl);
    const unsigned long long M = __ldcg(&B->m);
    const bool all = M <= (unsigned long long)kBelCand;
    unsigned long long hT = ~0ull, lT = ~0ull;
    if (!all) {
        int k = kBelCand, pass = 0;
        const unsigned long long h_and = __ldcg(&B->hi_and), h_or = __ldcg(&B->hi_or);
        bel_select_word(P, S, pass, false, 0ull, h_and, h_or ^ h_and, hT, k, i0, i1);
        const unsigned long long l_and = __ldcg(&B->lo_and), l_or = __ldcg(&B->lo_or);
        bel_select_word(P, S, pass, true, hT, l_and, l_or ^ l_and, lT, k, i0, i1);
    }
    for (long long i = i0 + tid; i < i1; i += T) {
        const unsigned long long hi = __ldcg(P.bel_hi + i);
        if (hi == ~0ull) continue;
        const unsigned long long lo = __ldcg(P.bel_lo + i);
        if (all || hi < hT || (hi == hT && lo <= lT)) {
            const int q = atomicAdd(&B->n_cand, 1);
            if (q < kBelCand) P.bel_cand[q] = BelCand{hi, lo, (unsigned int)i, 0u};
        }
    }
    if (tid == 0 && blockIdx.x == 0) {
        P.ctrl->scans += 1;
        P.ctrl->scanned_slots += P.cap;
        B->scans += 1;
    }
    grid_barrier(P.ctrl);
}

// CTA 0: sort the pass's candidates by (score, last_touch), then admit_pinned from B->pos on.
__device__ void bel_replay(const DevPool& P, const AdmitArgs& a, unsigned char* dsm, bool scanned) {
    BelCtl* B = P.bel_ctl;
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    unsigned long long* shi = reinterpret_cast<unsigned long long*>(dsm);
    unsigned long long* slo = shi + kBelCand;
    unsigned int* ssl = reinterpret_cast<unsigned int*>(slo + kBelCand);
    const int n = scanned ? min(B->n_cand, kBelCand) : 0;
    int N = 1;
    while (N < n) N <<= 1;
    for (int i = tid; i < N; i += T) {
        if (i < n) {
            const BelCand c = P.bel_cand[i];
            shi[i] = c.hi;
            slo[i] = c.lo;
            ssl[i] = c.slot;
        } else {
            shi[i] = ~0ull;
            slo[i] = ~0ull;
            ssl[i] = kNoSlot;
        }
    }
    __syncthreads();
    for (int k = 2; k <= N; k <<= 1) {  // bitonic sort, ascending (hi, lo)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < N; i += T) {
                const int p = i ^ j;
                if (p <= i) continue;
                const bool gt = shi[i] > shi[p] || (shi[i] == shi[p] && slo[i] > slo[p]);
                if (gt == ((i & k) == 0)) {
                    const unsigned long long th = shi[i], tl = slo[i];
                    const unsigned int ts = ssl[i];
                    shi[i] = shi[p];
                    slo[i] = slo[p];
                    ssl[i] = ssl[p];
                    shi[p] = th;
                    slo[p] = tl;
                    ssl[p] = ts;
                }
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        const bool all = scanned && B->m <= (unsigned long long)kBelCand;
        const int an = B->admit_n, anchor = B->anchor;
        const unsigned long long t0 = B->tick;
        long long res = C->resident, pin = C->pinned, top = C->free_top;
        unsigned long long ev = C->n_ev;
        long long erased = 0, reused = 0, nev = 0;
        int cp = 0, i = B->pos, more = 0, err = 0;
        for (; i < an; ++i) {
            const unsigned long long key = a.keys[i];
            unsigned int s = table_find(P, key);
            if (s == kNoSlot) {
                while (res >= P.cap) {  // EngineSim::evict_one over the sorted candidates
                    while (cp < n && P.refs[ssl[cp]] != 0u) ++cp;  // pinned by this admission
                    if (cp == n) break;
                    const unsigned int v = ssl[cp++];
                    const unsigned long long vk = P.key[v];
                    table_erase(P, vk);
                    ++erased;
                    P.evlog[ev % (unsigned long long)P.evlog_cap] = vk;
                    ++ev;
                    ++nev;
                    P.bel_kid_slot[P.bel_kid[v]] = kNoSlot;
                    P.lt[v] = kFreeTick;
                    P.agent[v] = kNoAgent;
                    P.pk[v] = kPkFreeWord;
                    P.free_stack[top++] = v;
                    --res;
                }
                if (res >= P.cap) {
                    if (all) err = 1;  // "evict_one: all resident blocks are pinned"
                    else more = 1;     // out of candidates: another pass over the pool as it is now
                    break;
                }
                s = P.free_stack[--top];
                P.key[s] = key;
                P.tokens[s] = a.counts[i];
                P.agent[s] = (a.agent != kNoAgent && i < anchor) ? a.agent : kNoAgent;  // engine.cpp:155-157
                P.lt[s] = t0 + 1 + (unsigned long long)i;
                P.refs[s] = 1u;
                P.pk[s] = pk_make(t0 + 1 + (unsigned long long)i, P.agent[s], true);
                ++pin;
                ++res;
                reused += table_insert(P, key, s);
                const unsigned int kid = a.kids[i];
                P.bel_kid[s] = kid;
                P.bel_kid_slot[kid] = s;
                P.bel_nu[s] = bel_next(P, kid, a.cursor);
            } else {
                P.lt[s] = t0 + 1 + (unsigned long long)i;  // EngineSim::touch
                if (P.refs[s]++ == 0u) ++pin;
                P.pk[s] = pk_make(t0 + 1 + (unsigned long long)i, P.agent[s], true);
            }
            if (a.pins_out) a.pins_out[i] = s;
        }
        C->resident = res;
        C->pinned = pin;
        C->free_top = top;
        C->n_ev = ev;
        C->tombstones += erased - reused;
        B->n_ev_adm += nev;
        B->pos = err ? an : i;
        B->more = more;
        if (err) B->error = 1;
    }
    __syncthreads();
    if (B->more) bel_reset_pass(B, tid, T);
}

__global__ void __launch_bounds__(kBelThreads, 1) belady_admit_kernel(DevPool P, AdmitArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ BelSmem S;
    Ctrl* C = P.ctrl;
    BelCtl* B = P.bel_ctl;
    const int tid = threadIdx.x, T = blockDim.x;
    const long long gt = (long long)blockIdx.x * T + tid, gs = (long long)gridDim.x * T;

    // BeladyPolicy::observe(RequestArrival) (baselines.cpp:48-52) since the last launch: a block
    // whose next use the cursor passed is one of the arrived requests' blocks
    for (long long f = a.adv_lo + gt; f < a.adv_hi; f += gs) {
        const unsigned int kid = P.bel_kid_of[f];
        const unsigned int s = P.bel_kid_slot[kid];
        if (s != kNoSlot) P.bel_nu[s] = bel_next(P, kid, a.cursor);
    }

    if (blockIdx.x == 0) {
        if (tid == 0) {
            B->started = 1;
            B->error = 0;
            B->cached = 0;
            B->n_ev_adm = 0;
            B->first_miss = 0;
            B->admit_n = 0;
            B->anchor = 0;
            B->needed = 0;
            B->scans = 0;
            B->pos = 0;
            B->more = 0;
            B->tick = a.tick_base;
        }
        apply_table_queue(P, S.red);
        long long dec = 0;
        const int nu = unpin_total(a, false);
        for (int i = tid; i < nu; i += T) {  // EngineSim::unpin of completed requests (engine.cpp:170-180)
            const unsigned int us = unpin_at(a, i);
            if (us != kNoSlot && atomicSub(&P.refs[us], 1u) == 1u) {
                ++dec;
                pk_unpinned(P, us);
            }
        }
        dec = block_sum(dec, S.red);
        if (tid == 0) C->pinned -= dec;
        long long miss = a.n, need = 0;
        for (int i = tid; i < a.n; i += T) {
            const unsigned int s = table_find(P, a.keys[i]);
            P.p_slot[i] = s;
            if (s == kNoSlot && i < miss) miss = i;
            if (s == kNoSlot || P.refs[s] == 0u) ++need;
        }
        need = block_sum(need, S.red);
        miss = block_min(miss, S.red);
        if (tid == 0) {
            B->needed = (int)need;
            if ((a.flags & kFeasible) && C->pinned + need > P.cap) {
                B->started = 0;  // try_start_head: wait for in-flight pins to clear
            } else {
                unsigned long long tick = a.tick_base;
                if (a.flags & kDispatch) tick += 1;  // emit(AgentDispatch): BeladyPolicy ignores it
                const int f = (a.flags & kLookup) ? (int)miss : 0;
                int an = (a.flags & kAdmit) ? a.n : 0;
                const long long room = P.cap - C->pinned;
                if (a.flags & kTruncate) an = (int)room;
                if (a.flags & kWarmupRoom) an = (int)min((long long)a.n, room);
                B->first_miss = f;
                B->admit_n = an;
                B->anchor = a.anchor < 0 ? an : a.anchor;
                B->tick = tick + (unsigned long long)f;  // the lookup's touches
            }
        }
        __syncthreads();
        if (B->started) {
            const int f = B->first_miss, pre = min(f, B->admit_n);
            const unsigned long long t0 = B->tick;
            long long cached = 0, pinc = 0;
            for (int i = tid; i < f; i += T) {
                cached += a.counts[i];
                if (a.touch_agent) a.touch_agent[i] = P.agent[P.p_slot[i]];  // BlockTouch{key, agent}
            }
            for (int i = tid; i < pre; i += T) {  // admit_pinned over the resident prefix
                const unsigned int s = P.p_slot[i];
                P.lt[s] = t0 + 1 + (unsigned long long)i;
                if (atomicAdd(&P.refs[s], 1u) == 0u) ++pinc;
                P.pk[s] = pk_make(t0 + 1 + (unsigned long long)i, P.agent[s], true);
                if (a.pins_out) a.pins_out[i] = s;
            }
            cached = block_sum(cached, S.red);
            pinc = block_sum(pinc, S.red);
            if (tid == 0) {
                B->cached = cached;
                C->pinned += pinc;
                B->pos = pre;
            }
        }
        bel_reset_pass(B, tid, T);
    }
    grid_barrier(C);

    for (;;) {
        const int started = __ldcg(&B->started), pos = __ldcg(&B->pos), an = __ldcg(&B->admit_n);
        if (!started || pos >= an) break;
        // each remaining block inserts at most one: no eviction is possible below the budget
        const bool scan = __ldcg(&C->resident) + (long long)(an - pos) > P.cap;
        if (scan) bel_pass(P, a, S);
        if (blockIdx.x == 0) bel_replay(P, a, dsm, scan);
        grid_barrier(C);
    }

    if (blockIdx.x == 0) {
        const int an = B->admit_n;
        if (B->started && !B->error && (a.flags & kUnpinAfter) && a.pins_out) {
            long long dec = 0;
            for (int i = tid; i < an; i += T)
                if (atomicSub(&P.refs[a.pins_out[i]], 1u) == 1u) {
                    ++dec;
                    pk_unpinned(P, a.pins_out[i]);
                }
            dec = block_sum(dec, S.red);
            if (tid == 0) C->pinned -= dec;
        }
        __syncthreads();
        if (tid == 0) {
            AdmitStatus* st = a.status;
            st->started = B->started;
            st->error = B->error;
            st->first_miss = B->first_miss;
            st->admit_n = B->started ? an : 0;
            st->cached = B->cached;
            st->n_evicted = B->n_ev_adm;
            st->resident = C->resident;
            st->pinned = C->pinned;
            st->tick_after = B->started ? B->tick + (unsigned long long)an : a.tick_base;
            st->ev_total = C->n_ev;
            st->n_pend = 0;
            st->warm_issued = -1;
            st->scans = B->scans;
            st->needed = B->needed;
            st->tombstones = C->tombstones;
            for (int k = 0; k < kPhases; ++k) st->phase_ns[k] = 0ull;
        }
    }
}

LaunchCfg belady_launch_config(const DevPool& P, int device) {
    (void)P;
    LaunchCfg lc{};
    if (cudaFuncSetAttribute(belady_admit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBelSmem) !=
        cudaSuccess)
        return lc;
    cudaDeviceProp prop{};
    int occ = 0;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, belady_admit_kernel, kBelThreads, kBelSmem) !=
            cudaSuccess ||
        occ < 1)
        return lc;
    lc.grid = prop.multiProcessorCount * occ;
    lc.threads = kBelThreads;
    lc.smem = kBelSmem;
    return lc;
}

cudaError_t launch_belady_admit(const DevPool& P, const AdmitArgs& a, const LaunchCfg& lc, int grid, cudaStream_t s) {
    DevPool p = P;
    AdmitArgs aa = a;
    void* args[] = {&p, &aa};
    if (grid <= 1) return cudaLaunchKernel((const void*)belady_admit_kernel, dim3(1), dim3(lc.threads), args, lc.smem, s);
    return cudaLaunchCooperativeKernel((const void*)belady_admit_kernel, dim3(grid), dim3(lc.threads), args, lc.smem,
                                       s);
}
