// Hash-sharded admission. Included at the end of cs_admit.cu: it reuses the
// scan (scan_pass), the exact per-list select (finalize_list), observe_dispatch and the
// deferred table updates of the single-pool admission kernel.
//
// The pool of GLOBAL budget N is split over G GPUs, block key k living on shard
// owner(k) = (k >> 40) % G (shard_owner). Per admission (EngineSim::start_request /
// execute_warmup, engine.cpp:141-323, paths relative to /root/reference/proj), every shard runs
//
//   front   (1 CTA)   probe: this shard's unpins (and any table updates still queued), a probe
//                     of the prompt positions this shard owns        -> exchange 1
//                     decide, replicated: global residency of every position, try_start_head
//                     feasibility, observe(AgentDispatch) on the replicated learner, lookup
//                     (owners touch their prefix blocks)
//   per chunk of <= 128 prompt blocks that can evict:
//     scan  (grid)    the shard's keep oldest unpinned per survival class + keep+1 oldest
//                     resident (the single-pool K4/K5a)              -> exchange 2
//     replay (1 CTA)  replicated: per list the global keep oldest = the keep smallest of the
//                     union of the shard lists; the exact evict_one replay
//                     (engine.cpp:102-125); owners apply their victims, touches and inserts;
//                     the status goes to the host, then the queued table updates are applied
//
// Exchanges: with the peer transport they are fused into these kernels (fx_push / fx_wait: the
// front's probe record and the scan's lists are stored into the peers' windows, the front's
// decide and the replay read the peers' messages in place); other transports allgather between
// separate probe / decide kernels and between scan and replay; one shard exchanges nothing.
//
// Exactness: the global keep oldest of a list are among the union of every shard's keep oldest
// of that list (a global member is beaten by at most keep-1 members, so by at most keep-1 of its
// own shard), and the replay is the single-pool replay over global slot names, so every shard
// reaches the same decisions as one pool of budget N. The learner is replicated: the dispatch
// stream is global and sequential (engine.cpp:280-281), so each shard applies the same update.

__device__ __forceinline__ unsigned int gslot_of(const DevPool& P, unsigned int s) {
    return ((unsigned int)P.rank << kShardBits) | s;
}
__device__ __forceinline__ bool own_gslot(const DevPool& P, unsigned int g) {
    return g < kNewRemote && (int)(g >> kShardBits) == P.rank;
}

// Instrumentation: %globaltimer at sharded-admission phase k (< 18), thread 0 of CTA 0, in the
// unused words 10..15 of CTAs 8..10's debug rows (tools/shard_timeline.py reads them).
__device__ __forceinline__ void shstamp(const DevPool& P, int k) {
    if (blockIdx.x == 0 && threadIdx.x == 0) P.dbg[(8 + k / 6) * 16 + 10 + k % 6] = gtimer();
}

__device__ __forceinline__ size_t shard_rec1(int n) { return sizeof(ShardHdr) + sizeof(ShardPos) * (size_t)n; }

// ---- the fused exchange (peer transport, ShardX.fused): one CTA of an admission kernel stores
// this shard's message into every peer's window slot [seq & 1][rank] over NVLink / NVSwitch and
// releases the peer's flag word for this rank (system scope); a later kernel of the same
// admission waits for every peer's flag and reads the peers' messages in place. A window slot
// is reused two exchanges later, by which time every peer has waited on the exchange between,
// so it has finished reading (every shard runs the same sequence of exchanges, and waits in each).
__device__ __forceinline__ const unsigned char* fx_msg(const DevPool& P, const ShardX& X, int r) {
    return X.t.win[P.rank] + (size_t)(X.seq & 1ull) * (size_t)P.world * X.cap + (size_t)r * X.cap;
}

// All threads of the CTA; bytes a multiple of 8.
__device__ void fx_push(const DevPool& P, const ShardX& X, const unsigned char* src, size_t bytes) {
    const size_t off = (size_t)(X.seq & 1ull) * (size_t)P.world * X.cap + (size_t)P.rank * X.cap;
    const unsigned long long* s8 = reinterpret_cast<const unsigned long long*>(src);
    for (int p = 0; p < P.world; ++p) {
        if (p == P.rank) continue;
        unsigned long long* d8 = reinterpret_cast<unsigned long long*>(X.t.win[p] + off);
        for (size_t i = threadIdx.x; i < bytes / 8; i += blockDim.x) d8[i] = s8[i];
    }
    __threadfence_system();
    __syncthreads();
    const int p = (int)threadIdx.x;
    if (p < P.world && p != P.rank)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(X.t.flags[p] + P.rank * kPeerParts), "l"(X.seq)
                     : "memory");
}

// All threads of the CTA: returns once every peer's message of exchange X.seq is in this
// shard's window.
__device__ void fx_wait(const DevPool& P, const ShardX& X) {
    const int p = (int)threadIdx.x;
    if (p < P.world && p != P.rank) {
        const unsigned long long* f = X.t.flags[P.rank] + p * kPeerParts;
        unsigned long long spins = 0, v;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
            if (v == ~0ull) trap_at(404);  // the peer aborted its admission (PeerComm::abort)
            if (v >= X.seq) break;
            if (++spins > 64) __nanosleep(100);
            if (spins > (1ull << 27)) trap_at(403);
        }
    }
    __syncthreads();
}

// The exchanged messages as this shard reads them: its own from its send buffer; a peer's from
// this shard's window (fused) or the allgathered receive buffer.
__device__ __forceinline__ const unsigned char* shard_rec1_of(const DevPool& P, const ShardX& X, int r, int n) {
    if (r == P.rank) return P.sh_send1;
    if (X.fused) return fx_msg(P, X, r);
    return P.sh_recv1 + (size_t)r * shard_rec1(n);
}
__device__ __forceinline__ const ShardLists* shard_in(const DevPool& P, const ShardX& X, int r) {
    if (r == P.rank) return P.sh_send2;
    if (X.fused) return reinterpret_cast<const ShardLists*>(fx_msg(P, X, r));
    return reinterpret_cast<const ShardLists*>(reinterpret_cast<const unsigned char*>(P.sh_recv2) +
                                               (size_t)r * shard_lists_bytes(P.n_lists));
}

// Deferred EngineSim::unpin calls (engine.cpp:170-180) of this shard's slots; kNoSlot entries
// are positions another shard owns. All threads of one CTA.
__device__ void shard_unpins(const DevPool& P, const AdmitArgs& a, RedSmem& Red) {
    if (a.n_unpin_ranges <= 0) return;
    long long dec = 0;
#pragma unroll
    for (int r = 0; r < kMaxUnpinRanges; ++r)
        if (r < a.n_unpin_ranges)
            for (int i = threadIdx.x; i < a.unpin_n[r]; i += blockDim.x) {
                const unsigned int us = a.unpin_ptr[r][i];
                if (us != kNoSlot && atomicSub(&P.refs[us], 1u) == 1u) {
                    ++dec;
                    pk_unpinned(P, us);
                }
            }
    dec = block_sum(dec, Red);
    if (threadIdx.x == 0) P.ctrl->pinned -= dec;
    __syncthreads();
}

// ---- probe: this shard's part of EngineSim::lookup / try_start_head (engine.cpp:127-139, 337-346)
__device__ void shard_probe_body(const DevPool& P, const AdmitArgs& a, RedSmem& Red) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    shstamp(P, 0);
    apply_table_queue(P, Red);
    shstamp(P, 1);
    shard_unpins(P, a, Red);
    shstamp(P, 2);
    ShardHdr* hdr = reinterpret_cast<ShardHdr*>(P.sh_send1);
    ShardPos* pos = reinterpret_cast<ShardPos*>(P.sh_send1 + sizeof(ShardHdr));
    for (int i = tid; i < a.n; i += T) {
        const unsigned long long k = a.keys[i];
        ShardPos q{kNoSlot, 0u};
        if (shard_owner(k, P.world) == P.rank) {
            const unsigned int s = table_find(P, k);
            if (s != kNoSlot) {
                q.gslot = gslot_of(P, s);
                q.refs0 = P.refs[s];
            }
        }
        pos[i] = q;
    }
    if (tid == 0) {
        hdr->resident = C->resident;
        hdr->pinned = C->pinned;
    }
    shstamp(P, 3);
}

__global__ void __launch_bounds__(512, 1) shard_probe_kernel(DevPool P, AdmitArgs a) {
    __shared__ RedSmem Red;
    shard_probe_body(P, a, Red);
}

__device__ void shard_write_status(const DevPool& P, const AdmitArgs& a, const ShardState& s) {
    Ctrl* C = P.ctrl;
    AdmitStatus* st = a.status;
    st->started = s.started;
    st->error = s.error;
    st->first_miss = s.first_miss;
    st->admit_n = s.admit_n;
    st->cached = s.cached;
    st->n_evicted = s.n_ev_adm;
    st->resident = s.res_g;
    st->pinned = s.pinned_g;
    st->tick_after = s.tick;
    st->ev_total = C->n_ev;
    st->warm_issued = s.warm_issued;
    st->needed = s.needed;
    st->scans = s.scans;
    st->tombstones = C->tombstones;
    for (int k = 0; k < kPhases; ++k) st->phase_ns[k] = 0ull;
    st->n_pend = C->n_pend;
    for (int k = 0; k < C->n_pend && k < kMaxPending; ++k) {
        st->pend_target[k] = C->pend_target[k];
        st->pend_tick[k] = C->pend_tick[k];
    }
    // early status: the host schedules the next admission while this kernel finishes (the
    // replay's table updates); every field above and the pins are written by now
    __threadfence_system();
    *(volatile unsigned long long*)&st->done_seq = a.seq;
}

// number of absent positions in [lo, hi) of the replicated position table
__device__ long long shard_absent(const DevPool& P, int lo, int hi, RedSmem& Red) {
    long long absent = 0;
    for (int j = lo + (int)threadIdx.x; j < hi; j += blockDim.x) absent += P.sh_gslot[j] == kNoSlot ? 1 : 0;
    return block_sum(absent, Red);
}

// ---- decide: replicated feasibility, observe and lookup (the single-pool phase 0)
__device__ void shard_decide_body(const DevPool& P, const AdmitArgs& a, const ShardX& X, unsigned char* dsm,
                                  RedSmem& Red, AdmSmem& A) {
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int G = P.world, n = a.n;
    shstamp(P, 4);
    if (tid == 0) {
        A.started = 1;
        A.error = 0;
        A.cached = 0;
        A.first_miss = 0;
        A.admit_n = 0;
        A.anchor = 0;
        A.needed = 0;
        A.warm_issued = -1;
        A.tick = a.tick_base;
        long long res = 0, pin = 0;
        for (int r = 0; r < G; ++r) {
            const ShardHdr* h = reinterpret_cast<const ShardHdr*>(shard_rec1_of(P, X, r, n));
            res += h->resident;
            pin += h->pinned;
        }
        A.resident = res;
        A.pinned = pin;
        C->done = 0;
        C->error = 0;
        C->rescan = 0;  // the scans of this admission start from clean bounds (no grid barrier)
        C->fin_done = 0u;
        if (a.flags & kPollReset) {
            C->step_warmups = 0;
            C->n_pend = 0;
        }
    }
    if (tid < kMaxLists) {
        P.gbound[tid] = kNoBound;
        P.gcount[tid] = 0;
        P.gmaxk[tid] = 0ull;
    }
    __syncthreads();
    // the replicated position table: at most one shard owns (and reports) each position
    long long miss_min = n, need = 0;
    for (int i = tid; i < n; i += T) {
        unsigned int gs = kNoSlot, r0 = 0u;
        for (int r = 0; r < G; ++r) {
            const ShardPos q =
                reinterpret_cast<const ShardPos*>(shard_rec1_of(P, X, r, n) + sizeof(ShardHdr))[i];
            if (q.gslot != kNoSlot) {
                gs = q.gslot;
                r0 = q.refs0;
            }
        }
        P.sh_gslot[i] = gs;
        P.sh_grefs0[i] = r0;
        if (gs == kNoSlot && i < miss_min) miss_min = i;
        if (gs == kNoSlot || r0 == 0u) ++need;
    }
    need = block_sum(need, Red);
    miss_min = block_min(miss_min, Red);
    if (tid == 0) {
        A.needed = (int)need;
        if ((a.flags & kFeasible) && A.pinned + need > P.gbudget) A.started = 0;  // try_start_head waits
    }
    __syncthreads();
    if (A.started) {
        if (a.flags & kDispatch) {
            if (tid == 0) A.tick = A.tick + 1;
            __syncthreads();
            observe_dispatch(P, a.prev, a.next, A.tick, a.n_agents, dsm, Red, A);
        }
        if (a.flags & kLookup) {
            const int f = (int)miss_min;
            long long cached = 0;
            for (int i = tid; i < f; i += T) {
                cached += a.counts[i];
                const unsigned int gs = P.sh_gslot[i];
                if (own_gslot(P, gs)) {  // EngineSim::touch
                    P.lt[gs & kShardMask] = A.tick + 1 + (unsigned long long)i;
                    pk_touch(P, gs & kShardMask, A.tick + 1 + (unsigned long long)i);
                }
            }
            cached = block_sum(cached, Red);
            if (tid == 0) {
                A.first_miss = f;
                A.cached = cached;
                A.tick += (unsigned long long)f;
            }
        }
        if (tid == 0) {
            int an = (a.flags & kAdmit) ? n : 0;
            const long long room = P.gbudget - A.pinned;
            if (a.flags & kTruncate) an = (int)room;
            if (a.flags & kWarmupRoom) an = (int)min((long long)n, room);
            A.admit_n = an;
            A.anchor = a.anchor < 0 ? an : a.anchor;
        }
    }
    __syncthreads();
    const long long absent = shard_absent(P, 0, min(A.admit_n, kChunk), Red);
    if (tid == 0) {
        ShardState s;
        s.tick = A.tick;
        s.first_touch = ~0ull;
        s.cached = A.cached;
        s.res_g = A.resident;
        s.pinned_g = A.pinned;
        s.n_ev_adm = 0;
        s.started = A.started;
        s.error = 0;
        s.first_miss = A.first_miss;
        s.admit_n = A.started ? A.admit_n : 0;
        s.anchor = A.anchor;
        s.needed = A.needed;
        s.warm_issued = A.warm_issued;
        s.chunk = 0;
        s.need_scan = A.started && A.admit_n > 0 && A.resident + absent > P.gbudget ? 1 : 0;
        s.scans = 0;
        *P.sh_state = s;
        if (!A.started || A.admit_n <= 0) shard_write_status(P, a, s);  // nothing to admit
    }
    shstamp(P, 5);
}

__global__ void __launch_bounds__(512, 1) shard_decide_kernel(DevPool P, AdmitArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ RedSmem Red;
    __shared__ AdmSmem A;
    ShardX X{};
    shard_decide_body(P, a, X, dsm, Red, A);
}

// ---- front: probe, exchange 1 and decide in one kernel (one CTA per shard). At world 1 there
// is nothing to exchange; with the fused exchange the probe's record goes straight into the
// peers' windows and decide reads theirs in place.
__global__ void __launch_bounds__(512, 1) shard_front_kernel(DevPool P, AdmitArgs a, ShardX X) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ RedSmem Red;
    __shared__ AdmSmem A;
    shard_probe_body(P, a, Red);
    __syncthreads();
    if (X.fused) {
        fx_push(P, X, P.sh_send1, shard_rec1(a.n));
        fx_wait(P, X);
    }
    shard_decide_body(P, a, X, dsm, Red, A);
}

// ---- scan: this shard's per-list keep oldest (the single-pool K4 + K5a), packed for exchange 2
// The host enqueues one scan + exchange + replay per possible chunk without waiting; a chunk
// that does not exist (admission smaller, not started) or cannot evict sends empty lists.
__global__ void __launch_bounds__(kThreads + 32, 1) shard_scan_kernel(DevPool P, AdmitArgs a, int chunk, ShardX X) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ ScanSmem S;
    __shared__ SelectSmem Sel;
    Ctrl* C = P.ctrl;
    const int tid = threadIdx.x, T = blockDim.x;
    const int NL = P.n_lists;
    const ScanBufs B = scan_bufs(dsm);
    const ShardState* SS = P.sh_state;
    const int admit_n = SS->admit_n;
    if (SS->error || SS->chunk != chunk || chunk * kChunk >= admit_n || !SS->need_scan) {
        if (blockIdx.x == 0) {
            for (int l = tid; l < kMaxLists; l += T) P.sh_send2->n[l] = 0;
            if (X.fused) {  // every shard's replay waits for this exchange: send the empty counts
                __syncthreads();
                fx_push(P, X, reinterpret_cast<const unsigned char*>(P.sh_send2), offsetof(ShardLists, c));
            }
        }
        return;  // uniform across the grid: SS is not written during this kernel
    }
    const int keep = min(kChunk, admit_n - chunk * kChunk);
    shstamp(P, 6);
    if (tid == 0) {
        S.spec = 0;
        S.cls_ready = 1;
    }
    for (int pass = 0;; ++pass) {
        int fast = 0;
        if (pass == 0) {
            // no grid barrier: the bounds and counters were reset before this kernel (decide, or
            // the previous chunk's scan), and every CTA derives the fast flag from the same hints
            fast = !__syncthreads_or(tid < NL && !(P.ghint[tid] < kNoBound) && !P.gsmall[tid]);
            if (blockIdx.x == 0 && tid == 0) {
                C->pass = 0;
                C->fast = fast;
                C->scans += 1;
                C->scanned_slots += P.cap;
            }
        } else {
            if (blockIdx.x == 0) {
                if (tid < NL) {
                    P.ghint[tid] = kNoBound;  // a hint was too tight: safe pass without hints
                    P.gbound[tid] = kNoBound;
                    P.gcount[tid] = 0;
                    P.gmaxk[tid] = 0ull;
                }
                __syncthreads();
                if (tid == 0) {
                    C->rescan = 0;
                    C->fin_done = 0u;
                    C->pass = pass;
                    C->fast = 0;
                    C->rescans += 1;
                }
            }
            grid_barrier(C);
        }
        for (int x = tid; x < a.n_agents; x += T) B.cls[x] = P.cls[x];
        __syncthreads();
        scan_pass(P, NL, keep, B, S, Sel, dsm, fast != 0, a);
        grid_barrier(C);
        shstamp(P, 7);
        int mine = 0;
        for (int l = blockIdx.x; l < NL; l += gridDim.x) {
            finalize_list(P, l, NL, keep, B, Sel);
            ++mine;
        }
        if (blockIdx.x != 0) {
            if (tid == 0 && mine) {
                __threadfence();
                atomicAdd(&C->fin_done, (unsigned int)mine);
            }
        } else {
            if (tid == 0) {
                const unsigned int want = (unsigned int)(NL - mine);
                unsigned long long spins = 0;
                while (ld_acquire(&C->fin_done) < want) {
                    if (++spins > 4096) __nanosleep(64);
                    if (spins > (1ull << 27)) trap_at(301);
                }
                __threadfence();
                C->done = (pass == 0 && *(volatile int*)&C->rescan) ? 0 : 1;
            }
        }
        grid_barrier(C);
        shstamp(P, 8);
        if (*(volatile int*)&C->done) break;
    }
    if (blockIdx.x == 0) {
        ShardLists* out = P.sh_send2;
        for (int q = tid; q < NL * (kChunk + 1); q += T) {
            const int l = q / (kChunk + 1), j = q - l * (kChunk + 1);
            if (j < P.fin_n[l]) {
                const unsigned int s = P.fin_slot[(long long)l * (kChunk + 2) + j];
                ShardCand c;
                c.lt = P.fin_lt[(long long)l * (kChunk + 2) + j];
                c.key = P.key[s];
                c.gslot = gslot_of(P, s);
                c.pad = 0u;
                out->c[l][j] = c;
            }
        }
        for (int l = tid; l < kMaxLists; l += T) out->n[l] = l < NL ? P.fin_n[l] : 0;
        if (tid < kMaxLists) {
            P.gbound[tid] = kNoBound;
            P.gcount[tid] = 0;
            P.gmaxk[tid] = 0ull;
        }
        if (tid == 0) {
            C->fin_done = 0u;
            C->rescan = 0;
        }
        if (X.fused) {  // exchange 2: the lists in use straight into the peers' windows
            __syncthreads();
            fx_push(P, X, reinterpret_cast<const unsigned char*>(P.sh_send2), shard_lists_bytes(NL));
        }
    }
    shstamp(P, 9);
}

struct ShardReplaySmem {
    ReplaySmem R;
    unsigned long long L_key[kMaxLists][kChunk + 2];
    unsigned char vreused[kChunk];  // victim k's slot was reused by a new block of this shard
    unsigned char own_key[kChunk];  // chunk position i's key lives on this shard
    int n_in[kMaxShards][kMaxLists];  // received list lengths
    int n_own_erase;
};

// ---- replay: replicated exact evict_one loop over the merged lists; owners apply
__global__ void __launch_bounds__(512, 1) shard_replay_kernel(DevPool P, AdmitArgs a, ShardX Xc) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ RedSmem Red;
    __shared__ AdmSmem A;
    ShardReplaySmem& X = *reinterpret_cast<ShardReplaySmem*>(dsm);
    ReplaySmem& R = X.R;
    Ctrl* C = P.ctrl;
    ShardState* SS = P.sh_state;
    const int tid = threadIdx.x, T = blockDim.x;
    const int NL = P.n_lists, Rl = NL - 1, G = P.world;
    shstamp(P, 10);
    if (Xc.fused) fx_wait(P, Xc);  // always, even for a chunk that does not exist (see fx_push)
    if (tid == 0) {
        A.tick = SS->tick;
        A.first_touch = SS->first_touch;
        A.resident = SS->res_g;
        A.pinned = SS->pinned_g;
        A.chunk = SS->chunk;
        A.admit_n = SS->admit_n;
        A.anchor = SS->anchor;
        A.error = 0;
#pragma unroll
        for (int c = 0; c < kMaxLists; ++c) A.wsurv[c] = P.wsurv[c];
    }
    __syncthreads();
    if (SS->error || !SS->started || A.chunk * kChunk >= A.admit_n) return;  // no such chunk
    const int lo = A.chunk * kChunk;
    const int hi = min(A.admit_n, lo + kChunk);
    const int len = hi - lo;
    const bool scanned = SS->need_scan != 0;

    // ---- prologue: the chunk's positions (replicated), this shard's free slots
    for (int j = tid; j < 512; j += T) {
        R.ph_key[j] = kNoSlot;
        R.vh_key[j] = kNoSlot;
    }
    const long long ftop = C->free_top;
    int absent = 0, pre_unpinned = 0;
    for (int i = tid; i < len; i += T) {
        const unsigned int gs = P.sh_gslot[lo + i];
        const unsigned int r0 = P.sh_grefs0[lo + i];
        R.c_slot[i] = gs;
        R.c_refs0[i] = r0;
        R.touched[i] = 0;
        R.pevict[i] = 0;
        X.own_key[i] = shard_owner(a.keys[lo + i], G) == P.rank ? 1 : 0;
        if (gs == kNoSlot) ++absent;
        else if (r0 == 0u) ++pre_unpinned;
    }
    for (int j = tid; j < kChunk + 2; j += T) R.rremoved[j] = 0;
    for (int j = tid; j < kChunk; j += T) X.vreused[j] = 0;
    for (int j = tid; j < len && j < ftop; j += T) R.freeslots[j] = P.free_stack[ftop - 1 - j];
    const long long both = block_sum(((long long)absent << 32) | (long long)pre_unpinned, Red);
    for (int i = tid; i < len; i += T) {  // gslot -> chunk position of the chunk's resident blocks
        const unsigned int s = R.c_slot[i];
        if (s == kNoSlot) continue;
        unsigned int h = hslot(s);
        for (int q = 0; q < 512; ++q) {
            const unsigned int old = atomicCAS(&R.ph_key[h], kNoSlot, s);
            if (old == kNoSlot || old == s) {
                R.ph_val[h] = (short)i;
                break;
            }
            h = (h + 1) & 511u;
        }
    }
    if (tid == 0) {
        R.absent = (int)(both >> 32);
        R.pre_unpinned = (int)(both & 0xffffffffll);
        R.n_vict = 0;
        R.n_new_global = 0;
        R.n_reused = 0;
        R.n_ins = 0;
        X.n_own_erase = 0;
    }

    // ---- the global lists: per list the keep smallest of the union of the shard lists. Every
    // shard list is sorted and ticks are distinct across shards, so an entry's global rank is
    // its own index plus, per other shard, the number of that shard's entries below it.
    shstamp(P, 11);
    // One round over every (list, shard, entry) instead of a round per list.
    for (int l = tid; l < kMaxLists; l += T) R.L_n[l] = 0;
    for (int q = tid; q < G * kMaxLists; q += T) {
        const int r = q / kMaxLists, l = q - r * kMaxLists;
        X.n_in[r][l] = l < NL ? shard_in(P, Xc, r)->n[l] : 0;
    }
    __syncthreads();
    if (scanned) {
        const int per_list = G * (kChunk + 1);
        for (int q = tid; q < NL * per_list; q += T) {
            const int l = q / per_list, q2 = q - l * per_list;
            const int r = q2 / (kChunk + 1), j = q2 - r * (kChunk + 1);
            if (j >= X.n_in[r][l]) continue;
            const ShardCand c = shard_in(P, Xc, r)->c[l][j];
            int rank = j;
            for (int o = 0; o < G; ++o) {
                if (o == r) continue;
                const ShardCand* co = shard_in(P, Xc, o)->c[l];
                int lo2 = 0, hi2 = X.n_in[o][l];
                while (lo2 < hi2) {
                    const int mid = (lo2 + hi2) >> 1;
                    if (co[mid].lt < c.lt) lo2 = mid + 1;
                    else hi2 = mid;
                }
                rank += lo2;
            }
            if (rank < keep_of(l, NL, len)) {
                R.L_lt[l][rank] = c.lt;
                R.L_slot[l][rank] = c.gslot;
                X.L_key[l][rank] = c.key;
            }
        }
        for (int l = tid; l < NL; l += T) {
            int tot = 0;
            for (int r = 0; r < G; ++r) tot += X.n_in[r][l];
            R.L_n[l] = min(tot, keep_of(l, NL, len));
        }
    }
    __syncthreads();
    auto prompt_index = [&](unsigned int s) -> short {
        unsigned int h = hslot(s);
        for (int q = 0; q < 512; ++q) {
            const unsigned int k = R.ph_key[h];
            if (k == kNoSlot) return -1;
            if (k == s) return R.ph_val[h];
            h = (h + 1) & 511u;
        }
        return -1;
    };
    {  // per list entry: prompt index (a touch removes it), position in the resident list
        const int nres = R.L_n[Rl];
        for (int l = 0; l < NL; ++l) {
            const int nl = R.L_n[l];
            for (int j = tid; j < nl; j += T) {
                R.L_pidx[l][j] = prompt_index(R.L_slot[l][j]);
                short rp = -1;
                if (l == Rl) {
                    rp = (short)j;
                } else {
                    const unsigned long long x = R.L_lt[l][j];
                    int lo2 = 0, hi2 = nres;
                    while (lo2 < hi2) {
                        const int mid = (lo2 + hi2) >> 1;
                        if (R.L_lt[Rl][mid] < x) lo2 = mid + 1;
                        else hi2 = mid;
                    }
                    if (lo2 < nres && R.L_lt[Rl][lo2] == x) rp = (short)lo2;
                }
                R.L_rpos[l][j] = rp;
            }
        }
    }
    __syncthreads();

    shstamp(P, 12);
    // ---- the sequential replay of admit_pinned (engine.cpp:141-168), warp 0; lane l owns list l
    if (warp_id() == 0) {
        const int lane = lane_id();
        int cursor = 0;
        const int my_n = lane < NL ? R.L_n[lane] : 0;
        const double my_ws = lane < kMaxLists ? A.wsurv[lane] : 0.0;
        unsigned long long tick = A.tick;
        unsigned long long first_touch = A.first_touch;
        long long resident = A.resident;
        long long pinned = A.pinned;
        int nv = 0, nglob = 0, own_cur = 0;
        int error = 0;
        long long ev_cyc = 0;  // (instrumentation: SM cycles in evict_one loops)
        const long long loop_t0 = clock64();
        for (int i = 0; i < len; ++i) {
            {  // the run of resident positions from i (touch + pin), up to 32 per round, one lane each:
               // evictions happen only at absent positions, so the run's flags are settled here
                const int j = i + lane;
                const bool res = j < len && R.c_slot[j] != kNoSlot && !R.pevict[j];
                const unsigned int bal = __ballot_sync(0xffffffffu, res);
                const int run = bal == 0xffffffffu ? 32 : __ffs(~bal) - 1;
                if (run > 0) {
                    if (lane < run) {
                        R.out_slot[j] = R.c_slot[j];
                        R.out_lt[j] = tick + 1 + (unsigned long long)lane;
                        R.out_new[j] = 0;
                        R.touched[j] = 1;
                    }
                    pinned += __popc(__ballot_sync(0xffffffffu, lane < run && R.c_refs0[j] == 0u));
                    if (first_touch == ~0ull) first_touch = tick + 1;
                    tick += (unsigned long long)run;
                    i += run - 1;
                    __syncwarp();
                    continue;
                }
            }
            const long long ev_t0 = clock64();
            while (resident >= P.gbudget) {  // evict_one (engine.cpp:102-125)
                if (lane < NL) {  // skip entries touched (pinned) or evicted via another list
                    while (cursor < my_n) {
                        const short pi = R.L_pidx[lane][cursor];
                        const bool gone = (pi >= 0 && R.touched[pi]) || (lane == Rl && R.rremoved[cursor]);
                        if (!gone) break;
                        ++cursor;
                    }
                }
                const unsigned long long rhead =
                    __shfl_sync(0xffffffffu, (lane == Rl && cursor < my_n) ? R.L_lt[Rl][cursor] : ~0ull, Rl);
                unsigned long long old = tick;  // oldest_live_touch (engine.cpp:90-100)
                if (rhead < old) old = rhead;
                if (first_touch < old) old = first_touch;
                unsigned long long sk = ~0ull, lk = ~0ull;
                if (lane < Rl && cursor < my_n) {
                    lk = R.L_lt[lane][cursor];
                    const double rho = recency(lk, tick, old);
                    sk = (unsigned long long)__double_as_longlong(P.policy == 0 ? rho : __dadd_rn(my_ws, rho));
                }
                const unsigned int m1 = __reduce_min_sync(0xffffffffu, (unsigned int)(sk >> 32));
                if (m1 == 0xffffffffu) {
                    error = 1;  // evict_one: all resident blocks are pinned
                    break;
                }
                bool c = (unsigned int)(sk >> 32) == m1;
                const unsigned int m2 = __reduce_min_sync(0xffffffffu, c ? (unsigned int)sk : 0xffffffffu);
                c = c && (unsigned int)sk == m2;
                unsigned int ball = __ballot_sync(0xffffffffu, c);
                if (__popc(ball) > 1) {  // equal scores: the older block wins (engine.cpp:111-114)
                    const unsigned int m3 = __reduce_min_sync(0xffffffffu, c ? (unsigned int)(lk >> 32) : 0xffffffffu);
                    c = c && (unsigned int)(lk >> 32) == m3;
                    const unsigned int m4 = __reduce_min_sync(0xffffffffu, c ? (unsigned int)lk : 0xffffffffu);
                    c = c && (unsigned int)lk == m4;
                    ball = __ballot_sync(0xffffffffu, c);
                }
                const int w = __ffs(ball) - 1;
                if (lane == w) {
                    const short pi = R.L_pidx[lane][cursor];
                    const short rp = R.L_rpos[lane][cursor];
                    if (pi >= 0) R.pevict[pi] = 1;  // reached later in this chunk: absent then
                    if (rp >= 0) R.rremoved[rp] = 1;
                    R.victims[nv] = R.L_slot[lane][cursor];
                    R.vkey[nv] = X.L_key[lane][cursor];
                    ++cursor;
                }
                ++nv;
                --resident;
                __syncwarp();
            }
            ev_cyc += clock64() - ev_t0;
            if (error) break;
            // the new block lives on its key's shard: that shard reuses its own victims of this
            // chunk first, then its free stack; the other shards only count it
            unsigned int ns = kNewRemote;
            if (X.own_key[i]) {
                while (own_cur < nv && !own_gslot(P, R.victims[own_cur])) ++own_cur;
                if (own_cur < nv) {
                    ns = R.victims[own_cur];
                    if (lane == 0) X.vreused[own_cur] = 1;
                    ++own_cur;
                } else if (nglob < ftop) {
                    ns = gslot_of(P, R.freeslots[nglob++]);
                } else {
                    error = 2;  // this shard has no free slot left (shard capacity too small)
                    break;
                }
            }
            ++tick;
            if (lane == 0) {
                R.out_slot[i] = ns;
                R.out_lt[i] = tick;
                R.out_new[i] = 1;
            }
            ++resident;
            ++pinned;
            if (first_touch == ~0ull) first_touch = tick;
            __syncwarp();
        }
        if (lane == 0 && blockIdx.x == 0) {
            P.dbg[10 * 16 + 14] = (unsigned long long)ev_cyc;
            P.dbg[10 * 16 + 15] = (unsigned long long)(clock64() - loop_t0) | ((unsigned long long)nv << 48);
        }
        if (lane == 0) {
            A.tick = tick;
            A.first_touch = first_touch;
            A.resident = resident;
            A.pinned = pinned;
            R.n_vict = nv;
            R.n_new_global = nglob;
            A.error = error;
        }
    }
    __syncthreads();

    shstamp(P, 13);
    // ---- apply: every shard logs every victim; owners erase / free / touch / insert
    const int err = A.error;
    const int nv = R.n_vict;
    const unsigned long long ev0 = C->n_ev;
    const int q_e = C->tq_erase, q_i = C->tq_insert;
    long long own_ev = 0;
    for (int k = tid; k < nv; k += T) {
        const unsigned int v = R.victims[k];
        const unsigned long long kk = R.vkey[k];
        P.evlog[(ev0 + k) % (unsigned long long)P.evlog_cap] = kk;
        unsigned int h = hslot(v);
        for (int q = 0; q < 512; ++q) {
            if (atomicCAS(&R.vh_key[h], kNoSlot, v) == kNoSlot) break;
            h = (h + 1) & 511u;
        }
        if (own_gslot(P, v)) {
            ++own_ev;
            P.tq_key[q_e + atomicAdd(&X.n_own_erase, 1)] = kk;
            if (!X.vreused[k]) {
                const unsigned int ls = v & kShardMask;
                P.lt[ls] = kFreeTick;
                P.refs[ls] = 0u;
                P.agent[ls] = kNoAgent;
                P.pk[ls] = kPkFreeWord;
            }
        }
    }
    __syncthreads();  // a reused victim's reset lands before the new block's writes
    const int done_len = err ? 0 : len;  // an erroring chunk is not applied
    long long own_new = 0, own_pin = 0;
    for (int i = tid; i < done_len; i += T) {
        const unsigned int s = R.out_slot[i];
        if (R.out_new[i]) {
            if (s != kNewRemote) {
                const unsigned int ls = s & kShardMask;
                const int gi = lo + i;
                P.key[ls] = a.keys[gi];
                P.tokens[ls] = a.counts[gi];
                P.agent[ls] = (a.agent != kNoAgent && gi < A.anchor) ? a.agent : kNoAgent;
                P.lt[ls] = R.out_lt[i];
                P.refs[ls] = 1u;
                P.pk[ls] = pk_make(R.out_lt[i], P.agent[ls], true);
                const int q = q_i + atomicAdd(&R.n_ins, 1);
                P.tq_key[P.p_cap + q] = a.keys[gi];
                P.tq_slot[q] = ls;
                ++own_new;
                ++own_pin;
            }
        } else if (own_gslot(P, s)) {
            const unsigned int ls = s & kShardMask;
            P.lt[ls] = R.out_lt[i];
            if (atomicAdd(&P.refs[ls], 1u) == 0u) ++own_pin;
            P.pk[ls] = pk_make(R.out_lt[i], P.agent[ls], true);
        }
        P.sh_gslot[lo + i] = s;
    }
    if (nv > 0) {  // blocks of later chunks evicted here are absent when reached
        for (int j = hi + tid; j < A.admit_n; j += T) {
            const unsigned int s = P.sh_gslot[j];
            if (s == kNoSlot || s == kNewRemote) continue;
            unsigned int h = hslot(s);
            for (int q = 0; q < 512; ++q) {
                const unsigned int k = R.vh_key[h];
                if (k == kNoSlot) break;
                if (k == s) {
                    P.sh_gslot[j] = kNoSlot;
                    break;
                }
                h = (h + 1) & 511u;
            }
        }
    }
    const long long sums = block_sum((own_ev << 42) | (own_new << 21) | own_pin, Red);
    own_ev = sums >> 42;
    own_new = (sums >> 21) & ((1ll << 21) - 1);
    own_pin = sums & ((1ll << 21) - 1);
    if (tid == 0) {
        long long top = ftop - R.n_new_global;
        long long own_reused = 0;
        for (int k = 0; k < nv; ++k) {
            if (!own_gslot(P, R.victims[k])) continue;
            if (X.vreused[k]) ++own_reused;
            else P.free_stack[top++] = R.victims[k] & kShardMask;
        }
        C->resident += own_new - own_ev;
        C->pinned += own_pin;
        C->free_top = top;
        C->n_ev = ev0 + nv;
        C->tq_erase = q_e + X.n_own_erase;
        C->tq_insert = q_i + R.n_ins;
        (void)own_reused;
    }
    __syncthreads();
    shstamp(P, 14);
    // ---- next chunk, or the admission's epilogue (EngineSim::admit unpins at once)
    const int next_lo = hi;
    const bool last = err || next_lo >= A.admit_n;
    const long long absent2 = last ? 0 : shard_absent(P, next_lo, min(A.admit_n, next_lo + kChunk), Red);
    long long dec_g = 0, dec_own = 0;
    if (last && !err) {
        for (int i = tid; i < A.admit_n; i += T) {
            const unsigned int s = P.sh_gslot[i];
            const bool own = own_gslot(P, s);
            if (a.pins_out) a.pins_out[i] = own ? (s & kShardMask) : kNoSlot;
            if (a.flags & kUnpinAfter) {
                // the block's pin count drops back to its value before this admission: it becomes
                // unpinned iff it was new or unpinned then (decidable on every shard)
                if (P.sh_grefs0[i] == 0u) ++dec_g;  // new blocks were absent at the probe: refs0 0
                if (own && atomicSub(&P.refs[s & kShardMask], 1u) == 1u) {
                    ++dec_own;
                    pk_unpinned(P, s & kShardMask);
                }
            }
        }
    }
    dec_g = block_sum(dec_g, Red);
    dec_own = block_sum(dec_own, Red);
    if (tid == 0) {
        ShardState s = *SS;
        s.tick = A.tick;
        s.first_touch = A.first_touch;
        s.res_g = A.resident;
        s.pinned_g = A.pinned - dec_g;
        s.n_ev_adm += nv;
        s.chunk = A.chunk + 1;
        s.error = err;
        s.scans += scanned ? 1 : 0;
        s.need_scan = (!last && A.resident + absent2 > P.gbudget) ? 1 : 0;
        C->pinned -= dec_own;
        *SS = s;
        if (last) shard_write_status(P, a, s);
    }
    shstamp(P, 15);
    // the admission's queued block-table updates, applied behind its early status (the host's
    // turnaround hides them; the next probe would otherwise apply them first)
    __syncthreads();
    if (last) apply_table_queue(P, Red);
}

cudaError_t launch_shard_probe(const DevPool& P, const AdmitArgs& a, cudaStream_t s) {
    shard_probe_kernel<<<1, 512, 0, s>>>(P, a);
    return cudaGetLastError();
}

cudaError_t launch_shard_decide(const DevPool& P, const AdmitArgs& a, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(shard_decide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(BfsSmem));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    shard_decide_kernel<<<1, 512, sizeof(BfsSmem), s>>>(P, a);
    return cudaGetLastError();
}

cudaError_t launch_shard_front(const DevPool& P, const AdmitArgs& a, const ShardX& x, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(shard_front_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(BfsSmem));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    shard_front_kernel<<<1, 512, sizeof(BfsSmem), s>>>(P, a, x);
    return cudaGetLastError();
}

cudaError_t launch_shard_scan(const DevPool& P, const AdmitArgs& a, int chunk, const ShardX& x, const LaunchCfg& lc,
                              cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(shard_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lc.smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    DevPool p = P;
    AdmitArgs aa = a;
    int k = chunk;
    ShardX xx = x;
    void* args[] = {&p, &aa, &k, &xx};
    return cudaLaunchCooperativeKernel((const void*)shard_scan_kernel, dim3(lc.grid), dim3(lc.threads), args, lc.smem,
                                       s);
}

cudaError_t launch_shard_replay(const DevPool& P, const AdmitArgs& a, const ShardX& x, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(shard_replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(ShardReplaySmem));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    shard_replay_kernel<<<1, 512, sizeof(ShardReplaySmem), s>>>(P, a, x);
    return cudaGetLastError();
}
