// Device-resident scheduler: one persistent cooperative launch runs whole
// EngineSim steps (engine.cpp:262-392, paths relative to /root/reference/proj), so an admission
// costs no kernel launch and no host round trip. Included at the end of cs_admit.cu (it calls
// admit_body). CTA 0's thread 0 runs the scheduler below, a line-for-line restatement of the
// host scheduler in cs_engine.cpp (itself the reference's EngineSim), with its state on chip;
// every admission it issues runs on the whole grid through admit_body.

enum EngPhase { kPhStep = 0, kPhTry, kPhTryResult, kPhNoProg, kPhDrain, kPhWarm, kPhWarmResult, kPhStepEnd };

__device__ __forceinline__ bool flight_later(const EngFlight& a, const EngFlight& b) {
    return a.end_us > b.end_us || (a.end_us == b.end_us && a.seq > b.seq);
}

// std::push_heap / std::pop_heap with `later` (a min-heap on (end_us, seq)): the same element
// order as the host's std heap is not needed, only the same top, which is unique per (end, seq).
__device__ void heap_push(EngState& s, const EngFlight& f) {
    int i = s.n_flight++;
    s.flight[i] = f;
    while (i > 0) {
        const int p = (i - 1) >> 1;
        if (!flight_later(s.flight[p], s.flight[i])) break;
        const EngFlight t = s.flight[p];
        s.flight[p] = s.flight[i];
        s.flight[i] = t;
        i = p;
    }
}

__device__ EngFlight heap_pop(EngState& s) {
    const EngFlight top = s.flight[0];
    s.flight[0] = s.flight[--s.n_flight];
    int i = 0;
    for (;;) {
        const int l = 2 * i + 1, r = l + 1;
        int m = i;
        if (l < s.n_flight && flight_later(s.flight[m], s.flight[l])) m = l;
        if (r < s.n_flight && flight_later(s.flight[m], s.flight[r])) m = r;
        if (m == i) break;
        const EngFlight t = s.flight[m];
        s.flight[m] = s.flight[i];
        s.flight[i] = t;
        i = m;
    }
    return top;
}

__device__ void eng_arrive(const EngDev& E, EngState& s, int idx) {  // cs_engine::arrive
    E.t_arrival[idx] = s.sim_now;
    ++s.tick;  // emit(RequestArrival)
    s.ready[(s.ready_head + s.ready_n) % (kMaxConc + 1)] = idx;
    ++s.ready_n;
}

__device__ void eng_activate(const EngDev& E, EngState& s) {  // cs_engine::activate_sessions
    while (s.active_sessions < s.conc && s.next_session < s.n_sessions) {
        const int sid = s.next_session++;
        ++s.active_sessions;
        E.session_pos[sid] = 0;
        eng_arrive(E, s, E.sess_reqs[E.sess_off[sid]]);
    }
}

__device__ void eng_complete(const DevPool& P, const EngDev& E, EngState& s) {  // cs_engine::complete_earliest
    const EngFlight f = heap_pop(s);
    s.sim_now = f.end_us;
    ++s.tick;  // emit(TurnComplete)
    const EngReq r = E.reqs[f.req];
    // defer the unpin to the next admission (cs_pool::defer_unpin)
    if (f.npins > 0) {
        if (s.n_unpin == kMaxUnpinRanges) {  // more completions than ranges: unpin here (rare)
            long long dec = 0;
            for (int k = 0; k < s.n_unpin; ++k)
                for (int i = 0; i < s.unpin_n[k]; ++i) {
                    const unsigned int us = s.unpin_ptr[k][i];
                    if (us != kNoSlot && atomicSub(&P.refs[us], 1u) == 1u) {
                        pk_unpinned(P, us);
                        ++dec;
                        if (P.dbg_unpin) P.dbg_unpin[us] = (s.seq << 8) | 4u;
                    }
                }
            P.ctrl->pinned -= dec;
            s.n_unpin = 0;
            s.unpin_slots = 0;
            s.pre_ok = 0;  // pool changed outside an admission launch
        }
        s.unpin_ptr[s.n_unpin] = E.pins + r.blk_off;
        s.unpin_n[s.n_unpin] = f.npins;
        ++s.n_unpin;
        s.unpin_slots += f.npins;
    }
    const int sid = r.session;
    const int pos = ++E.session_pos[sid];
    if (pos < E.sess_off[sid + 1] - E.sess_off[sid]) {
        eng_arrive(E, s, E.sess_reqs[E.sess_off[sid] + pos]);
    } else {
        --s.active_sessions;
    }
    E.t_cached[f.req] = f.cached;
    E.t_prompt[f.req] = r.prompt_tokens;
    E.t_start[f.req] = f.start_us;
    E.t_end[f.req] = f.end_us;
    E.t_done[f.req] = 1;
    s.tot_prompt += r.prompt_tokens;
    s.tot_cached += f.cached;
    ++s.completed;
}

// Fills E.args for one admission (cs_engine::try_start_head / execute_warmup through
// cs_pool::admit): the deferred unpins, the poll reset, speculation / prescan flags.
__device__ void eng_issue(const DevPool& P, const EngDev& E, EngState& s, long long blk_off, int nb, int flags,
                          int prev, int next, unsigned int agent, int anchor) {
    AdmitArgs& a = *E.args;
    a.keys = E.keys + blk_off;
    a.counts = E.counts + blk_off;
    a.n = nb;
    a.prev = prev;
    a.next = next;
    a.agent = agent;
    a.anchor = anchor;
    a.tick_base = s.tick;
    a.n_agents = 0;  // set by the kernel (the pool's agent count)
    a.pins_out = E.pins + blk_off;
    if (s.poll_reset_pending) flags |= kPollReset;
    a.n_unpin_ranges = s.n_unpin;
    for (int k = 0; k < s.n_unpin; ++k) {
        a.unpin_ptr[k] = s.unpin_ptr[k];
        a.unpin_n[k] = s.unpin_n[k];
    }
    const int cur_unpins = s.unpin_slots;
    s.n_unpin = 0;
    s.unpin_slots = 0;
    a.seq = ++s.seq;
    if (s.speculate && nb + cur_unpins <= kXsetMax) flags |= kSpeculate;
    if (s.prescan) flags |= kPrescan;
    a.n_prev_ranges = 0;
    if ((flags & kPrescan) && s.use_prescan && s.pre_ok && cur_unpins + s.prev_slots <= kXsetMax && s.n_prev <= kMaxUnpinRanges + 1) {
        flags |= kUsePrescan;
        for (int k = 0; k < s.n_prev; ++k) {
            a.prev_ptr[k] = s.prev_ptr[k];
            a.prev_n[k] = s.prev_n[k];
        }
        a.n_prev_ranges = s.n_prev;
    }
    a.flags = flags;
    s.pre_ok = 0;
    ++s.admissions;
}

// After an admission (cs_pool::admit's epilogue): the next prescan reuse, the poll reset.
__device__ void eng_admitted(const DevPool& P, const EngDev& E, EngState& s, const AdmSmem& A) {
    const AdmitArgs& a = *E.args;
    s.poll_reset_pending = 0;
    s.n_prev = 0;
    s.prev_slots = 0;
    for (int r = 0; r < a.n_unpin_ranges; ++r) {
        s.prev_ptr[s.n_prev] = a.unpin_ptr[r];
        s.prev_n[s.n_prev] = a.unpin_n[r];
        ++s.n_prev;
        s.prev_slots += a.unpin_n[r];
    }
    if ((a.flags & kUnpinAfter) && A.started && !A.error && A.admit_n > 0) {
        s.prev_ptr[s.n_prev] = a.pins_out;
        s.prev_n[s.n_prev] = A.admit_n;
        ++s.n_prev;
        s.prev_slots += A.admit_n;
    }
    s.pre_ok = (a.flags & kPrescan) && !A.error ? 1 : 0;
    if (A.error) s.error = 2;  // evict_one: all resident blocks are pinned
}

// One scheduler move on CTA 0 thread 0: advances the step coroutine until it needs an admission
// (returns 0 with E.args filled), the launch's admission budget is reached or the trace is done
// (returns 1). `last` is the status of the admission just run (first call: none).
__device__ int eng_schedule(const DevPool& P, const EngDev& E, EngState& s, const AdmSmem& A, bool have_last,
                            long long stop_at, long long max_steps, long long steps0) {
    if (have_last) eng_admitted(P, E, s, A);
    for (;;) {
        if (s.error) return 1;
        switch (s.phase) {
            case kPhStep: {  // EngineSim::step (engine.cpp:372-392) / cs_engine::step
                const bool done = s.n_flight == 0 && s.ready_n == 0 && s.next_session >= s.n_sessions;
                if (done || s.admissions >= stop_at || s.steps - steps0 >= max_steps) return 1;
                eng_activate(E, s);
                s.progressed = 0;
                s.phase = kPhTry;
                break;
            }
            case kPhTry: {  // try_start_head (engine.cpp:328-370)
                if (s.ready_n == 0 || s.n_flight >= s.conc) {
                    s.phase = kPhNoProg;
                    break;
                }
                const int idx = s.ready[s.ready_head];
                const EngReq r = E.reqs[idx];
                const bool oversized = r.nb > s.budget;
                if (oversized && s.n_flight > 0) {  // oversized prompts run solo
                    s.phase = kPhNoProg;
                    break;
                }
                s.cur_req = idx;
                eng_issue(P, E, s, r.blk_off, r.nb,
                          kDispatch | kAdmit | (oversized ? kTruncate : (kFeasible | kLookup)), s.last_dispatched,
                          r.agent, (unsigned int)r.agent, r.anchor_blocks);
                s.phase = kPhTryResult;
                return 0;
            }
            case kPhTryResult: {
                if (!A.started) {  // wait for in-flight pins to clear
                    s.phase = kPhNoProg;
                    break;
                }
                const int idx = s.cur_req;
                const EngReq r = E.reqs[idx];
                const bool oversized = r.nb > s.budget;
                s.ready_head = (s.ready_head + 1) % (kMaxConc + 1);
                --s.ready_n;
                s.last_dispatched = r.agent;
                s.tick = A.tick;
                if (oversized) ++s.truncated;
                EngFlight f;
                f.seq = s.flight_seq++;
                f.req = idx;
                f.npins = A.admit_n;
                f.cached = oversized ? 0 : A.cached;
                f.start_us = s.sim_now;
                const double ttft =
                    __dadd_rn(s.cost_base, __dmul_rn(s.cost_tok, (double)(r.prompt_tokens - f.cached)));
                f.end_us = __dadd_rn(__dadd_rn(s.sim_now, ttft), __dmul_rn(s.cost_dec, (double)r.decode));
                f.pad = 0;
                heap_push(s, f);
                s.progressed = 1;
                s.phase = kPhTry;
                break;
            }
            case kPhNoProg: {
                if (!s.progressed) {
                    if (s.n_flight > 0) {
                        eng_complete(P, E, s);
                    } else if (s.ready_n > 0) {
                        s.error = 1;  // scheduler stalled with an idle engine
                        return 1;
                    }
                }
                s.phase = kPhDrain;
                break;
            }
            case kPhDrain: {  // drain_and_run_warmups (engine.cpp:230-238) via poll_actions
                Ctrl* C = P.ctrl;
                // the host drains the last admission's status list; with no admission since the
                // previous drain that list is empty (the device list is reset lazily, kPollReset)
                const int np = s.poll_reset_pending ? 0 : min(C->n_pend, kMaxPending);
                s.n_fx = np;
                for (int k = 0; k < np; ++k) {
                    s.fx[k] = C->pend_target[k];
                    s.fx_tick[k] = C->pend_tick[k];
                    if (s.n_warm >= E.w_cap) {
                        s.error = 3;
                        return 1;
                    }
                    E.w_step[s.n_warm] = s.steps;
                    E.w_target[s.n_warm] = E.agent_ids[s.fx[k]];
                    E.w_tick[s.n_warm] = s.fx_tick[k];
                    ++s.n_warm;
                }
                s.poll_reset_pending = 1;
                s.warm_i = 0;
                s.phase = s.prefetch ? kPhWarm : kPhStepEnd;
                break;
            }
            case kPhWarm: {  // execute_warmup (engine.cpp:197-228)
                if (s.warm_i >= s.n_fx) {
                    s.phase = kPhStepEnd;
                    break;
                }
                const int t = s.fx[s.warm_i];
                const EngCat c = E.cat[t];
                if (c.nb == 0) {
                    ++s.warm_drop;
                    ++s.warm_i;
                    break;
                }
                eng_issue(P, E, s, c.blk_off, c.nb, kLookup | kAdmit | kWarmupRoom | kUnpinAfter, -1, -1,
                          (unsigned int)t, -1);
                s.phase = kPhWarmResult;
                return 0;
            }
            case kPhWarmResult: {
                s.tick = A.tick;
                ++s.warm_exec;
                s.warm_prompt += E.cat[s.fx[s.warm_i]].prompt_tokens;
                ++s.warm_i;
                s.phase = kPhWarm;
                break;
            }
            case kPhStepEnd: {
                ++s.steps;
                s.phase = kPhStep;
                break;
            }
        }
    }
}

// The grid-wide table rebuild (launch_table_rebuild) inside the persistent launch.
__device__ void eng_table_rebuild(const DevPool& P) {
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long e = i0; e <= (long long)P.tmask; e += stride) {
        P.table[e].slot = kSlotEmpty;
        P.table[e].key = 0ull;
    }
    grid_barrier(P.ctrl);
    for (long long s = i0; s < P.cap; s += stride)
        if (P.lt[s] != kFreeTick) table_insert(P, P.key[s], (unsigned int)s);
    grid_barrier(P.ctrl);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.ctrl->tombstones = 0;
        P.ctrl->tq_erase = 0;
        P.ctrl->tq_insert = 0;
    }
}

__global__ void __launch_bounds__(kThreads + 32, 1) engine_kernel(DevPool P, EngDev E, long long stop_at,
                                                                  long long max_steps, int n_agents) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ ScanSmem S;
    __shared__ SelectSmem Sel;
    __shared__ RedSmem Red;
    __shared__ AdmSmem A;
    __shared__ AdmitArgs a;
    __shared__ long long steps0;
    const int tid = threadIdx.x, T = blockDim.x;
    // The scheduler state lives in global memory across admissions (admit_body owns all of the
    // dynamic shared memory); CTA 0 stages it on chip, in the TMA ring, around each decision.
    EngState& es = *reinterpret_cast<EngState*>(dsm + kOffRing);
    static_assert(sizeof(EngState) <= kRing * kRingStage, "scheduler state must fit the TMA ring");
    if (blockIdx.x == 0 && tid == 0) {
        steps0 = E.st->steps;
        A.srv_t0 = 0;
    }
    bool have_last = false;
    for (;;) {
        if (blockIdx.x == 0) {
            {
                const int* src = reinterpret_cast<const int*>(E.st);
                int* dst = reinterpret_cast<int*>(&es);
                for (int i = tid; i < (int)(sizeof(EngState) / 4); i += T) dst[i] = __ldcg(src + i);
            }
            __syncthreads();
            if (tid == 0) {
                int cmd = eng_schedule(P, E, es, A, have_last, stop_at, max_steps, steps0);
                if (cmd == 0 && (unsigned long long)(P.ctrl->resident + P.ctrl->tombstones) > (P.tmask + 1) / 2) {
                    // table rebuild first (the host driver rebuilds after the admission that
                    // crossed the bound; here it runs before the next one: same table contents)
                    cmd = 2;
                    ++es.table_rebuilds;
                }
                *E.cmd = cmd;
            }
            __syncthreads();
            {
                const int* src = reinterpret_cast<const int*>(&es);
                int* dst = reinterpret_cast<int*>(E.st);
                for (int i = tid; i < (int)(sizeof(EngState) / 4); i += T) dst[i] = src[i];
            }
            __threadfence();
            __syncthreads();
        }
        grid_barrier(P.ctrl);
        const int cmd = *(volatile int*)E.cmd;
        if (cmd == 1) break;
        if (cmd == 2) {
            eng_table_rebuild(P);
            grid_barrier(P.ctrl);  // CTA 0 re-decides (the pending admission args stay in E.args)
            if (blockIdx.x == 0 && tid == 0) {
                *E.cmd = 0;
                __threadfence();
            }
            grid_barrier(P.ctrl);
        }
        {  // this admission's arguments, on chip in every CTA
            const int* src = reinterpret_cast<const int*>(E.args);
            int* dst = reinterpret_cast<int*>(&a);
            for (int i = tid; i < (int)(sizeof(AdmitArgs) / 4); i += T) dst[i] = __ldcg(src + i);
            __syncthreads();
            if (tid == 0) {
                a.n_agents = n_agents;
                a.status = nullptr;
            }
            __syncthreads();
        }
        admit_body(P, a, dsm, S, Sel, Red, A);
        __syncthreads();
        fence_proxy_async_smem();  // this admission's generic writes before the next TMA reads
        have_last = true;
    }
}

cudaError_t launch_engine(const DevPool& P, const EngDev& E, long long stop_at, long long max_steps, int n_agents,
                          const LaunchCfg& lc, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lc.smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    DevPool p = P;
    // In one persistent launch, bulk (TMA) reads of pool slots could return values older than
    // the L2 loads see after the previous admission's writes (observed on small pools; a kernel
    // boundary per admission never showed it): the engine kernel streams with L2 loads.
    p.stream_generic = 1;
    EngDev e = E;
    long long sa = stop_at, ms = max_steps;
    int na = n_agents;
    void* args[] = {&p, &e, &sa, &ms, &na};
    return cudaLaunchCooperativeKernel((const void*)engine_kernel, dim3(lc.grid), dim3(lc.threads), args, lc.smem, s);
}
