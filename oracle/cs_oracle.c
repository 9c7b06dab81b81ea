/* TEST INFRASTRUCTURE ONLY — plain-C CPU oracle for the CacheSage per-step hot path.
 * See cs_oracle.h for the contract. Every function cites the reference file:line (relative to
 * /root/reference/proj) whose behaviour it restates. Deliberately simple: the eviction scan is
 * the reference's O(N)-per-eviction argmin, not the GPU's batched design, so the two are
 * independent derivations of the same decisions.
 * Build with -ffp-contract=off: w_pred*S + rho must not become an FMA. */
#include "cs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- hashing (L0) */

/* hashing.hpp:13-14 */
static const uint64_t kSeed = 0x5ca9e5a6e0f1c3b7ULL;
static const uint64_t kRoot = 0x9d2c5680f0a5b4d1ULL;
static const uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

/* splitmix64 finalizer, hashing.hpp:17-22 */
uint64_t cso_mix64(uint64_t x) {
    x += kGolden;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* hashing.cpp:26-35 */
uint64_t cso_chain_hash(int has_parent, uint64_t parent, const uint32_t* t, size_t n, int* err) {
    if (n == 0) {
        if (err) *err = 1;
        return 0;
    }
    uint64_t h = cso_mix64(kSeed ^ (has_parent ? parent : kRoot));
    for (size_t i = 0; i < n; ++i) h = cso_mix64(h ^ ((uint64_t)t[i] + kGolden));
    return h;
}

/* hashing.cpp:37-51 */
long cso_block_keys(const uint32_t* t, size_t n, int bs, uint64_t* keys, int32_t* counts) {
    if (bs <= 0) return -1;
    long nb = 0;
    int has_parent = 0;
    uint64_t parent = 0;
    for (size_t off = 0; off < n; off += (size_t)bs) {
        size_t m = n - off < (size_t)bs ? n - off : (size_t)bs;
        uint64_t k = cso_chain_hash(has_parent, parent, t + off, m, NULL);
        keys[nb] = k;
        counts[nb] = (int32_t)m;
        ++nb;
        parent = k;
        has_parent = 1;
    }
    return nb;
}

/* derive_agent_identity, cachesage_policy.cpp:9-31 */
int cso_identity(const uint64_t* keys, size_t n, int skip, int take, uint64_t* out) {
    if (skip < 0 || take < 1 || n == 0) return -1;
    size_t lo = 0, hi = n;
    if (n >= (size_t)skip + (size_t)take) {
        lo = (size_t)skip;
        hi = (size_t)skip + (size_t)take;
    } else if (n > (size_t)skip) {
        lo = (size_t)skip;
    }
    uint64_t h = cso_mix64(kSeed ^ 0xa9e0c7d35b1f64e9ULL);
    for (size_t i = lo; i < hi; ++i) h = cso_mix64(h ^ keys[i]);
    *out = h;
    return 0;
}

/* ---------------------------------------------------------------- generator (L4) */

/* std::mt19937_64 (the standard's published recurrence; workload.cpp:161 seeds one per session) */
typedef struct {
    uint64_t mt[312];
    int mti;
} mt64;

static void mt64_seed(mt64* r, uint64_t s) {
    r->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
}

static uint64_t mt64_next(mt64* r) {
    static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (r->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag[x & 1ULL];
        }
        for (; i < 311; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1ULL];
        }
        x = (r->mt[311] & UM) | (r->mt[0] & LM);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag[x & 1ULL];
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* draw_uniform_int, workload.cpp:134-136 */
static int draw_uniform_int(mt64* r, int lo, int hi) {
    return lo + (int)(mt64_next(r) % (uint64_t)(hi - lo + 1));
}

/* draw_categorical, workload.cpp:138-153 */
static int draw_categorical(mt64* r, const double* row, int n) {
    const double u = (double)(mt64_next(r) >> 11) * 0x1.0p-53;
    double acc = 0.0;
    int last = 0;
    for (int i = 0; i < n; ++i) {
        if (row[i] <= 0.0) continue;
        last = i;
        acc += row[i];
        if (u < acc) return last;
    }
    return last;
}

/* generate_trace, workload.cpp:156-182 */
long cso_generate(const cso_spec* s, int64_t* turns7, long cap) {
    long n = 0;
    const int start = s->supervisor >= 0 ? s->supervisor : 0;
    for (int sess = 0; sess < s->sessions; ++sess) {
        mt64 r;
        mt64_seed(&r, cso_mix64(s->seed ^ cso_mix64(0x5e5510ULL + (uint64_t)sess)));
        const int turns = draw_uniform_int(&r, s->turns_min, s->turns_max);
        int agent = start;
        if (s->supervisor == -2 && s->start_dist) agent = draw_categorical(&r, s->start_dist, s->n_agents);
        for (int t = 0; t < turns; ++t) {
            if (t > 0) agent = draw_categorical(&r, s->transition + (size_t)agent * s->n_agents, s->n_agents);
            if (n < cap && turns7) {
                int64_t* o = turns7 + 7 * n;
                o[0] = sess;
                o[1] = t;
                o[2] = agent;
                o[3] = s->anchor_tokens[agent];
                o[4] = (int64_t)s->task_tokens + (int64_t)t * s->history_growth;
                o[5] = s->template_tokens + o[3] + o[4];
                o[6] = s->decode_tokens;
            }
            ++n;
        }
    }
    return n;
}

static uint32_t anchor_stride(const cso_spec* s) { return s->anchor_stride ? s->anchor_stride : 0x00010000u; }
static int pos_bits(const cso_spec* s) { return s->hist_pos_bits ? s->hist_pos_bits : 20; }

/* Trace::turn_tokens, workload.cpp:125-140 (history_token :126-129) */
long cso_turn_tokens(const cso_spec* s, const int64_t* t7, uint32_t* out, long cap) {
    long n = 0;
    for (int j = 0; j < s->template_tokens; ++j) {
        if (n < cap) out[n] = 0x00100000u + (uint32_t)j;
        ++n;
    }
    const uint32_t ab = 0x01000000u + (uint32_t)t7[2] * anchor_stride(s);
    for (int64_t j = 0; j < t7[3]; ++j) {
        if (n < cap) out[n] = ab + (uint32_t)j;
        ++n;
    }
    for (int64_t p = 0; p < t7[4]; ++p) {
        if (n < cap) out[n] = 0x80000000u | ((uint32_t)t7[0] << pos_bits(s)) | (uint32_t)p;
        ++n;
    }
    return n;
}

/* Trace::warmup_tokens, workload.cpp:142-154 */
static long warmup_tokens(const cso_spec* s, int agent, uint32_t* out) {
    long n = 0;
    for (int j = 0; j < s->template_tokens; ++j) out[n++] = 0x00100000u + (uint32_t)j;
    const uint32_t ab = 0x01000000u + (uint32_t)agent * anchor_stride(s);
    for (int j = 0; j < s->anchor_tokens[agent]; ++j) out[n++] = ab + (uint32_t)j;
    out[n++] = 0x02000000u;
    return n;
}

/* ---------------------------------------------------------------- policy (L1/L2) */

typedef struct {
    uint64_t* ids; /* agent id per index */
    long n, cap;
    long* tab; /* open addressing: index+1, 0 empty */
    long tcap;
} agent_map;

static long amap_get(agent_map* m, uint64_t id, int insert) {
    uint64_t h = cso_mix64(id) & (uint64_t)(m->tcap - 1);
    for (;;) {
        long v = m->tab[h];
        if (v == 0) {
            if (!insert || m->n >= m->cap) return -1;
            m->ids[m->n] = id;
            m->tab[h] = m->n + 1;
            return m->n++;
        }
        if (m->ids[v - 1] == id) return v - 1;
        h = (h + 1) & (uint64_t)(m->tcap - 1);
    }
}

typedef struct {
    cso_cfg cfg;
    agent_map am;
    long A;            /* capacity */
    uint64_t* counts;  /* A*A */
    uint64_t* totals;  /* A */
    /* per row, its nonzero columns (any order; hops and argmax are order-independent):
     * nz[a*A + k], k < nnz[a]; nzpos[a*A + b] = k */
    long* nz;
    long* nzpos;
    long* nnz;
    long* win_a;       /* ring */
    long* win_b;
    long win_head, win_size, win_cap;
    int* hops; /* A */
    int reach_built;
    long current; /* -1 none */
    int step_warmups;
    uint64_t* pend_target;
    uint64_t* pend_tick;
    long n_pend, pend_cap;
    uint64_t rebuilds;
    /* BeladyPolicy (baselines.cpp:34-46): every request block as (key, request id, chain
     * position), sorted, and the cursor (highest arrived request id, :48-52) */
    uint64_t* bel_key;
    uint64_t* bel_req;
    int* bel_pos;
    long bel_n;
    uint64_t cursor;
} policy;

static void cell_inc(policy* p, long a, long b) {
    if (p->counts[a * p->A + b]++ == 0) {
        p->nzpos[a * p->A + b] = p->nnz[a];
        p->nz[a * p->A + p->nnz[a]++] = b;
    }
    p->totals[a]++;
}

/* erase zero cells (transition_learner.cpp:40-47) */
static void cell_dec(policy* p, long a, long b) {
    p->totals[a]--;
    if (--p->counts[a * p->A + b] == 0) {
        const long k = p->nzpos[a * p->A + b];
        const long last = p->nz[a * p->A + --p->nnz[a]];
        p->nz[a * p->A + k] = last;
        p->nzpos[a * p->A + last] = k;
    }
}

/* TransitionLearner::record, transition_learner.cpp:22-51 (note_agent :16-20 is the alphabet,
 * which does not influence any decision; indices come from the agent map). */
static void learner_record(policy* p, long a, long b) {
    long pos = (p->win_head + p->win_size) % p->win_cap;
    if (p->win_size == p->win_cap) {
        /* window full: the appended pair overwrites the oldest slot after it is retired */
        long oa = p->win_a[p->win_head], ob = p->win_b[p->win_head];
        p->win_a[p->win_head] = a;
        p->win_b[p->win_head] = b;
        cell_inc(p, a, b);
        cell_dec(p, oa, ob);
        p->win_head = (p->win_head + 1) % p->win_cap;
        return;
    }
    p->win_a[pos] = a;
    p->win_b[pos] = b;
    p->win_size++;
    cell_inc(p, a, b);
}

/* rebuild_reachability, reachability.cpp:39-81: FIFO BFS from current over edges with
 * count/total >= tau; no expansion when depth+1 >= e_max; unknown agents stay at e_max. */
static void rebuild(policy* p, long cur) {
    const int e = p->cfg.e_max;
    for (long i = 0; i < p->am.n; ++i) p->hops[i] = e;
    p->hops[cur] = 0;
    long* q = (long*)malloc(sizeof(long) * (size_t)(p->am.n + 1) * 2);
    long qh = 0, qt = 0;
    q[qt++] = cur;
    while (qh < qt) {
        long a = q[qh++];
        int d = p->hops[a];
        if (d + 1 >= e) continue;
        if (p->totals[a] == 0) continue;
        const double total = (double)p->totals[a];
        for (long k = 0; k < p->nnz[a]; ++k) {
            const long b = p->nz[a * p->A + k];
            uint64_t c = p->counts[a * p->A + b];
            if ((double)c / total < p->cfg.tau) continue;
            if (p->hops[b] > d + 1) {
                p->hops[b] = d + 1;
                q[qt++] = b;
            }
        }
    }
    free(q);
    p->reach_built = 1;
}

/* argmax_row, transition_learner.cpp:79-96: max count, ties -> smaller AgentId value */
static int argmax_row(const policy* p, long a, long* best, double* prob) {
    if (p->totals[a] == 0) return 0;
    uint64_t bc = 0;
    long bi = -1;
    for (long k = 0; k < p->nnz[a]; ++k) {
        const long b = p->nz[a * p->A + k];
        uint64_t c = p->counts[a * p->A + b];
        if (bi < 0 || c > bc || (c == bc && p->am.ids[b] < p->am.ids[bi])) {
            bi = b;
            bc = c;
        }
    }
    if (bi < 0) return 0;
    *best = bi;
    *prob = (double)bc / (double)p->totals[a];
    return 1;
}

/* CacheSagePolicy::observe(AgentDispatch), cachesage_policy.cpp:57-72, with maybe_prefetch
 * :109-123. LRU (baselines.cpp:10) observes nothing. */
static void observe_dispatch(policy* p, long prev, long next, uint64_t tick) {
    if (p->cfg.policy != 1) return; /* LruPolicy / TtlPolicy / BeladyPolicy ignore dispatches */
    if (prev >= 0) learner_record(p, prev, next);
    const int changed = p->current < 0 || p->current != next;
    p->current = next;
    if (changed) {
        rebuild(p, next);
        p->rebuilds++;
    }
    if (p->step_warmups >= p->cfg.budget_per_step) return;
    if (p->totals[next] < p->cfg.min_row_count) return;
    long best;
    double prob;
    if (!argmax_row(p, next, &best, &prob) || prob < p->cfg.min_confidence) return;
    p->step_warmups++;
    if (p->n_pend == p->pend_cap) {
        p->pend_cap = p->pend_cap ? p->pend_cap * 2 : 16;
        p->pend_target = (uint64_t*)realloc(p->pend_target, sizeof(uint64_t) * (size_t)p->pend_cap);
        p->pend_tick = (uint64_t*)realloc(p->pend_tick, sizeof(uint64_t) * (size_t)p->pend_cap);
    }
    p->pend_target[p->n_pend] = p->am.ids[best];
    p->pend_tick[p->n_pend] = tick;
    p->n_pend++;
}

/* recency_residual, runtime.cpp:23-32 */
static double recency(uint64_t lt, uint64_t now, uint64_t old) {
    if (now <= old) return 1.0;
    const double span = (double)(now - old);
    const double off = lt >= old ? (double)(lt - old) : 0.0;
    double r = off / span;
    if (r < 0.0) r = 0.0;
    if (r > 1.0) r = 1.0;
    return r;
}

/* CacheSagePolicy::score, cachesage_policy.cpp:79-85 (+ ReachabilityState::survival,
 * reachability.cpp:12-20); LruPolicy::score, baselines.cpp:12-14 */
/* BeladyPolicy::score, baselines.cpp:54-70 */
static double belady_score(const policy* p, uint64_t key) {
    long lo = 0, hi = p->bel_n;
    while (lo < hi) { /* first entry of the key */
        long m = (lo + hi) / 2;
        if (p->bel_key[m] < key) lo = m + 1;
        else hi = m;
    }
    if (lo == p->bel_n || p->bel_key[lo] != key) return 0.0;
    const int depth = p->bel_pos[lo]; /* depth_.emplace: the first occurrence */
    long j = lo, e = p->bel_n;
    while (j < e) { /* std::upper_bound of the cursor in the key's request ids (:60) */
        long m = (j + e) / 2;
        if (p->bel_key[m] < key || (p->bel_key[m] == key && p->bel_req[m] <= p->cursor)) j = m + 1;
        else e = m;
    }
    if (j == p->bel_n || p->bel_key[j] != key) return 0.0; /* never referenced again */
    const double nudge = 1e-10 * (double)depth;
    return 1.0 / (1.0 + (double)(p->bel_req[j] - p->cursor)) - nudge;
}

static double score(const policy* p, long agent, uint64_t lt, uint64_t now, uint64_t old) {
    const double rho = recency(lt, now, old);
    if (p->cfg.policy == 0) return rho;
    double surv = 0.0;
    if (agent >= 0 && p->reach_built) {
        int h = p->hops[agent];
        if (h > p->cfg.e_max) h = p->cfg.e_max;
        surv = 1.0 - (double)h / (double)p->cfg.e_max;
    }
    return p->cfg.w_pred * surv + rho;
}

/* ---------------------------------------------------------------- engine pool (L3) */

typedef struct {
    uint64_t key, lt;
    double lt_us;
    long agent;
    int32_t tokens, refs, used;
} entry;

struct cso_engine {
    cso_cfg cfg;
    policy pol;
    entry* ent;
    long n_ent_cap;
    long* free_stack;
    long n_free;
    long* tab; /* entry index + 1, 0 = empty */
    long tcap;
    long resident, pinned;
    uint64_t tick;
    double sim_now;
    long last_dispatched; /* agent index or -1 */
    uint64_t* ev;
    long n_ev, ev_cap;
    int error;
    /* fast_evict index (see lheap below): grp[g] holds the unpinned resident blocks of agent
     * index g (g = A: agentless) keyed by last_touch; all holds every resident block. */
    int fast;
    struct lheap* grp;
    long n_grp;
    struct lheap* all;
};

static long tab_find(const cso_engine* e, uint64_t key) {
    uint64_t h = cso_mix64(key) & (uint64_t)(e->tcap - 1);
    for (;;) {
        long v = e->tab[h];
        if (v == 0) return -1;
        if (e->ent[v - 1].key == key) return v - 1;
        h = (h + 1) & (uint64_t)(e->tcap - 1);
    }
}

static void tab_insert(cso_engine* e, uint64_t key, long idx) {
    uint64_t h = cso_mix64(key) & (uint64_t)(e->tcap - 1);
    while (e->tab[h]) h = (h + 1) & (uint64_t)(e->tcap - 1);
    e->tab[h] = idx + 1;
}

/* linear-probing delete with backward shift */
static void tab_erase(cso_engine* e, uint64_t key) {
    const uint64_t m = (uint64_t)(e->tcap - 1);
    uint64_t h = cso_mix64(key) & m;
    while (e->ent[e->tab[h] - 1].key != key) h = (h + 1) & m;
    uint64_t hole = h, j = h;
    for (;;) {
        j = (j + 1) & m;
        long v = e->tab[j];
        if (v == 0) break;
        uint64_t home = cso_mix64(e->ent[v - 1].key) & m;
        /* move v into the hole if its home is not in (hole, j] cyclically */
        int in_range = hole <= j ? (home > hole && home <= j) : (home > hole || home <= j);
        if (!in_range) {
            e->tab[hole] = v;
            hole = j;
        }
    }
    e->tab[hole] = 0;
}

/* ---------------------------------------------------------------- indexed evict_one
 *
 * The class-head lemma: a block's score is f(survival(hop(agent)), rho(lt)) with
 * rho monotone in last_touch (runtime.cpp:23-32) and fp64 rounding monotone, so among the
 * unpinned blocks of ONE agent the reference's argmin (engine.cpp:106-118, tie on
 * (score, last_touch, key)) is the one with the smallest last_touch. evict_one therefore only
 * needs each agent's oldest unpinned block: it scores those heads with the same score() and
 * picks the (score, last_touch, key) minimum — the reference's own comparison over a subset
 * that provably contains its victim. oldest_live_touch (engine.cpp:90-96) is the top of a heap
 * of every resident block. This is an independent derivation from the GPU's (one scan per
 * admission, per-class lists, dominance replay); both must agree with the O(N) argmin, which
 * the tests check on every golden fixture.
 *
 * Lazy heaps: an entry (lt, idx) is live iff ent[idx] is resident with that last_touch (and,
 * for the group heaps, unpinned). last_touch values are never reused, so a stale entry can
 * never become live again. Heaps are compacted when stale entries outnumber live ones. */
typedef struct {
    uint64_t lt;
    long idx;
} hnode;

typedef struct lheap {
    hnode* a;
    long n, cap, live;
    /* cached live top (group heaps): valid unless dirty; hidx < 0 = empty */
    uint64_t hlt;
    long hidx;
    int dirty;
} lheap;

static void lh_push_raw(lheap* h, uint64_t lt, long idx) {
    if (h->n == h->cap) {
        h->cap = h->cap ? h->cap * 2 : 16;
        h->a = (hnode*)realloc(h->a, sizeof(hnode) * (size_t)h->cap);
    }
    h->a[h->n].lt = lt;
    h->a[h->n].idx = idx;
    h->n++;
}

static void lh_down(lheap* h, long i) {
    const hnode x = h->a[i];
    for (;;) {
        long l = 2 * i + 1;
        if (l >= h->n) break;
        if (l + 1 < h->n && h->a[l + 1].lt < h->a[l].lt) ++l;
        if (h->a[l].lt >= x.lt) break;
        h->a[i] = h->a[l];
        i = l;
    }
    h->a[i] = x;
}

static void lh_up(lheap* h, long i) {
    const hnode x = h->a[i];
    while (i > 0) {
        long p = (i - 1) / 2;
        if (h->a[p].lt <= x.lt) break;
        h->a[i] = h->a[p];
        i = p;
    }
    h->a[i] = x;
}

static void lh_heapify(lheap* h) {
    for (long i = h->n / 2 - 1; i >= 0; --i) lh_down(h, i);
}

static void lh_pop(lheap* h) {
    h->a[0] = h->a[--h->n];
    if (h->n > 0) lh_down(h, 0);
}

static int live_all(const cso_engine* e, const hnode* x) {
    return e->ent[x->idx].used && e->ent[x->idx].lt == x->lt;
}

static int live_grp(const cso_engine* e, const hnode* x) {
    return live_all(e, x) && e->ent[x->idx].refs == 0;
}

static void lh_compact(cso_engine* e, lheap* h, int grp) {
    long m = 0;
    for (long i = 0; i < h->n; ++i)
        if (grp ? live_grp(e, &h->a[i]) : live_all(e, &h->a[i])) h->a[m++] = h->a[i];
    h->n = m;
    lh_heapify(h);
    h->dirty = 1;
}

static void lh_push(cso_engine* e, lheap* h, uint64_t lt, long idx, int grp) {
    lh_push_raw(h, lt, idx);
    lh_up(h, h->n - 1);
    h->live++;
    h->dirty = 1;
    if (h->n > 2 * h->live + 64) lh_compact(e, h, grp);
}

static lheap* grp_of(cso_engine* e, long idx) {
    const long a = e->ent[idx].agent;
    return &e->grp[a >= 0 ? a : e->n_grp - 1];
}

/* hooks: the index follows every change of (resident, last_touch, refs == 0) */
static void ix_touched(cso_engine* e, long idx, int was_resident) {
    if (!e->fast) return;
    if (was_resident) e->all->live--; /* the previous (lt, idx) entry went stale */
    lh_push(e, e->all, e->ent[idx].lt, idx, 0);
}

static void ix_join_grp(cso_engine* e, long idx) { /* unpinned member at its current last_touch */
    if (e->fast) lh_push(e, grp_of(e, idx), e->ent[idx].lt, idx, 1);
}

static void ix_leave_grp(cso_engine* e, long idx) { /* pinned, touched, or evicted while unpinned */
    if (!e->fast) return;
    lheap* h = grp_of(e, idx);
    h->live--;
    if (h->hidx == idx) h->dirty = 1;
}

static void ix_evicted(cso_engine* e, long idx) {
    if (!e->fast) return;
    e->all->live--;
    if (e->ent[idx].refs == 0) ix_leave_grp(e, idx);
}

cso_engine* cso_engine_new(const cso_cfg* cfg, long agent_cap) {
    cso_engine* e = (cso_engine*)calloc(1, sizeof(cso_engine));
    e->cfg = *cfg;
    e->n_ent_cap = cfg->budget_blocks;
    e->ent = (entry*)calloc((size_t)e->n_ent_cap, sizeof(entry));
    e->free_stack = (long*)malloc(sizeof(long) * (size_t)e->n_ent_cap);
    for (long i = 0; i < e->n_ent_cap; ++i) e->free_stack[i] = e->n_ent_cap - 1 - i;
    e->n_free = e->n_ent_cap;
    e->tcap = 16;
    while (e->tcap < 2 * e->n_ent_cap + 16) e->tcap *= 2;
    e->tab = (long*)calloc((size_t)e->tcap, sizeof(long));
    e->last_dispatched = -1;
    policy* p = &e->pol;
    p->cfg = *cfg;
    if (agent_cap < 1) agent_cap = 1;
    p->A = agent_cap;
    p->am.cap = agent_cap;
    p->am.ids = (uint64_t*)calloc((size_t)agent_cap, sizeof(uint64_t));
    p->am.tcap = 16;
    while (p->am.tcap < 2 * agent_cap + 16) p->am.tcap *= 2;
    p->am.tab = (long*)calloc((size_t)p->am.tcap, sizeof(long));
    p->counts = (uint64_t*)calloc((size_t)(agent_cap * agent_cap), sizeof(uint64_t));
    p->totals = (uint64_t*)calloc((size_t)agent_cap, sizeof(uint64_t));
    p->nz = (long*)malloc(sizeof(long) * (size_t)(agent_cap * agent_cap));
    p->nzpos = (long*)malloc(sizeof(long) * (size_t)(agent_cap * agent_cap));
    p->nnz = (long*)calloc((size_t)agent_cap, sizeof(long));
    p->win_cap = cfg->window > 0 ? cfg->window : 1024;
    p->win_a = (long*)malloc(sizeof(long) * (size_t)p->win_cap);
    p->win_b = (long*)malloc(sizeof(long) * (size_t)p->win_cap);
    p->hops = (int*)calloc((size_t)agent_cap, sizeof(int));
    p->current = -1;
    e->fast = cfg->fast_evict && cfg->policy != 3;
    if (e->fast) {
        e->n_grp = agent_cap + 1;
        e->grp = (lheap*)calloc((size_t)e->n_grp, sizeof(lheap));
        for (long g = 0; g < e->n_grp; ++g) e->grp[g].dirty = 1;
        e->all = (lheap*)calloc(1, sizeof(lheap));
    }
    return e;
}

void cso_engine_free(cso_engine* e) {
    if (!e) return;
    free(e->ent);
    free(e->free_stack);
    free(e->tab);
    free(e->ev);
    free(e->pol.am.ids);
    free(e->pol.am.tab);
    free(e->pol.counts);
    free(e->pol.totals);
    free(e->pol.nz);
    free(e->pol.nzpos);
    free(e->pol.nnz);
    free(e->pol.win_a);
    free(e->pol.win_b);
    free(e->pol.hops);
    free(e->pol.pend_target);
    free(e->pol.pend_tick);
    free(e->pol.bel_key);
    free(e->pol.bel_req);
    free(e->pol.bel_pos);
    if (e->fast) {
        for (long g = 0; g < e->n_grp; ++g) free(e->grp[g].a);
        free(e->grp);
        free(e->all->a);
        free(e->all);
    }
    free(e);
}

static long agent_index(cso_engine* e, uint64_t id) { return amap_get(&e->pol.am, id, 1); }


/* EngineSim::touch, engine.cpp:79-88 (BlockTouch events are no-ops for both policies).
 * was_resident = 0 for a block admit_pinned just inserted. */
static void touch(cso_engine* e, long idx, int was_resident) {
    e->ent[idx].lt = ++e->tick;
    e->ent[idx].lt_us = e->sim_now;
    ix_touched(e, idx, was_resident);
}

/* the fast_evict victim: the (score, last_touch, key) minimum over each agent group's oldest
 * unpinned block (see the lemma above); -1 when every resident block is pinned. Groups that
 * share a survival value score by the same function of last_touch, so only the oldest head per
 * survival class is scored (LRU and TTL scores do not depend on the agent: one class). */
static long fast_victim(cso_engine* e) {
    uint64_t old = e->tick;
    lheap* all = e->all;
    while (all->n > 0 && !live_all(e, &all->a[0])) lh_pop(all);
    if (all->n > 0 && all->a[0].lt < old) old = all->a[0].lt;
    const policy* p = &e->pol;
    const int cs = p->cfg.policy == 1 && p->reach_built;
    const int emax = p->cfg.e_max;
    long cand[65];
    const int ncls = cs ? (emax < 64 ? emax : 64) + 1 : 1;
    for (int c = 0; c < ncls; ++c) cand[c] = -1;
    for (long g = 0; g < e->n_grp; ++g) {
        lheap* h = &e->grp[g];
        if (h->dirty) {
            while (h->n > 0 && !live_grp(e, &h->a[0])) lh_pop(h);
            h->hidx = h->n > 0 ? h->a[0].idx : -1;
            h->hlt = h->n > 0 ? h->a[0].lt : 0;
            h->dirty = 0;
        }
        if (h->hidx < 0) continue;
        int c = 0;
        if (cs) {
            const int hop = g < e->n_grp - 1 ? p->hops[g] : emax;
            c = hop < emax ? hop : emax;
            if (c > 64) c = 64;
        }
        if (cand[c] < 0 || h->hlt < e->ent[cand[c]].lt) cand[c] = h->hidx;
    }
    long v = -1;
    double vs = 0.0;
    for (int c = 0; c < ncls; ++c) {
        if (cand[c] < 0) continue;
        const entry* x = &e->ent[cand[c]];
        double s;
        if (p->cfg.policy == 2) { /* TtlPolicy::score, baselines.cpp:22-28 */
            const double rho = recency(x->lt, e->tick, old);
            s = e->sim_now - x->lt_us < 5000000.0 ? 1.0e6 + rho : rho;
        } else {
            s = score(p, x->agent, x->lt, e->tick, old);
        }
        if (v < 0 || s < vs ||
            (s == vs && (x->lt < e->ent[v].lt || (x->lt == e->ent[v].lt && x->key < e->ent[v].key)))) {
            v = cand[c];
            vs = s;
        }
    }
    return v;
}

/* EngineSim::evict_one, engine.cpp:102-125 with score_context/oldest_live_touch :90-100 */
static int evict_one(cso_engine* e) {
    if (e->fast) {
        const long v = fast_victim(e);
        if (v < 0) return -1; /* "evict_one: all resident blocks are pinned" */
        ix_evicted(e, v);
        tab_erase(e, e->ent[v].key);
        if (e->n_ev == e->ev_cap) {
            e->ev_cap = e->ev_cap ? e->ev_cap * 2 : 1024;
            e->ev = (uint64_t*)realloc(e->ev, sizeof(uint64_t) * (size_t)e->ev_cap);
        }
        e->ev[e->n_ev++] = e->ent[v].key;
        e->ent[v].used = 0;
        e->free_stack[e->n_free++] = v;
        e->resident--;
        return 0;
    }
    uint64_t old = e->tick;
    for (long i = 0; i < e->n_ent_cap; ++i)
        if (e->ent[i].used && e->ent[i].lt < old) old = e->ent[i].lt;
    long v = -1;
    double vs = 0.0;
    for (long i = 0; i < e->n_ent_cap; ++i) {
        const entry* x = &e->ent[i];
        if (!x->used || x->refs > 0) continue;
        double s;
        if (e->pol.cfg.policy == 3) {
            s = belady_score(&e->pol, x->key);
        } else if (e->pol.cfg.policy == 2) { /* TtlPolicy::score, baselines.cpp:22-28 */
            const double rho = recency(x->lt, e->tick, old);
            s = e->sim_now - x->lt_us < 5000000.0 ? 1.0e6 + rho : rho;
        } else {
            s = score(&e->pol, x->agent, x->lt, e->tick, old);
        }
        if (v < 0 || s < vs ||
            (s == vs && (x->lt < e->ent[v].lt || (x->lt == e->ent[v].lt && x->key < e->ent[v].key)))) {
            v = i;
            vs = s;
        }
    }
    if (v < 0) return -1; /* "evict_one: all resident blocks are pinned" */
    tab_erase(e, e->ent[v].key);
    if (e->n_ev == e->ev_cap) {
        e->ev_cap = e->ev_cap ? e->ev_cap * 2 : 1024;
        e->ev = (uint64_t*)realloc(e->ev, sizeof(uint64_t) * (size_t)e->ev_cap);
    }
    e->ev[e->n_ev++] = e->ent[v].key;
    e->ent[v].used = 0;
    e->free_stack[e->n_free++] = v;
    e->resident--;
    return 0;
}

/* EngineSim::lookup, engine.cpp:127-139 */
long cso_engine_lookup(cso_engine* e, const uint64_t* keys, const int32_t* counts, long n, long* first_miss) {
    long cached = 0, i = 0;
    for (; i < n; ++i) {
        long idx = tab_find(e, keys[i]);
        if (idx < 0) break;
        cached += counts[i];
        const int unpinned = e->ent[idx].refs == 0;
        if (unpinned) ix_leave_grp(e, idx);
        touch(e, idx, 1);
        if (unpinned) ix_join_grp(e, idx);
    }
    if (first_miss) *first_miss = i;
    return cached;
}

int cso_engine_dispatch(cso_engine* e, uint64_t agent) {
    long a = agent_index(e, agent);
    if (a < 0) return -1;
    const uint64_t t = ++e->tick;
    observe_dispatch(&e->pol, e->last_dispatched, a, t);
    e->last_dispatched = a;
    return 0;
}

/* EngineSim::admit_pinned, engine.cpp:141-168 (budget assert :190-195) */
static long admit_pinned(cso_engine* e, const uint64_t* keys, const int32_t* counts, long n, long agent,
                         int anchor, long* pins) {
    for (long i = 0; i < n; ++i) {
        long idx = tab_find(e, keys[i]);
        const int fresh = idx < 0;
        if (idx < 0) {
            while (e->resident >= e->cfg.budget_blocks) {
                if (evict_one(e) != 0) {
                    e->error = 1;
                    return -1;
                }
            }
            idx = e->free_stack[--e->n_free];
            entry* x = &e->ent[idx];
            x->key = keys[i];
            x->tokens = counts[i];
            x->agent = (agent >= 0 && i < anchor) ? agent : -1;
            x->refs = 0;
            x->used = 1;
            tab_insert(e, keys[i], idx);
            e->resident++;
        }
        if (!fresh && e->ent[idx].refs == 0) ix_leave_grp(e, idx);
        touch(e, idx, !fresh);
        if (e->ent[idx].refs++ == 0) e->pinned++;
        if (pins) pins[i] = idx;
    }
    return n;
}

int cso_engine_admit_pinned(cso_engine* e, const uint64_t* keys, const int32_t* counts, long n, int has_agent,
                            uint64_t agent, int anchor) {
    long a = has_agent ? agent_index(e, agent) : -1;
    return admit_pinned(e, keys, counts, n, a, anchor, NULL) < 0 ? -1 : 0;
}

/* EngineSim::unpin, engine.cpp:170-180 */
static int unpin_idx(cso_engine* e, const long* idx, long n) {
    for (long i = 0; i < n; ++i)
        if (--e->ent[idx[i]].refs == 0) {
            e->pinned--;
            ix_join_grp(e, idx[i]);
        }
    return 0;
}

int cso_engine_unpin(cso_engine* e, const uint64_t* keys, long n) {
    for (long i = 0; i < n; ++i) {
        long idx = tab_find(e, keys[i]);
        if (idx < 0) return -1; /* "unpin: block vanished while referenced" */
        if (--e->ent[idx].refs == 0) {
            e->pinned--;
            ix_join_grp(e, idx);
        }
    }
    return 0;
}

int cso_engine_restore(cso_engine* e, const uint64_t* keys, const uint64_t* lt, const int32_t* has_agent,
                       const uint64_t* agents, const int32_t* refs, long n, uint64_t tick) {
    for (long i = 0; i < n; ++i) {
        if (e->n_free == 0 || tab_find(e, keys[i]) >= 0) return -1;
        long idx = e->free_stack[--e->n_free];
        entry* x = &e->ent[idx];
        x->key = keys[i];
        x->lt = lt[i];
        x->lt_us = 0.0;
        x->tokens = 16;
        x->agent = has_agent[i] ? agent_index(e, agents[i]) : -1;
        x->refs = refs ? refs[i] : 0;
        x->used = 1;
        if (x->refs > 0) e->pinned++;
        tab_insert(e, keys[i], idx);
        e->resident++;
        if (e->fast) {
            lh_push(e, e->all, x->lt, idx, 0);
            if (x->refs == 0) ix_join_grp(e, idx);
        }
    }
    if (tick > e->tick) e->tick = tick;
    return 0;
}

long cso_engine_evictions(const cso_engine* e, uint64_t* out, long cap) {
    for (long i = 0; i < e->n_ev && i < cap; ++i) out[i] = e->ev[i];
    return e->n_ev;
}
uint64_t cso_engine_tick(const cso_engine* e) { return e->tick; }
long cso_engine_resident(const cso_engine* e) { return e->resident; }
long cso_engine_pinned(const cso_engine* e) { return e->pinned; }

/* CacheSagePolicy::poll_actions, cachesage_policy.cpp:125-130 */
long cso_engine_poll(cso_engine* e, uint64_t* targets, uint64_t* ticks, long cap) {
    policy* p = &e->pol;
    p->step_warmups = 0;
    long n = p->n_pend;
    for (long i = 0; i < n && i < cap; ++i) {
        if (targets) targets[i] = p->pend_target[i];
        if (ticks) ticks[i] = p->pend_tick[i];
    }
    p->n_pend = 0;
    return n;
}

int cso_engine_hops(const cso_engine* e, const uint64_t* agents, long n, int* hops) {
    for (long i = 0; i < n; ++i) {
        if (!e->pol.reach_built) {
            hops[i] = -1;
            continue;
        }
        long a = amap_get((agent_map*)&e->pol.am, agents[i], 0);
        hops[i] = a < 0 ? e->cfg.e_max : e->pol.hops[a];
    }
    return 0;
}

long cso_engine_scores(const cso_engine* e, uint64_t* keys, double* scores, long cap) {
    uint64_t old = e->tick;
    for (long i = 0; i < e->n_ent_cap; ++i)
        if (e->ent[i].used && e->ent[i].lt < old) old = e->ent[i].lt;
    long n = 0;
    for (long i = 0; i < e->n_ent_cap; ++i) {
        if (!e->ent[i].used) continue;
        if (n < cap) {
            keys[n] = e->ent[i].key;
            scores[n] = score(&e->pol, e->ent[i].agent, e->ent[i].lt, e->tick, old);
        }
        ++n;
    }
    return n;
}

/* ---------------------------------------------------------------- scheduler (L3) */

typedef struct {
    uint64_t* keys;
    int32_t* counts;
    long nb;
    long prompt_tokens;
    int decode_tokens;
    int anchor_blocks;
    int session;
    uint64_t agent;
} req_t;

typedef struct {
    double end_us;
    uint64_t seq;
    long req;
    long* pins;
    long npins;
    long cached;
    double start_us;
} flight_t;

/* min-heap on (end_us, seq): InFlight::later, engine.hpp:153-155 */
static int flight_less(const flight_t* a, const flight_t* b) {
    return a->end_us < b->end_us || (a->end_us == b->end_us && a->seq < b->seq);
}

static void heap_push(flight_t* h, long* n, flight_t f) {
    long i = (*n)++;
    h[i] = f;
    while (i > 0) {
        long p = (i - 1) / 2;
        if (!flight_less(&h[i], &h[p])) break;
        flight_t t = h[i];
        h[i] = h[p];
        h[p] = t;
        i = p;
    }
}

static flight_t heap_pop(flight_t* h, long* n) {
    flight_t top = h[0];
    h[0] = h[--(*n)];
    long i = 0;
    for (;;) {
        long l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && flight_less(&h[l], &h[m])) m = l;
        if (r < *n && flight_less(&h[r], &h[m])) m = r;
        if (m == i) break;
        flight_t t = h[i];
        h[i] = h[m];
        h[m] = t;
        i = m;
    }
    return top;
}

/* CostModel defaults, engine.hpp:20-24 */
static const double kPrefillPerTok = 50.0, kPrefillBase = 1000.0, kDecodePerTok = 20000.0;

static void push_u64(uint64_t** a, long* n, long* cap, uint64_t v) {
    if (*n == *cap) {
        *cap = *cap ? *cap * 2 : 64;
        *a = (uint64_t*)realloc(*a, sizeof(uint64_t) * (size_t)*cap);
    }
    (*a)[(*n)++] = v;
}

typedef struct {
    uint64_t key, req;
    int pos;
} bel_t;

static int bel_cmp(const void* x, const void* y) {
    const bel_t* a = (const bel_t*)x;
    const bel_t* b = (const bel_t*)y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->req != b->req) return a->req < b->req ? -1 : 1;
    return a->pos < b->pos ? -1 : a->pos > b->pos;
}

/* run_cell (experiment.cpp:355-379) -> EngineSim::run (engine.cpp:415-421): load (:240-255),
 * step (:372-392), activate/arrive (:262-276), try_start_head (:325-351), start_request
 * (:278-323), complete_earliest (:353-370), drain_and_run_warmups/execute_warmup (:197-238). */
int cso_run(const cso_spec* s, const cso_cfg* cfg_in, cso_run_out* out) {
    return cso_run_ex(s, cfg_in, NULL, -1, out);
}

int cso_run_ex(const cso_spec* s, const cso_cfg* cfg_in, const cso_snapshot* snap, long max_steps,
               cso_run_out* out) {
    memset(out, 0, sizeof(*out));
    cso_cfg cfg = *cfg_in;
    if (cfg.budget_blocks <= 0) cfg.budget_blocks = s->budget_blocks;
    if (cfg.concurrency <= 0) cfg.concurrency = s->concurrency;
    /* EngineSim ctor validation, engine.cpp:57-63 (0 selects the CostModel default) */
    const double c_base = cfg.prefill_base_us != 0.0 ? cfg.prefill_base_us : kPrefillBase;
    const double c_tok = cfg.prefill_per_token_us != 0.0 ? cfg.prefill_per_token_us : kPrefillPerTok;
    const double c_dec = cfg.decode_per_token_us != 0.0 ? cfg.decode_per_token_us : kDecodePerTok;
    if (c_base <= 0.0 || c_tok <= 0.0 || c_dec <= 0.0) return -3; /* invalid_argument */
    const int bs = cfg.block_size;
    const long nt = cso_generate(s, NULL, 0);
    int64_t* t7 = (int64_t*)malloc(sizeof(int64_t) * 7 * (size_t)(nt > 0 ? nt : 1));
    cso_generate(s, t7, nt);

    /* materialize_requests, engine.cpp:8-35 */
    req_t* rq = (req_t*)calloc((size_t)(nt > 0 ? nt : 1), sizeof(req_t));
    long tokcap = 1 << 16;
    uint32_t* tok = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)tokcap);
    for (long i = 0; i < nt; ++i) {
        long m = cso_turn_tokens(s, t7 + 7 * i, tok, tokcap);
        if (m > tokcap) {
            tokcap = m;
            tok = (uint32_t*)realloc(tok, sizeof(uint32_t) * (size_t)tokcap);
            cso_turn_tokens(s, t7 + 7 * i, tok, tokcap);
        }
        long nb = (m + bs - 1) / bs;
        rq[i].keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nb > 0 ? nb : 1));
        rq[i].counts = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nb > 0 ? nb : 1));
        rq[i].nb = cso_block_keys(tok, (size_t)m, bs, rq[i].keys, rq[i].counts);
        rq[i].prompt_tokens = m;
        rq[i].decode_tokens = (int)t7[7 * i + 6];
        rq[i].anchor_blocks = (int)((s->template_tokens + t7[7 * i + 3]) / bs);
        rq[i].session = (int)t7[7 * i + 0];
        cso_identity(rq[i].keys, (size_t)rq[i].nb, cfg.skip, cfg.take, &rq[i].agent);
    }
    /* build_warmup_catalog, engine.cpp:37-54 */
    req_t* cat = (req_t*)calloc((size_t)s->n_agents, sizeof(req_t));
    for (int a = 0; a < s->n_agents; ++a) {
        long need = s->template_tokens + s->anchor_tokens[a] + 1;
        if (need > tokcap) {
            tokcap = need;
            tok = (uint32_t*)realloc(tok, sizeof(uint32_t) * (size_t)tokcap);
        }
        long m = warmup_tokens(s, a, tok);
        long nb = (m + bs - 1) / bs;
        cat[a].keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)nb);
        cat[a].counts = (int32_t*)malloc(sizeof(int32_t) * (size_t)nb);
        cat[a].nb = cso_block_keys(tok, (size_t)m, bs, cat[a].keys, cat[a].counts);
        cat[a].prompt_tokens = m;
        cso_identity(cat[a].keys, (size_t)cat[a].nb, cfg.skip, cfg.take, &cat[a].agent);
    }
    free(tok);

    /* size the agent alphabet: distinct identities over requests + catalog */
    long distinct = 0;
    {
        agent_map tmp;
        memset(&tmp, 0, sizeof(tmp));
        tmp.cap = nt + s->n_agents + 1;
        tmp.ids = (uint64_t*)calloc((size_t)tmp.cap, sizeof(uint64_t));
        tmp.tcap = 16;
        while (tmp.tcap < 2 * tmp.cap + 16) tmp.tcap *= 2;
        tmp.tab = (long*)calloc((size_t)tmp.tcap, sizeof(long));
        for (long i = 0; i < nt; ++i) amap_get(&tmp, rq[i].agent, 1);
        for (int a = 0; a < s->n_agents; ++a) amap_get(&tmp, cat[a].agent, 1);
        distinct = tmp.n;
        free(tmp.ids);
        free(tmp.tab);
    }
    cso_engine* e = cso_engine_new(&cfg, distinct + 1);
    int rc = 0;
    if (snap && snap->n > 0) {
        uint64_t mx = 0;
        for (long i = 0; i < snap->n; ++i)
            if (snap->last_touch[i] > mx) mx = snap->last_touch[i];
        if (snap->n > cfg.budget_blocks ||
            cso_engine_restore(e, snap->keys, snap->last_touch, snap->has_agent, snap->agents, snap->refs, snap->n,
                               mx) != 0)
            rc = -4; /* invalid snapshot */
    }
    if (cfg.policy == 3) {
        long nb = 0;
        for (long i = 0; i < nt; ++i) nb += rq[i].nb;
        bel_t* t = (bel_t*)malloc(sizeof(bel_t) * (size_t)(nb > 0 ? nb : 1));
        long k = 0;
        for (long i = 0; i < nt; ++i)
            for (long b = 0; b < rq[i].nb; ++b) {
                t[k].key = rq[i].keys[b];
                t[k].req = (uint64_t)i;
                t[k].pos = (int)b;
                ++k;
            }
        qsort(t, (size_t)nb, sizeof(bel_t), bel_cmp);
        policy* p = &e->pol;
        p->bel_n = nb;
        p->bel_key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nb > 0 ? nb : 1));
        p->bel_req = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nb > 0 ? nb : 1));
        p->bel_pos = (int*)malloc(sizeof(int) * (size_t)(nb > 0 ? nb : 1));
        for (long i = 0; i < nb; ++i) {
            p->bel_key[i] = t[i].key;
            p->bel_req[i] = t[i].req;
            p->bel_pos[i] = t[i].pos;
        }
        free(t);
    }

    /* sessions ascending (std::map order); requests per session in trace order */
    int max_sess = 0;
    for (long i = 0; i < nt; ++i)
        if (rq[i].session > max_sess) max_sess = rq[i].session;
    long* sess_cnt = (long*)calloc((size_t)max_sess + 2, sizeof(long));
    for (long i = 0; i < nt; ++i) sess_cnt[rq[i].session + 1]++;
    for (int k = 1; k <= max_sess + 1; ++k) sess_cnt[k] += sess_cnt[k - 1];
    long* sess_req = (long*)malloc(sizeof(long) * (size_t)(nt > 0 ? nt : 1));
    long* fill = (long*)calloc((size_t)max_sess + 1, sizeof(long));
    for (long i = 0; i < nt; ++i) sess_req[sess_cnt[rq[i].session] + fill[rq[i].session]++] = i;
    free(fill);
    long* pending = (long*)malloc(sizeof(long) * ((size_t)max_sess + 1));
    long np_head = 0, np_tail = 0;
    for (int k = 0; k <= max_sess; ++k)
        if (sess_cnt[k + 1] > sess_cnt[k]) pending[np_tail++] = k;
    long* sess_pos = (long*)calloc((size_t)max_sess + 1, sizeof(long));
    long* ready = (long*)malloc(sizeof(long) * (size_t)(nt + 1));
    long rd_head = 0, rd_tail = 0;
    double* arrival = (double*)calloc((size_t)(nt > 0 ? nt : 1), sizeof(double));
    flight_t* heap = (flight_t*)malloc(sizeof(flight_t) * (size_t)(cfg.concurrency + 1));
    long nheap = 0;
    uint64_t flight_seq = 0;
    int active = 0;

    out->n_turns = nt;
    out->cached_tokens = (long*)calloc((size_t)(nt > 0 ? nt : 1), sizeof(long));
    out->prompt_tokens = (long*)calloc((size_t)(nt > 0 ? nt : 1), sizeof(long));
    out->start_us = (double*)calloc((size_t)(nt > 0 ? nt : 1), sizeof(double));
    out->end_us = (double*)calloc((size_t)(nt > 0 ? nt : 1), sizeof(double));
    long w_cap = 0, w_n = 0;
    uint64_t *w_target = NULL, *w_tick = NULL, *w_step = NULL;
    long wt_cap = 0, wt_n = 0, ws_cap = 0, ws_n = 0;
    out->completed = (uint8_t*)calloc((size_t)(nt > 0 ? nt : 1), 1);
    long long tot_prompt = 0, tot_cached = 0;
    long steps = 0, completed = 0;
    if (rc != 0) goto done;
    (void)w_cap;
    (void)w_n;

    for (;;) {
        if (max_steps >= 0 && steps >= max_steps) break;
        /* done() */
        if (nheap == 0 && rd_head == rd_tail && np_head == np_tail) break;
        /* activate_sessions */
        while (active < cfg.concurrency && np_head < np_tail) {
            int sid = (int)pending[np_head++];
            ++active;
            sess_pos[sid] = 0;
            long idx = sess_req[sess_cnt[sid]];
            arrival[idx] = e->sim_now;
            ++e->tick; /* RequestArrival: note_agent only; BeladyPolicy::observe moves the cursor */
            if ((uint64_t)idx > e->pol.cursor) e->pol.cursor = (uint64_t)idx;
            agent_index(e, rq[idx].agent);
            ready[rd_tail++] = idx;
        }
        int progressed = 0;
        for (;;) {
            /* try_start_head */
            if (rd_head == rd_tail || nheap >= cfg.concurrency) break;
            long idx = ready[rd_head];
            req_t* r = &rq[idx];
            const int oversized = r->nb > cfg.budget_blocks;
            if (oversized) {
                if (nheap > 0) break;
            } else {
                long needed = 0;
                for (long b = 0; b < r->nb; ++b) {
                    long x = tab_find(e, r->keys[b]);
                    if (x < 0 || e->ent[x].refs == 0) ++needed;
                }
                if (e->pinned + needed > cfg.budget_blocks) break;
            }
            ++rd_head;
            progressed = 1;
            /* start_request */
            cso_engine_dispatch(e, r->agent);
            long cached = 0, admit_n = r->nb;
            if (oversized) {
                out->truncated++;
                admit_n = cfg.budget_blocks - e->pinned;
            } else {
                cached = cso_engine_lookup(e, r->keys, r->counts, r->nb, NULL);
            }
            flight_t f;
            f.seq = flight_seq++;
            f.req = idx;
            f.pins = (long*)malloc(sizeof(long) * (size_t)(admit_n > 0 ? admit_n : 1));
            f.npins = admit_n;
            long ai = agent_index(e, r->agent);
            if (admit_pinned(e, r->keys, r->counts, admit_n, ai, r->anchor_blocks, f.pins) < 0) {
                rc = -1;
                goto done;
            }
            out->n_admissions++;
            const double ttft = c_base + c_tok * (double)(r->prompt_tokens - cached);
            f.end_us = e->sim_now + ttft + c_dec * r->decode_tokens;
            f.cached = cached;
            f.start_us = e->sim_now;
            heap_push(heap, &nheap, f);
        }
        if (!progressed) {
            if (nheap > 0) {
                /* complete_earliest */
                flight_t f = heap_pop(heap, &nheap);
                e->sim_now = f.end_us;
                ++e->tick; /* TurnComplete */
                unpin_idx(e, f.pins, f.npins);
                free(f.pins);
                int sid = rq[f.req].session;
                if (++sess_pos[sid] < sess_cnt[sid + 1] - sess_cnt[sid]) {
                    long nx = sess_req[sess_cnt[sid] + sess_pos[sid]];
                    arrival[nx] = e->sim_now;
                    ++e->tick;
                    if ((uint64_t)nx > e->pol.cursor) e->pol.cursor = (uint64_t)nx;
                    agent_index(e, rq[nx].agent);
                    ready[rd_tail++] = nx;
                } else {
                    --active;
                }
                out->cached_tokens[f.req] = f.cached;
                out->prompt_tokens[f.req] = rq[f.req].prompt_tokens;
                out->start_us[f.req] = f.start_us;
                out->end_us[f.req] = f.end_us;
                out->completed[f.req] = 1;
                tot_prompt += rq[f.req].prompt_tokens;
                tot_cached += f.cached;
                ++completed;
            } else if (rd_head != rd_tail) {
                rc = -2; /* "scheduler stalled with an idle engine" */
                goto done;
            }
        }
        /* drain_and_run_warmups */
        {
            policy* p = &e->pol;
            long nfx = p->n_pend;
            uint64_t* fx = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nfx > 0 ? nfx : 1));
            for (long i = 0; i < nfx; ++i) {
                fx[i] = p->pend_target[i];
                push_u64(&w_target, &wt_n, &wt_cap, p->pend_target[i]);
                push_u64(&w_tick, &ws_n, &ws_cap, p->pend_tick[i]);
                push_u64(&w_step, &w_n, &w_cap, (uint64_t)steps);
            }
            p->n_pend = 0;
            p->step_warmups = 0;
            if (cfg.prefetch) {
                for (long i = 0; i < nfx; ++i) {
                    req_t* c = NULL;
                    for (int a = 0; a < s->n_agents; ++a)
                        if (cat[a].agent == fx[i]) {
                            c = &cat[a];
                            break;
                        }
                    if (!c) {
                        out->warmups_dropped++;
                        continue;
                    }
                    long room = cfg.budget_blocks - e->pinned;
                    long admit_n = c->nb < room ? c->nb : room;
                    cso_engine_lookup(e, c->keys, c->counts, c->nb, NULL);
                    long* pins = (long*)malloc(sizeof(long) * (size_t)(admit_n > 0 ? admit_n : 1));
                    long ai = agent_index(e, c->agent);
                    if (admit_pinned(e, c->keys, c->counts, admit_n, ai, (int)admit_n, pins) < 0) {
                        free(pins);
                        free(fx);
                        rc = -1;
                        goto done;
                    }
                    unpin_idx(e, pins, admit_n);
                    free(pins);
                    out->warmups_executed++;
                    out->n_admissions++;
                }
            }
            free(fx);
        }
        ++steps;
    }
done:
    out->n_evictions = e->n_ev;
    out->evictions = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(e->n_ev > 0 ? e->n_ev : 1));
    if (e->n_ev) memcpy(out->evictions, e->ev, sizeof(uint64_t) * (size_t)e->n_ev);
    out->n_warmups = wt_n;
    out->warmup_target = w_target;
    out->warmup_tick = w_tick;
    out->warmup_step = (long*)malloc(sizeof(long) * (size_t)(w_n > 0 ? w_n : 1));
    for (long i = 0; i < w_n; ++i) out->warmup_step[i] = (long)w_step[i];
    free(w_step);
    out->hit_rate = tot_prompt > 0 ? (double)tot_cached / (double)tot_prompt : 0.0;
    out->sim_us = e->sim_now;
    out->n_steps = steps;
    (void)completed;
    for (long i = 0; i < nt; ++i) {
        free(rq[i].keys);
        free(rq[i].counts);
    }
    for (int a = 0; a < s->n_agents; ++a) {
        free(cat[a].keys);
        free(cat[a].counts);
    }
    while (nheap > 0) free(heap[--nheap].pins);
    free(rq);
    free(cat);
    free(t7);
    free(sess_cnt);
    free(sess_req);
    free(pending);
    free(sess_pos);
    free(ready);
    free(arrival);
    free(heap);
    cso_engine_free(e);
    return rc;
}

void cso_free_run(cso_run_out* o) {
    free(o->cached_tokens);
    free(o->prompt_tokens);
    free(o->start_us);
    free(o->end_us);
    free(o->evictions);
    free(o->warmup_step);
    free(o->warmup_target);
    free(o->warmup_tick);
    free(o->completed);
    memset(o, 0, sizeof(*o));
}
