/*
 * semsched_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded-per-trace restatement of the reference
 * scheduler (arXiv 2506.12204 package `semsched`, /root/reference/pkg/src/
 * semsched) used (a) as the parity checker for the CUDA path in tests/ and
 * __graft_entry__.smoke(), and (b) as the bench's CPU baseline ("port").
 * It is never linked into, imported by, or called from the product path.
 *
 * It follows the reference's own data structures: an indexed binary
 * min-heap for dispatch, the same heap over negated keys for eviction and a
 * FIFO arrival buffer (heaps.py:32-237), tuple keys compared
 * lexicographically exactly like Python tuples (requests.py:81-97), and the
 * engine loop statement by statement (engine.py:169-421).
 *
 * Parity pinned against the reference itself: tests/golden/make_golden.py
 * imports /root/reference and records outputs; tests/test_oracle_golden.py
 * checks this file reproduces them bit-for-bit.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (see oracle/Makefile).
 * -ffp-contract=off matters: the reference's float64 chains must not be
 * fused into FMAs (SURVEY.md §7 hard part 1).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/semsched_b200.h"

/* ------------------------------------------------------------------ */
/* Request state: requests.py:100-125                                 */
/* ------------------------------------------------------------------ */
enum { ST_WAITING = 0, ST_PREFILLING = 1, ST_DECODING = 2, ST_EVICTED_OFF = 3,
       ST_EVICTED_DIS = 4, ST_COMPLETED = 5 };

typedef struct {
    /* static (ground truth + predictions) */
    int64_t id;
    double arrival, ready;
    int64_t prompt, true_out, mid;
    int frank, trank;
    /* dynamic */
    double f_t;
    int64_t prefilled, decoded, kv_dev, kv_host;
    int stage;
    int64_t evictions;
    double first_sched, finish; /* NaN == None */
    /* heap bookkeeping */
    int hpos, gpos, in_buffer, unservable;
} oreq;

/* Dispatch key, a Python tuple. The policy decides which fields exist
 * (engine.py:114-123); absent leading fields are held at 0 so the
 * lexicographic comparison degenerates to the policy's tuple. */
typedef struct {
    int64_t rank;
    double ft;
    double arrival;
    int64_t id;
} okey;

static int key_lt(const okey* a, const okey* b) {
    if (a->rank != b->rank) return a->rank < b->rank;
    if (a->ft != b->ft) return a->ft < b->ft;
    if (a->arrival != b->arrival) return a->arrival < b->arrival;
    return a->id < b->id;
}

/* eviction_priority: negate every component (requests.py:94-97). */
static okey key_neg(okey k) {
    okey r;
    r.rank = -k.rank;
    r.ft = -k.ft;
    r.arrival = -k.arrival;
    r.id = -k.id;
    return r;
}

/* ------------------------------------------------------------------ */
/* cost model: costs.py:99-191                                         */
/* ------------------------------------------------------------------ */
typedef ss_profile prof;

static double prefill_time(int64_t n, const prof* p) {            /* costs.py:99-102 */
    double dn = (double)n;
    return p->alpha1 * dn * dn + p->alpha2 * dn;
}
static double decode_step_time(int64_t n, int64_t j, const prof* p) { /* :105-109 */
    return p->gamma1 * (double)(n + j - 1) + p->gamma2;
}
static double decode_total_time(int64_t n, int64_t m, const prof* p) { /* :112-116 */
    double dm = (double)m;
    /* 0.5*m*m + n*m + 0.5*m : n*m is a Python int product, then int->float */
    double inner = 0.5 * dm * dm + (double)(n * m);
    inner = inner + 0.5 * dm;
    return p->gamma1 * inner + p->gamma2 * dm;
}
static double reload_time(int64_t tokens, const prof* p) {         /* :119-122 */
    return p->beta_load * (double)tokens;
}
static int should_cache_prefill(int64_t n, const prof* p) {        /* :125-130 */
    return p->beta_load < p->alpha1 * (double)n + p->alpha2;
}
static double resume_cost(int64_t n, int64_t m_done, int64_t m_saved, const prof* p) { /* :133-139 */
    int64_t k = m_done - m_saved;
    return p->beta_load * (double)m_saved + decode_total_time(n, k, p);
}
static int64_t clamp_floor_ceil(double s_real, int64_t m_done, int use_ceil) {
    /* min(m_done, max(0, math.floor/ceil(s_real))) with Python ints */
    double v = use_ceil ? ceil(s_real) : floor(s_real);
    if (v <= 0.0) return 0;
    if (v >= (double)m_done) return m_done;
    return (int64_t)v;
}
static int64_t optimal_save_tokens(int64_t n, int64_t m_done, const prof* p) { /* :142-171 */
    if (m_done == 0) return 0;
    if (p->gamma1 == 0.0) {
        double lo = resume_cost(n, m_done, 0, p), hi = resume_cost(n, m_done, m_done, p);
        return hi <= lo ? m_done : 0;
    }
    double k_star = (p->beta_load - p->gamma1 * (double)n - p->gamma1 / 2 - p->gamma2) / p->gamma1;
    double s_real = (double)m_done - k_star;
    int64_t a = clamp_floor_ceil(s_real, m_done, 0);
    int64_t b = clamp_floor_ceil(s_real, m_done, 1);
    /* sorted(set) iterated ascending; ties -> larger s ("<=") */
    int64_t cands[2];
    int nc = 0;
    if (a == b) { cands[nc++] = a; }
    else { cands[nc++] = a < b ? a : b; cands[nc++] = a < b ? b : a; }
    int64_t best = -1;
    double best_cost = INFINITY;
    for (int i = 0; i < nc; i++) {
        double c = resume_cost(n, m_done, cands[i], p);
        if (c <= best_cost) { best = cands[i]; best_cost = c; }
    }
    return best;
}
static double estimate_remaining_time(const oreq* r, const prof* p) { /* :174-191 */
    double total = reload_time(r->kv_host, p);
    total += prefill_time(r->prompt - r->prefilled, p);
    int64_t remaining = r->mid - r->decoded;
    if (remaining < 1) remaining = 1;
    total += decode_total_time(r->prompt + r->decoded, remaining, p);
    return total;
}

/* CPython >= 3.12 builtin sum() over floats (Neumaier compensation),
 * the arithmetic behind sum(step_times) (engine.py:148) and the metrics. */
typedef struct { double s, c; int n; } pysum;
static void pysum_add(pysum* a, double x) {
    if (a->n == 0) { a->s = x; a->c = 0.0; a->n = 1; return; }  /* 0 + x */
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else a->c += (x - t) + a->s;
    a->s = t;
    a->n++;
}
static double pysum_value(const pysum* a) {
    if (a->n == 0) return 0.0;
    double s = a->s;
    if (a->c != 0.0 && isfinite(a->c)) s += a->c;
    return s;
}

/* ------------------------------------------------------------------ */
/* IndexedMinHeap: heaps.py:32-130                                    */
/* ------------------------------------------------------------------ */
typedef struct {
    okey* keys;
    int* items;     /* request indices */
    int n;
    int which;      /* 0 dispatch (hpos), 1 eviction (gpos) */
    oreq* reqs;
} oheap;

static int* posp(oheap* h, int item) {
    return h->which == 0 ? &h->reqs[item].hpos : &h->reqs[item].gpos;
}
static void h_swap(oheap* h, int i, int j) {
    if (i == j) return;
    okey tk = h->keys[i]; h->keys[i] = h->keys[j]; h->keys[j] = tk;
    int ti = h->items[i]; h->items[i] = h->items[j]; h->items[j] = ti;
    *posp(h, h->items[i]) = i;
    *posp(h, h->items[j]) = j;
}
static void h_sift_up(oheap* h, int i) {
    while (i > 0) {
        int parent = (i - 1) / 2;
        if (key_lt(&h->keys[i], &h->keys[parent])) { h_swap(h, i, parent); i = parent; }
        else break;
    }
}
static void h_sift_down(oheap* h, int i) {
    int n = h->n;
    for (;;) {
        int l = 2 * i + 1, r = 2 * i + 2, s = i;
        if (l < n && key_lt(&h->keys[l], &h->keys[s])) s = l;
        if (r < n && key_lt(&h->keys[r], &h->keys[s])) s = r;
        if (s == i) return;
        h_swap(h, i, s);
        i = s;
    }
}
static void h_insert(oheap* h, int item, okey k) {
    h->keys[h->n] = k;
    h->items[h->n] = item;
    *posp(h, item) = h->n;
    h->n++;
    h_sift_up(h, h->n - 1);
}
static int h_remove_at(oheap* h, int i) {
    int last = h->n - 1;
    h_swap(h, i, last);
    int item = h->items[last];
    h->n--;
    *posp(h, item) = -1;
    if (i < h->n) { h_sift_down(h, i); h_sift_up(h, i); }
    return item;
}
static int h_contains(oheap* h, int item) { return *posp(h, item) >= 0; }

/* ------------------------------------------------------------------ */
/* simulator                                                           */
/* ------------------------------------------------------------------ */
typedef struct {
    int victim, action;
    int64_t saved, discarded, freed;
    double ftb, fta;
} odecision;

typedef struct {
    const ss_params* P;
    prof p;
    int n;
    oreq* r;
    oheap heap, evq;
    int* buffer; int nbuf;
    int* ongoing; int nongoing;
    int64_t cap, used;
    double clock;
    /* outputs */
    uint32_t* unserv; int nunserv;
    int64_t eviction_count, rounds, peak;
    uint64_t digest;
    uint32_t* log; int64_t log_cap, log_len; int log_overflow;
    int status;
    int last_granted;
    int64_t lost_evictions, anomalies;
    int64_t sum_pool, sum_granted, sum_victims, sum_res_evict;
    int evict_round;
    /* scratch */
    int* cand; int* merged; int* granted; int* pushed;
    odecision* dec; int ndec, dec_cap;
    char* evicted_flag;
} osim;

static okey key_of(const osim* s, int i) {                 /* engine.py:114-123 */
    const oreq* r = &s->r[i];
    okey k;
    switch (s->P->policy) {
    case SS_POLICY_FCFS: k.rank = 0; k.ft = 0.0; break;
    case SS_POLICY_SJF: k.rank = 0; k.ft = r->f_t; break;
    case SS_POLICY_HPJF: k.rank = r->frank; k.ft = 0.0; break;
    default: k.rank = r->frank; k.ft = r->f_t; break;          /* priority_key */
    }
    k.arrival = r->arrival;
    k.id = r->id;
    return k;
}
static void heap_insert(osim* s, int i) {
    if (h_contains(&s->heap, i)) { s->status = SS_TRACE_REF_ERROR; return; } /* DuplicateRequestError */
    h_insert(&s->heap, i, key_of(s, i));
}
static void evq_insert(osim* s, int i) { h_insert(&s->evq, i, key_neg(key_of(s, i))); }
static void evq_update(osim* s, int i) {                       /* heaps.py:72-76,191-192 */
    if (h_contains(&s->evq, i)) h_remove_at(&s->evq, s->r[i].gpos);
    evq_insert(s, i);
}

static void push_dec(osim* s, odecision d) {
    if (s->ndec == s->dec_cap) {
        s->dec_cap = s->dec_cap ? 2 * s->dec_cap : 64;
        s->dec = (odecision*)realloc(s->dec, sizeof(odecision) * s->dec_cap);
    }
    s->dec[s->ndec++] = d;
}

/* stable insertion sort by key (total order -> same as Python sorted) */
static void sort_by_key(osim* s, int* a, int n) {
    for (int i = 1; i < n; i++) {
        int x = a[i];
        okey kx = key_of(s, x);
        int j = i - 1;
        while (j >= 0) {
            okey kj = key_of(s, a[j]);
            if (key_lt(&kx, &kj)) { a[j + 1] = a[j]; j--; }
            else break;
        }
        a[j + 1] = x;
    }
}

/* ArrivalBuffer.drain_into: FIFO into the dispatch heap (heaps.py:229-237) */
static void drain(osim* s) {
    for (int k = 0; k < s->nbuf; k++) { s->r[s->buffer[k]].in_buffer = 0; heap_insert(s, s->buffer[k]); }
    s->nbuf = 0;
}

static int needs_prefill(const oreq* r) { return r->stage != ST_DECODING; }  /* batching.py:39-43 */

/* Returns batch size; members written to s->merged[0..m), *kind set. */
static int schedule(osim* s, int* kind) {
    int b = s->P->batch_size;
    for (int k = 0; k < s->nongoing; k++) {                      /* engine.py:248-249 */
        oreq* r = &s->r[s->ongoing[k]];
        r->f_t = estimate_remaining_time(r, &s->p);
    }
    if (s->P->policy == SS_POLICY_SEMANTIC) {
        /* extract_top_b (batching.py:46-54) */
        drain(s);
        int nc = 0;
        while (nc < b && s->heap.n > 0) s->cand[nc++] = h_remove_at(&s->heap, 0);
        int np = nc + s->nongoing;
        if (np == 0) { *kind = SS_KIND_DECODE; return 0; }
        /* p* = min(pool) (batching.py:73-74) */
        int pstar = -1;
        okey kbest;
        for (int k = 0; k < np; k++) {
            int i = k < nc ? s->cand[k] : s->ongoing[k - nc];
            okey ki = key_of(s, i);
            if (pstar < 0 || key_lt(&ki, &kbest)) { pstar = i; kbest = ki; }
        }
        int nm = 0;
        if (needs_prefill(&s->r[pstar])) {                      /* :76-78 */
            for (int k = 0; k < nc; k++) s->merged[nm++] = s->cand[k];
            for (int k = 0; k < s->nongoing; k++) s->merged[nm++] = s->ongoing[k];
            *kind = SS_KIND_PREFILL;
        } else {                                                 /* :79-84 */
            for (int k = 0; k < nc; k++) {
                int i = s->cand[k];
                if (!needs_prefill(&s->r[i])) s->merged[nm++] = i;
            }
            for (int k = 0; k < nc; k++) {                       /* push_back prefill candidates */
                int i = s->cand[k];
                if (needs_prefill(&s->r[i])) heap_insert(s, i);
            }
            for (int k = 0; k < s->nongoing; k++) s->merged[nm++] = s->ongoing[k];
            *kind = SS_KIND_DECODE;
        }
        sort_by_key(s, s->merged, nm);
        int m = nm < b ? nm : b;
        for (int k = m; k < nm; k++) heap_insert(s, s->merged[k]);  /* :86-87 */
        return m;
    }
    if (s->P->policy == SS_POLICY_FCFS) {                       /* engine.py:256-268 */
        drain(s);
        int m = 0;
        for (int k = 0; k < s->nongoing; k++) s->merged[m++] = s->ongoing[k];
        while (m < b && s->heap.n > 0) s->merged[m++] = h_remove_at(&s->heap, 0);
        int anyp = 0;
        for (int k = 0; k < m; k++) anyp |= s->r[s->merged[k]].stage != ST_DECODING;
        *kind = anyp ? SS_KIND_PREFILL : SS_KIND_DECODE;
        return m;
    }
    /* SJF / HPJF: engine.py:270-285 */
    drain(s);
    int nc = 0;
    while (nc < b && s->heap.n > 0) s->cand[nc++] = h_remove_at(&s->heap, 0);
    int nm = 0;
    for (int k = 0; k < nc; k++) s->merged[nm++] = s->cand[k];
    for (int k = 0; k < s->nongoing; k++) s->merged[nm++] = s->ongoing[k];
    sort_by_key(s, s->merged, nm);
    int m = nm < b ? nm : b;
    for (int k = m; k < nm; k++) heap_insert(s, s->merged[k]);
    int anyp = 0;
    for (int k = 0; k < m; k++) anyp |= s->r[s->merged[k]].stage != ST_DECODING;
    *kind = anyp ? SS_KIND_PREFILL : SS_KIND_DECODE;
    return m;
}

/* should_recompute: kvcache.py:81-134 */
static odecision should_recompute(osim* s, int v) {
    oreq* r = &s->r[v];
    odecision d;
    d.victim = v;
    d.freed = r->kv_dev;
    d.ftb = r->f_t;
    int64_t prefill_saved;
    if (r->prefilled > 0 && should_cache_prefill(r->prefilled, &s->p)) {
        d.action = 0;
        prefill_saved = r->prefilled;
    } else {
        d.action = 1;
        prefill_saved = 0;
        r->prefilled = 0;
    }
    int64_t saved = r->decoded > 0 ? optimal_save_tokens(r->prompt, r->decoded, &s->p) : 0;
    if (d.action == 1 && s->P->dependency_rule) saved = 0;
    d.discarded = r->decoded - saved;
    r->decoded = saved;
    d.saved = saved;
    r->kv_dev = 0;
    r->kv_host = prefill_saved + saved;
    r->stage = ST_WAITING;   /* EVICTED_* -> WAITING, immediately re-queued */
    r->evictions += 1;
    r->f_t = estimate_remaining_time(r, &s->p);
    d.fta = r->f_t;
    return d;
}

/* priority_based_eviction: kvcache.py:137-179. Returns 0 ok, -1 AdmissionFailure. */
static int priority_based_eviction(osim* s, int ri, int64_t demand, const int* prot, int nprot) {
    int skipped_cap = s->evq.n + 1;
    int* skipped = (int*)malloc(sizeof(int) * skipped_cap);
    int nsk = 0, rc = 0;
    if (demand + s->used > s->cap && !s->evict_round) {
        s->evict_round = 1;
        s->sum_res_evict += s->evq.n;
    }
    while (demand + s->used > s->cap) {
        int victim = -1;
        while (s->evq.n > 0) {
            int cand = h_remove_at(&s->evq, 0);
            int is_prot = cand == ri;
            for (int k = 0; k < nprot && !is_prot; k++) is_prot = prot[k] == cand;
            if (is_prot) skipped[nsk++] = cand;
            else { victim = cand; break; }
        }
        if (victim < 0) { rc = -1; break; }
        if (h_contains(&s->heap, victim)) h_remove_at(&s->heap, s->r[victim].hpos);
        s->used -= s->r[victim].kv_dev;                          /* mem.release */
        s->sum_victims++;
        push_dec(s, should_recompute(s, victim));
        heap_insert(s, victim);
    }
    for (int k = 0; k < nsk; k++) evq_insert(s, skipped[k]);     /* finally: reinsert */
    free(skipped);
    return rc;
}

static int64_t estimate_kv_size(const oreq* r) {                 /* kvcache.py:70-78 */
    int64_t need = r->prompt + r->mid - r->kv_dev;
    return need > 0 ? need : 0;
}

static void log_words(osim* s, const uint32_t* w, int64_t nw) {
    if (!s->log || s->log_overflow) return;
    if (s->log_len + nw > s->log_cap) { s->log_overflow = 1; return; }
    memcpy(s->log + s->log_len, w, sizeof(uint32_t) * nw);
    s->log_len += nw;
}

static void record_round(osim* s, int kind, const int* g, int m, const int* c, int nc,
                         double t) {
    int v = s->ndec;
    uint64_t r = (uint64_t)s->rounds;
    if (s->P->flags & SS_FLAG_DIGEST) {
        uint64_t tb; memcpy(&tb, &t, 8);
        uint64_t d = ss_round_fields(r, ss_hdr_word(kind, m, nc, v), (uint64_t)s->used, tb);
        uint64_t gh = 0;
        for (int j = 0; j < m; j++) gh += ss_grant_term((uint32_t)j, (uint64_t)g[j]);
        d += gh * ss_round_mul(r);
        for (int j = 0; j < nc; j++) d += ss_term(r, SS_TAG_DONE, j, (uint64_t)c[j]);
        for (int k = 0; k < v; k++) {
            odecision* e = &s->dec[k];
            uint64_t fb, fa; memcpy(&fb, &e->ftb, 8); memcpy(&fa, &e->fta, 8);
            d += ss_decision_term(r, (uint32_t)k, (uint64_t)(uint32_t)e->victim | ((uint64_t)e->action << 32),
                                  (uint64_t)(uint32_t)e->saved | ((uint64_t)(uint32_t)e->discarded << 32),
                                  (uint64_t)e->freed, fb, fa);
        }
        s->digest += d;
    }
    /* the reference appends an ITERATION_END only for granted rounds or
     * rounds with decisions (engine.py:329-344, 368-380) */
    if ((m > 0 || v > 0) && s->used > s->peak) s->peak = s->used;
    if ((s->P->flags & SS_FLAG_ROUND_LOG) && (m > 0 || v > 0)) {
        uint32_t h[SS_LOG_HEADER_WORDS];
        uint64_t mu = (uint64_t)s->used, tb;
        memcpy(&tb, &t, 8);
        h[0] = (uint32_t)kind; h[1] = (uint32_t)m; h[2] = (uint32_t)nc; h[3] = (uint32_t)v;
        h[4] = (uint32_t)mu; h[5] = (uint32_t)(mu >> 32);
        h[6] = (uint32_t)tb; h[7] = (uint32_t)(tb >> 32);
        log_words(s, h, SS_LOG_HEADER_WORDS);
        for (int k = 0; k < v; k++) {
            odecision* e = &s->dec[k];
            uint32_t w[SS_LOG_DECISION_WORDS];
            uint64_t fb, fa; memcpy(&fb, &e->ftb, 8); memcpy(&fa, &e->fta, 8);
            w[0] = (uint32_t)e->victim; w[1] = (uint32_t)e->action; w[2] = (uint32_t)e->saved;
            w[3] = (uint32_t)e->discarded; w[4] = (uint32_t)e->freed;
            w[5] = (uint32_t)fb; w[6] = (uint32_t)(fb >> 32); w[7] = (uint32_t)fa; w[8] = (uint32_t)(fa >> 32);
            log_words(s, w, SS_LOG_DECISION_WORDS);
        }
        for (int j = 0; j < m; j++) { uint32_t w = (uint32_t)g[j]; log_words(s, &w, 1); }
        for (int j = 0; j < nc; j++) { uint32_t w = (uint32_t)c[j]; log_words(s, &w, 1); }
    }
}

static void mark_unservable(osim* s, int i) {                    /* engine.py:402-412 */
    oreq* r = &s->r[i];
    if (h_contains(&s->evq, i)) h_remove_at(&s->evq, r->gpos);
    if (h_contains(&s->heap, i)) h_remove_at(&s->heap, r->hpos);
    if (r->kv_dev) { s->used -= r->kv_dev; r->kv_dev = 0; }
    r->unservable = 1;
    s->unserv[s->nunserv++] = (uint32_t)i;
}

/* _execute: engine.py:288-380 */
static void execute(osim* s, int kind, int m) {
    const ss_params* P = s->P;
    int ng = 0;
    s->ndec = 0;
    int64_t reserved = 0;
    int* batch = s->merged;
    for (int k = 0; k < m; k++) {
        int i = batch[k];
        oreq* r = &s->r[i];
        if (s->evicted_flag[i]) continue;                          /* :297-298 */
        if (r->stage == ST_COMPLETED) {                            /* estimate_kv_size: ValueError */
            s->status = SS_TRACE_REF_ERROR;
            return;
        }
        int64_t immediate = r->stage == ST_DECODING ? 1 : r->kv_host + (r->prompt - r->prefilled) + 1;
        int64_t est = estimate_kv_size(r);
        int64_t demand = est > immediate ? est : immediate;
        if (demand + reserved > s->cap) demand = immediate;       /* :304-305 */
        int d0 = s->ndec;
        int rc = priority_based_eviction(s, i, demand + reserved, s->granted, ng);
        if (rc < 0) {                                              /* AdmissionFailure */
            /* the decisions of a failed call live in a local list of
             * priority_based_eviction and are lost with the exception: the
             * evictions stand but are neither logged, counted nor added to
             * evicted_ids (kvcache.py:157-179, engine.py:307-323) */
            s->lost_evictions += s->ndec - d0;
            s->ndec = d0;
            if (r->kv_dev + immediate > s->cap) mark_unservable(s, i);
            else if (!h_contains(&s->heap, i)) heap_insert(s, i);
            continue;
        }
        for (int q = d0; q < s->ndec; q++) s->evicted_flag[s->dec[q].victim] = 1;
        /* a lost-decision victim that is a later batch member is processed as a
         * normal member; granting it leaves it queued in the heap as well */
        if (h_contains(&s->heap, i)) s->anomalies++;
        s->granted[ng++] = i;
        reserved += immediate;
    }
    for (int q = 0; q < s->ndec; q++) s->evicted_flag[s->dec[q].victim] = 0;

    s->last_granted = ng;
    s->sum_granted += ng;
    if (ng == 0) {                                                 /* :329-344 */
        s->nongoing = 0;
        s->eviction_count += s->ndec;
        record_round(s, SS_KIND_NONE, NULL, 0, NULL, 0, s->clock);
        return;
    }
    /* batch_duration (engine.py:126-149) over the granted members */
    double total = 0.0;
    double mx = 0.0; int nsteps = 0;
    pysum ssum = {0, 0, 0};
    for (int k = 0; k < ng; k++) {
        oreq* r = &s->r[s->granted[k]];
        if (r->stage == ST_DECODING) {
            double st = decode_step_time(r->prompt + r->decoded + 1, 1, &s->p);
            if (nsteps == 0 || st > mx) mx = st;
            pysum_add(&ssum, st);
            nsteps++;
        } else {
            total += reload_time(r->kv_host, &s->p);
            total += prefill_time(r->prompt - r->prefilled, &s->p);
        }
    }
    if (nsteps) total += P->decode_cost_sum ? pysum_value(&ssum) : mx;
    double end = s->clock + total;
    int nc = 0;
    int* completed = s->pushed;
    for (int k = 0; k < ng; k++) {                                 /* :351-363 */
        int i = s->granted[k];
        oreq* r = &s->r[i];
        if (isnan(r->first_sched)) r->first_sched = s->clock;
        if (r->stage == ST_COMPLETED) {                            /* transition(PREFILLING) */
            s->status = SS_TRACE_REF_ERROR;
            return;
        }
        if (r->stage == ST_DECODING) {                             /* _decode_step */
            if (1 > s->cap - s->used) s->status = SS_TRACE_REF_ERROR;
            s->used += 1; r->kv_dev += 1; r->decoded += 1;
        } else {                                                   /* _prefill_round */
            if (r->kv_host > 0) {
                if (r->kv_host > s->cap - s->used) s->status = SS_TRACE_REF_ERROR;
                s->used += r->kv_host; r->kv_dev += r->kv_host; r->kv_host = 0;
            }
            int64_t to_prefill = r->prompt - r->prefilled;
            if (to_prefill > 0) {
                if (to_prefill > s->cap - s->used) s->status = SS_TRACE_REF_ERROR;
                s->used += to_prefill; r->kv_dev += to_prefill; r->prefilled = r->prompt;
            }
            r->stage = ST_DECODING;                                /* PREFILLING -> DECODING */
        }
        if (r->decoded >= r->true_out) {                           /* _complete */
            if (r->stage == ST_COMPLETED) { s->status = SS_TRACE_REF_ERROR; return; } /* IllegalTransition */
            if (h_contains(&s->evq, i)) h_remove_at(&s->evq, r->gpos);
            s->used -= r->kv_dev; r->kv_dev = 0;
            r->finish = end; r->f_t = 0.0; r->stage = ST_COMPLETED;
            completed[nc++] = i;
        } else {
            r->f_t = estimate_remaining_time(r, &s->p);
            evq_update(s, i);
        }
    }
    s->clock = end;
    s->nongoing = 0;
    for (int k = 0; k < ng; k++)
        if (s->r[s->granted[k]].stage != ST_COMPLETED) s->ongoing[s->nongoing++] = s->granted[k];
    s->eviction_count += s->ndec;
    record_round(s, kind, s->granted, ng, completed, nc, end);
}

static void run_trace(const ss_params* P, const ss_trace_batch* B, const int64_t* ids,
                      const ss_outputs* O, int t) {
    int64_t off = B->trace_offsets[t];
    int n = (int)(B->trace_offsets[t + 1] - off);
    osim S;
    memset(&S, 0, sizeof(S));
    osim* s = &S;
    s->P = P;
    s->p = P->profile;
    s->n = n;
    s->cap = P->memory_capacity;
    s->r = (oreq*)calloc(n > 0 ? n : 1, sizeof(oreq));
    int nn = n > 0 ? n : 1;
    s->heap.keys = (okey*)malloc(sizeof(okey) * nn); s->heap.items = (int*)malloc(sizeof(int) * nn);
    s->heap.which = 0; s->heap.reqs = s->r;
    s->evq.keys = (okey*)malloc(sizeof(okey) * nn); s->evq.items = (int*)malloc(sizeof(int) * nn);
    s->evq.which = 1; s->evq.reqs = s->r;
    s->buffer = (int*)malloc(sizeof(int) * nn);
    s->ongoing = (int*)malloc(sizeof(int) * nn);
    int bcap = 2 * P->batch_size + 2;
    s->cand = (int*)malloc(sizeof(int) * bcap);
    s->merged = (int*)malloc(sizeof(int) * (bcap + nn));
    s->granted = (int*)malloc(sizeof(int) * bcap);
    s->pushed = (int*)malloc(sizeof(int) * bcap);
    s->evicted_flag = (char*)calloc(nn, 1);
    s->unserv = O->unservable_slots ? O->unservable_slots + off : (uint32_t*)malloc(sizeof(uint32_t) * nn);
    if ((P->flags & SS_FLAG_ROUND_LOG) && O->round_log && O->log_offsets) {
        s->log = O->round_log + O->log_offsets[t];
        s->log_cap = O->log_offsets[t + 1] - O->log_offsets[t];
    }
    for (int i = 0; i < n; i++) {
        oreq* r = &s->r[i];
        r->id = ids ? ids[off + i] : (int64_t)B->tie_rank[off + i];
        r->arrival = B->arrival_time[off + i];
        r->ready = B->ready_time[off + i];
        r->prompt = B->prompt_len[off + i];
        r->true_out = B->true_output_len[off + i];
        r->mid = B->pred_len[off + i];
        r->frank = B->pred_urgency[off + i];
        r->trank = B->true_urgency[off + i];
        r->stage = ST_WAITING;
        r->first_sched = NAN; r->finish = NAN;
        r->hpos = r->gpos = -1;
        r->f_t = estimate_remaining_time(r, &s->p);               /* engine.py:183-184 */
    }
    /* unservable pre-filter, in ready order (engine.py:193-199) */
    int* pending = (int*)malloc(sizeof(int) * nn);
    int npend = 0;
    for (int i = 0; i < n; i++) {
        if (s->r[i].prompt + 1 > s->cap) { s->r[i].unservable = 1; s->unserv[s->nunserv++] = (uint32_t)i; }
        else pending[npend++] = i;
    }
    int next = 0;
    s->clock = 0.0;
    int64_t max_rounds = P->max_rounds;
    if (max_rounds <= 0) {                 /* same automatic cap as the device */
        int64_t tokens = 0;
        for (int i = 0; i < n; i++) tokens += s->r[i].true_out;
        max_rounds = 64 * (tokens + n) + 100000;
    }
    if (max_rounds > 0x7fffffffll) max_rounds = 0x7fffffffll;
    for (;;) {                                                       /* engine.py:202-224 */
        while (next < npend && s->r[pending[next]].ready <= s->clock + 1e-12) {
            s->buffer[s->nbuf++] = pending[next]; s->r[pending[next]].in_buffer = 1; next++;
        }
        int live = s->heap.n + s->nbuf + s->nongoing;
        if (live == 0) {
            if (next >= npend) break;
            s->clock = s->r[pending[next]].ready;
            continue;
        }
        int kind;
        int had_ongoing = s->nongoing;
        s->sum_pool += live;
        s->evict_round = 0;
        int m = schedule(s, &kind);
        if (m == 0) {
            if (next < npend) { s->clock = s->r[pending[next]].ready; continue; }
            break;
        }
        int unserv_before = s->nunserv;
        execute(s, kind, m);
        s->rounds++;
        if (s->status) break;
        /* The reference would spin forever here: nothing granted,
         * nothing evicted, nobody removed and no ongoing carried in means the
         * next round starts from exactly the same state. */
        if (s->last_granted == 0 && s->ndec == 0 && s->nunserv == unserv_before && had_ongoing == 0) {
            s->status = SS_TRACE_LIVELOCK;
            break;
        }
        if (s->rounds >= max_rounds) { s->status = SS_TRACE_ROUND_CAP; break; }
    }
    free(pending);
    if (s->log_overflow && !s->status) s->status = SS_TRACE_LOG_OVERFLOW;

    /* records (engine.py:228-242) and statistics (metrics.py:35-56, 137-157) */
    ss_trace_stats st;
    memset(&st, 0, sizeof(st));
    pysum sw = {0, 0, 0}, sn = {0, 0, 0};
    pysum lv[SS_MAX_LEVELS];
    memset(lv, 0, sizeof(lv));
    for (int i = 0; i < n; i++) {
        oreq* r = &s->r[i];
        if (O->req.first_scheduled) O->req.first_scheduled[off + i] = r->first_sched;
        if (O->req.finish_time) O->req.finish_time[off + i] = r->finish;
        if (O->req.generated) O->req.generated[off + i] = (uint32_t)r->decoded;
        if (O->req.evictions) O->req.evictions[off + i] = (uint32_t)r->evictions;
        if (O->req.f_t) O->req.f_t[off + i] = r->f_t;
        if (O->req.state) {
            uint32_t stg = r->unservable ? SS_STAGE_UNSERVABLE
                         : (r->stage == ST_COMPLETED ? SS_STAGE_COMPLETED
                         : (r->stage == ST_DECODING ? SS_STAGE_DECODING : SS_STAGE_WAITING));
            O->req.state[off + i] = stg | ((r->prefilled > 0 ? 1u : 0u) << 8) |
                                    ((r->unservable && r->stage == ST_DECODING ? 1u : 0u) << 9);
        }
        if (!isnan(r->finish)) {
            double w = r->finish - r->arrival;
            double nw = w / (double)r->decoded;
            pysum_add(&sw, w);
            pysum_add(&sn, nw);
            if (r->trank < SS_MAX_LEVELS) { pysum_add(&lv[r->trank], nw); st.level_count[r->trank]++; }
            st.completed++;
        }
    }
    st.digest = s->digest;
    st.rounds = s->rounds;
    st.evictions = s->eviction_count;
    st.mem_used_peak = s->peak;
    st.log_words = s->log_len;
    st.unservable = s->nunserv;
    st.status = s->status;
    st.lost_evictions = (int32_t)s->lost_evictions;
    st.anomalies = (int32_t)s->anomalies;
    st.sum_pool = s->sum_pool;
    st.sum_granted = s->sum_granted;
    st.sum_victims = s->sum_victims;
    st.sum_resident_evict = s->sum_res_evict;
    st.final_clock = s->clock;
    st.sum_wait = pysum_value(&sw);
    st.sum_norm_wait = pysum_value(&sn);
    for (int l = 0; l < SS_MAX_LEVELS; l++) st.level_norm_sum[l] = pysum_value(&lv[l]);
    if (O->stats) O->stats[t] = st;

    if (!O->unservable_slots) free(s->unserv);
    free(s->r); free(s->heap.keys); free(s->heap.items); free(s->evq.keys); free(s->evq.items);
    free(s->buffer); free(s->ongoing); free(s->cand); free(s->merged); free(s->granted);
    free(s->pushed); free(s->evicted_flag); free(s->dec);
}

/* ------------------------------------------------------------------ */
/* batch driver: traces are independent, so they run on a thread pool  */
/* ------------------------------------------------------------------ */
typedef struct {
    const ss_params* P; const ss_trace_batch* B; const int64_t* ids; const ss_outputs* O;
    int next; pthread_mutex_t mu;
} pool_t;

static void* worker(void* arg) {
    pool_t* pl = (pool_t*)arg;
    for (;;) {
        pthread_mutex_lock(&pl->mu);
        int t = pl->next++;
        pthread_mutex_unlock(&pl->mu);
        if (t >= pl->B->n_traces) break;
        run_trace(pl->P, pl->B, pl->ids, pl->O, t);
    }
    return NULL;
}

/* Run every trace of `batch` (host pointers). `ids` (nullable) are the
 * reference request ids in the same order, used for the (arrival, id)
 * tie-break exactly as the reference's tuple key; when NULL the tie rank
 * stands in for the id. Returns SS_OK or SS_ERR_TRACE_FAILED. */
int so_run_traces(const ss_params* P, const ss_trace_batch* B, const int64_t* ids,
                  const ss_outputs* O, int n_threads) {
    if (!P || !B || !O || P->batch_size < 1 || P->memory_capacity < 1) return SS_ERR_INVALID_ARG;
    if (n_threads <= 1 || B->n_traces <= 1) {
        for (int t = 0; t < B->n_traces; t++) run_trace(P, B, ids, O, t);
    } else {
        pool_t pl;
        pl.P = P; pl.B = B; pl.ids = ids; pl.O = O; pl.next = 0;
        pthread_mutex_init(&pl.mu, NULL);
        int nt = n_threads < B->n_traces ? n_threads : B->n_traces;
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nt);
        for (int k = 0; k < nt; k++) pthread_create(&th[k], NULL, worker, &pl);
        for (int k = 0; k < nt; k++) pthread_join(th[k], NULL);
        free(th);
        pthread_mutex_destroy(&pl.mu);
    }
    if (O->stats)
        for (int t = 0; t < B->n_traces; t++)
            if (O->stats[t].status != SS_TRACE_OK) return SS_ERR_TRACE_FAILED;
    return SS_OK;
}

/* Known-answer hooks for the cost model (tests pin them to the
 * reference's own test vectors, tests/test_costs.py in the reference). */
double so_prefill_time(int64_t n, const ss_profile* p) { return prefill_time(n, p); }
double so_decode_step_time(int64_t n, int64_t j, const ss_profile* p) { return decode_step_time(n, j, p); }
double so_decode_total_time(int64_t n, int64_t m, const ss_profile* p) { return decode_total_time(n, m, p); }
int64_t so_optimal_save_tokens(int64_t n, int64_t m, const ss_profile* p) { return optimal_save_tokens(n, m, p); }
double so_resume_cost(int64_t n, int64_t m, int64_t s, const ss_profile* p) { return resume_cost(n, m, s, p); }
int so_should_cache_prefill(int64_t n, const ss_profile* p) { return should_cache_prefill(n, p); }
double so_estimate_remaining_time(int64_t prompt, int64_t mid, int64_t prefilled, int64_t decoded,
                                  int64_t kv_host, const ss_profile* p) {
    oreq r;
    memset(&r, 0, sizeof(r));
    r.prompt = prompt; r.mid = mid; r.prefilled = prefilled; r.decoded = decoded; r.kv_host = kv_host;
    return estimate_remaining_time(&r, p);
}
double so_pysum(const double* x, int64_t n) {
    pysum a = {0, 0, 0};
    for (int64_t i = 0; i < n; i++) pysum_add(&a, x[i]);
    return pysum_value(&a);
}

/* metrics.constraint_audit (metrics.py:59-91), counts only: completed
 * records (finish not NaN) sorted by finish time, every pair a < b with
 * f_a < f_b is comparable, a violation when f_a >= arrival_b and
 * rank_a > rank_b. Ties in f are skipped, so the sort order does not change
 * the counts; this restatement walks all ordered pairs directly. */
void so_audit(int32_t n_traces, const int64_t* off, const double* fin, const double* arr, const int32_t* rank,
              int64_t* violations, int64_t* comparable) {
    for (int32_t t = 0; t < n_traces; t++) {
        int64_t v = 0, c = 0;
        for (int64_t i = off[t]; i < off[t + 1]; i++) {
            const double fi = fin[i];
            if (isnan(fi)) continue;
            for (int64_t j = off[t]; j < off[t + 1]; j++) {
                if (!(fi < fin[j])) continue;
                c++;
                if (fi < arr[j]) continue;
                if (rank[i] <= rank[j]) continue;
                v++;
            }
        }
        violations[t] = v;
        comparable[t] = c;
    }
}
