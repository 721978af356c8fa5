/*
 * oracle/oracle.c -- plain sequential CPU oracle for Scalene trace replay.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled with -O2
 * -ffp-contract=off so that the fp64 expressions below are evaluated exactly
 * as written (IEEE division, no FMA contraction).
 *
 * Everything here is the plain definition of SURVEY.md §8(c), executed one
 * event at a time in trace order, with no blocking, fusion or reordering.
 * Every function cites the PAPER.md passage it follows.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define SIZE_MASK ((1ull << 40) - 1)

static inline uint64_t ev_size(const orc_event* e) { return e->meta & SIZE_MASK; }
static inline unsigned ev_kind(const orc_event* e) { return (unsigned)((e->meta >> 40) & 3u); }
static inline uint32_t ev_site(const orc_event* e) { return (uint32_t)(e->meta >> 43); }

/*
 * One trace, in event order.
 *
 * (a1) footprint: F_i = F_{i-1} + d_i, d_i = +size (alloc) / -size (free)
 *      -- "maintains a count of all memory allocations and frees, in bytes"
 *      (P:430-431); "tracks the current memory footprint".
 * (a2) high-water mark: M_i = max(M_{i-1}, F_i), M_{-1} = 0.
 * (a3) threshold sampler: c accumulates d since the last sample; "Once the
 *      absolute difference between allocations and frees crosses a threshold
 *      (|A - F| >= T), Scalene triggers a sample ... and resets the counters"
 *      (P:430-434).  Readings Q1 (>=), Q2 (reset after every sample, one
 *      sample per event).
 * (a4) leak tracker: "Whenever the threshold-based sampler triggers because
 *      of memory growth, Scalene checks to see if this growth has led to a
 *      new high-water mark ... If so, Scalene records the sampled allocation.
 *      Every call to free then checks to see whether this object is ever
 *      reclaimed ... a pointer comparison".  Leak score: "first
 *      increments the mallocs field when it starts tracking an object, and
 *      then increments the frees field only if it reclaimed the allocated
 *      object. It then resumes tracking with a newly sampled object"
 *      (P:31-39).  Readings Q3 (PREFIX: F_i > M_{i-1}), Q4 (strict), Q5
 *      (the triggering alloc), Q6 (settle at next new max and at trace end),
 *      Q7 (first match only).
 * (a5) per-site reduce (readings Q13, Q14): per event
 *      n_malloc/malloc_bytes or n_free/free_bytes at the event's site; per
 *      sample n_growth/growth_bytes or n_decline/decline_bytes at the
 *      triggering event's site.
 */
int orc_replay_trace(const orc_event* ev, uint64_t n, uint64_t T, int hwm_mode,
                     orc_sample* samples, uint64_t cap,
                     orc_trace_summary* summary,
                     uint64_t* site_table, uint32_t n_sites,
                     orc_sample_domain* dom)
{
    int64_t F = 0, M = 0, c = 0;
    int64_t Msample = 0;                 /* max over sample footprints (hwm_mode SAMPLE) */
    int have_ep = 0, reclaimed = 0;
    uint64_t ep_ptr = 0; uint32_t ep_site = 0;
    uint64_t ns = 0, n_ep = 0;
    int64_t f_first = 0, f_last = 0;
    uint64_t a_since = 0, m_since = 0;   /* allocated / managed allocated bytes since the reset */
    const int64_t Ti = (int64_t)T;

    for (uint64_t i = 0; i < n; ++i) {
        const orc_event* e = &ev[i];
        unsigned kind = ev_kind(e);
        uint32_t site = ev_site(e);
        uint64_t size = ev_size(e);
        if (kind == 3 || site >= n_sites) return -1;
        if (kind == 2) continue;                     /* copies do not change footprint */

        int64_t d = (kind == 0) ? (int64_t)size : -(int64_t)size;
        if (kind == 0) { a_since += size; if ((e->meta >> 42) & 1u) m_since += size; }
        int64_t Mprev = M;
        F += d;
        if (F > M) M = F;
        c += d;

        /* free path: the pointer comparison against the tracked object */
        if (kind == 1 && have_ep && !reclaimed && e->ptr == ep_ptr) reclaimed = 1;

        if (c >= Ti || c <= -Ti) {
            int growth = c > 0;
            int new_max;
            if (hwm_mode == ORC_HWM_SAMPLE) new_max = growth && F > Msample;
            else                            new_max = growth && F > Mprev;
            if (ns < cap) {
                orc_sample* s = &samples[ns];
                s->idx = i; s->net = c; s->footprint = F; s->site = site;
                s->kind = growth ? 0 : 1; s->new_max = (uint8_t)new_max; s->pad = 0;
                if (dom) { dom[ns].alloc_bytes = a_since; dom[ns].managed_bytes = m_since; }
            }
            a_since = 0; m_since = 0;
            if (ns == 0) f_first = F;
            f_last = F;
            ++ns;
            if (F > Msample) Msample = F;
            uint64_t* row = &site_table[(size_t)site * ORC_NCOL];
            if (growth) { row[ORC_N_GROWTH] += 1; row[ORC_GROWTH_BYTES] += (uint64_t)c; }
            else        { row[ORC_N_DECLINE] += 1; row[ORC_DECLINE_BYTES] += (uint64_t)(-c); }
            if (new_max) {
                if (have_ep && reclaimed) site_table[(size_t)ep_site * ORC_NCOL + ORC_LEAK_FREES] += 1;
                have_ep = 1; reclaimed = 0; ep_ptr = e->ptr; ep_site = site;
                row[ORC_LEAK_MALLOCS] += 1;
                ++n_ep;
            }
            c = 0;
        }
        uint64_t* row = &site_table[(size_t)site * ORC_NCOL];
        if (kind == 0) { row[ORC_N_MALLOC] += 1; row[ORC_MALLOC_BYTES] += size; }
        else           { row[ORC_N_FREE]   += 1; row[ORC_FREE_BYTES]   += size; }
    }
    /* settle the in-flight episode at trace end (reading Q6) */
    if (have_ep && reclaimed) site_table[(size_t)ep_site * ORC_NCOL + ORC_LEAK_FREES] += 1;

    summary->f_final = F; summary->hwm = M;
    summary->n_samples = ns; summary->n_episodes = n_ep;
    summary->f_first_sample = f_first; summary->f_last_sample = f_last;
    return 0;
}

/* ---- many traces, one per task on a pthread pool (SURVEY §8(d) "Oracle timing") ---- */
typedef struct {
    const orc_event* ev; const uint64_t* offsets; uint32_t n_traces; uint32_t n_sites;
    uint64_t T; int hwm_mode; orc_sample* samples; const uint64_t* sample_off; orc_sample_domain* dom;
    orc_trace_summary* summaries; uint64_t* table; int err; uint32_t* next;
} orc_job;

static void* orc_worker(void* arg)
{
    orc_job* j = (orc_job*)arg;
    for (;;) {
        uint32_t t = __atomic_fetch_add(j->next, 1u, __ATOMIC_RELAXED);
        if (t >= j->n_traces) break;
        uint64_t b = j->offsets[t], e = j->offsets[t + 1];
        uint64_t so = j->sample_off[t], cap = j->sample_off[t + 1] - so;
        if (orc_replay_trace(j->ev + b, e - b, j->T, j->hwm_mode, j->samples + so, cap,
                             &j->summaries[t], j->table, j->n_sites, j->dom ? j->dom + so : NULL) != 0) j->err = -1;
    }
    return NULL;
}

int orc_replay_all(const orc_event* ev, const uint64_t* offsets, uint32_t n_traces,
                   uint32_t n_sites, uint64_t T, int hwm_mode, int n_threads,
                   orc_sample* samples, const uint64_t* sample_off,
                   orc_trace_summary* summaries, uint64_t* site_table,
                   orc_sample_domain* dom)
{
    if (n_threads < 1) n_threads = 1;
    size_t tab = (size_t)n_sites * ORC_NCOL;
    uint32_t next = 0;
    orc_job* jobs = (orc_job*)calloc((size_t)n_threads, sizeof(orc_job));
    pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -1; }
    int err = 0;
    for (int k = 0; k < n_threads; ++k) {
        orc_job* j = &jobs[k];
        j->ev = ev; j->offsets = offsets; j->n_traces = n_traces; j->n_sites = n_sites;
        j->T = T; j->hwm_mode = hwm_mode; j->samples = samples; j->sample_off = sample_off; j->dom = dom;
        j->summaries = summaries; j->err = 0; j->next = &next;
        j->table = (k == 0) ? site_table : (uint64_t*)calloc(tab ? tab : 1, sizeof(uint64_t));
        if (!j->table) err = -1;
    }
    memset(site_table, 0, tab * sizeof(uint64_t));
    if (!err) {
        for (int k = 1; k < n_threads; ++k) pthread_create(&th[k], NULL, orc_worker, &jobs[k]);
        orc_worker(&jobs[0]);
        for (int k = 1; k < n_threads; ++k) pthread_join(th[k], NULL);
        for (int k = 0; k < n_threads; ++k) if (jobs[k].err) err = -1;
        for (int k = 1; k < n_threads; ++k)                 /* integer sums: order-free */
            for (size_t x = 0; x < tab; ++x) site_table[x] += jobs[k].table[x];
    }
    for (int k = 1; k < n_threads; ++k) free(jobs[k].table);
    free(jobs); free(th);
    return err;
}

/* ---- gate: "only when the slope of overall memory growth is at least 1%", reading Q10 ---- */
void orc_gate(const orc_trace_summary* s, uint32_t n_traces, int64_t* num, int64_t* den, int* open)
{
    int64_t gn = 0, gd = 0; int any = 0;
    for (uint32_t t = 0; t < n_traces; ++t) {
        if (s[t].n_samples < 2) continue;
        any = 1;
        gn += s[t].f_last_sample - s[t].f_first_sample;
        gd += s[t].f_first_sample > 1 ? s[t].f_first_sample : 1;
    }
    *num = gn; *den = gd;
    *open = any && ((__int128)100 * (__int128)gn >= (__int128)gd);
}

/*
 * Leak probability: "computes the leak probability as
 * 1.0 - (frees + 1) / (mallocs - frees + 2)" -- as printed, unclamped
 * (reading Q8).  TEXTBOOK = Laplace's rule 1 - (f+1)/(m+2) (NEXT-4 switch).
 * Flag: "only reports leaks whose likelihood exceeds a 95%
 * threshold" -- p > 0.95, decided exactly on integers (reading Q9):
 * PAPER: (f+1)/(m-f+2) < 1/20  <=>  m > 21 f + 18;
 * TEXTBOOK: (f+1)/(m+2) < 1/20 <=>  m > 20 f + 18.
 * Rate: "average amount of memory allocated at a given line divided
 * by time elapsed, in MB per second" -- malloc_bytes / 2^20 / (elapsed_ns/1e9)
 * (reading Q11).
 */
void orc_finalize(const uint64_t* site_table, uint32_t n_sites, int gate_open,
                  uint64_t elapsed_ns, int formula,
                  double* prob, double* rate, uint8_t* flag)
{
    for (uint32_t s = 0; s < n_sites; ++s) {
        const uint64_t* row = &site_table[(size_t)s * ORC_NCOL];
        uint64_t m = row[ORC_LEAK_MALLOCS], f = row[ORC_LEAK_FREES];
        double p; int over;
        if (formula == ORC_FORMULA_TEXTBOOK) {
            p = 1.0 - (double)(f + 1) / (double)(m + 2);
            over = (unsigned __int128)m > (unsigned __int128)20 * f + 18;
        } else {
            p = 1.0 - (double)(f + 1) / (double)(m - f + 2);
            over = (unsigned __int128)m > (unsigned __int128)21 * f + 18;
        }
        prob[s] = p;
        /* reading Q20: an elapsed time of 0 (every trace empty, so no site has bytes) counts as 1 ns */
        rate[s] = ((double)row[ORC_MALLOC_BYTES] / 1048576.0) / ((double)(elapsed_ns ? elapsed_ns : 1) / 1e9);
        flag[s] = (uint8_t)(gate_open && over);
    }
}

/* ---- report order: "focus their attention on high-confidence leaks with a high leak rate" ---- */
static const double* g_rate; static const uint8_t* g_flag;
static int cmp_site(const void* a, const void* b)
{
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    if (g_flag[x] != g_flag[y]) return g_flag[x] ? -1 : 1;
    if (g_flag[x] && g_rate[x] != g_rate[y]) return g_rate[x] > g_rate[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}
void orc_report_order(const double* rate, const uint8_t* flag, uint32_t n_sites, uint32_t* order)
{
    for (uint32_t s = 0; s < n_sites; ++s) order[s] = s;
    g_rate = rate; g_flag = flag;
    qsort(order, n_sites, sizeof(uint32_t), cmp_site);
}

/* ---- "a prime number slightly above 10MB" ---- */
uint64_t orc_next_prime(uint64_t base)
{
    for (uint64_t x = base < 2 ? 2 : base;; ++x) {
        int prime = 1;
        for (uint64_t q = 2; q * q <= x; ++q) if (x % q == 0) { prime = 0; break; }
        if (prime) return x;
    }
}

/* ---- trace validity (reading Q16), open-addressing set of live pointers ---- */
int64_t orc_validate_trace(const orc_event* ev, uint64_t n, uint32_t n_sites)
{
    uint64_t cap = 16; while (cap < 2 * n + 16) cap <<= 1;
    uint64_t* key = (uint64_t*)calloc(cap, sizeof(uint64_t));
    uint64_t* val = (uint64_t*)calloc(cap, sizeof(uint64_t));   /* size; 0 = empty/tombstone */
    uint8_t* used = (uint8_t*)calloc(cap, 1);                    /* 0 empty, 1 live, 2 tombstone */
    int64_t bad = -1;
    if (!key || !val || !used) { free(key); free(val); free(used); return 0; }
    for (uint64_t i = 0; i < n && bad < 0; ++i) {
        unsigned kind = ev_kind(&ev[i]); uint64_t size = ev_size(&ev[i]);
        if (kind == 3 || ev_site(&ev[i]) >= n_sites || (kind != 2 && size == 0)) { bad = (int64_t)i; break; }
        if (kind == 2) continue;
        uint64_t p = ev[i].ptr, h = (p * 0x9E3779B97F4A7C15ull) & (cap - 1);
        uint64_t slot = cap, first_tomb = cap;
        for (;;) {                                               /* probe */
            if (used[h] == 0) { slot = cap; break; }
            if (used[h] == 1 && key[h] == p) { slot = h; break; }
            if (used[h] == 2 && first_tomb == cap) first_tomb = h;
            h = (h + 1) & (cap - 1);
        }
        if (kind == 0) {
            if (slot != cap) { bad = (int64_t)i; break; }        /* ptr already live */
            uint64_t ins = first_tomb != cap ? first_tomb : h;
            used[ins] = 1; key[ins] = p; val[ins] = size;
        } else {
            if (slot == cap || val[slot] != size) { bad = (int64_t)i; break; }
            used[slot] = 2;
        }
    }
    free(key); free(val); free(used);
    return bad;
}
