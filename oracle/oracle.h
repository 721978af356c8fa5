/*
 * oracle/oracle.h -- CPU ORACLE FOR THE SCALENE TRACE-REPLAY HOT PATH.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this
 * code.  The product (paper_2212_07597_b200/, include/scl.h) never links it,
 * and this file shares no header, struct or helper with the CUDA path: the
 * structs below are declared here independently (same byte layout as the
 * C-ABI's, because both describe the same trace file format).
 *
 * Paper: Berger, Stern, Altmayer Pizzorno, "Triangulating Python Performance
 * Issues with Scalene" (arXiv 2212.07597), cited as P:<lines of PAPER.md>.
 *   - threshold sampler ...................... P:429-438 (sec:memory-sampling)
 *   - footprint + max footprint .............. P:490-494
 *   - leak tracker + leak score .............. P:20-39   (sec:memory-leak-detector)
 *   - leak probability ....................... P:49-57
 *   - report filter / leak rate .............. P:59-71
 * Readings where the paper is silent are SURVEY.md §8(c) Q1..Q16 and are
 * listed in DESIGN.md §3.
 */
#ifndef SCL_ORACLE_H
#define SCL_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One trace event, 16 bytes: meta bits 0..39 size, 40..41 kind
 * (0 alloc, 1 free, 2 copy = ignored), 42 domain, 43..63 site id. */
typedef struct { uint64_t ptr; uint64_t meta; } orc_event;

/* One threshold-sampler entry (the "sampling file" entry of P:433-434,
 * P:475-478), 32 bytes. kind 0 = growth, 1 = decline. */
typedef struct {
    uint64_t idx; int64_t net; int64_t footprint;
    uint32_t site; uint8_t kind; uint8_t new_max; uint16_t pad;
} orc_sample;

typedef struct {
    int64_t  f_final;          /* F_{n-1} = sum of signed sizes          */
    int64_t  hwm;              /* M_{n-1} = max(0, max_i F_i)             */
    uint64_t n_samples;
    uint64_t n_episodes;
    int64_t  f_first_sample;   /* footprint at the first sample (0 if none) */
    int64_t  f_last_sample;    /* footprint at the last sample (0 if none)  */
} orc_trace_summary;

/* Site-table columns. */
enum {
    ORC_N_MALLOC = 0, ORC_N_FREE, ORC_MALLOC_BYTES, ORC_FREE_BYTES,
    ORC_N_GROWTH, ORC_N_DECLINE, ORC_GROWTH_BYTES, ORC_DECLINE_BYTES,
    ORC_LEAK_MALLOCS, ORC_LEAK_FREES, ORC_NCOL
};

enum { ORC_HWM_PREFIX = 0, ORC_HWM_SAMPLE = 1 };
enum { ORC_FORMULA_PAPER = 0, ORC_FORMULA_TEXTBOOK = 1 };

/* Replay ONE trace sequentially, in event order.  Adds into site_table
 * (n_sites x ORC_NCOL, row-major, caller-zeroed once).  Writes at most
 * `cap` samples; *summary->n_samples is the true count.
 * Returns 0, or -1 if an event's site >= n_sites or kind == 3. */
/* Per sample (NEXT-2, SPEC S:121 / S:146): allocated bytes and managed-domain (meta bit 42)
 * allocated bytes since the previous sample (the counters "reset" at P:434), the triggering
 * event included; managed fraction = managed / max(alloc, 1) ("the fraction of Python (vs.
 * native) allocations in the total sample"). */
typedef struct { uint64_t alloc_bytes; uint64_t managed_bytes; } orc_sample_domain;

int orc_replay_trace(const orc_event* ev, uint64_t n, uint64_t T, int hwm_mode,
                     orc_sample* samples, uint64_t cap,
                     orc_trace_summary* summary,
                     uint64_t* site_table, uint32_t n_sites,
                     orc_sample_domain* dom /* [cap] or NULL */);

/* Replay all traces (offsets[n_traces+1]) on n_threads host threads (one
 * trace per task).  samples for trace t go to samples + sample_off[t],
 * capacity sample_off[t+1]-sample_off[t].  site_table is overwritten.
 * Returns 0 or -1. */
int orc_replay_all(const orc_event* ev, const uint64_t* offsets, uint32_t n_traces,
                   uint32_t n_sites, uint64_t T, int hwm_mode, int n_threads,
                   orc_sample* samples, const uint64_t* sample_off,
                   orc_trace_summary* summaries, uint64_t* site_table,
                   orc_sample_domain* dom /* parallel to samples, or NULL */);

/* Gate of P:62-65 ("slope of overall memory growth is at least 1%"), reading
 * Q10: num = sum_t (F_last - F_first), den = sum_t max(F_first, 1) over traces
 * with >= 2 samples; open iff 100*num >= den and some trace qualified. */
void orc_gate(const orc_trace_summary* s, uint32_t n_traces,
              int64_t* num, int64_t* den, int* open);

/* Per-site leak probability, leak rate and report flag
 * (P:62-63).  elapsed_ns > 0. */
void orc_finalize(const uint64_t* site_table, uint32_t n_sites, int gate_open,
                  uint64_t elapsed_ns, int formula,
                  double* prob, double* rate, uint8_t* flag);

/* Report order: flagged sites by (rate desc, site asc), then the others by
 * site asc.  order[] receives n_sites site ids. */
void orc_report_order(const double* rate, const uint8_t* flag, uint32_t n_sites,
                      uint32_t* order);

/* Smallest prime >= base, by trial division ("a prime number
 * slightly above 10MB"). */
uint64_t orc_next_prime(uint64_t base);

/* Trace validity (reading Q16): every free matches a live prior alloc of the
 * same trace with equal size; pointers are unique among live allocations;
 * size >= 1; kind <= 2; site < n_sites.  Returns -1 if valid, else the index
 * of the first bad event. */
int64_t orc_validate_trace(const orc_event* ev, uint64_t n, uint32_t n_sites);

/* ---- rate-based byte sampler (NEXT-1 baseline, NEXT-3 copy volume): oracle/rate.c ---- */
typedef struct { uint64_t idx; uint64_t draw_sum; uint32_t site; uint32_t kind; } orc_rate_sample;   /* 24 B */
double   orc_soft_log(double x);
uint64_t orc_rate_draw(uint64_t R, uint64_t seed, uint32_t trace, uint64_t k);
int      orc_rate_trace(const orc_event* ev, uint64_t n, uint64_t R, uint64_t seed, uint32_t trace,
                        unsigned kinds, orc_rate_sample* out, uint64_t cap, uint64_t* n_samples);

#ifdef __cplusplus
}
#endif
#endif
