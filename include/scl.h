/*
 * include/scl.h -- C-ABI of the B200 trace-replay library (libscl.so).
 *
 * What it computes: batched replay of recorded malloc/free traces through
 * Scalene's memory-profiling method (Berger et al., arXiv 2212.07597;
 * "P:a-b" = lines of PAPER.md):
 *   a1 footprint prefix sum ........ P:430-431
 *   a2 high-water-mark prefix max .. P:24-25
 *   a3 threshold sampler ........... P:429-438 ("|A - F| >= T" then reset)
 *   a4 leak tracker + ptr match .... P:20-39
 *   a5 per-(file,line) reduce ...... P:488-494
 *   a6 leak probability/filter/rate
 * Every trace is replayed independently (its own sampler and tracker); only
 * the per-site table is summed over traces (and over GPUs).  Readings where
 * the paper is silent are DESIGN.md §3.
 *
 * Conventions
 *  - Every call returns scl_status (0 = OK, negative = error);
 *    scl_last_error() returns a thread-local message for the last failure.
 *  - Pointers passed IN may be host or device memory (detected with
 *    cudaPointerGetAttributes); the library copies what it keeps.  The
 *    caller always owns its arrays; the library owns handles until *_free.
 *  - Size queries: pass cap = 0 (out buffer may be NULL) to get the count.
 *  - All work is queued on opts->cuda_stream (NULL = the legacy default
 *    stream) and is complete when the call returns, unless stated otherwise.
 *  - A handle is not safe for concurrent use from several threads.
 *  - There is no CPU fallback: without a CUDA device every compute call
 *    fails with SCL_ECUDA.
 */
#ifndef SCL_H
#define SCL_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SCL_OK = 0,
    SCL_EINVAL = -1,     /* bad argument: threshold 0, site >= n_sites, size 0, kind 3, NULL ... */
    SCL_ENOMEM = -2,     /* device or host allocation failed */
    SCL_ECUDA = -3,      /* CUDA runtime error or no device */
    SCL_ETRACE = -4,     /* invalid trace (validate = 1): message names trace and first bad event */
    SCL_EOVERFLOW = -5,  /* a result does not fit (e.g. > 2^21 sites) */
    SCL_EIO = -6,        /* trace file unreadable or malformed */
    SCL_ENCCL = -7       /* NCCL unavailable or a collective failed (scl_run_opts.nccl_comm) */
} scl_status;

/* One trace event, 16 bytes, 16-byte aligned, array-of-structs.
 *   ptr : the address passed to / returned by the allocator (pointer identity)
 *   meta: bits  0..39  size in bytes, 1 .. 2^40-1
 *         bits 40..41  kind: 0 alloc, 1 free, 2 copy (ignored by a1..a6: copies
 *                      do not change the footprint), 3 invalid
 *         bit  42      domain (0 native, 1 Python-managed; carried, unused by a1..a6)
 *         bits 43..63  site id (< 2^21): dense index of a (file, line) pair */
typedef struct { uint64_t ptr; uint64_t meta; } scl_event;

#define SCL_META(kind, size, site) \
    (((uint64_t)(size) & 0xFFFFFFFFFFull) | ((uint64_t)(kind) << 40) | ((uint64_t)(site) << 43))

/* One threshold-sampler entry (the sampling-file entry of P:433-434), 32 bytes.
 *   idx       event index within its trace that triggered the sample
 *   net       signed bytes since the previous sample (the counter value, |net| >= T)
 *   footprint F at that event
 *   site      site of the triggering event (reading Q14)
 *   kind      0 growth (net > 0, always an alloc), 1 decline (always a free)
 *   new_max   1 if a growth sample reached a new high-water mark (episode start) */
typedef struct {
    uint64_t idx; int64_t net; int64_t footprint;
    uint32_t site; uint8_t kind; uint8_t new_max; uint16_t pad;
} scl_sample;

/* Site-table columns (one uint64 row of SCL_NCOL per site, a5). */
enum {
    SCL_COL_N_MALLOC = 0, SCL_COL_N_FREE, SCL_COL_MALLOC_BYTES, SCL_COL_FREE_BYTES,
    SCL_COL_N_GROWTH, SCL_COL_N_DECLINE, SCL_COL_GROWTH_BYTES, SCL_COL_DECLINE_BYTES,
    SCL_COL_LEAK_MALLOCS, SCL_COL_LEAK_FREES, SCL_NCOL
};

/* One report row (a6).  leak_prob = 1 - (f+1)/(m-f+2), fp64, unclamped (P:55-57,
 * reading Q8); leak_rate_mbps = malloc_bytes / 2^20 / elapsed_s (Q11);
 * leak_flag = gate open AND p > 0.95, decided as m > 21 f + 18 (Q9). */
typedef struct {
    uint32_t site; uint32_t leak_flag;
    uint64_t col[SCL_NCOL];
    double leak_prob; double leak_rate_mbps;
} scl_site_row;

typedef struct {
    int64_t f_final;          /* footprint after the last event = sum of signed sizes (a1) */
    int64_t hwm;              /* max(0, max_i F_i) (a2) */
    uint64_t n_samples;       /* threshold samples in the trace (a3) */
    uint64_t n_episodes;      /* leak-tracking episodes = new-max growth samples (a4) */
    int64_t f_first_sample;   /* footprint at the first / last sample (0 if none): */
    int64_t f_last_sample;    /*   the footprint trend endpoints used by the gate */
} scl_trace_summary;

enum { SCL_HWM_PREFIX = 0,                            /* reading Q3: new maximum = above the prefix max M_{i-1} */
       SCL_HWM_SAMPLE = 1 };                          /* alternative: above every earlier sample footprint (NEXT-4) */
enum { SCL_FORMULA_PAPER = 0, SCL_FORMULA_TEXTBOOK = 1 };

typedef struct {
    uint64_t tick_ns;        /* synthetic time base: event i at (i+1)*tick_ns; 0 -> 1000 */
    int hwm_mode;            /* SCL_HWM_PREFIX (default) or SCL_HWM_SAMPLE: what a "new high-water
                                mark" is compared against at a growth sample */
    int formula;             /* SCL_FORMULA_PAPER (default) or SCL_FORMULA_TEXTBOOK (Laplace) */
    int defer_finalize;      /* 1: stop after the site table (a1-a5); the caller may sum the
                                device table across GPUs (scl_result_device_table) and then
                                call scl_finalize.  0: finalize immediately. */
    int timing;              /* 1: record CUDA events around the phases and the replay kernel
                                (scl_result_timing, scl_result_kernel_times); 0: one completion
                                event only (each event record costs ~2.5 us of stream time) */
    uint64_t elapsed_ns;     /* 0: max_t n_t * tick_ns over this handle's traces (over every rank's
                                traces when nccl_comm is set) */
    void* cuda_stream;       /* cudaStream_t, NULL = default stream */
    void* nccl_comm;         /* ncclComm_t of the ranks that hold the other trace shards, or NULL
                                (single GPU).  Set: after a1-a5 the summable table is SUM
                                all-reduced and the elapsed time MAX all-reduced over the ranks on
                                cuda_stream, then a6 runs (unless defer_finalize) -- every rank
                                ends with the global report; samples stay rank-local.  Every rank
                                must make the matching call.  The library loads libnccl.so.2
                                (already in the process, or from the system) on first use;
                                SCL_ENCCL if it cannot or a collective fails. */
    int chain_mode;          /* how the sampler's sequential chain (a3) is evaluated:
                                SCL_CHAIN_AUTO (0, default): the library chooses;
                                SCL_CHAIN_RUNNERS (1): one runner lane per trace, overlapped with
                                the stream pass;  SCL_CHAIN_SPLIT (2): each trace cut into
                                independent pieces at its sync events (|d| >= 2T-1: a sample from
                                any state), the pieces chained in parallel
                                after the stream pass (hwm_mode PREFIX only; SAMPLE mode always
                                uses the runners).  Results are identical. */
} scl_run_opts;
enum { SCL_CHAIN_AUTO = 0, SCL_CHAIN_RUNNERS = 1, SCL_CHAIN_SPLIT = 2 };

typedef struct scl_traces scl_traces;  /* opaque: device copy of events + offsets + segment plan */
typedef struct scl_result scl_result;  /* opaque: samples, summaries, site table, report */

/* Load traces into library-owned device memory (a copy: 16 B per event, rounded up to
 * 8-event rows, plus 32 zeroed rows the kernels may read past the last trace).
 *   path      binary trace file ("SCLTRC01" format) or NULL to use the arrays
 *   events    n = offsets[n_traces] events (host or device pointer)
 *   offsets   n_traces+1 uint64 event offsets, offsets[0] = 0, non-decreasing (host or device)
 *   n_sites   number of distinct sites (1 .. 2^21); every event site must be < n_sites
 *   device    CUDA device ordinal
 *   validate  1: host-side validity check (reading Q16); returns SCL_ETRACE naming the trace
 *             and first bad event.  0: skip (an invalid trace gives undefined results).
 * Errors: SCL_EINVAL (NULL, n_sites 0 or > 2^21, bad offsets), SCL_ETRACE, SCL_ENOMEM,
 *         SCL_ECUDA, SCL_EIO. */
scl_status scl_trace_load(const char* path, const scl_event* events, const uint64_t* offsets,
                          uint32_t n_traces, uint32_t n_sites, int device, int validate,
                          scl_traces** out);

/* Refill an existing handle with new traces (same meaning of the arguments as
 * scl_trace_load, events/offsets host or device pointers).  The handle's device buffers
 * are reused while the new traces fit and grown otherwise; the copy, the load checks and
 * the unit plan are ordered on cuda_stream (cudaStream_t, NULL = default stream), and the
 * call returns after one synchronisation of that stream (the per-trace sample bounds come
 * back to the host).  Runs of this handle still in flight on ANOTHER stream must have
 * finished.  Results of the handle stay valid handles (re-sized on their next run); their
 * earlier contents are stale.  On SCL_EINVAL from the event check, and on SCL_ENOMEM (a
 * buffer could not grow: the old traces may already be overwritten), the handle holds no
 * traces until the next successful reload (a run of it replays nothing).
 * Errors: as scl_trace_load. */
scl_status scl_trace_reload(scl_traces* traces, const scl_event* events, const uint64_t* offsets,
                            uint32_t n_traces, uint32_t n_sites, int validate, void* cuda_stream);

/* Replay every trace at threshold T (used verbatim; P:436-438 picks a prime slightly
 * above 10 MB -- see scl_next_prime).  Runs a1..a5 on the GPU and, unless
 * opts->defer_finalize, a6.  threshold == 0 -> SCL_EINVAL.
 * Asynchronous: the work is enqueued on opts->cuda_stream and the call returns without
 * waiting (it blocks only when the sample buffer must grow).  The accessors below
 * (report, samples, summaries, gate, timing) wait for the run themselves.
 * *out: NULL -> a new result; else a result of the same handle, reused. */
scl_status scl_replay_run(uint64_t threshold, const scl_traces* traces,
                          const scl_run_opts* opts, scl_result** out);

/* The same replay at another threshold over the handle's LAST stream pass (the scl_replay_run
 * that produced `base`): the per-unit summaries, Bloom filters and per-event (Tier E) site
 * counters of that pass are reused (the handle keeps this rank's Tier E as the pass computed
 * it, so a base whose table was since all-reduced, in the library or by the caller, does not
 * count the other ranks twice), so the events are not streamed again -- only the runners
 * re-chain every trace (re-reading the rows where a sample fires) and the reclaim pass, the
 * per-sample reduce and a6 run for the new threshold (several thresholds, one
 * read of the events).  Output contract, options and errors as scl_replay_run; in addition
 * SCL_EINVAL when base is NULL, belongs to another handle, is not of the handle's last stream
 * pass (another scl_replay_run or a reload came after it) or is *out.  Ordered on
 * opts->cuda_stream after the base run when both use the same stream. */
scl_status scl_replay_rethreshold(uint64_t threshold, const scl_traces* traces, const scl_result* base,
                                  const scl_run_opts* opts, scl_result** out);

/* Device pointer to the result's summable int64 table: n_sites*SCL_NCOL site-table
 * values followed by 3 gate values (sum of F_last-F_first, sum of max(F_first,1),
 * number of traces with >= 2 samples).  Summing it element-wise across GPUs (an
 * int64 all-reduce) gives the multi-GPU table. */
scl_status scl_result_device_table(scl_result* r, int64_t** dev_ptr, size_t* n_int64);

/* a6 on the (possibly all-reduced) table: probabilities, rates, flags, report order.
 * elapsed_ns 0 -> keep the run's value (use the global max across GPUs otherwise). */
scl_status scl_finalize(scl_result* r, uint64_t elapsed_ns);

/* Report rows in report order: flagged sites by (rate desc, site asc), then the rest by
 * site asc (a6).  rows may be NULL with cap 0; *n_rows = n_sites. */
scl_status scl_site_report(const scl_result* r, scl_site_row* rows, size_t cap, size_t* n_rows);

/* Samples of one trace, in event order (host buffer).  *n = the trace's sample count. */
scl_status scl_samples(const scl_result* r, uint32_t trace, scl_sample* out, size_t cap, size_t* n);

/* All traces' summaries (host buffer of n_traces). */
scl_status scl_trace_summaries(const scl_result* r, scl_trace_summary* out, size_t cap, size_t* n);
/* One trace's summary (SURVEY §8(b)'s scl_trace_summary; that name is the struct here): any output
 * pointer may be NULL.  Errors: SCL_EINVAL
 * for a NULL result or trace >= n_traces. */
scl_status scl_trace_summary_of(const scl_result* r, uint32_t trace, int64_t* f_final, int64_t* hwm,
                                uint64_t* n_samples, uint64_t* n_episodes);

/* Gate of P:62-65 (reading Q10): num = sum(F_last - F_first), den = sum max(F_first,1)
 * over traces with >= 2 samples; open iff some trace qualifies and 100*num >= den. */
scl_status scl_gate(const scl_result* r, int64_t* num, int64_t* den, int* open);

/* Device time of the last run, in ms, from CUDA events on the run's stream (waits for it);
 * -1 for the phases of a run made without opts->timing:
 *   replay_kernel_ms  the streaming a1..a5 kernel alone (the roofline kernel)
 *   run_ms            a1..a5 including the per-run clears, the reclaim pass and the per-sample reduce
 *   finalize_ms       a6 (probabilities, flags, report order, rows) */
scl_status scl_result_timing(const scl_result* r, float* replay_kernel_ms, float* run_ms, float* finalize_ms);

/* Replay-kernel durations (ms) of the runs made with opts->timing since the previous call (at
 * most the latest 128), oldest first; waits for them.  Lets a caller time many back-to-back runs
 * without synchronising between them.  *n = number written (<= cap). */
scl_status scl_result_kernel_times(const scl_result* r, float* ms, size_t cap, size_t* n);

/* The same for the whole stream pass of each run: from the replay kernel's start to the end of the
 * kernels that complete a1-a5 after it (the cold-site Tier-E reduce, the split chains) -- before
 * the post pass.  Read independently of scl_result_kernel_times. */
scl_status scl_result_pass_times(const scl_result* r, float* ms, size_t cap, size_t* n);

/* Number of kernels the library launched for the result's last run and finalize (replay or
 * re-chain kernel, the cold-site Tier-E reduce when n_sites > 4096, the post pass, and the a6
 * kernels of a deferred finalize).  Host bookkeeping only: does not wait.
 * Errors: SCL_EINVAL (NULL). */
scl_status scl_result_launches(const scl_result* r, uint32_t* n);

/* ---- Per-sample Python / native split ("the fraction of Python
 * (vs. native) allocations in the total sample"): for each threshold sample,
 * the bytes allocated since the previous sample (the triggering event included, frees
 * excluded) and the part of them allocated in the managed domain (meta bit 42).  managed
 * fraction = managed_bytes / max(alloc_bytes, 1). */
typedef struct { uint64_t alloc_bytes; uint64_t managed_bytes; } scl_sample_domain;   /* 16 B */
/* One trace's values, parallel to scl_samples (computed on the first call after a run; waits
 * for it). */
scl_status scl_sample_domains(const scl_result* r, uint32_t trace, scl_sample_domain* out, size_t cap, size_t* n);

/* ---- Footprint trend: the samples' (idx, footprint) are
 * the trend series.  Per trace, its exact maximum reconstruction error: max over events i of
 * |F_i - footprint of the latest sample at or before i| (0 before the first sample); below T by
 * the reset semantics.  n_traces values; computed on the first call after a run. */
scl_status scl_trace_recon_error(const scl_result* r, uint64_t* err, size_t cap, size_t* n);

/* ---- Rate-based byte sampler: the paper's comparison baseline (Table
 * tab:sampling-comparison) and copy-volume sampling (NEXT-3).
 * Per trace a counter drawn from a geometric distribution with mean R is decremented by the
 * bytes of every counted event; each time it drops below 0 a sample is taken and a new draw is
 * added (one event may take several samples).  Draw k of trace t comes from a counter-based
 * generator keyed by (seed, t, k) (Q17-Q19); seed 0 = deterministic mode (every
 * draw = R).  Sample k fires at the first event whose cumulative counted bytes exceed
 * S_k = G_1 + ... + G_k. */
typedef struct {
    uint64_t idx;        /* event index within the trace */
    uint64_t draw_sum;   /* S_k */
    uint32_t site;       /* the event's site */
    uint32_t kind;       /* the event's kind (0 alloc, 1 free, 2 copy) */
} scl_rate_sample;       /* 24 B */
enum { SCL_RATE_ALLOC_FREE = 3, SCL_RATE_COPY = 4 };
typedef struct scl_rate_result scl_rate_result;

/* Run the rate sampler over every trace of the handle.  rate_bytes R >= 1; kinds: nonzero mask
 * of {1 alloc, 2 free, 4 copy} (SCL_RATE_ALLOC_FREE: the baseline; SCL_RATE_COPY: copy volume).
 * cuda_stream: cudaStream_t or NULL.  Synchronises once (the sample counts size the output).
 * *out: NULL -> a new result; else a result of the same handle, reused.
 * Errors: SCL_EINVAL (R = 0, bad kinds, NULL), SCL_EOVERFLOW (more than 2^32 samples), SCL_ENOMEM,
 * SCL_ECUDA. */
scl_status scl_rate_run(uint64_t rate_bytes, uint64_t seed, unsigned kinds, const scl_traces* traces,
                        void* cuda_stream, scl_rate_result** out);
/* Samples per trace (n_traces values). */
scl_status scl_rate_counts(const scl_rate_result* r, uint64_t* counts, size_t cap, size_t* n);
/* One trace's samples in order (k = 1, 2, ...). */
scl_status scl_rate_samples(const scl_rate_result* r, uint32_t trace, scl_rate_sample* out, size_t cap, size_t* n);
/* Samples per site (n_sites values); x R = the bytes credited to the site (copy volume). */
scl_status scl_rate_site_counts(const scl_rate_result* r, uint64_t* counts, size_t cap, size_t* n);
/* Device time of the run's kernels (ms), excluding the one host synchronisation. */
scl_status scl_rate_timing(const scl_rate_result* r, float* ms);
void scl_rate_free(scl_rate_result* r);

void scl_traces_free(scl_traces* t);
void scl_result_free(scl_result* r);
const char* scl_last_error(void);

/* Smallest prime >= base ("a prime number slightly above 10MB"). */
uint64_t scl_next_prime(uint64_t base);

/* Number of events / traces / sites held by a handle. */
scl_status scl_traces_info(const scl_traces* t, uint64_t* n_events, uint32_t* n_traces,
                           uint32_t* n_sites);

#ifdef __cplusplus
}
#endif
#endif /* SCL_H */
