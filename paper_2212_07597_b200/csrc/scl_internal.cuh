// scl_internal.cuh -- device-side layout shared by the replay kernels and the
// host API of libscl.so (not part of the public ABI; see include/scl.h).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../include/scl.h"

// SCL_CHECKED builds (libscl_checked.so, tools/checked.sh): every computed index of a global write is
// bounds-checked on the device and a violation traps with its source line -- the stand-in for
// compute-sanitizer memcheck, which this GPU pool does not allow.
#ifdef SCL_CHECKED
#include <cstdio>
#define SCL_CHECK(c) do { if (!(c)) { printf("SCL_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); __trap(); } } while (0)
#else
#define SCL_CHECK(c) do { } while (0)
#endif

namespace scl {

// ---- geometry and CTA roles -----------------------------------
// Events are viewed as 128-B rows of 8.  A TMA box is 256 rows (2048 events,
// 32 KiB), staged in shared memory with the 128-byte swizzle so that each
// compute lane reads its own row with conflict-free LDS.128.  A chain UNIT
// (the runners' granule) is kSub = 4 boxes = 8192 events = 32 chunks of 256
// events (one chunk per compute warp per box).  One persistent CTA per SM:
//   warps 0..15  compute: two groups of 8 alternate boxes (one chunk per warp), no CTA barriers;
//                one arrival per chunk on the unit slot's completion mbarrier
//   warp  16     producer: tickets (one per unit) + TMA issue into a kStages ring
//   warp  17     publisher: composes and publishes each complete unit
//   warps 18..19 runners: advance their traces over the published units, resolve samples
constexpr int kThreads = 256;                 // rows per box = compute threads
constexpr int kEpt = 8;                       // events per row
constexpr int kSeg = kThreads * kEpt;         // events per box
constexpr int kSegBytes = kSeg * 16;
constexpr int kSub = 4;                       // boxes per unit
constexpr int kUnitRows = kThreads * kSub;
constexpr int kUnit = kSeg * kSub;            // events per unit (8192)
constexpr int kChunks = 32;                   // 256-event chunks per unit (one per runner lane)
constexpr int kComputeWarps = 16;                // two groups of 8, alternating boxes
constexpr int kLBWarps = 3;                   // publisher + 2 runner warps (20 warps total, 96 registers)
constexpr int kEmbeddedRunners = 2;           // warps 18-19 of every CTA run traces
constexpr int kProducerWarp = kComputeWarps;
constexpr int kCtaThreads = (kComputeWarps + 1 + kLBWarps) * 32;
#ifndef SCL_STAGES
#define SCL_STAGES 4
#endif
#ifndef SCL_WARM
#define SCL_WARM 2048
#endif
#ifndef SCL_RUNNER_NAP
#define SCL_RUNNER_NAP 1024
#endif
#ifndef SCL_BLOOM_LOG2
#define SCL_BLOOM_LOG2 5
#endif
constexpr int kStages = SCL_STAGES;           // TMA ring depth
constexpr int kSlots = 6;                     // compute -> publisher unit summary ring (smem)
constexpr int kBloomLog2 = SCL_BLOOM_LOG2;
constexpr unsigned kBloomBig = 4096;          // the filter's halves: frees under / from this size (replay_kernel.cu)
constexpr int kBloomWords = 1 << kBloomLog2;  // Bloom filter of freed pointers per chunk (32 words = 1024 bits; 64
                                              //   measured 6-7 % slower on configs 2 and 3: the records and their zeroing)
constexpr int kHot = 1024;                    // sites with shared-memory Tier-E counters (all 4 kinds)
constexpr int kWarm = SCL_WARM;               // n_sites > kHot: the allocs and frees of the kWarm lowest site ids;
                                              //   the other sites' events go to the cold-record stream
constexpr int kRecChunk = 4096;               // cold-record stream: records per chunk (one warp's, at a time)
constexpr int kColdSites = 28672;             // cold_hist_kernel: sites per range (2 kinds x 4 B = 224 KiB)
constexpr long long kNeg = -(1ll << 62);      // "no event" sentinels for max / min
constexpr long long kPos = (1ll << 62);
constexpr unsigned long long kNoEp = ~0ull;
constexpr unsigned kInvalid = 0xffffffffu;
constexpr long long kAggBig = -(1ll << 47);   // tagged aggregate word: the value does not fit in 48 bits

// ---- event decoding (include/scl.h) ----------------------------------------
__host__ __device__ inline uint64_t ev_size(uint64_t meta) { return meta & 0xFFFFFFFFFFull; }
__host__ __device__ inline unsigned ev_kind(uint64_t meta) { return (unsigned)(meta >> 40) & 3u; }
__host__ __device__ inline uint32_t ev_site(uint64_t meta) { return (uint32_t)(meta >> 43); }

// ---- exact sequential state of one trace between units (owned by the trace's runner) ----
struct __align__(16) RunState {
    long long F, M, B;                // footprint, high-water mark, footprint at the last sample
    unsigned long long n, nep, ep1;   // samples, episodes, current episode (sample slot + 1; 0 none)
    unsigned long long eptr;          // pointer of the current episode's allocation
    long long Ms;                     // max footprint over the samples so far (hwm_mode SAMPLE)
    unsigned next, pad;               // next unit index to run
};

// One unit's leak-tracker entry, written by its trace's runner for the reclaim pass: the episode
// in progress when the unit starts (sample slot + 1; 0 none) and its pointer, and the absolute
// sample slots [s_in, s_out) taken inside the unit.
struct __align__(16) UnitEntry { unsigned long long ep1, eptr, s_in, s_out; };

struct SegInfo {                     // one unit ticket, as the producer resolved it
    unsigned u, t, kraw, slot;       // ticket, trace, unit index (| last << 31), state slot
    long long off_t, n_t, row_base;  // trace start, trace length, first global row of the unit
    unsigned nbox, pad;              // boxes of this unit that overlap the trace
};
struct __align__(16) Slot {          // compute -> publisher -> runners / post pass: one unit record (urec)
    SegInfo info;
    long long Pc[kChunks], ax[kChunks], an[kChunks];       // chunk prefix; max/min relative to the unit start
                                                           // (before the compose: chunk sum, max, min
                                                           // relative to the chunk start)
    long long usum, umx, umn;                              // unit aggregate
    unsigned pad0, pad1;
    unsigned bloom[kChunks][kBloomWords];
};

// One unit ticket, resolved on the host at load time (one 32-B load per ticket).
struct __align__(16) TicketInfo {
    long long off_t, n_t;             // trace start (global event index), trace length
    unsigned t, kraw, slot, nbox;     // trace, unit index (| last << 31), state slot, boxes overlapping the trace
};

struct FinalParams {
    const unsigned long long* table;  // [n_sites*SCL_NCOL + 3]
    unsigned int n_sites;
    int formula;
    double elapsed_ns;
    unsigned long long* gate_out;     // [3] host-mapped pinned buffer: the gate sums (written by one thread)
    unsigned long long* prof;         // debug build only: phase timestamps of a6
};

// Per-run preparation, done by CTA 0 of the replay kernel before the other CTAs' producers and
// runners start: zero the site table, the trace summaries, the runner states and the counters;
// sample slot bases sbase[t] = sum_{t'<t} min(n_t', floor(sum|d|_t' / T)) (the host computes the
// same bound).
struct PrepParams {
    unsigned long long* table; size_t table_words;
    unsigned long long* summ; size_t summ_words;
    unsigned long long* run; size_t run_words;
    unsigned int* ticket;             // [8] (the replay kernel's counters; [0..6] zeroed here)
    unsigned* rsbcnt; unsigned n_sb;  // a6 scratch superblock counts (zeroed here)
    unsigned long long* sbase;        // [n_traces]
    const unsigned long long* off;    // [n_traces + 1]
    const unsigned long long* sabs;   // [n_traces]
    unsigned int n_traces;
    unsigned long long T;
};

// One exact re-check of the reclaim pass: chunk rows [row0, row0 + 32) of a unit, unit positions
// [sbeg, send), does any free of `ptr` occur?  (pos0: unit position of the chunk's first event;
// site: the episode's sample site, its leak-frees column.)
struct __align__(16) RTask {
    unsigned long long ep1, ptr;
    long long row0, off_t, n_t;
    unsigned pos0, sbeg, send, site;
};

struct ReplayParams {
    const scl_event* ev;              // padded device copy (multiple of 8 events)
    const unsigned long long* off;    // [n_traces+1]
    const TicketInfo* tk;             // [n_segs] in ticket order (unit index, trace)
    void* urec;                       // [n_segs] unit records (copied out by the publisher warps)
    unsigned long long* uagg;         // [n_segs][4] unit sum, max, min as (value << 16 | epoch tag), published
                                      // after the unit record (value kAggBig: read it from the record)
    RunState* run;                    // [n_traces] per-trace runner state (zeroed per run)
    UnitEntry* uent;                  // [n_segs] state entering each unit (runner -> reclaim pass)
    const unsigned int* tr_nseg;      // [n_traces] units per trace
    const unsigned int* tr_base;      // [n_traces] first unit id of the trace
    unsigned int* ticket;             // [8]: unit tickets; post pass: units settled, task tail, blocks done (zeroed
                                      //      per run); [7] = epoch once the run is prepared (never zeroed)
    RTask* rtask;                     // [rtask_cap] exact re-checks queued by the reclaim pass
    unsigned int rtask_cap;
    int rechain;                      // runners only, over the handle's last stream pass (prepared by the host)
    PrepParams prep;                  // CTA 0 prepares the run; ticket[7] = epoch once done
    int fuse_report;                  // post_kernel runs a6 over all its blocks (fin -> rows)
    unsigned* rbits;                  // [max(n_sites, kReportSites)/32] a6 scratch: flag bitmask words
    unsigned* rsbcnt;                 //   flags per kSuper bitmask words (zeroed by the preparation)
    double* rlrate; unsigned* rlsite; //   flagged sites' rates and ids (kReportList)
    FinalParams fin;
    scl_site_row* rows;
    unsigned int n_segs;
    unsigned int n_runners;           // gridDim.x * kEmbeddedRunners
    unsigned int epoch;               // run number on this traces handle (ready tag)
    unsigned int zc_target;           // ticket[8] once every CTA of this replay launch zeroed its slice
    unsigned int n_sites;
    unsigned int n_traces;
    int hwm_sample;                   // 1: new maximum against earlier sample footprints (SCL_HWM_SAMPLE)
    long long T;
    unsigned long long* table;        // [n_sites*SCL_NCOL + 3]
    scl_sample* samples;              // [capacity]
    unsigned long long sample_cap;    // slots of samples / ep_flag (SCL_CHECKED bounds)
    unsigned int* ep_flag;            // [capacity]  reclaimed flag per episode-start sample
    const unsigned long long* sbase;  // trace -> first sample slot
    scl_trace_summary* summ;          // [n_traces]
    unsigned long long* prof;         // debug build only (SCL_PROFILE): per-role cycle sums, else NULL
    // cold-record stream (n_sites > kWarm): the meta word of every fast-path alloc / free of a site
    // >= kWarm, in chunks of kRecChunk records taken by one compute warp at a time (cold_hist_kernel
    // reduces them per site after the stream pass)
    unsigned long long* crec;         // [crec_cap] records (the events' meta words)
    unsigned long long crec_cap;      // records (a multiple of kRecChunk)
    unsigned long long* cctr;         // [2]: records allocated (chunk granules), spare (zeroed per run)
    unsigned* crec_fill;              // [crec_cap / kRecChunk] records written to each allocated chunk
    unsigned long long* covf;         // host-mapped: set when the pool was exhausted (the host grows it)
    unsigned* cpart;                  // [max(nsm, R) * 2 * kColdSites] cold_hist's partial tables
    unsigned long long* tierE;        // [n_sites * 4] Tier-E columns of the stream pass (post pass copy; re-thresholds)
    // chain split at sync events (pchain.cu; hwm_mode PREFIX): the embedded runners stand down
    int no_chain;                     // 1: runner warps exit at once (the pchain kernels run the chains)
    struct UnitStart* ust;            // [n_segs] F at each unit start, max F before it
    struct SyncInfo* sync;            // [n_segs] the unit's first sync event (|d| >= 2T - 1)
    struct PieceCount* pc;            // [n_traces + n_segs] the chain's results per piece
    struct PieceRun* pr;              // [n_traces + n_segs] placement of each piece (slot base, entering episode)
    struct UnitLocal* ul;             // [n_segs] piece-local sample counts / episode at each unit's ends
    scl_sample* pscr;                 // [pblocks * kPBlock] samples as the pieces found them (blocks)
    unsigned* pnext;                  // [pblocks] next block of the same piece
    unsigned* pctr;                   // [2] scratch blocks taken, pieces taken (zeroed by pc_prefix)
    unsigned pblocks;
};

// Chain pieces (pchain.cu).  A sync event (|d| >= 2T - 1) takes a sample from
// any counter state, after which the state is B = F there: each trace splits into independent
// pieces, one starting at the trace start and one after the first sync event of every unit that
// has one (piece id n_traces + unit), each ending at the first sync event of a later unit (included)
// or at the trace end.
struct UnitStart { long long F0, M0; };                  // F before the unit's first event; max F before it (M_-1 = 0)
struct SyncInfo { long long Fs, pad2; int pos, pad0; long long pad1; };  // pos: unit position (-1: none); F through it, relative to the unit start
constexpr int kPBlock = 64;                              // samples per scratch block of a piece
struct PieceCount {                                      // one piece's chain (pc_run)
    unsigned long long n, nep;                           // samples, new-maximum samples (episode starts)
    unsigned long long lep, lep_ptr;                     // local index + 1 of the last episode start (0: none), its pointer
    long long ffirst, flast;                             // footprint at the first / last sample
    unsigned active, first_blk;                          // the piece exists; its first scratch block
    unsigned u_first, u_last;                            // its units (the first from its window start, the last
    unsigned end_sync, pad;                              //   up to its end: a sync event of u_last, or the unit end)
};
struct UnitLocal {                                       // piece-local state at a unit's start / end (pc_run)
    unsigned long long n_start, lep_start, lep_ptr_start;   // samples before; last episode start before (+1, 0 none)
    unsigned long long n_end;                            // samples through the unit end
};
struct PieceRun { unsigned long long base, ep1, eptr, pad; };   // pass 2: first slot; episode entering (slot + 1, 0 none)
cudaError_t launch_pchain(const ReplayParams& p, cudaStream_t st);




#ifdef __CUDACC__
// The 8 events of one global row, through L2 (re-read path).  A row past the end of its trace
// (a chunk's lanes beyond the last event, masked by the caller) is still read: the event buffer
// carries 32 zeroed rows past its last row for exactly these lanes (scl_trace_load).
__device__ __forceinline__ void load_row_global(const scl_event* ev, long long row,
                                                unsigned long long* ptr, unsigned long long* meta) {
    // 32-B loads (two events each, LDG.256 on sm_100): each sector of the row is requested once
    const scl_event* q = ev + row * kEpt;
    #pragma unroll
    for (int j = 0; j < kEpt; j += 2)
        asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(ptr[j]), "=l"(meta[j]), "=l"(ptr[j + 1]), "=l"(meta[j + 1]) : "l"(q + j));
}

__device__ __forceinline__ void load_row_meta(const scl_event* ev, long long row, unsigned long long* meta) {
    const scl_event* q = ev + row * kEpt;
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) meta[j] = __ldcg(&q[j].meta);
}

// Tier S of one sample (a5: n_growth / growth_bytes or n_decline / decline_bytes of the
// sample's site -- a decline at the free's site, reading Q14) and, at an episode start, the site's
// leak mallocs (the frees are counted by the reclaim pass).  Fire-and-forget L2 reductions
// by the runner lane that takes the sample.
__device__ __forceinline__ void sample_counters(const ReplayParams& p, unsigned site, bool growth, long long net, bool nm)
{
    SCL_CHECK(site < p.n_sites);
    unsigned long long* row = p.table + (size_t)site * SCL_NCOL;
    atomicAdd(&row[growth ? SCL_COL_N_GROWTH : SCL_COL_N_DECLINE], 1ull);
    atomicAdd(&row[growth ? SCL_COL_GROWTH_BYTES : SCL_COL_DECLINE_BYTES], (unsigned long long)(growth ? net : -net));
    if (nm) atomicAdd(&row[SCL_COL_LEAK_MALLOCS], 1ull);
}

#endif

constexpr int kUCols = 4;               // per-unit byte sums: alloc, free, copy, managed alloc (rate.cu)

// Per-sample Python / native split (rate.cu; NEXT-2).
struct DomainParams {
    const scl_event* ev;
    const TicketInfo* tk;
    unsigned n_segs, n_traces;
    const unsigned long long* ustart;  // [n_segs][kUCols]
    const scl_sample* samples;
    const unsigned long long* sbase;
    const scl_trace_summary* summ;
    unsigned long long* P;             // [slots][2] inclusive (alloc, managed) prefix at each sample event
    scl_sample_domain* dom;            // [slots]
};
cudaError_t launch_domains(const DomainParams& p, cudaStream_t st);
cudaError_t launch_recon(const DomainParams& p, unsigned long long* err, cudaStream_t st);

// Rate-based byte sampler (rate.cu; NEXT-1 / NEXT-3).
struct RateParams {
    const scl_event* ev;
    const TicketInfo* tk;              // [n_segs] unit placement (as the replay kernel's tickets)
    unsigned n_segs, n_traces;
    unsigned long long R, seed;
    unsigned kinds;                    // counted event kinds: bit 0 alloc, 1 free, 2 copy
    const unsigned long long* ttot;    // [n_traces][kUCols] alloc / free / copy / managed bytes per trace
    const unsigned long long* ustart;  // [n_segs][kUCols] the same before each unit (exclusive, within its trace)
    unsigned long long* count;         // [n_traces] samples per trace
    const unsigned long long* sbase;   // [n_traces] first sample slot
    unsigned long long* S;             // [total] draw prefix sums S_k of the samples
    unsigned long long* kfirst;        // [n_segs] index (within its trace) of each unit's first sample
    scl_rate_sample* samples;          // [total]
    unsigned long long* site_count;    // [n_sites] samples per site
};
cudaError_t launch_unit_sums(const scl_event* ev, const TicketInfo* tk, unsigned n_segs, unsigned long long* usum,
                             const unsigned* tr_base, const unsigned* tr_nseg, unsigned n_traces,
                             unsigned long long* ustart, unsigned long long* ttot, cudaStream_t st);
cudaError_t launch_rate(const RateParams& p, int phase, cudaStream_t st);   // 0 count, 1 fill S, 2 place

// launch wrappers (replay.cu)
cudaError_t launch_load_stats(const scl_event* ev, const unsigned long long* off, unsigned n_traces,
                              unsigned long long n_events, unsigned n_sites, unsigned long long* sabs,
                              unsigned long long* err, scl_event* dst, unsigned long long* shist,
                              const unsigned* remap, cudaStream_t st);
cudaError_t launch_site_sample(const scl_event* src, unsigned long long stride, unsigned long long m,
                               unsigned n_sites, unsigned* cnt, cudaStream_t st);
cudaError_t launch_permute_table(const unsigned long long* tin, unsigned long long* tout, const unsigned* remap,
                                 unsigned n_sites, cudaStream_t st);
cudaError_t launch_replay(const CUtensorMap* tmap, const ReplayParams& p, int grid, cudaStream_t st);
cudaError_t launch_post(const ReplayParams& p, cudaStream_t st);
cudaError_t launch_rechain(const ReplayParams& p, cudaStream_t st);   // runner warps alone
cudaError_t launch_cold_hist(const ReplayParams& p, cudaStream_t st);  // Tier E of the cold-record stream
bool cold_hist_launched(const ReplayParams& p);
unsigned cold_hist_launches(const ReplayParams& p);   // kernels of launch_cold_hist (hist + partial sum)
unsigned cold_ranges(unsigned n_sites);       // cold_hist ranges of kColdSites sites
bool report_fused(unsigned n_sites);   // a6 in one block (report_kernel) for tables this small
cudaError_t launch_report(const FinalParams& p, scl_site_row* rows, cudaStream_t st);
size_t replay_smem_bytes();
size_t replay_urec_bytes();            // bytes of one unit record
int replay_occupancy(int* grid);

}  // namespace scl
