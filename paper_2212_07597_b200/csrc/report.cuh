// report.cuh -- a6: per-site probability, rate and flag, the report order and the rows (
// readings Q8-Q11 of DESIGN.md §3).  report_block: one block (report_kernel, deferred runs);
// report_grid_*: spread over post_kernel's blocks when the run finalizes at once.
#pragma once
#include <cstddef>
#include "scl_internal.cuh"
#include "ptx.cuh"

namespace scl {

// Probability, rate and flag of one site, from the summed table.
// The flag is an integer decision (no division); bytes / 2^20 is an exact scaling.
struct SiteStat { double prob, rate; bool flag; };
__device__ __forceinline__ bool site_over(const FinalParams& p, unsigned long long m, unsigned long long f) {
    return p.formula == SCL_FORMULA_TEXTBOOK ? (unsigned __int128)m > (unsigned __int128)20 * f + 18    // 1-(f+1)/(m+2) > 0.95
                                             : (unsigned __int128)m > (unsigned __int128)21 * f + 18;   // reading Q9
}
__device__ __forceinline__ double site_prob(const FinalParams& p, unsigned long long m, unsigned long long f) {
    return p.formula == SCL_FORMULA_TEXTBOOK ? __dsub_rn(1.0, __ddiv_rn((double)(f + 1), (double)(m + 2)))
                                             : __dsub_rn(1.0, __ddiv_rn((double)(f + 1), (double)(m - f + 2)));   // Q8
}
__device__ __forceinline__ double site_rate(unsigned long long bytes, double elapsed_s) {
    return __ddiv_rn(__dmul_rn((double)bytes, 1.0 / 1048576.0), elapsed_s);     // MB / s (Q11)
}
__device__ __forceinline__ double elapsed_s(const FinalParams& p) { return __ddiv_rn(p.elapsed_ns, 1e9); }
__device__ __forceinline__ SiteStat site_stat(const FinalParams& p, unsigned sidx, bool open)
{
    const unsigned long long* row = p.table + (size_t)sidx * SCL_NCOL;
    const unsigned long long m = __ldcg(&row[SCL_COL_LEAK_MALLOCS]), f = __ldcg(&row[SCL_COL_LEAK_FREES]);
    SiteStat r;
    r.prob = site_prob(p, m, f);
    r.rate = site_rate(__ldcg(&row[SCL_COL_MALLOC_BYTES]), elapsed_s(p));
    r.flag = open && site_over(p, m, f);
    return r;
}

__device__ __forceinline__ bool gate_open(const FinalParams& p) {
    const unsigned long long* g = p.table + (size_t)p.n_sites * SCL_NCOL;
    const long long gnum = (long long)__ldcg(&g[0]), gden = (long long)__ldcg(&g[1]);
    return __ldcg(&g[2]) > 0 && (__int128)100 * (__int128)gnum >= (__int128)gden;
}

__device__ __forceinline__ void gate_copy(const FinalParams& p) {   // to the host-mapped buffer
    const unsigned long long* g = p.table + (size_t)p.n_sites * SCL_NCOL;
    p.gate_out[0] = __ldcg(&g[0]); p.gate_out[1] = __ldcg(&g[1]); p.gate_out[2] = __ldcg(&g[2]);
}


constexpr unsigned kReportSites = 16384, kReportList = 2048, kRowWords = sizeof(scl_site_row) / 8;   // 13
static_assert(sizeof(scl_site_row) == 104 && offsetof(scl_site_row, leak_flag) == 4 && offsetof(scl_site_row, col) == 8 &&
              offsetof(scl_site_row, leak_prob) == 88 && offsetof(scl_site_row, leak_rate_mbps) == 96,
              "report_block writes scl_site_row as 13 words: {site, flag}, col[10], prob, rate");
template <int NT> struct ReportSmem {
    double lrate[kReportList]; unsigned lsite[kReportList];          // flagged sites (any order)
    unsigned bits[kReportSites / 32], wpre[kReportSites / 32];        // flag bitmask, flags before each word
    unsigned wsum[32], nflag;
    unsigned long long stage[NT / 32][32 * kRowWords];                // per-warp row staging (coalesced writes)
};
template <int NT> constexpr size_t report_smem_bytes() { return sizeof(ReportSmem<NT>); }

// Report order: flagged sites by (rate desc, site asc), then the others by site (a6).  Rank of a
// flagged site = flagged sites with a larger rate, or the same rate and a smaller site; rank of an
// unflagged site = #flagged + unflagged sites before it, so the unflagged sites of a warp's 32
// consecutive sites take consecutive ranks: their rows are staged in shared memory and written
// with lane-contiguous stores.  Four sites per thread and pass are in flight at once (the passes
// are latency-bound).  n_sites <= kReportSites; blockDim.x == NT.
#ifndef SCL_RU
#define SCL_RU 1
#endif
constexpr int kRU = SCL_RU;                  // sites per thread and pass in flight: pass 2 (rows)
constexpr int kRU1 = 4;                      //   and pass 1 (two words per site: flags)
template <int NT>
__device__ void report_block(const FinalParams& p, scl_site_row* rows, ReportSmem<NT>& sm)
{
    const unsigned tid = threadIdx.x, lane = tid & 31, wrp = tid >> 5, S = p.n_sites, nw = (S + 31) / 32;
#ifdef SCL_PROFILE
#define RPT_T(i) if (p.prof && tid == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); p.prof[46 + (i)] = t_; }
#else
#define RPT_T(i)
#endif
    const bool open = gate_open(p);
    const double es = elapsed_s(p);
    if (tid == 0) { sm.nflag = 0; gate_copy(p); }
    __syncthreads();
    RPT_T(0)
    for (unsigned base = 0; base < S; base += kRU1 * NT) {    // pass 1: flags (integer only), flagged list
        unsigned long long m[kRU1], f[kRU1];
        #pragma unroll
        for (int k = 0; k < kRU1; ++k) {
            const unsigned sidx = base + k * NT + tid;
            m[k] = f[k] = 0;
            if (sidx < S) {
                const unsigned long long* row = p.table + (size_t)sidx * SCL_NCOL;
                m[k] = __ldcg(&row[SCL_COL_LEAK_MALLOCS]); f[k] = __ldcg(&row[SCL_COL_LEAK_FREES]);
            }
        }
        #pragma unroll
        for (int k = 0; k < kRU1; ++k) {
            const unsigned sidx = base + k * NT + tid;
            const bool fl = sidx < S && open && site_over(p, m[k], f[k]);
            if (fl) {
                const unsigned q = atomicAdd(&sm.nflag, 1u);
                if (q < kReportList) {
                    sm.lrate[q] = site_rate(__ldcg(&p.table[(size_t)sidx * SCL_NCOL + SCL_COL_MALLOC_BYTES]), es);
                    sm.lsite[q] = sidx;
                }
            }
            const unsigned word = __ballot_sync(kFull, fl);
            const unsigned wi = ((base + k * NT) >> 5) + wrp;
            if (lane == 0 && wi < nw) sm.bits[wi] = word;
        }
    }
    __syncthreads();
    for (unsigned w0 = 0; w0 < nw; w0 += NT) {              // exclusive prefix of flags per word
        const unsigned w = w0 + tid;
        const unsigned c = w < nw ? __popc(sm.bits[w]) : 0u;
        unsigned inc = c;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) { const unsigned o = __shfl_up_sync(kFull, inc, d); if (lane >= (unsigned)d) inc += o; }
        if (lane == 31) sm.wsum[wrp] = inc;
        __syncthreads();
        unsigned wb = w0 ? sm.wpre[w0 - 1] + __popc(sm.bits[w0 - 1]) : 0u;
        for (unsigned q = 0; q < wrp; ++q) wb += sm.wsum[q];
        if (w < nw) sm.wpre[w] = wb + inc - c;
        __syncthreads();
    }
    const unsigned F = sm.nflag;
    RPT_T(1)
    unsigned long long* stg = sm.stage[wrp];
    for (unsigned base = 0; base < S; base += kRU * NT) {    // pass 2: stats, ranks, rows
        ulonglong2 rv[kRU][SCL_NCOL / 2];                   // the table rows, one load each
        #pragma unroll
        for (int k = 0; k < kRU; ++k) {
            const unsigned sidx = base + k * NT + tid;
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(p.table + (size_t)min(sidx, S - 1) * SCL_NCOL);
            #pragma unroll
            for (int c = 0; c < SCL_NCOL / 2; ++c) rv[k][c] = __ldcg(src + c);
        }
        #pragma unroll
        for (int k = 0; k < kRU; ++k) {
            const unsigned sidx = base + k * NT + tid;
            const bool in = sidx < S;
            const unsigned word = in ? sm.bits[sidx >> 5] : 0u;
            const bool fl = in && ((word >> lane) & 1u);
            const unsigned um = __ballot_sync(kFull, in && !fl);  // unflagged lanes: consecutive ranks
            if (in) {
                const unsigned long long m = SCL_COL_LEAK_MALLOCS % 2 ? rv[k][SCL_COL_LEAK_MALLOCS / 2].y : rv[k][SCL_COL_LEAK_MALLOCS / 2].x;
                const unsigned long long f = SCL_COL_LEAK_FREES % 2 ? rv[k][SCL_COL_LEAK_FREES / 2].y : rv[k][SCL_COL_LEAK_FREES / 2].x;
                const unsigned long long by = SCL_COL_MALLOC_BYTES % 2 ? rv[k][SCL_COL_MALLOC_BYTES / 2].y : rv[k][SCL_COL_MALLOC_BYTES / 2].x;
                const double prob = site_prob(p, m, f), rate = site_rate(by, es);
                // the row's 13 words: {site, flag}, col[0..9], prob, rate  (scl_site_row layout)
                auto word_at = [&](int q) -> unsigned long long {
                    if (q == 0) return (unsigned long long)sidx | ((unsigned long long)(fl ? 1u : 0u) << 32);
                    if (q == 11) return (unsigned long long)__double_as_longlong(prob);
                    if (q == 12) return (unsigned long long)__double_as_longlong(rate);
                    return (q - 1) % 2 ? rv[k][(q - 1) / 2].y : rv[k][(q - 1) / 2].x;
                };
                if (fl) {
                    unsigned rank = 0;
                    if (F <= kReportList) {
                        for (unsigned q = 0; q < F; ++q)
                            rank += (sm.lrate[q] > rate || (sm.lrate[q] == rate && sm.lsite[q] < sidx)) ? 1u : 0u;
                    } else {                                // many flagged sites: compare against all
                        for (unsigned j = 0; j < S; ++j) {
                            const SiteStat o = site_stat(p, j, open);
                            rank += (o.flag && (o.rate > rate || (o.rate == rate && j < sidx))) ? 1u : 0u;
                        }
                    }
                    unsigned long long* dst = reinterpret_cast<unsigned long long*>(rows + rank);
                    #pragma unroll
                    for (int q = 0; q < (int)kRowWords; ++q) dst[q] = word_at(q);
                } else {
                    const unsigned j = __popc(um & ((1u << lane) - 1u));      // slot among the warp's unflagged
                    #pragma unroll
                    for (int q = 0; q < (int)kRowWords; ++q) stg[j * kRowWords + q] = word_at(q);
                }
            }
            __syncwarp();
            if (um) {
                const unsigned s_first = base + k * NT + (wrp << 5) + (unsigned)(__ffs(um) - 1);
                const unsigned r0 = F + s_first - (sm.wpre[s_first >> 5] + __popc(sm.bits[s_first >> 5] & ((1u << (s_first & 31)) - 1u)));
                unsigned long long* dst = reinterpret_cast<unsigned long long*>(rows + r0);
                const unsigned nwds = (unsigned)__popc(um) * kRowWords;
                for (unsigned q = lane; q < nwds; q += 32) dst[q] = stg[q];
            }
            __syncwarp();
        }
    }
}

// ---- a6 spread over a whole grid (post_kernel, fused; or report_flags_kernel + report_rows_kernel
// after a deferred finalize of a table above kReportSites): warp w owns the 32 sites of word w.
// Any table size: bits has one word per 32 sites and sbcnt one flag count per kSuper words (both
// zeroed before C1, like nflag), so the flagged sites before a word are <= n/2^15 + kSuper terms.
constexpr unsigned kSuper = 1024;                              // bitmask words per superblock count
struct ReportScratch { unsigned* bits; double* lrate; unsigned* lsite; unsigned* nflag; unsigned* sbcnt; };

// C1: integer flags (bitmask word per warp), flagged sites (rate, site) appended to a global list.
static __device__ void report_grid_flags(const FinalParams& p, const ReportScratch& x, unsigned wid, unsigned nw, int lane)
{
    const unsigned S = p.n_sites, nwd = (S + 31) / 32;
    const bool open = gate_open(p);
    const double es = elapsed_s(p);
    if (wid == 0 && lane == 0) gate_copy(p);
    for (unsigned w = wid; w < nwd; w += nw) {
        const unsigned sidx = w * 32 + (unsigned)lane;
        bool fl = false;
        if (sidx < S) {
            const unsigned long long* row = p.table + (size_t)sidx * SCL_NCOL;
            fl = open && site_over(p, __ldcg(&row[SCL_COL_LEAK_MALLOCS]), __ldcg(&row[SCL_COL_LEAK_FREES]));
            if (fl) {
                const unsigned q = atomicAdd(x.nflag, 1u);
                if (q < kReportList) { x.lrate[q] = site_rate(__ldcg(&row[SCL_COL_MALLOC_BYTES]), es); x.lsite[q] = sidx; }
            }
        }
        const unsigned word = __ballot_sync(kFull, fl);
        if (lane == 0) { x.bits[w] = word; if (word) atomicAdd(&x.sbcnt[w / kSuper], (unsigned)__popc(word)); }
    }
}

// C2: ranks and rows (after a grid barrier): flagged sites against the flagged list, unflagged
// sites = #flagged + unflagged sites before them (staged, lane-contiguous stores).
static __device__ void report_grid_rows(const FinalParams& p, scl_site_row* rows, const ReportScratch& x,
                                 unsigned long long* stg, unsigned wid, unsigned nw, int lane)
{
    const unsigned S = p.n_sites, nwd = (S + 31) / 32;
    const bool open = gate_open(p);
    const double es = elapsed_s(p);
    const unsigned F = __ldcg(x.nflag);
    for (unsigned w = wid; w < nwd; w += nw) {
        unsigned fbw = 0;                                      // flagged sites before word w
        for (unsigned q = (unsigned)lane; q < w / kSuper; q += 32) fbw += __ldcg(&x.sbcnt[q]);
        for (unsigned q = w / kSuper * kSuper + (unsigned)lane; q < w; q += 32) fbw += __popc(__ldcg(&x.bits[q]));
        fbw = (unsigned)warp_sum((long long)fbw);
        const unsigned word = __ldcg(&x.bits[w]);
        const unsigned sidx = w * 32 + (unsigned)lane;
        const bool in = sidx < S, fl = in && ((word >> lane) & 1u);
        const unsigned um = __ballot_sync(kFull, in && !fl);
        if (in) {
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(p.table + (size_t)sidx * SCL_NCOL);
            ulonglong2 rv[SCL_NCOL / 2];
            #pragma unroll
            for (int c = 0; c < SCL_NCOL / 2; ++c) rv[c] = __ldcg(src + c);
            auto col = [&](int c) { return (c & 1) ? rv[c >> 1].y : rv[c >> 1].x; };
            const double prob = site_prob(p, col(SCL_COL_LEAK_MALLOCS), col(SCL_COL_LEAK_FREES));
            const double rate = site_rate(col(SCL_COL_MALLOC_BYTES), es);
            auto word_at = [&](int q) -> unsigned long long {
                if (q == 0) return (unsigned long long)sidx | ((unsigned long long)(fl ? 1u : 0u) << 32);
                if (q == 11) return (unsigned long long)__double_as_longlong(prob);
                if (q == 12) return (unsigned long long)__double_as_longlong(rate);
                return col(q - 1);
            };
            if (fl) {
                unsigned rank = 0;
                if (F <= kReportList) {
                    for (unsigned q = 0; q < F; ++q) {
                        const double r2 = __ldcg(&x.lrate[q]);
                        rank += (r2 > rate || (r2 == rate && __ldcg(&x.lsite[q]) < sidx)) ? 1u : 0u;
                    }
                } else {                                       // many flagged sites: compare against all
                    for (unsigned j = 0; j < S; ++j) {
                        const SiteStat o = site_stat(p, j, open);
                        rank += (o.flag && (o.rate > rate || (o.rate == rate && j < sidx))) ? 1u : 0u;
                    }
                }
                unsigned long long* dst = reinterpret_cast<unsigned long long*>(rows + rank);
                #pragma unroll
                for (int q = 0; q < (int)kRowWords; ++q) dst[q] = word_at(q);
            } else {
                const unsigned j = __popc(um & ((1u << lane) - 1u));
                #pragma unroll
                for (int q = 0; q < (int)kRowWords; ++q) stg[j * kRowWords + q] = word_at(q);
            }
        }
        __syncwarp();
        if (um) {
            const int l1 = __ffs(um) - 1;                      // the first unflagged lane
            const unsigned r0 = F + w * 32 + (unsigned)l1 - (fbw + __popc(word & ((1u << l1) - 1u)));
            unsigned long long* dst = reinterpret_cast<unsigned long long*>(rows + r0);
            const unsigned nwds = (unsigned)__popc(um) * kRowWords;
            for (unsigned q = (unsigned)lane; q < nwds; q += 32) dst[q] = stg[q];
        }
        __syncwarp();
    }
}

cudaError_t launch_report_grid(const FinalParams& p, const ReportScratch& x, scl_site_row* rows, cudaStream_t st);

}  // namespace scl
