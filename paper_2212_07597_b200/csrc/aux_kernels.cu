// aux_kernels.cu -- small sm_100a kernels around the streaming replay kernel:
//   load_stats_kernel  per-trace sum|d| (sample-capacity bound) + argument check, at load time
//   finalize_kernel    a6: leak probability, rate, flag, sort key
//   rows_kernel        report rows in report order
#include "scl_internal.cuh"
#include "ptx.cuh"
#include <algorithm>

namespace scl {

// ============================================================================ load statistics
// Per trace: sum |d| over alloc/free events (the sample-capacity bound floor(sum|d|/T)), and
// the first invalid event (size 0, kind 3, site >= n_sites).  One warp per 256-event chunk
// (grid-stride, 8 events = one 128-B row per lane); a chunk inside one trace is reduced in the
// warp before its single atomic.
__global__ void __launch_bounds__(256) load_stats_kernel(const scl_event* ev, const unsigned long long* off,
                                                         unsigned n_traces, unsigned long long n_events,
                                                         unsigned n_sites, unsigned long long* sabs,
                                                         unsigned long long* err)
{
    const int lane = threadIdx.x & 31;
    const unsigned long long wid = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    for (unsigned long long base = wid * 256; base < n_events; base += nw * 256) {
        const unsigned long long i0 = base + (unsigned long long)lane * 8;
        // trace of event i0: last t with off[t] <= i0 (traces may be empty)
        unsigned lo = 0, hi = n_traces;                      // invariant: off[lo] <= i0 < off[hi]
        while (hi - lo > 1) { const unsigned mid = (lo + hi) >> 1; if (off[mid] <= i0) lo = mid; else hi = mid; }
        unsigned t = lo;
        unsigned long long tend = off[t + 1];
        const ulonglong2* q = reinterpret_cast<const ulonglong2*>(ev + i0);
        ulonglong2 v[8];
        #pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = i0 + j < n_events ? __ldcs(q + j) : make_ulonglong2(0, 0);
        unsigned long long acc = 0;
        bool split = false;
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            const unsigned long long i = i0 + j;
            if (i >= n_events) break;
            while (i >= tend) {                             // trace boundary inside this lane's row
                if (acc) atomicAdd(&sabs[t], acc);
                acc = 0; split = true; ++t; tend = off[t + 1];
            }
            const unsigned long long m = v[j].y;
            const unsigned kind = ev_kind(m);
            const unsigned long long sz = ev_size(m);
            if (kind == 3 || ev_site(m) >= n_sites || (kind < 2 && sz == 0)) atomicMin(err, i);
            if (kind < 2) acc += sz;
        }
        const unsigned t_lane0 = __shfl_sync(kFull, t, 0);  // every lane shuffles (never inside a short circuit)
        const bool uni = __all_sync(kFull, !split && t == t_lane0);
        if (uni) {
            #pragma unroll
            for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
            if (lane == 0 && acc) atomicAdd(&sabs[t], acc);
        } else if (acc) {
            atomicAdd(&sabs[t], acc);
        }
    }
}

// ============================================================================ per-run preparation
__global__ void __launch_bounds__(1024) prep_kernel(const __grid_constant__ PrepParams p)
{
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
    for (size_t i = tid; i < p.table_words; i += nth) p.table[i] = 0;
    for (size_t i = tid; i < p.summ_words; i += nth) p.summ[i] = 0;
    for (size_t i = tid; i < p.run_words; i += nth) p.run[i] = 0;
    if (tid < 4) p.ticket[tid] = 0;
    if (blockIdx.x != 0) return;
    // block 0: exclusive scan of the per-trace sample capacities (thread j: a contiguous run of traces)
    __shared__ unsigned long long part[1024];
    const unsigned per = (p.n_traces + blockDim.x - 1) / blockDim.x;
    const unsigned t0 = threadIdx.x * per, t1 = min(p.n_traces, t0 + per);
    auto cap = [&](unsigned t) {
        const unsigned long long n = p.off[t + 1] - p.off[t], b = p.sabs[t] / p.T;
        return n < b ? n : b;
    };
    unsigned long long acc = 0;
    for (unsigned t = t0; t < t1; ++t) acc += cap(t);
    part[threadIdx.x] = acc;
    __syncthreads();
    for (unsigned d = 1; d < blockDim.x; d <<= 1) {          // Hillis-Steele inclusive scan
        const unsigned long long v = threadIdx.x >= d ? part[threadIdx.x - d] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned long long base = part[threadIdx.x] - acc;
    for (unsigned t = t0; t < t1; ++t) { p.sbase[t] = base; base += cap(t); }
}

// ============================================================================ a6
// Probability, rate and flag of one site, from the summed table.
struct SiteStat { double prob, rate; bool flag; };
__device__ __forceinline__ SiteStat site_stat(const FinalParams& p, unsigned sidx, bool open)
{
    const unsigned long long* row = p.table + (size_t)sidx * SCL_NCOL;
    const unsigned long long m = row[SCL_COL_LEAK_MALLOCS], f = row[SCL_COL_LEAK_FREES];
    SiteStat r;
    bool over;
    if (p.formula == SCL_FORMULA_TEXTBOOK) {
        r.prob = __dsub_rn(1.0, __ddiv_rn((double)(f + 1), (double)(m + 2)));
        over = (unsigned __int128)m > (unsigned __int128)20 * f + 18;
    } else {   // P:55-57, exactly as printed (reading Q8); flag p > 0.95 <=> m > 21 f + 18 (Q9)
        r.prob = __dsub_rn(1.0, __ddiv_rn((double)(f + 1), (double)(m - f + 2)));
        over = (unsigned __int128)m > (unsigned __int128)21 * f + 18;
    }
    r.rate = __ddiv_rn(__ddiv_rn((double)row[SCL_COL_MALLOC_BYTES], 1048576.0), __ddiv_rn(p.elapsed_ns, 1e9));
    r.flag = open && over;
    return r;
}

__device__ __forceinline__ bool gate_open(const FinalParams& p) {
    const unsigned long long* g = p.table + (size_t)p.n_sites * SCL_NCOL;
    const long long gnum = (long long)g[0], gden = (long long)g[1];
    return g[2] > 0 && (__int128)100 * (__int128)gnum >= (__int128)gden;
}

__device__ __forceinline__ void gate_copy(const FinalParams& p) {   // to the host-mapped buffer
    const unsigned long long* g = p.table + (size_t)p.n_sites * SCL_NCOL;
    p.gate_out[0] = g[0]; p.gate_out[1] = g[1]; p.gate_out[2] = g[2];
}

__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ FinalParams p)
{
    const bool open = gate_open(p);
    if (blockIdx.x == 0 && threadIdx.x == 0) gate_copy(p);
    for (unsigned sidx = blockIdx.x * blockDim.x + threadIdx.x; sidx < p.n_sites; sidx += gridDim.x * blockDim.x) {
        const SiteStat st = site_stat(p, sidx, open);
        p.prob[sidx] = st.prob; p.rate[sidx] = st.rate; p.flag[sidx] = st.flag ? 1 : 0;
        // report order key: flagged by rate desc (rate >= 0, so ~bits is descending), others last;
        // a stable radix sort over site-ordered input breaks ties by site asc.
        p.key1[sidx] = st.flag ? ~(unsigned long long)__double_as_longlong(st.rate) : ~0ull;
        p.val[sidx] = sidx;
    }
}

__device__ __forceinline__ void write_row(const FinalParams& p, scl_site_row* rows, unsigned rank, unsigned sidx,
                                          const SiteStat& st)
{
    scl_site_row r;
    r.site = sidx; r.leak_flag = st.flag ? 1u : 0u;
    #pragma unroll
    for (int c = 0; c < SCL_NCOL; ++c) r.col[c] = p.table[(size_t)sidx * SCL_NCOL + c];
    r.leak_prob = st.prob; r.leak_rate_mbps = st.rate;
    rows[rank] = r;
}

// Whole a6 in one block (n_sites <= kReportSites): stats, report order, rows.  Rank of a flagged
// site = flagged sites with a larger rate, or the same rate and a smaller site; rank of the
// others = #flagged + unflagged sites before it (site order).
constexpr unsigned kReportSites = 16384, kReportList = 2048;
__global__ void __launch_bounds__(1024) report_kernel(const __grid_constant__ FinalParams p, scl_site_row* rows)
{
    __shared__ double lrate[kReportList];
    __shared__ unsigned lsite[kReportList];
    __shared__ unsigned nflag, part[1024];
    const unsigned tid = threadIdx.x, S = p.n_sites;
    const unsigned per = (S + 1023) / 1024, s0 = min(S, tid * per), s1 = min(S, s0 + per);
    const bool open = gate_open(p);
    if (tid == 0) { nflag = 0; gate_copy(p); }
    __syncthreads();
    unsigned cf = 0;
    for (unsigned sidx = s0; sidx < s1; ++sidx) {
        const SiteStat st = site_stat(p, sidx, open);
        if (st.flag) {
            ++cf;
            const unsigned k = atomicAdd(&nflag, 1u);
            if (k < kReportList) { lrate[k] = st.rate; lsite[k] = sidx; }
        }
    }
    part[tid] = cf;
    __syncthreads();
    for (unsigned d = 1; d < 1024; d <<= 1) {               // inclusive scan of the flag counts
        const unsigned v = tid >= d ? part[tid - d] : 0;
        __syncthreads();
        part[tid] += v;
        __syncthreads();
    }
    const unsigned F = nflag;
    unsigned fb = part[tid] - cf;                           // flagged sites before s0
    for (unsigned sidx = s0; sidx < s1; ++sidx) {
        const SiteStat st = site_stat(p, sidx, open);
        unsigned rank;
        if (!st.flag) {
            rank = F + (sidx - fb);
        } else {
            rank = 0;
            if (F <= kReportList) {
                for (unsigned k = 0; k < F; ++k)
                    rank += (lrate[k] > st.rate || (lrate[k] == st.rate && lsite[k] < sidx)) ? 1u : 0u;
            } else {                                        // many flagged sites: compare against all
                for (unsigned j = 0; j < S; ++j) {
                    const SiteStat o = site_stat(p, j, open);
                    rank += (o.flag && (o.rate > st.rate || (o.rate == st.rate && j < sidx))) ? 1u : 0u;
                }
            }
            ++fb;
        }
        write_row(p, rows, rank, sidx, st);
    }
}

__global__ void __launch_bounds__(256) rows_kernel(const unsigned long long* table, const double* prob, const double* rate,
                                                   const unsigned char* flag, const unsigned int* order, unsigned n_sites,
                                                   scl_site_row* rows)
{
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n_sites; i += gridDim.x * blockDim.x) {
        const unsigned sidx = order[i];
        scl_site_row r;
        r.site = sidx; r.leak_flag = flag[sidx];
        #pragma unroll
        for (int c = 0; c < SCL_NCOL; ++c) r.col[c] = table[(size_t)sidx * SCL_NCOL + c];
        r.leak_prob = prob[sidx]; r.leak_rate_mbps = rate[sidx];
        rows[i] = r;
    }
}

// ============================================================================ launch wrappers
cudaError_t launch_load_stats(const scl_event* ev, const unsigned long long* off, unsigned n_traces,
                              unsigned long long n_events, unsigned n_sites, unsigned long long* sabs,
                              unsigned long long* err, cudaStream_t st)
{
    if (n_traces == 0 || n_events == 0) return cudaSuccess;
    const unsigned long long warps = (n_events + 255) / 256;
    const unsigned blocks = (unsigned)std::min<unsigned long long>((warps + 7) / 8, 148ull * 8);
    load_stats_kernel<<<blocks, 256, 0, st>>>(ev, off, n_traces, n_events, n_sites, sabs, err);
    return cudaGetLastError();
}

cudaError_t launch_prep(const PrepParams& p, cudaStream_t st)
{
    size_t words = p.table_words > p.summ_words ? p.table_words : p.summ_words;
    words = words > p.run_words ? words : p.run_words;
    unsigned blocks = (unsigned)std::min<size_t>((words + 1023) / 1024, 148);
    prep_kernel<<<blocks ? blocks : 1, 1024, 0, st>>>(p);
    return cudaGetLastError();
}

bool report_fused(unsigned n_sites) { return n_sites <= kReportSites; }

cudaError_t launch_report(const FinalParams& p, scl_site_row* rows, cudaStream_t st)
{
    report_kernel<<<1, 1024, 0, st>>>(p, rows);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalParams& p, cudaStream_t st)
{
    unsigned blocks = (p.n_sites + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    if (blocks == 0) blocks = 1;
    finalize_kernel<<<blocks, 256, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_rows(const unsigned long long* table, const double* prob, const double* rate,
                        const unsigned char* flag, const unsigned int* order, unsigned n_sites,
                        scl_site_row* rows, cudaStream_t st)
{
    unsigned blocks = (n_sites + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    if (blocks == 0) blocks = 1;
    rows_kernel<<<blocks, 256, 0, st>>>(table, prob, rate, flag, order, n_sites, rows);
    return cudaGetLastError();
}

}  // namespace scl
