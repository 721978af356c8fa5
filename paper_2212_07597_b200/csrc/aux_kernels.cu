// aux_kernels.cu -- small sm_100a kernels around the streaming replay kernel:
//   load_stats_kernel  per-trace sum|d| (sample-capacity bound) + argument check, at load time
//   finalize_kernel    a6: leak probability, rate, flag, sort key
//   rows_kernel        report rows in report order
#include "scl_internal.cuh"
#include "ptx.cuh"
#include "report.cuh"
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

// ============================================================================ a6
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

// Whole a6 in one block (n_sites <= kReportSites): report.cuh.
__global__ void __launch_bounds__(512) report_kernel(const __grid_constant__ FinalParams p, scl_site_row* rows)
{
    extern __shared__ __align__(16) unsigned char report_smem[];
    report_block<512>(p, rows, *reinterpret_cast<ReportSmem<512>*>(report_smem));
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

bool report_fused(unsigned n_sites) { return n_sites <= kReportSites; }

cudaError_t launch_report(const FinalParams& p, scl_site_row* rows, cudaStream_t st)
{
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(report_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)report_smem_bytes<512>());
        if (e != cudaSuccess) return e;
        attr = true;
    }
    report_kernel<<<1, 512, report_smem_bytes<512>(), st>>>(p, rows);
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
