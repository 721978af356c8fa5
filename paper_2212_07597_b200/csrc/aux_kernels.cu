// aux_kernels.cu -- small sm_100a kernels around the streaming replay kernel:
//   load_stats_kernel  per-trace sum|d| (sample-capacity bound) + argument check, at load time
//   report_kernel      a6 in one block (tables <= kReportSites): probability, rate
//                      (P:65-69), flag, report order and rows
//   report_flags_kernel / report_rows_kernel   the same over a grid, for larger tables
#include "scl_internal.cuh"
#include "ptx.cuh"
#include "report.cuh"
#include <algorithm>

namespace scl {

// ============================================================================ load statistics
// Per trace: sum |d| over alloc/free events (the sample-capacity bound floor(sum|d|/T)), and
// the first invalid event (size 0, kind 3, site >= n_sites).  One warp per 256-event chunk
// (grid-stride, 8 events = one 128-B row per lane); a chunk inside one trace is reduced in the
// warp before its single atomic.  dst != NULL: the same pass is the load's copy (ev: the caller's
// device buffer or pinned host memory mapped into the device's address space; dst: the handle's
// device copy), so the events reach HBM once and are not read back for the statistics.
__global__ void __launch_bounds__(256) load_stats_kernel(const scl_event* ev, const unsigned long long* off,
                                                         unsigned n_traces, unsigned long long n_events,
                                                         unsigned n_sites, unsigned long long* sabs,
                                                         unsigned long long* err, scl_event* dst,
                                                         unsigned long long* shist, const unsigned* remap)
{
    // histogram of floor(log2(size)) over the alloc / free events (how many sync events |d| >= 2T - 1
    // a threshold T has: the chain-split heuristic of scl_replay_run), per block in shared memory
    __shared__ unsigned hist[64];
    if (threadIdx.x < 64) hist[threadIdx.x] = 0;
    __syncthreads();
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
        if (remap) {                                         // site ids by load-time frequency (see upload)
            ulonglong2* o = reinterpret_cast<ulonglong2*>((dst ? dst : const_cast<scl_event*>(ev)) + i0);
            #pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (i0 + j < n_events) {
                    const unsigned long long m = v[j].y;
                    const unsigned site = ev_site(m);
                    const unsigned long long m2 = site < n_sites
                        ? (m & ((1ull << 43) - 1ull)) | ((unsigned long long)__ldg(remap + site) << 43) : m;
                    if (dst) o[j] = make_ulonglong2(v[j].x, m2);
                    else if (m2 != m) o[j].y = m2;
                }
            }
        } else if (dst) {
            ulonglong2* o = reinterpret_cast<ulonglong2*>(dst + i0);
            #pragma unroll
            for (int j = 0; j < 8; ++j) if (i0 + j < n_events) o[j] = v[j];
        }
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
            if (kind < 2) { acc += sz; if (sz) atomicAdd(&hist[63 - __clzll(sz)], 1u); }
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
    __syncthreads();
    if (threadIdx.x < 64 && hist[threadIdx.x]) atomicAdd(&shist[threadIdx.x], (unsigned long long)hist[threadIdx.x]);
}

// ============================================================================ a6 (report.cuh)
// Tables above kReportSites after a deferred finalize: C1 (flags, flagged list) and C2 (ranks, rows)
// as two stream-ordered grid kernels (the launch boundary is the grid barrier of the fused path).
constexpr int kRptThreads = 256;
__global__ void __launch_bounds__(kRptThreads) report_flags_kernel(const __grid_constant__ FinalParams p, ReportScratch x)
{
    const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    report_grid_flags(p, x, wid, nw, threadIdx.x & 31);
}
__global__ void __launch_bounds__(kRptThreads) report_rows_kernel(const __grid_constant__ FinalParams p, ReportScratch x,
                                                                 scl_site_row* rows)
{
    __shared__ unsigned long long stg[kRptThreads / 32][32 * kRowWords];
    const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    report_grid_rows(p, rows, x, stg[threadIdx.x >> 5], wid, nw, threadIdx.x & 31);
}

// Whole a6 in one block (n_sites <= kReportSites): report.cuh.
__global__ void __launch_bounds__(512) report_kernel(const __grid_constant__ FinalParams p, scl_site_row* rows)
{
    extern __shared__ __align__(16) unsigned char report_smem[];
    report_block<512>(p, rows, *reinterpret_cast<ReportSmem<512>*>(report_smem));
}

// ============================================================================ launch wrappers
cudaError_t launch_load_stats(const scl_event* ev, const unsigned long long* off, unsigned n_traces,
                              unsigned long long n_events, unsigned n_sites, unsigned long long* sabs,
                              unsigned long long* err, scl_event* dst, unsigned long long* shist,
                              const unsigned* remap, cudaStream_t st)
{
    if (n_traces == 0 || n_events == 0) return cudaSuccess;
    const unsigned long long warps = (n_events + 255) / 256;
    const unsigned blocks = (unsigned)std::min<unsigned long long>((warps + 7) / 8, 148ull * 8);
    load_stats_kernel<<<blocks, 256, 0, st>>>(ev, off, n_traces, n_events, n_sites, sabs, err, dst, shist, remap);
    return cudaGetLastError();
}

// Load-time site frequencies (the site renumbering, api.cu site_remap) from a device source: every
// stride-th event's site (allocs and frees), counted in cnt[n_sites] -- one kernel and one small
// copy back instead of a strided 16-B-row copy of the sample to the host.
__global__ void site_sample_kernel(const scl_event* src, unsigned long long stride, unsigned long long m,
                                   unsigned n_sites, unsigned* cnt)
{
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long meta = __ldg(&src[i * stride].meta);
        const unsigned site = ev_site(meta);
        if (site < n_sites && ev_kind(meta) < 2) atomicAdd(&cnt[site], 1u);
    }
}

cudaError_t launch_site_sample(const scl_event* src, unsigned long long stride, unsigned long long m,
                               unsigned n_sites, unsigned* cnt, cudaStream_t st)
{
    if (m == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)std::min<unsigned long long>((m + 255) / 256, 148ull * 8);
    site_sample_kernel<<<blocks, 256, 0, st>>>(src, stride, m, n_sites, cnt);
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

// The summable table in the caller's site order: tout[c] = tin[remap[c]] (+ the gate words).
__global__ void __launch_bounds__(256) permute_table_kernel(const unsigned long long* tin, unsigned long long* tout,
                                                            const unsigned* remap, unsigned n_sites)
{
    const size_t n = (size_t)n_sites * SCL_NCOL + 3;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t c = i / SCL_NCOL;
        tout[i] = c < n_sites ? __ldcg(tin + (size_t)__ldg(remap + c) * SCL_NCOL + i % SCL_NCOL) : __ldcg(tin + i);
    }
}

cudaError_t launch_permute_table(const unsigned long long* tin, unsigned long long* tout, const unsigned* remap,
                                 unsigned n_sites, cudaStream_t st)
{
    const size_t n = (size_t)n_sites * SCL_NCOL + 3;
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
    permute_table_kernel<<<blocks, 256, 0, st>>>(tin, tout, remap, n_sites);
    return cudaGetLastError();
}

cudaError_t launch_report_grid(const FinalParams& p, const ReportScratch& x, scl_site_row* rows, cudaStream_t st)
{
    const unsigned words = (p.n_sites + 31) / 32;
    const unsigned blocks = std::max(1u, std::min((words + kRptThreads / 32 - 1) / (kRptThreads / 32), 148u * 8));
    report_flags_kernel<<<blocks, kRptThreads, 0, st>>>(p, x);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    report_rows_kernel<<<blocks, kRptThreads, 0, st>>>(p, x, rows);
    return cudaGetLastError();
}

}  // namespace scl
