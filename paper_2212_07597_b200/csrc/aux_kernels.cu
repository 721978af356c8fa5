// aux_kernels.cu -- small sm_100a kernels around the streaming replay kernel:
//   load_stats_kernel  per-trace sum|d| (sample-capacity bound) + argument check, at load time
//   samples_kernel     Tier-S, leak (mallocs, frees) and gate sums from the sample lists
//   finalize_kernel    a6: leak probability, rate, flag, sort key
//   rows_kernel        report rows in report order
#include "scl_internal.cuh"
#include "ptx.cuh"

namespace scl {

// ============================================================================ load statistics
// Per trace: sum |d| over alloc/free events (the sample-capacity bound
// floor(sum|d|/T)), and the first invalid event (size 0, kind 3, site >= n_sites).
__global__ void __launch_bounds__(256) load_stats_kernel(const scl_event* ev, const unsigned long long* off,
                                                         unsigned n_traces, unsigned n_sites,
                                                         unsigned long long* sabs, unsigned long long* err)
{
    __shared__ unsigned long long red[8];
    for (unsigned t = blockIdx.x; t < n_traces; t += gridDim.x) {
        const unsigned long long b = off[t], e = off[t + 1];
        unsigned long long acc = 0;
        for (unsigned long long i = b + threadIdx.x; i < e; i += blockDim.x) {
            const unsigned long long m = ev[i].meta;
            const unsigned kind = ev_kind(m);
            const unsigned long long sz = ev_size(m);
            if (kind == 3 || ev_site(m) >= n_sites || (kind < 2 && sz == 0)) atomicMin(err, i);
            if (kind < 2) acc += sz;
        }
        #pragma unroll
        for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long tot = 0;
            for (int w = 0; w < 8; ++w) tot += red[w];
            sabs[t] = tot;
        }
        __syncthreads();
    }
}

// ============================================================================ per-sample reduce
// One warp per trace: Tier-S columns, leak score (mallocs at episode start,
// frees if the episode's object was reclaimed), footprint-trend
// endpoints and the gate sums (reading Q10).
__global__ void __launch_bounds__(256) samples_kernel(const __grid_constant__ ReplayParams p)
{
    const int lane = threadIdx.x & 31;
    const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nw = (gridDim.x * blockDim.x) >> 5;
    unsigned long long* gate = p.table + (size_t)p.n_sites * SCL_NCOL;
    for (unsigned t = wid; t < p.n_traces; t += nw) {
        const unsigned long long n = p.summ[t].n_samples, sb = p.sbase[t];
        for (unsigned long long i = lane; i < n; i += 32) {
            const scl_sample sm = p.samples[sb + i];
            unsigned long long* row = p.table + (size_t)sm.site * SCL_NCOL;
            if (sm.kind == 0) { atomicAdd(&row[SCL_COL_N_GROWTH], 1ull); atomicAdd(&row[SCL_COL_GROWTH_BYTES], (unsigned long long)sm.net); }
            else              { atomicAdd(&row[SCL_COL_N_DECLINE], 1ull); atomicAdd(&row[SCL_COL_DECLINE_BYTES], (unsigned long long)(-sm.net)); }
            if (sm.new_max) {
                atomicAdd(&row[SCL_COL_LEAK_MALLOCS], 1ull);
                if (p.ep_flag[sb + i]) atomicAdd(&row[SCL_COL_LEAK_FREES], 1ull);
            }
        }
        if (lane == 0) {
            long long ff = 0, fl = 0;
            if (n > 0) { ff = p.samples[sb].footprint; fl = p.samples[sb + n - 1].footprint; }
            p.summ[t].f_first_sample = ff; p.summ[t].f_last_sample = fl;
            if (n >= 2) {
                atomicAdd(&gate[0], (unsigned long long)(fl - ff));
                atomicAdd(&gate[1], (unsigned long long)(ff > 1 ? ff : 1));
                atomicAdd(&gate[2], 1ull);
            }
        }
    }
}

// ============================================================================ a6
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ FinalParams p)
{
    const unsigned long long* g = p.table + (size_t)p.n_sites * SCL_NCOL;
    const long long gnum = (long long)g[0], gden = (long long)g[1];
    const bool open = g[2] > 0 && (__int128)100 * (__int128)gnum >= (__int128)gden;
    for (unsigned sidx = blockIdx.x * blockDim.x + threadIdx.x; sidx < p.n_sites; sidx += gridDim.x * blockDim.x) {
        const unsigned long long* row = p.table + (size_t)sidx * SCL_NCOL;
        const unsigned long long m = row[SCL_COL_LEAK_MALLOCS], f = row[SCL_COL_LEAK_FREES];
        double prob; bool over;
        if (p.formula == SCL_FORMULA_TEXTBOOK) {
            prob = __dsub_rn(1.0, __ddiv_rn((double)(f + 1), (double)(m + 2)));
            over = (unsigned __int128)m > (unsigned __int128)20 * f + 18;
        } else {   // P:55-57, exactly as printed (reading Q8); flag p > 0.95 <=> m > 21 f + 18 (Q9)
            prob = __dsub_rn(1.0, __ddiv_rn((double)(f + 1), (double)(m - f + 2)));
            over = (unsigned __int128)m > (unsigned __int128)21 * f + 18;
        }
        const double rate = __ddiv_rn(__ddiv_rn((double)row[SCL_COL_MALLOC_BYTES], 1048576.0),
                                      __ddiv_rn(p.elapsed_ns, 1e9));
        const bool fl = open && over;
        p.prob[sidx] = prob; p.rate[sidx] = rate; p.flag[sidx] = fl ? 1 : 0;
        // report order key: flagged by rate desc (rate >= 0, so ~bits is descending), others last;
        // a stable radix sort over site-ordered input breaks ties by site asc.
        p.key1[sidx] = fl ? ~(unsigned long long)__double_as_longlong(rate) : ~0ull;
        p.val[sidx] = sidx;
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
                              unsigned n_sites, unsigned long long* sabs, unsigned long long* err, cudaStream_t st)
{
    if (n_traces == 0) return cudaSuccess;
    unsigned grid = n_traces < 4096 ? n_traces : 4096;
    load_stats_kernel<<<grid, 256, 0, st>>>(ev, off, n_traces, n_sites, sabs, err);
    return cudaGetLastError();
}

cudaError_t launch_samples(const ReplayParams& p, cudaStream_t st)
{
    if (p.n_traces == 0) return cudaSuccess;
    unsigned warps = p.n_traces, blocks = (warps + 7) / 8;
    if (blocks > 2048) blocks = 2048;
    samples_kernel<<<blocks, 256, 0, st>>>(p);
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
