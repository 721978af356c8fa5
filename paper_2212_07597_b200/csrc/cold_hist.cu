// cold_hist.cu -- Tier E (a5: per-site malloc / free counts and bytes) of the sites that
// do not fit the replay kernel's shared-memory table (site >= kWarm when n_sites > kHot).
//
// The stream pass writes the meta word of every such alloc / free to the cold-record stream
// (chunks of kRecChunk records, one compute warp's at a time); this kernel reduces the stream per
// (site, kind) in shared memory and adds the sums to the site table.  The cold sites are split into
// ranges of kColdSites sites (2 kinds x 4 B packed count:8 | bytes:24 per site = 224 KiB); CTA b
// takes range b % R of the chunks of group b / R, so the R CTAs that read the same chunks are
// adjacent and run together (the second read of a chunk hits L2).  Carries out of a packed field
// are corrected exactly in the L2 table (as in replay_kernel); a size >= 2^24 goes to L2 directly.
// Each pass issues the next pass's loads before reducing its own records.
#include "scl_internal.cuh"
#include "ptx.cuh"
#include <algorithm>

namespace scl {

__global__ void __launch_bounds__(1024, 1) cold_hist_kernel(const __grid_constant__ ReplayParams p, unsigned R)
{
    extern __shared__ __align__(16) unsigned ctab[];          // [2][kColdSites]
    const unsigned r = blockIdx.x % R, G = gridDim.x / R, g = blockIdx.x / R;
    if (g >= G) return;
    const unsigned lo = (unsigned)kWarm + r * (unsigned)kColdSites;
    const unsigned ns = min((unsigned)kColdSites, p.n_sites - lo);   // sites of this range
    for (unsigned i = threadIdx.x; i < 2 * (unsigned)kColdSites; i += blockDim.x) ctab[i] = 0;
    __syncthreads();
    const unsigned long long used = min(ld_relaxed_u64(p.cctr), p.crec_cap);
    const unsigned long long nchunks = used / kRecChunk;
    auto one = [&](unsigned long long m) {                       // one record (an alloc or a free)
        const unsigned hi = (unsigned)(m >> 32), lo32 = (unsigned)m;
        const unsigned site = (hi >> 11) - lo;
        if (site >= ns) return;                                   // another range (or an invalid id)
        const unsigned kind = (hi >> 8) & 1u;
        if ((hi & 0xFFu) == 0 && lo32 < (1u << 24)) {             // size < 2^24: the packed word
            const unsigned ad = (1u << 24) + lo32;
            const unsigned o = atomicAdd(&ctab[kind * kColdSites + site], ad);
            if ((o & 0xFFFFFFu) + lo32 > 0xFFFFFFu || o > ~ad) {  // rare: a field carried -- exact fix in L2
                const unsigned c1 = ((o & 0xFFFFFFu) + lo32) >> 24;
                const unsigned w = (unsigned)(((unsigned long long)o + ad) >> 32);
                unsigned long long* row = p.table + (size_t)(site + lo) * SCL_NCOL;
                atomicAdd(&row[SCL_COL_N_MALLOC + kind], ((unsigned long long)w << 8) - c1);
                if (c1) atomicAdd(&row[SCL_COL_MALLOC_BYTES + kind], 1ull << 24);
            }
        } else {
            unsigned long long* row = p.table + (size_t)(site + lo) * SCL_NCOL;
            atomicAdd(&row[SCL_COL_N_MALLOC + kind], 1ull);
            atomicAdd(&row[SCL_COL_MALLOC_BYTES + kind], ev_size(m));
        }
    };
    // two chunks per pass, each thread 2 x 16 B of each; the next pass's loads are issued before this
    // pass's records are reduced (the records past a chunk's fill are read and ignored: the loads do
    // not wait for the fill word)
    constexpr unsigned kPer = kRecChunk / 2 / 1024;              // 16-B loads per thread per chunk (2)
    auto load = [&](unsigned long long c0, ulonglong2* v, unsigned* fill) {
        #pragma unroll
        for (int q = 0; q < 2; ++q) {
            const unsigned long long c = c0 + (unsigned long long)q * G;
            const bool ok = c < nchunks;
            fill[q] = ok ? min(__ldcg(p.crec_fill + c), (unsigned)kRecChunk) : 0u;
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(p.crec + (ok ? c : 0) * kRecChunk);
            #pragma unroll
            for (unsigned k = 0; k < kPer; ++k)
                v[q * kPer + k] = ok ? __ldcg(src + threadIdx.x + k * 1024u) : make_ulonglong2(0, 0);
        }
    };
    ulonglong2 v[2 * kPer], w[2 * kPer];
    unsigned fv[2], fw[2];
    load(g, v, fv);
    for (unsigned long long c0 = g; c0 < nchunks; c0 += 2ull * G) {
        load(c0 + 2ull * G, w, fw);                              // in flight while v is reduced
        #pragma unroll
        for (int q = 0; q < 2; ++q) {
            #pragma unroll
            for (unsigned k = 0; k < kPer; ++k) {
                const unsigned i = (threadIdx.x + k * 1024u) * 2u;
                if (i < fv[q]) one(v[q * kPer + k].x);
                if (i + 1 < fv[q]) one(v[q * kPer + k].y);
            }
        }
        #pragma unroll
        for (int q = 0; q < 2 * (int)kPer; ++q) v[q] = w[q];
        fv[0] = fw[0]; fv[1] = fw[1];
    }
    __syncthreads();
    // the CTA's partial table goes out with plain coalesced stores; cold_sum_kernel adds the G partials
    // of each range (one L2 atomic pair per word of every CTA cost ~70 us on config 3: 13.6 M reductions)
    if (p.cpart) {
        uint4* dst = reinterpret_cast<uint4*>(p.cpart + (size_t)blockIdx.x * 2 * kColdSites);
        const uint4* srcw = reinterpret_cast<const uint4*>(ctab);
        for (unsigned i = threadIdx.x; i < 2 * (unsigned)kColdSites / 4; i += blockDim.x) dst[i] = srcw[i];
        return;
    }
    for (unsigned i = threadIdx.x; i < 2 * ns; i += blockDim.x) {     // (no partial-table buffer: L2 atomics)
        const unsigned kind = i / ns, site = i % ns;
        const unsigned cw = ctab[kind * kColdSites + site];
        if (cw) {
            unsigned long long* row = p.table + (size_t)(site + lo) * SCL_NCOL;
            atomicAdd(&row[SCL_COL_N_MALLOC + kind], (unsigned long long)(cw >> 24));
            atomicAdd(&row[SCL_COL_MALLOC_BYTES + kind], (unsigned long long)(cw & 0xFFFFFFu));
        }
    }
}

// Sum of the G partial tables of every range -> the site table (thread per (range, kind, site); the
// partials of one word are G apart).  No other kernel writes Tier E of the cold sites at this point,
// so the add needs no atomic.
__global__ void __launch_bounds__(256) cold_sum_kernel(const __grid_constant__ ReplayParams p, unsigned R, unsigned G)
{
    const size_t n = (size_t)R * 2 * kColdSites;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
        const unsigned r = (unsigned)(idx / (2 * kColdSites)), k = (unsigned)(idx % (2 * kColdSites));
        const unsigned kind = k / kColdSites, site = k % kColdSites;
        const unsigned lo = (unsigned)kWarm + r * (unsigned)kColdSites;
        if (lo + site >= p.n_sites) continue;
        unsigned long long cnt = 0, bytes = 0;
        for (unsigned g = 0; g < G; ++g) {
            const unsigned w = __ldcg(p.cpart + ((size_t)g * R + r) * 2 * kColdSites + k);
            cnt += w >> 24; bytes += w & 0xFFFFFFu;
        }
        if (cnt | bytes) {
            unsigned long long* row = p.table + (size_t)(lo + site) * SCL_NCOL;
            row[SCL_COL_N_MALLOC + kind] += cnt;
            row[SCL_COL_MALLOC_BYTES + kind] += bytes;
        }
    }
}

bool cold_hist_launched(const ReplayParams& p) { return p.n_sites > (unsigned)kWarm && p.n_segs > 0; }
unsigned cold_hist_launches(const ReplayParams& p) { return cold_hist_launched(p) ? (p.cpart ? 2u : 1u) : 0u; }
unsigned cold_ranges(unsigned n_sites) { return n_sites > (unsigned)kWarm ? (n_sites - kWarm + kColdSites - 1) / kColdSites : 0; }

cudaError_t launch_cold_hist(const ReplayParams& p, cudaStream_t st)
{
    if (!cold_hist_launched(p)) return cudaSuccess;
    static int nsm = 0;
    constexpr size_t smem = 2 * (size_t)kColdSites * 4;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaFuncSetAttribute(cold_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) { nsm = 0; return e; }
    }
    const unsigned R = cold_ranges(p.n_sites);
    const unsigned G = std::max(1u, (unsigned)nsm / R);
    cold_hist_kernel<<<R * G, 1024, smem, st>>>(p, R);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !p.cpart) return e;
    const size_t n = (size_t)R * 2 * kColdSites;
    cold_sum_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(p, R, G);
    return cudaGetLastError();
}

}  // namespace scl
