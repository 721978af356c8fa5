// rate.cu -- the classical rate-based byte sampler (SURVEY §8(f) NEXT-1 baseline, NEXT-3 copy
// volume): a counter drawn from a geometric distribution with mean R, decremented by
// the bytes of every counted event, a sample each time it drops below 0, then re-drawn (the draw
// is added to the residual).  Unlike the threshold sampler there is no
// data-dependent chain: with S_k = G_1 + ... + G_k and A_j = counted bytes up to event j, sample k
// fires at the first event j with A_j > S_k -- the draws do not depend on the trace, so every
// sample is placed independently:
//   unit_sums_kernel   per unit (8192 events): alloc / free / copy byte sums   (once per handle)
//   unit_scan_kernel   per trace: their exclusive prefix over the trace's units
//   rate_count_kernel  per trace (warp): draws 32 at a time until S_k >= A_total -> sample count
//   rate_fill_kernel   per trace (warp): the draw prefix sums S_k
//   rate_place_kernel  per unit (block, lane = row of 8 events): the samples whose S_k falls in the
//                      unit, each placed in its row by the row's counted-byte prefix; per-site counts
// Draw k of trace t: splitmix64 keyed by (seed, t, k), u in (0, 1], G = 1 + floor(ln u / ln(1-1/R))
// with a fixed-order logarithm (explicit round-to-nearest operations, no FMA contraction), so the
// draws are reproducible; seed 0 = deterministic mode (G = R).
#include "scl_internal.cuh"
#include "ptx.cuh"

namespace scl {

// ln x, x > 0: x = m 2^e, m in [sqrt(1/2), sqrt(2)), ln m = 2 atanh((m-1)/(m+1)) by its series
// (terms up to f^23, Horner from the highest), every operation rounded separately.
__device__ __forceinline__ double rate_log(double x)
{
    const double c[12] = {
        0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
        0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4,
        0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5 };
    int e = 0;
    double m = frexp(x, &e);
    if (m < 0x1.6a09e667f3bcdp-1) { m = __dmul_rn(m, 2.0); e -= 1; }
    const double f = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
    const double f2 = __dmul_rn(f, f);
    double s = c[11];
    #pragma unroll
    for (int j = 10; j >= 0; --j) s = __dadd_rn(__dmul_rn(s, f2), c[j]);
    return __dadd_rn(__dmul_rn(__dmul_rn(2.0, f), s), __dmul_rn((double)e, 0x1.62e42fefa39efp-1));
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// the k-th counter reload of trace t (k >= 1); lq = ln(1 - 1/R)
__device__ __forceinline__ unsigned long long rate_draw(unsigned long long R, unsigned long long seed, unsigned t,
                                                        unsigned long long k, double lq)
{
    if (seed == 0) return R;
    if (R <= 1) return 1;
    const unsigned long long x = mix64(seed ^ mix64(((unsigned long long)t << 40) ^ k));
    const double u = __dmul_rn((double)((x >> 11) + 1), 0x1.0p-53);
    return (unsigned long long)floor(__ddiv_rn(rate_log(u), lq)) + 1;
}

__device__ __forceinline__ unsigned long long counted(unsigned long long meta, unsigned kinds) {
    const unsigned kind = ev_kind(meta);
    return ((kinds >> kind) & 1u) && kind < 3 ? ev_size(meta) : 0ull;
}

// ---------------------------------------------------------------- unit byte sums (per handle)
__global__ void __launch_bounds__(1024) unit_sums_kernel(const scl_event* ev, const TicketInfo* tk, unsigned long long* usum)
{
    const TicketInfo ti = tk[blockIdx.x];
    const long long row = (ti.off_t >> 3) + (long long)(ti.kraw & 0x7fffffffu) * kUnitRows + threadIdx.x;
    unsigned long long s[3] = {0, 0, 0};                    // alloc, free, copy (registers: no dynamic index)
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) {
        const long long g = row * kEpt + j, ie = g - ti.off_t;
        if (ie >= 0 && ie < ti.n_t) {
            const unsigned long long m = __ldcs(&ev[g].meta), z = ev_size(m);
            const unsigned kind = ev_kind(m);
            s[0] += kind == 0 ? z : 0ull; s[1] += kind == 1 ? z : 0ull; s[2] += kind == 2 ? z : 0ull;
        }
    }
    __shared__ unsigned long long red[3][32];
    #pragma unroll
    for (int q = 0; q < 3; ++q) {
        unsigned long long v = warp_sum((long long)s[q]);
        if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < 3 * 32) {
        const int q = threadIdx.x >> 5, l = threadIdx.x & 31;
        const unsigned long long v = (unsigned long long)warp_sum((long long)red[q][l]);
        if (l == 0) usum[(size_t)ti.slot * 3 + q] = v;
    }
}

// per trace (warp): exclusive prefix of the unit sums over the trace's units, and the totals
__global__ void __launch_bounds__(256) unit_scan_kernel(const unsigned long long* usum, const unsigned* tr_base,
                                                        const unsigned* tr_nseg, unsigned n_traces,
                                                        unsigned long long* ustart, unsigned long long* ttot)
{
    const int lane = threadIdx.x & 31;
    const unsigned t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t >= n_traces) return;
    const unsigned base = tr_base[t], ns = tr_nseg[t];
    unsigned long long carry[3] = {0, 0, 0};
    for (unsigned k0 = 0; k0 < ns; k0 += 32) {
        const unsigned k = k0 + lane;
        #pragma unroll
        for (int q = 0; q < 3; ++q) {
            const long long v = k < ns ? (long long)usum[(size_t)(base + k) * 3 + q] : 0;
            long long inc = v;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { const long long o = shfl_up_ll(inc, d); if (lane >= d) inc += o; }
            if (k < ns) ustart[(size_t)(base + k) * 3 + q] = carry[q] + (unsigned long long)(inc - v);
            carry[q] += (unsigned long long)shfl_ll(inc, 31);
        }
    }
    if (lane < 3) ttot[(size_t)t * 3 + lane] = lane == 0 ? carry[0] : (lane == 1 ? carry[1] : carry[2]);
}

__device__ __forceinline__ unsigned long long mask_sum(const unsigned long long* v3, unsigned kinds) {
    return ((kinds & 1u) ? v3[0] : 0ull) + ((kinds & 2u) ? v3[1] : 0ull) + ((kinds & 4u) ? v3[2] : 0ull);
}

// ---------------------------------------------------------------- draws
// One warp per trace: draws k = k0+1 .. k0+32 (lane-parallel), their prefix sums; the samples are
// the k with S_k < A_total.  fill == nullptr: count only.
__global__ void __launch_bounds__(256) rate_draws_kernel(const RateParams p, bool fill)
{
    const int lane = threadIdx.x & 31;
    const unsigned t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t >= p.n_traces) return;
    const unsigned long long A = mask_sum(p.ttot + (size_t)t * 3, p.kinds);
    const double lq = (p.seed != 0 && p.R > 1) ? rate_log(__dsub_rn(1.0, __ddiv_rn(1.0, (double)p.R))) : -1.0;
    unsigned long long S0 = 0, k0 = 0, n = 0;
    const unsigned long long cap = fill ? p.count[t] : ~0ull;
    for (;;) {
        const unsigned long long g = rate_draw(p.R, p.seed, t, k0 + lane + 1, lq);
        long long inc = (long long)g;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) { const long long o = shfl_up_ll(inc, d); if (lane >= d) inc += o; }
        const unsigned long long S = S0 + (unsigned long long)inc;           // S_{k0+lane+1}
        const bool below = S < A;
        if (fill && below && k0 + lane < cap) p.S[p.sbase[t] + k0 + lane] = S;
        n += (unsigned long long)__popc(__ballot_sync(kFull, below));
        if (!__all_sync(kFull, below)) break;                                // S is increasing
        S0 = (unsigned long long)shfl_ll((long long)S, 31);
        k0 += 32;
    }
    if (!fill && lane == 0) p.count[t] = n;
}

// ---------------------------------------------------------------- placement
// One block per unit (thread = row of 8 events): the row's counted-byte range [a, b) (absolute
// within the trace); the samples k with a <= S_k < b fire in this row, each at its first event
// whose inclusive prefix exceeds S_k.
__global__ void __launch_bounds__(1024) rate_place_kernel(const RateParams p)
{
    const TicketInfo ti = p.tk[blockIdx.x];
    const unsigned t = ti.t, lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
    const long long row = (ti.off_t >> 3) + (long long)(ti.kraw & 0x7fffffffu) * kUnitRows + threadIdx.x;
    unsigned long long sz[kEpt], meta[kEpt], rs = 0;
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) {
        const long long g = row * kEpt + j, ie = g - ti.off_t;
        meta[j] = 0; sz[j] = 0;
        if (ie >= 0 && ie < ti.n_t) { meta[j] = __ldcs(&p.ev[g].meta); sz[j] = counted(meta[j], p.kinds); }
        rs += sz[j];
    }
    // block exclusive scan of the row sums
    __shared__ unsigned long long wsum[32];
    long long inc = (long long)rs;
    #pragma unroll
    for (int d = 1; d < 32; d <<= 1) { const long long o = shfl_up_ll(inc, d); if ((int)lane >= d) inc += o; }
    if (lane == 31) wsum[wrp] = (unsigned long long)inc;
    __syncthreads();
    unsigned long long wb = 0;
    for (unsigned q = 0; q < wrp; ++q) wb += wsum[q];
    const unsigned long long a = mask_sum(p.ustart + (size_t)ti.slot * 3, p.kinds) + wb + (unsigned long long)inc - rs;
    const unsigned long long b = a + rs;
    if (rs == 0) return;
    // samples of this row: lower_bound(S, a) .. lower_bound(S, b) within the trace's samples
    const unsigned long long* S = p.S + p.sbase[t];
    const unsigned long long K = p.count[t];
    auto lower = [&](unsigned long long v) {
        unsigned long long lo = 0, hi = K;
        while (lo < hi) { const unsigned long long mid = (lo + hi) >> 1; if (__ldcg(S + mid) < v) lo = mid + 1; else hi = mid; }
        return lo;
    };
    const unsigned long long k1 = lower(b);
    unsigned long long k = lower(a);
    const long long e0 = row * kEpt - ti.off_t;
    unsigned long long A = a;                                   // counted bytes before event j
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) {
        A += sz[j];                                             // inclusive prefix at event j
        while (k < k1 && __ldcg(S + k) < A) {                   // sample k+1 (1-based) fires here
            scl_rate_sample smp;
            smp.idx = (unsigned long long)(e0 + j); smp.draw_sum = __ldcg(S + k);
            smp.site = ev_site(meta[j]); smp.kind = ev_kind(meta[j]);
            p.samples[p.sbase[t] + k] = smp;
            atomicAdd(&p.site_count[ev_site(meta[j])], 1ull);
            ++k;
        }
    }
}

cudaError_t launch_unit_sums(const scl_event* ev, const TicketInfo* tk, unsigned n_segs, unsigned long long* usum,
                             const unsigned* tr_base, const unsigned* tr_nseg, unsigned n_traces,
                             unsigned long long* ustart, unsigned long long* ttot, cudaStream_t st)
{
    if (n_segs) unit_sums_kernel<<<n_segs, 1024, 0, st>>>(ev, tk, usum);
    if (n_traces) unit_scan_kernel<<<(n_traces + 7) / 8, 256, 0, st>>>(usum, tr_base, tr_nseg, n_traces, ustart, ttot);
    return cudaGetLastError();
}

cudaError_t launch_rate(const RateParams& p, int phase, cudaStream_t st)
{
    if (phase == 0 || phase == 1) {
        if (p.n_traces) rate_draws_kernel<<<(p.n_traces + 7) / 8, 256, 0, st>>>(p, phase == 1);
    } else if (p.n_segs) {
        rate_place_kernel<<<p.n_segs, 1024, 0, st>>>(p);
    }
    return cudaGetLastError();
}

}  // namespace scl
