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
//   rate_ranges_kernel per unit (thread): the index of its first sample
//   rate_place_kernel  per unit (block, lane = row of 8 events): the samples whose S_k falls in the
//                      unit, each placed in its row by the row's counted-byte prefix; per-site counts
// Draw k of trace t: splitmix64 keyed by (seed, t, k), u in (0, 1], G = 1 + floor(ln u / ln(1-1/R))
// with a fixed-order logarithm (explicit round-to-nearest operations, no FMA contraction), so the
// draws are reproducible; seed 0 = deterministic mode (G = R).
#include "scl_internal.cuh"
#include "ptx.cuh"

namespace scl {

// A unit's meta words in row order, loaded coalesced: warp w of the (1024-thread) block reads its 32
// rows (256 events) event-major (each load instruction covers 512 contiguous bytes), stages them in
// shared memory with an XOR swizzle (conflict-free 8-B stores and 16-B loads) and each lane takes
// its own row's 8 words.  Events outside the trace read as 0 (an alloc of 0 bytes).
constexpr size_t kRowStage = 32 * 256 * 8;                 // 64 KiB of dynamic shared memory per block
__device__ __forceinline__ void unit_rows_meta(const scl_event* ev, const TicketInfo& ti, unsigned long long* wsm,
                                               unsigned long long* meta)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long g0 = ((ti.off_t >> 3) + (long long)(ti.kraw & 0x7fffffffu) * kUnitRows + w * 32) * kEpt;
    unsigned long long* ws = wsm + w * 256;
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) {
        const int e = j * 32 + lane;
        const long long ie = g0 + e - ti.off_t;
        unsigned long long m = 0;
        if (ie >= 0 && ie < ti.n_t) m = __ldcs(reinterpret_cast<const unsigned long long*>(ev + g0 + e) + 1);
        const int r = e >> 3, q = (e & 7) >> 1;
        ws[(r * 4 + (q ^ ((r >> 1) & 3))) * 2 + (e & 1)] = m;
    }
    __syncwarp();
    const ulonglong2* w2 = reinterpret_cast<const ulonglong2*>(ws);
    #pragma unroll
    for (int q = 0; q < kEpt / 2; ++q) {
        const ulonglong2 v = w2[lane * 4 + (q ^ ((lane >> 1) & 3))];
        meta[2 * q] = v.x; meta[2 * q + 1] = v.y;
    }
}

// The 8 meta words of row `row` (128 B, 32-B aligned) with four 256-bit loads: a lane reading its own
// row issues 4 requests instead of 8 (measured -11 % on the rate sampler).  The caller guarantees
// the row overlaps its trace (the device copy is padded to whole rows).
__device__ __forceinline__ void row_meta(const scl_event* ev, long long row, unsigned long long* meta) {
    const unsigned long long* q = reinterpret_cast<const unsigned long long*>(ev + row * kEpt);
    #pragma unroll
    for (int i = 0; i < kEpt / 2; ++i) {
        unsigned long long m0, m1;                             // (the pointers are not needed)
        asm volatile("{\n\t.reg .b64 p0, p1;\n\tld.global.nc.v4.u64 {p0,%0,p1,%1}, [%2];\n}"
                     : "=l"(m0), "=l"(m1) : "l"(q + 4 * i));
        meta[2 * i] = m0; meta[2 * i + 1] = m1;
    }
}

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
    unsigned long long s[kUCols] = {0, 0, 0, 0};            // alloc, free, copy, managed alloc
    extern __shared__ unsigned long long rstage[];
    unsigned long long mr[kEpt];
    const long long r0 = row * kEpt - ti.off_t;
    unit_rows_meta(ev, ti, rstage, mr);
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) {
        const long long ie = r0 + j;
        if (ie >= 0 && ie < ti.n_t) {
            const unsigned long long m = mr[j], z = ev_size(m);
            const unsigned kind = ev_kind(m);
            s[0] += kind == 0 ? z : 0ull; s[1] += kind == 1 ? z : 0ull; s[2] += kind == 2 ? z : 0ull;
            s[3] += kind == 0 && ((m >> 42) & 1ull) ? z : 0ull;
        }
    }
    __shared__ unsigned long long red[kUCols][32];
    #pragma unroll
    for (int q = 0; q < kUCols; ++q) {
        unsigned long long v = warp_sum((long long)s[q]);
        if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < kUCols * 32) {
        const int q = threadIdx.x >> 5, l = threadIdx.x & 31;
        const unsigned long long v = (unsigned long long)warp_sum((long long)red[q][l]);
        if (l == 0) usum[(size_t)ti.slot * kUCols + q] = v;
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
    unsigned long long carry[kUCols] = {0, 0, 0, 0};
    for (unsigned k0 = 0; k0 < ns; k0 += 32) {
        const unsigned k = k0 + lane;
        #pragma unroll
        for (int q = 0; q < kUCols; ++q) {
            const long long v = k < ns ? (long long)usum[(size_t)(base + k) * kUCols + q] : 0;
            long long inc = v;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { const long long o = shfl_up_ll(inc, d); if (lane >= d) inc += o; }
            if (k < ns) ustart[(size_t)(base + k) * kUCols + q] = carry[q] + (unsigned long long)(inc - v);
            carry[q] += (unsigned long long)shfl_ll(inc, 31);
        }
    }
    #pragma unroll
    for (int q = 0; q < kUCols; ++q) if (lane == q) ttot[(size_t)t * kUCols + q] = carry[q];
}

__device__ __forceinline__ unsigned long long mask_sum(const unsigned long long* v3, unsigned kinds) {   // columns 0-2
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
    const unsigned long long A = mask_sum(p.ttot + (size_t)t * kUCols, p.kinds);
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
    // the unit's samples [kfirst[u], kfirst[u+1]) (rate_ranges_kernel) and its counted-byte base,
    // loaded first: a unit without a sample reads no event
    const bool last = (ti.kraw >> 31) != 0;
    const unsigned long long ukr[2] = {p.kfirst[ti.slot], last ? p.count[t] : p.kfirst[ti.slot + 1]};
    const unsigned long long ubase = mask_sum(p.ustart + (size_t)ti.slot * kUCols, p.kinds);
    const unsigned long long sb = p.sbase[t];
    if (ukr[0] == ukr[1]) return;
    extern __shared__ unsigned long long rstage[];
    unsigned long long sz[kEpt], meta[kEpt], rs = 0;
    const long long r0 = row * kEpt - ti.off_t;               // trace index of the row's first event
    unit_rows_meta(p.ev, ti, rstage, meta);
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) {
        const long long ie = r0 + j;
        const bool in = ie >= 0 && ie < ti.n_t;
        if (!in) meta[j] = 0;
        sz[j] = in ? counted(meta[j], p.kinds) : 0ull;
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
    const unsigned long long a = ubase + wb + (unsigned long long)inc - rs;
    const unsigned long long b = a + rs;
    // each row within the unit's samples
    const unsigned long long* S = p.S + sb;
    if (rs == 0) return;
    auto lower = [&](unsigned long long v) {
        unsigned long long lo = ukr[0], hi = ukr[1];
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
            p.samples[sb + k] = smp;
            atomicAdd(&p.site_count[ev_site(meta[j])], 1ull);
            ++k;
        }
    }
}

// ---------------------------------------------------------------- per-sample Python / native split (NEXT-2)
// Allocated and managed-domain allocated bytes since the previous sample: inclusive
// prefixes of both at every sample event (block per unit: its samples found by binary search in
// the trace's sorted sample list, the unit's row sums scanned), then differences per trace.
__global__ void __launch_bounds__(1024) domain_prefix_kernel(const DomainParams p)
{
    const TicketInfo ti = p.tk[blockIdx.x];
    const unsigned t = ti.t;
    const long long row_base = (ti.off_t >> 3) + (long long)(ti.kraw & 0x7fffffffu) * kUnitRows;
    const long long lo = max(0ll, row_base * kEpt - ti.off_t), hi = min(ti.n_t, (row_base + kUnitRows) * kEpt - ti.off_t);
    const scl_sample* smp = p.samples + p.sbase[t];
    const unsigned long long K = p.summ[t].n_samples;
    __shared__ unsigned long long k0s, k1s;
    if (threadIdx.x < 2) {                                    // samples with lo <= idx < hi
        const long long v = threadIdx.x == 0 ? lo : hi;
        unsigned long long a = 0, b = K;
        while (a < b) { const unsigned long long mid = (a + b) >> 1; if ((long long)smp[mid].idx < v) a = mid + 1; else b = mid; }
        if (threadIdx.x == 0) k0s = a; else k1s = a;
    }
    __syncthreads();
    const unsigned long long k0 = k0s, k1 = k1s;
    if (k0 == k1) return;
    // row sums of allocated / managed allocated bytes, block exclusive scan
    const long long row = row_base + threadIdx.x;
    unsigned long long ra = 0, rm = 0, mr[kEpt];
    const long long r0 = row * kEpt - ti.off_t;
    if (r0 + kEpt > 0 && r0 < ti.n_t) row_meta(p.ev, row, mr);
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) {
        const long long ie = r0 + j;
        if (ie >= 0 && ie < ti.n_t) {
            const unsigned long long m = mr[j];
            if (ev_kind(m) == 0) { ra += ev_size(m); rm += ((m >> 42) & 1ull) ? ev_size(m) : 0ull; }
        }
    }
    __shared__ unsigned long long wa[32], wm[32], pa[1024], pm[1024];
    const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
    long long ia = (long long)ra, im = (long long)rm;
    #pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const long long oa = shfl_up_ll(ia, d), om = shfl_up_ll(im, d);
        if (lane >= d) { ia += oa; im += om; }
    }
    if (lane == 31) { wa[wrp] = (unsigned long long)ia; wm[wrp] = (unsigned long long)im; }
    __syncthreads();
    unsigned long long ba = p.ustart[(size_t)ti.slot * kUCols + 0], bm = p.ustart[(size_t)ti.slot * kUCols + 3];
    for (int q = 0; q < wrp; ++q) { ba += wa[q]; bm += wm[q]; }
    pa[threadIdx.x] = ba + (unsigned long long)ia - ra;         // before the row
    pm[threadIdx.x] = bm + (unsigned long long)im - rm;
    __syncthreads();
    for (unsigned long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const long long g = ti.off_t + (long long)smp[k].idx;      // the sample's event
        const int r = (int)((g >> 3) - row_base);
        unsigned long long A = pa[r], M = pm[r];
        for (long long x = (g >> 3) << 3; x <= g; ++x) {
            if (x - ti.off_t < 0) continue;
            const unsigned long long m = __ldcg(&p.ev[x].meta);
            if (ev_kind(m) == 0) { A += ev_size(m); M += ((m >> 42) & 1ull) ? ev_size(m) : 0ull; }
        }
        p.P[(p.sbase[t] + k) * 2 + 0] = A;
        p.P[(p.sbase[t] + k) * 2 + 1] = M;
    }
}

__global__ void __launch_bounds__(256) domain_diff_kernel(const DomainParams p)
{
    const int lane = threadIdx.x & 31;
    const unsigned t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t >= p.n_traces) return;
    const unsigned long long K = p.summ[t].n_samples, b = p.sbase[t];
    for (unsigned long long k = lane; k < K; k += 32) {
        const unsigned long long a1 = p.P[(b + k) * 2], m1 = p.P[(b + k) * 2 + 1];
        const unsigned long long a0 = k ? p.P[(b + k - 1) * 2] : 0ull, m0 = k ? p.P[(b + k - 1) * 2 + 1] : 0ull;
        p.dom[b + k].alloc_bytes = a1 - a0;
        p.dom[b + k].managed_bytes = m1 - m0;
    }
}

// ---------------------------------------------------------------- reconstruction error (NEXT-4 trend)
// The samples' footprints are the footprint trend.  Per trace: max over events of
// |F_i - footprint of the latest sample at or before i| (0 before the first sample) -- below T by
// the reset semantics.  Block per unit (thread = row): F from the unit's alloc / free
// prefix plus a block scan, the latest sample before each row by binary search.
__global__ void __launch_bounds__(1024) recon_kernel(const DomainParams p, unsigned long long* err)
{
    const TicketInfo ti = p.tk[blockIdx.x];
    const unsigned t = ti.t;
    const long long row = (ti.off_t >> 3) + (long long)(ti.kraw & 0x7fffffffu) * kUnitRows + threadIdx.x;
    long long d[kEpt], rs = 0;
    unsigned live = 0;
    unsigned long long mr[kEpt];
    const long long r0 = row * kEpt - ti.off_t;
    if (r0 + kEpt > 0 && r0 < ti.n_t) row_meta(p.ev, row, mr);
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) {
        const long long ie = r0 + j;
        d[j] = 0;
        if (ie >= 0 && ie < ti.n_t) {
            const unsigned long long m = mr[j];
            const unsigned kind = ev_kind(m);
            d[j] = kind == 0 ? (long long)ev_size(m) : (kind == 1 ? -(long long)ev_size(m) : 0);
            live |= 1u << j;
        }
        rs += d[j];
    }
    __shared__ long long ws[32];
    const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
    long long inc = rs;
    #pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) { const long long o = shfl_up_ll(inc, dd); if (lane >= dd) inc += o; }
    if (lane == 31) ws[wrp] = inc;
    __syncthreads();
    long long F = (long long)(p.ustart[(size_t)ti.slot * kUCols + 0] - p.ustart[(size_t)ti.slot * kUCols + 1]);
    for (int q = 0; q < wrp; ++q) F += ws[q];
    F += inc - rs;                                           // footprint before the row
    unsigned long long e = 0;
    if (live) {
        const scl_sample* smp = p.samples + p.sbase[t];
        const unsigned long long K = p.summ[t].n_samples;
        const long long r_lo = row * kEpt - ti.off_t;        // trace index of the row's first slot
        unsigned long long a = 0, b = K;                     // first sample with idx >= r_lo
        while (a < b) { const unsigned long long mid = (a + b) >> 1; if ((long long)smp[mid].idx < r_lo) a = mid + 1; else b = mid; }
        long long B = a ? smp[a - 1].footprint : 0;
        unsigned long long kn = a;
        #pragma unroll
        for (int j = 0; j < kEpt; ++j) {
            if (!((live >> j) & 1u)) continue;
            F += d[j];
            if (kn < K && (long long)smp[kn].idx == r_lo + j) { B = F; ++kn; }
            else { const long long x = F > B ? F - B : B - F; e = e > (unsigned long long)x ? e : (unsigned long long)x; }
        }
    }
    #pragma unroll
    for (int dd = 16; dd > 0; dd >>= 1) { const unsigned long long o = __shfl_xor_sync(kFull, e, dd); e = e > o ? e : o; }
    if (lane == 0 && e) atomicMax(&err[t], e);
}

cudaError_t launch_recon(const DomainParams& p, unsigned long long* err, cudaStream_t st)
{
    if (p.n_segs) recon_kernel<<<p.n_segs, 1024, 0, st>>>(p, err);
    return cudaGetLastError();
}

cudaError_t launch_domains(const DomainParams& p, cudaStream_t st)
{
    if (p.n_segs) domain_prefix_kernel<<<p.n_segs, 1024, 0, st>>>(p);
    if (p.n_traces) domain_diff_kernel<<<(p.n_traces + 7) / 8, 256, 0, st>>>(p);
    return cudaGetLastError();
}

// Per unit: the index of its first sample, lower_bound(S_t, counted bytes before the unit)
// (thread per unit; the placement blocks read their unit's range with one load).
__global__ void __launch_bounds__(256) rate_ranges_kernel(const RateParams p)
{
    const unsigned q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= p.n_segs) return;
    const TicketInfo ti = p.tk[q];
    const unsigned long long v = mask_sum(p.ustart + (size_t)ti.slot * kUCols, p.kinds);
    const unsigned long long* S = p.S + p.sbase[ti.t];
    unsigned long long lo = 0, hi = p.count[ti.t];
    while (lo < hi) { const unsigned long long mid = (lo + hi) >> 1; if (__ldcg(S + mid) < v) lo = mid + 1; else hi = mid; }
    p.kfirst[ti.slot] = lo;
}

cudaError_t launch_unit_sums(const scl_event* ev, const TicketInfo* tk, unsigned n_segs, unsigned long long* usum,
                             const unsigned* tr_base, const unsigned* tr_nseg, unsigned n_traces,
                             unsigned long long* ustart, unsigned long long* ttot, cudaStream_t st)
{
    static const bool attr = cudaFuncSetAttribute(unit_sums_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)kRowStage) == cudaSuccess;
    if (!attr) return cudaErrorInvalidValue;
    if (n_segs) unit_sums_kernel<<<n_segs, 1024, kRowStage, st>>>(ev, tk, usum);
    if (n_traces) unit_scan_kernel<<<(n_traces + 7) / 8, 256, 0, st>>>(usum, tr_base, tr_nseg, n_traces, ustart, ttot);
    return cudaGetLastError();
}

cudaError_t launch_rate(const RateParams& p, int phase, cudaStream_t st)
{
    if (phase == 0 || phase == 1) {
        if (p.n_traces) rate_draws_kernel<<<(p.n_traces + 7) / 8, 256, 0, st>>>(p, phase == 1);
    } else if (p.n_segs) {
        rate_ranges_kernel<<<(p.n_segs + 255) / 256, 256, 0, st>>>(p);
        static const bool attr = cudaFuncSetAttribute(rate_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)kRowStage) == cudaSuccess;
        if (!attr) return cudaErrorInvalidValue;
        rate_place_kernel<<<p.n_segs, 1024, kRowStage, st>>>(p);
    }
    return cudaGetLastError();
}

}  // namespace scl
