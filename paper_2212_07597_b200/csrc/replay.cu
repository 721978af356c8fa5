// replay.cu -- sm_100a kernels of the Scalene trace-replay hot path.
//
//   replay_kernel   a1..a5 in ONE streaming pass over the events:
//                   footprint prefix sum, high-water-mark prefix max, threshold
//                   sampler, leak tracker with free-pointer match, Tier-E site
//                   reduce.  Persistent CTAs take 2048-event segments from a
//                   global ticket counter; each segment is staged in shared
//                   memory by a 2-D TMA load (128-B swizzle) into a 2-deep ring;
//                   segments of one trace are chained with a decoupled look-back
//                   whose aggregates (sum, max/min prefix) let a segment skip
//                   waiting whenever the sampler band provably stays closed.
//   samples_kernel  Tier-S, leak (mallocs, frees) and gate sums from the sample lists.
//   finalize_kernel a6: probability, rate, flag, sort key.
//   rows_kernel     report rows in report order.
//
// Paper (PAPER.md lines): sampler P:429-438, footprint P:430-431 / P:490-494,
// HWM P:24-25, leak tracker P:20-39, per-line stats P:488-494, leak score and
// probability P:31-57, filter and rate P:59-71.
#include "scl_internal.cuh"
#include <cub/device/device_radix_sort.cuh>

namespace scl {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "SCL_WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra SCL_WAIT_%=;\n}" :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_rows(void* dst, const CUtensorMap* map, int row, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(dst)), "l"((uint64_t)map), "r"(0), "r"(row), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ long long ldcg_ll(const long long* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ldcg_ull(const unsigned long long* p) { return __ldcg(p); }

__device__ __forceinline__ long long shfl_ll(long long v, int src) { return __shfl_sync(kFull, v, src); }
__device__ __forceinline__ long long shfl_up_ll(long long v, int d) { return __shfl_up_sync(kFull, v, d); }
__device__ __forceinline__ long long shfl_down_ll(long long v, int d) { return __shfl_down_sync(kFull, v, d); }
__device__ __forceinline__ long long llmax(long long a, long long b) { return a > b ? a : b; }
__device__ __forceinline__ long long llmin(long long a, long long b) { return a < b ? a : b; }

// ---------------------------------------------------------------- shared memory
struct __align__(16) ReplaySmem {
    unsigned int cnt[2 * kHot];          // Tier-E per (kind, hot site): event count
    unsigned int blo[2 * kHot];          //   bytes, low 32 bits
    unsigned int bhi[2 * kHot];          //   carries out of blo
    long long P[kThreads];               // thread exclusive prefix of d (relative to segment start)
    long long tmx[kThreads];             // thread max / min of its own running sum
    long long tmn[kThreads];
    long long PM[kThreads];              // max over earlier threads of (P + tmx)
    long long wsum[8], wmx[8], wmn[8], wpm[8];
    SegState in;                         // state before the current segment
    uint64_t bar[kStages];
    unsigned int tk[kStages];            // ticket held by each stage
    unsigned int n_list;                 // episodes started inside the current segment
    unsigned int pad;
};

size_t replay_smem_bytes() { return 1024 /*align slack*/ + (size_t)kStages * kSegBytes + sizeof(ReplaySmem); }

__device__ void flush_tier_e(ReplaySmem& s, const ReplayParams& p) {
    for (int x = threadIdx.x; x < 2 * kHot; x += kThreads) {
        unsigned c = s.cnt[x];
        int kind = x / kHot, site = x % kHot;
        if (c) {
            unsigned long long* row = p.table + (size_t)site * SCL_NCOL;
            atomicAdd(&row[SCL_COL_N_MALLOC + kind], (unsigned long long)c);
            atomicAdd(&row[SCL_COL_MALLOC_BYTES + kind],
                      ((unsigned long long)s.bhi[x] << 32) | (unsigned long long)s.blo[x]);
        }
        s.cnt[x] = 0; s.blo[x] = 0; s.bhi[x] = 0;
    }
}

// ============================================================================ replay kernel
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
replay_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ ReplayParams p)
{
    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* stage = base;                                          // kStages x 32 KiB, 1024-aligned
    ReplaySmem& s = *reinterpret_cast<ReplaySmem*>(base + (size_t)kStages * kSegBytes);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned want = p.epoch * 4u;
    EpStart* scratch = p.ep_scratch + (size_t)blockIdx.x * kSeg;

    for (int x = tid; x < 2 * kHot; x += kThreads) { s.cnt[x] = 0; s.blo[x] = 0; s.bhi[x] = 0; }
    if (tid == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(&s.bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"((uint64_t)&tmap) : "memory");
        for (int st = 0; st < kStages; ++st) {
            unsigned u = atomicAdd(p.ticket, 1u);
            s.tk[st] = u;
            if (u < p.n_segs) {
                unsigned t = p.tk_trace[u], k = p.tk_k[u] & 0x7fffffffu;
                int row = (int)(p.off[t] >> 3) + (int)k * kThreads;
                mbar_expect_tx(&s.bar[st], kSegBytes);
                tma_load_rows(stage + (size_t)st * kSegBytes, &tmap, row, &s.bar[st]);
            }
        }
    }
    __syncthreads();

    unsigned long long since_flush = 0;
    for (unsigned it = 0;; ++it) {
        const int st = it % kStages;
        const unsigned u = s.tk[st];
        if (u >= p.n_segs) break;
        const unsigned t = p.tk_trace[u];
        const unsigned kraw = p.tk_k[u];
        const unsigned k = kraw & 0x7fffffffu;
        const bool last_seg = (kraw >> 31) != 0;
        const unsigned slot = p.seg_base[t] + k;
        const long long off_t = (long long)p.off[t];
        const long long n_t = (long long)p.off[t + 1] - off_t;
        const long long row_base = (off_t >> 3) + (long long)k * kThreads;
        const long long e0_trace = (row_base + tid) * kEpt - off_t;       // trace index of this thread's event 0

        mbar_wait(&s.bar[st], (it / kStages) & 1u);

        // ---------------- phase 1: load 8 events, local scan, Tier-E (carry independent)
        const unsigned char* rowp = stage + (size_t)st * kSegBytes + (size_t)tid * 128;
        unsigned long long ptr[kEpt], meta[kEpt];
        #pragma unroll
        for (int j = 0; j < kEpt; ++j) {
            ulonglong2 v = *reinterpret_cast<const ulonglong2*>(rowp + ((j ^ (tid & 7)) << 4));
            ptr[j] = v.x; meta[j] = v.y;
        }
        unsigned vmask = 0;                 // bit j: event j is an alloc/free of this trace
        long long run = 0, tmx = kNeg, tmn = kPos;
        #pragma unroll
        for (int j = 0; j < kEpt; ++j) {
            const long long ie = e0_trace + j;
            const unsigned kind = ev_kind(meta[j]);
            const bool af = ie >= 0 && ie < n_t && kind < 2;
            const unsigned long long size = ev_size(meta[j]);
            const long long d = af ? (kind == 0 ? (long long)size : -(long long)size) : 0;
            run += d;
            if (af) {
                vmask |= 1u << j;
                tmx = llmax(tmx, run); tmn = llmin(tmn, run);
                const unsigned site = ev_site(meta[j]);
                if (site < (unsigned)kHot && size < (1ull << 32)) {       // a5 Tier E, shared-memory counters
                    const int x = kind * kHot + site;
                    atomicAdd(&s.cnt[x], 1u);
                    const unsigned sz = (unsigned)size;
                    const unsigned old = atomicAdd(&s.blo[x], sz);
                    if (old + sz < old) atomicAdd(&s.bhi[x], 1u);
                } else {                                                  // cold site / huge size: L2 reductions
                    unsigned long long* row = p.table + (size_t)site * SCL_NCOL;
                    atomicAdd(&row[SCL_COL_N_MALLOC + kind], 1ull);
                    atomicAdd(&row[SCL_COL_MALLOC_BYTES + kind], size);
                }
            }
        }
        // warp level: exclusive prefix, relative max / min, exclusive prefix max
        long long incl = run;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) { long long o = shfl_up_ll(incl, d); if (lane >= d) incl += o; }
        const long long Pw = incl - run;
        const long long hw = Pw + tmx, lw = Pw + tmn;
        long long hmx = hw, lmn = lw;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            long long o = shfl_up_ll(hmx, d); if (lane >= d) hmx = llmax(hmx, o);
            long long q = shfl_up_ll(lmn, d); if (lane >= d) lmn = llmin(lmn, q);
        }
        long long pmw = shfl_up_ll(hmx, 1);
        if (lane == 0) pmw = kNeg;
        if (lane == 31) { s.wsum[warp] = incl; s.wmx[warp] = hmx; s.wmn[warp] = lmn; }
        __syncthreads();                                                  // stage st fully consumed

        if (tid == 0) {                                                   // refill stage st (ring)
            unsigned un = atomicAdd(p.ticket, 1u);
            s.tk[st] = un;
            if (un < p.n_segs) {
                unsigned tn = p.tk_trace[un], kn = p.tk_k[un] & 0x7fffffffu;
                int row = (int)(p.off[tn] >> 3) + (int)kn * kThreads;
                mbar_expect_tx(&s.bar[st], kSegBytes);
                tma_load_rows(stage + (size_t)st * kSegBytes, &tmap, row, &s.bar[st]);
            }
        }
        // CTA level (every thread scans the 8 warp partials)
        long long Pwarp = 0, segsum = 0, segmx = kNeg, segmn = kPos, pm_prev = kNeg;
        #pragma unroll
        for (int w = 0; w < 8; ++w) {
            const long long ws = s.wsum[w], wx = s.wmx[w], wn = s.wmn[w];
            if (w < warp) { pm_prev = llmax(pm_prev, segsum + wx); Pwarp += ws; }
            segmx = llmax(segmx, segsum + wx);
            segmn = llmin(segmn, segsum + wn);
            segsum += ws;
        }
        s.P[tid] = Pwarp + Pw;
        s.tmx[tid] = tmx;
        s.tmn[tid] = tmn;
        s.PM[tid] = llmax(pm_prev, Pwarp + pmw);

        // ---------------- phase 2 (warp 0): publish aggregate, look back, resolve, publish inclusive
        if (warp == 0) {
            SegState* my = &p.state[slot];
            if (lane == 0) {
                my->sum = segsum; my->mx = segmx; my->mn = segmn;
                st_release(&my->flag, want + 1);
            }
            // --- state before this segment (a1, a2, a3, a4 carries)
            long long F0 = 0, M0 = 0, B0 = 0;
            unsigned long long n0 = 0, nep0 = 0, ep0 = kNoEp, eptr0 = 0;
            if (k > 0) {
                long long Rs = 0, Rmx = kNeg, Rmn = kPos;     // composition base+1 .. k-1
                int j = (int)k - 1;
                bool found_incl = false; int incl_idx = -1;
                for (;;) {
                    const int idx = j - lane;
                    unsigned fl = 0;
                    if (idx >= 0) {
                        const unsigned* fp = &p.state[slot - k + (unsigned)idx].flag;
                        do { fl = ld_acquire(fp); } while (fl < want + 1);
                    }
                    const bool inc = idx >= 0 && fl >= want + 2;
                    const unsigned im = __ballot_sync(kFull, inc);
                    const int stop = im ? __ffs(im) - 1 : 32;
                    long long a_s = 0, a_mx = kNeg, a_mn = kPos;
                    if (lane < stop && idx >= 0) {
                        const SegState* q = &p.state[slot - k + (unsigned)idx];
                        a_s = ldcg_ll(&q->sum); a_mx = ldcg_ll(&q->mx); a_mn = ldcg_ll(&q->mn);
                    }
                    #pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {            // ordered tree: higher lane = earlier
                        long long s2 = shfl_down_ll(a_s, d), x2 = shfl_down_ll(a_mx, d), n2 = shfl_down_ll(a_mn, d);
                        if ((lane & (2 * d - 1)) == 0 && lane + d < 32) {
                            a_mx = llmax(x2, s2 + a_mx); a_mn = llmin(n2, s2 + a_mn); a_s = s2 + a_s;
                        }
                    }
                    a_s = shfl_ll(a_s, 0); a_mx = shfl_ll(a_mx, 0); a_mn = shfl_ll(a_mn, 0);
                    Rmx = llmax(a_mx, a_s + Rmx); Rmn = llmin(a_mn, a_s + Rmn); Rs = a_s + Rs;
                    if (im) { found_incl = true; incl_idx = j - stop; break; }
                    if (j - 31 <= 0) break;                       // reached segment 0: base = trace start
                    j -= 32;
                }
                if (found_incl) {
                    const SegState* q = &p.state[slot - k + (unsigned)incl_idx];
                    F0 = ldcg_ll(&q->F); M0 = ldcg_ll(&q->M); B0 = ldcg_ll(&q->B);
                    n0 = ldcg_ull(&q->n); nep0 = ldcg_ull(&q->nep); ep0 = ldcg_ull(&q->ep); eptr0 = ldcg_ull(&q->ep_ptr);
                }
                const long long c = F0 - B0;
                if (c + Rmx < p.T && c + Rmn > -p.T) {            // no sample can fire in between
                    M0 = llmax(M0, F0 + Rmx); F0 = F0 + Rs;
                } else {                                          // wait for the predecessor's inclusive state
                    const SegState* q = &p.state[slot - 1];
                    unsigned fl;
                    do { fl = ld_acquire(&q->flag); } while (fl < want + 2);
                    F0 = ldcg_ll(&q->F); M0 = ldcg_ll(&q->M); B0 = ldcg_ll(&q->B);
                    n0 = ldcg_ull(&q->n); nep0 = ldcg_ull(&q->nep); ep0 = ldcg_ull(&q->ep); eptr0 = ldcg_ull(&q->ep_ptr);
                }
            }
            if (lane == 0) { s.in.F = F0; s.in.M = M0; s.in.B = B0; s.in.n = n0; s.in.nep = nep0; s.in.ep = ep0; s.in.ep_ptr = eptr0; }

            // --- a3 / a4: resolve the samples of this segment (rare: band-skip otherwise)
            long long B = B0;
            unsigned long long n = n0, nep = nep0, ep = ep0, eptr = eptr0;
            unsigned n_list = 0;
            const long long c0 = F0 - B0;
            __syncwarp();
            if (c0 + segmx >= p.T || c0 + segmn <= -p.T) {
                const unsigned long long sb = p.sbase[t];
                // cursor: threads < cur_t are resolved for the current base B
                int cur_t = 0;
                while (cur_t < kThreads) {
                    int found = -1;
                    for (int g = cur_t >> 5; g < 8; ++g) {
                        const int i = g * 32 + lane;
                        const long long Pi = s.P[i];
                        const bool cand = i >= cur_t &&
                            (F0 + Pi + s.tmx[i] >= B + p.T || F0 + Pi + s.tmn[i] <= B - p.T);
                        const unsigned msk = __ballot_sync(kFull, cand);
                        if (msk) { found = g * 32 + __ffs(msk) - 1; break; }
                    }
                    if (found < 0) break;
                    // detailed scan of thread `found`: lanes 0..7 take its events (re-read through L2)
                    const long long rowg = row_base + found;
                    const long long ie = rowg * kEpt + lane - off_t;
                    const bool inr = lane < kEpt && ie >= 0 && ie < n_t;
                    unsigned long long eptr_l = 0, emeta = 3ull << 40;
                    if (inr) {
                        const unsigned long long* q = reinterpret_cast<const unsigned long long*>(p.ev + rowg * kEpt + lane);
                        eptr_l = __ldcg(q); emeta = __ldcg(q + 1);
                    }
                    const unsigned ek = ev_kind(emeta);
                    const bool af = inr && ek < 2;
                    const long long esz = (long long)ev_size(emeta);
                    long long L = af ? (ek == 0 ? esz : -esz) : 0;
                    #pragma unroll
                    for (int d = 1; d < kEpt; d <<= 1) { long long o = shfl_up_ll(L, d); if (lane >= d) L += o; }
                    const long long Fe = F0 + s.P[found] + L;
                    const long long Mbase = llmax(M0, F0 + s.PM[found]);
                    int e0 = 0;
                    for (;;) {                                            // first exit of (B-T, B+T), repeatedly
                        const bool ex = af && lane >= e0 && (Fe >= B + p.T || Fe <= B - p.T);
                        const unsigned em = __ballot_sync(kFull, ex);
                        if (!em) break;
                        const int e = __ffs(em) - 1;
                        const long long Fs = shfl_ll(Fe, e);
                        long long mv = (af && lane < e) ? Fe : kNeg;
                        #pragma unroll
                        for (int d = 16; d > 0; d >>= 1) mv = llmax(mv, __shfl_xor_sync(kFull, mv, d));
                        const long long Mprev = llmax(Mbase, mv);         // M_{i-1}
                        const long long net = Fs - B;                     // counter value |A - F|
                        const bool growth = net > 0;
                        const bool nm = growth && Fs > Mprev;             // new high-water mark (Q3, Q4)
                        const unsigned long long slot_s = sb + n;
                        if (lane == e) {
                            scl_sample smp;
                            smp.idx = (unsigned long long)ie; smp.net = net; smp.footprint = Fs;
                            smp.site = ev_site(emeta); smp.kind = growth ? 0 : 1; smp.new_max = nm ? 1 : 0; smp.pad = 0;
                            p.samples[slot_s] = smp;
                            if (nm) {
                                p.ep_flag[slot_s] = 0u;
                                EpStart es; es.ep = slot_s; es.ptr = eptr_l; es.pos = (unsigned)(found * kEpt + e); es.pad = 0;
                                scratch[n_list] = es;
                            }
                        }
                        if (nm) { ep = slot_s; eptr = __shfl_sync(kFull, eptr_l, e); ++nep; ++n_list; }
                        ++n; B = Fs; e0 = e + 1;                          // "resets the counters"
                    }
                    cur_t = found + 1;
                }
            }
            if (lane == 0) {
                s.n_list = n_list;
                my->F = F0 + segsum; my->M = llmax(M0, F0 + segmx); my->B = B;
                my->n = n; my->nep = nep; my->ep = ep; my->ep_ptr = eptr;
                st_release(&my->flag, want + 2);
                if (last_seg) {
                    scl_trace_summary* sm = &p.summ[t];
                    sm->f_final = F0 + segsum; sm->hwm = llmax(M0, F0 + segmx);
                    sm->n_samples = n; sm->n_episodes = nep;
                }
            }
        }
        __syncthreads();

        // ---------------- phase 4: free-pointer match against the tracked object
        {
            unsigned long long cur_ep = s.in.ep, cur_ptr = s.in.ep_ptr;
            const unsigned nl = s.n_list;
            if (cur_ep != kNoEp || nl > 0) {
                unsigned li = 0;
                const unsigned first = (unsigned)tid * kEpt;
                while (li < nl && scratch[li].pos < first) { cur_ep = scratch[li].ep; cur_ptr = scratch[li].ptr; ++li; }
                #pragma unroll
                for (int j = 0; j < kEpt; ++j) {
                    while (li < nl && scratch[li].pos <= first + j) { cur_ep = scratch[li].ep; cur_ptr = scratch[li].ptr; ++li; }
                    if (((vmask >> j) & 1u) && ev_kind(meta[j]) == 1 && cur_ep != kNoEp && ptr[j] == cur_ptr)
                        atomicOr(&p.ep_flag[cur_ep], 1u);
                }
            }
        }
        since_flush += kSeg;
        if (since_flush > (1ull << 31)) {                         // keep u32 counters from wrapping
            __syncthreads();
            flush_tier_e(s, p);
            since_flush = 0;
        }
        __syncthreads();
    }
    __syncthreads();
    flush_tier_e(s, p);
}

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

int replay_occupancy(int* grid)
{
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)replay_smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, replay_kernel, kThreads, replay_smem_bytes());
    if (per < 1) per = 1;
    *grid = nsm * per;
    return per;
}

cudaError_t launch_replay(const CUtensorMap* tmap, const ReplayParams& p, int grid, cudaStream_t st)
{
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)replay_smem_bytes());
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (p.n_segs == 0) return cudaSuccess;
    replay_kernel<<<grid, kThreads, replay_smem_bytes(), st>>>(*tmap, p);
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
