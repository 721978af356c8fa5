// replay_kernel.cu -- the streaming hot path a1..a5 in one pass over the events.
//
// Paper (PAPER.md lines): threshold sampler P:429-438 ("|A - F| >= T ... resets
// the counters"), footprint P:430-431 / P:490-494, high-water mark P:24-25,
// leak tracker with the free-pointer comparison P:20-39, per-line statistics
// P:488-494.  Readings Q1-Q16: DESIGN.md §3.
//
// replay_kernel: one persistent CTA per SM, warp-specialised:
//   producer warp   CTA 0 first prepares the run (zeroes tables / states, scans the sample
//                   bases); then one ticket per 8192-event unit (tickets ordered (unit index,
//                   trace), so the units of one trace are spread over time), the unit's four
//                   2-D TMA boxes (32 KiB, 128-B swizzle, L2 evict_first) into a 4-stage ring;
//   16 compute warps in two groups alternating boxes, one 256-event chunk per warp per box:
//                   signed sizes, the chunk's sum and max/min prefix, Tier-E site counters
//                   (unconditional 32-bit shared atomics), a 2048-bit Bloom filter of freed
//                   pointers; one mbarrier arrival per chunk completes the unit's slot;
//   publisher warp  per complete unit (in order): composes the 32 chunk summaries, copies the
//                   unit record to global through the TMA engine, hands the slot back, and after
//                   one fence per batch publishes the unit's tagged aggregate words;
//   2 runner warps  each trace has one runner lane that advances it strictly in order over its
//                   published units: batches of units without a sample composed from their
//                   aggregates, units where a sample fires resolved chunk by chunk (32-bit when
//                   the chunk allows), entry states recorded for the reclaim pass.
// post_kernel (cooperative): the free-pointer comparison of every episode segment (Bloom query
// per chunk, exact re-checks of positives), the per-sample reduce, and a6 when fused.
#include <climits>
#include <algorithm>
#include "scl_internal.cuh"
#include "ptx.cuh"
#include "report.cuh"

namespace scl {

constexpr int kTabSlots = 4 * kHot > 2 * kWarm ? 4 * kHot : 2 * kWarm;   // the two table layouts share storage
constexpr int kESlots = kTabSlots + kComputeWarps * 32;              // + one sink slot per compute lane

constexpr uint32_t kBloOff = kESlots * 4;   // byte distance cnt -> blo

struct __align__(16) Smem {
    unsigned cnt[kESlots];           // Tier-E per (kind, hot site): event count    (slot kind*kHot + site, or
                                     //   (kind&1)*kWarm + site for the allocs and frees of n_sites > kHot;
    unsigned blo[kESlots];           //   bytes mod 2^32 (carries: straight to L2)  slots >= 4*kHot: per-lane
                                     //   sinks of the unconditional atomics; copies counted, not reported)
    Slot slot[kSlots];
    SegInfo info[kStages];
    unsigned sub[kStages];           // box index within the unit
    uint64_t full[kStages], empty[kStages];
    uint64_t sempty[kSlots];         // slot free again (publisher -> compute)
    uint64_t sdone[kSlots];          // the slot's unit is complete: one arrival per chunk (compute -> publisher)
    unsigned n_units;                // units handed to this CTA (known at the end of the tickets)
};

static_assert(sizeof(Slot) % 16 == 0, "unit records are copied by the TMA engine in 16-B units");
size_t replay_urec_bytes() { return sizeof(Slot); }
size_t replay_smem_bytes() { return 1024 + (size_t)kStages * kSegBytes + sizeof(Smem); }

// Blocked Bloom filter of freed pointers, 64 words (2048 bits) per 256-event chunk: one
// word per pointer, two bits in it (one shared-memory OR per free; ~1.4 % false positives
// at ~128 frees per chunk).  One multiply of the pointer's low word (16-B aligned pointers:
// its low 4 bits are zero): word = bits 26..31, bits = 21..25 and 16..20.
__device__ __forceinline__ unsigned bloom_hash(unsigned long long ptr) {
    return (unsigned)ptr * 0x9E3779B1u;
}
// The filter's two halves: frees of objects under kBloomBig bytes, and the larger ones.  A leak
// episode tracks the allocation of a new-maximum growth sample -- in our workloads >= 64 KiB in
// 97-100 % of the episodes, while 91-93 % of the frees are under 4 KiB -- so the query of a large
// tracked object meets a sparse half and few false positives (the free of an object has its
// allocation's size: reading Q16).
__device__ __forceinline__ unsigned bloom_word(unsigned long long ptr, bool big) {
    return (bloom_hash(ptr) >> (33 - kBloomLog2)) | (big ? (unsigned)kBloomWords / 2 : 0u);
}
__device__ __forceinline__ unsigned bloom_mask(unsigned long long ptr) {
    const unsigned h = bloom_hash(ptr);
#ifdef SCL_BLOOM_FUNNEL
    // bits (h >> 21) & 31 and (h >> 16) & 31: a wrapping funnel shift of 1 takes its count mod 32
    return __funnelshift_l(0u, 1u, h >> 21) | __funnelshift_l(0u, 1u, h >> 16);
#else
    return (1u << ((h >> 21) & 31u)) | (1u << ((h >> 16) & 31u));
#endif
}

// Optional per-role cycle accounting (debug build with -DSCL_PROFILE only).
#ifdef SCL_PROFILE
#define PROF_DECL unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long pt = clock64();
#define PROF_MARK(i) { const long long now_ = clock64(); pacc[i] += now_ - pt; pt = now_; }
#define PROF_FLUSH(base) if (lane == 0 && p.prof) { for (int q_ = 0; q_ < 8; ++q_) atomicAdd(&p.prof[(base) + q_], pacc[q_]); }
#define RPROF_ADD(i, v) if (p.prof && lane == 0) atomicAdd(&p.prof[24 + (i)], (unsigned long long)(v));
#define PROF_TOUCH(v) asm volatile("" : "+l"(v));      /* the value must have arrived before the next clock read */
#define PROF_UNIT_T(u, which) if (p.prof) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); p.prof[48 + 4 * (size_t)(u) + (which)] = t_; }
#else
#define PROF_DECL
#define PROF_MARK(i)
#define PROF_FLUSH(base)
#define PROF_UNIT_T(u, which)
#define RPROF_ADD(i, v)
#define PROF_TOUCH(v)
#endif

// ============================================================================ per-run preparation
// Every CTA zeroes its slice of the site table, trace summaries and runner states, then arrives on
// ticket[8] (never reset between launches: the host passes the count after this launch's arrivals,
// zc_target); wait_prepared also waits for all arrivals.  (One CTA zeroing config 3's 4-MB table
// held every producer ~20 us.)
__device__ void zero_slice(const ReplayParams& rp)
{
    const PrepParams& p = rp.prep;
    const size_t tid = threadIdx.x, nth = blockDim.x, b = blockIdx.x, nb = gridDim.x;
    auto slice = [&](unsigned long long* a, size_t n) {
        for (size_t i = n * b / nb + tid, hi = n * (b + 1) / nb; i < hi; i += nth) a[i] = 0;
    };
    slice(p.table, p.table_words); slice(p.summ, p.summ_words); slice(p.run, p.run_words);
    __syncthreads();
    if (tid == 0) { __threadfence(); atomicAdd(rp.ticket + 8, 1u); }
}

__device__ void prepare_run(const ReplayParams& rp, unsigned long long* scratch)   // CTA 0
{
    const PrepParams& p = rp.prep;
    const unsigned tid = threadIdx.x, nth = blockDim.x;
    if (tid < 7) p.ticket[tid] = 0;
    if (tid < 2 && rp.cctr) rp.cctr[tid] = 0;              // cold-record pool: allocated, exhausted
    for (unsigned i = tid; i < p.n_sb; i += nth) p.rsbcnt[i] = 0;
    // exclusive scan of the per-trace sample capacities (thread j: a contiguous run of traces)
    const unsigned per = (p.n_traces + nth - 1) / nth;
    const unsigned t0 = min(p.n_traces, tid * per), t1 = min(p.n_traces, t0 + per);
    auto cap = [&](unsigned t) {
        const unsigned long long n = p.off[t + 1] - p.off[t], b = p.sabs[t] / p.T;
        return n < b ? n : b;
    };
    unsigned long long acc = 0;
    for (unsigned t = t0; t < t1; ++t) acc += cap(t);
    scratch[tid] = acc;
    __syncthreads();
    for (unsigned d = 1; d < nth; d <<= 1) {                 // Hillis-Steele inclusive scan
        const unsigned long long v = tid >= d ? scratch[tid - d] : 0;
        __syncthreads();
        scratch[tid] += v;
        __syncthreads();
    }
    unsigned long long base = scratch[tid] - acc;
    for (unsigned t = t0; t < t1; ++t) { p.sbase[t] = base; base += cap(t); }
    __syncthreads();
    if (tid == 0) { __threadfence(); st_release(&rp.ticket[7], rp.epoch); }
}

__device__ __forceinline__ void wait_prepared(const ReplayParams& p) {
    while (ld_relaxed(&p.ticket[7]) != p.epoch) __nanosleep(32);
    while ((int)(ld_relaxed(&p.ticket[8]) - p.zc_target) < 0) __nanosleep(32);
    fence_acquire();
}

// ============================================================================ compute warps
// Fast path of one row (8 events) in a lane: sizes < 2^27 (size bits 27-39 zero).  Every shared
// atomic is unconditional (no branch around it): an event that does not count goes to the lane's
// sink slot (and adds 0 bytes, so the sink never wraps).  Tier-E slot of (kind, site) = kind*kHot +
// site (kind-major: a warp's random sites spread over all 32 banks), copies included -- with every
// site hot, no event needs a select.  Two counters per slot: the event count (a u32 that cannot wrap
// within one CTA) and the bytes mod 2^32, whose rare wrap is re-examined after the row (a packed
// count | bytes word was measured slower: its carries are frequent enough that nearly every warp
// takes the correction branch).  Kinds are read as bits: bit 41 set = copy (no footprint change),
// else bit 40 = free (kind 3 is rejected by the trace validation; unvalidated, it only widens the
// Bloom filter, which is re-checked).
// kAllHot: every site is in the shared-memory table (n_sites <= kHot), no cold-site bookkeeping;
// otherwise the table holds the allocs and frees of the kWarm lowest site ids, the others are
// returned in `cold` (bit j: event j) for the cold-record stream.
template <bool kAllHot>
__device__ __forceinline__ void fast_row(const unsigned long long* ptr, const unsigned long long* meta, uint32_t cnt_s,
                                         uint32_t bl_s, uint32_t dslot, unsigned long long* table, int& r32,
                                         int& mx32, int& mn32, unsigned& cold)
{
    unsigned old[kEpt], add[kEpt];
    bool anyc = false;
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) {
        const unsigned hi = (unsigned)(meta[j] >> 32), lo = (unsigned)meta[j];
        const bool isfree = (hi & 0x100u) != 0, af = (hi & 0x200u) == 0;
        const int d = isfree ? -(int)lo : (int)lo;
        if (af) r32 += d;                                                     // a1: signed size
        mx32 = max(mx32, r32); mn32 = min(mn32, r32);
        uint32_t a;
        if (kAllHot) {                                                        // site < kHot
            const uint32_t off = ((hi >> 9) & (uint32_t)(4 * kHot - 4)) | ((hi << 4) & (uint32_t)(3 * 4 * kHot));
            a = cnt_s + off; add[j] = lo;                                     // (kind*kHot + site)*4
        } else {
            const bool h = af && (hi >> 11) < (unsigned)kWarm;
            cold |= (af && !h ? 1u : 0u) << j;
            uint32_t offw;                                                    // ((kind&1)*kWarm + site)*4
            if constexpr ((kWarm & (kWarm - 1)) == 0)                         // (site < kWarm when used)
                offw = ((hi >> 9) & (uint32_t)(4 * kWarm - 4)) | (((hi >> 8) & 1u) * (uint32_t)(4 * kWarm));
            else
                offw = ((hi >> 9) & ~3u) + ((hi >> 8) & 1u) * (uint32_t)(4 * kWarm);
            a = cnt_s + (h ? offw : dslot); add[j] = h ? lo : 0u;                // ((kind&1)*kWarm + site)*4
        }
        red_add(a, 1u);                                                       // a5 Tier E
        old[j] = atom_add(a + kBloOff, add[j]);
        red_or(isfree ? bl_s + bloom_word(ptr[j], lo >= kBloomBig) * 4u : cnt_s + dslot, bloom_mask(ptr[j]));   // freed ptr -> Bloom
    }
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) anyc |= old[j] + add[j] < old[j];
    if (anyc) {                                       // rare: a 32-bit byte counter wrapped: 2^32 to L2
        #pragma unroll
        for (int j = 0; j < kEpt; ++j) {
            const unsigned kind = ev_kind(meta[j]);
            if (old[j] + add[j] < old[j] && kind < 2)
                atomicAdd(&table[(size_t)ev_site(meta[j]) * SCL_NCOL + SCL_COL_MALLOC_BYTES + kind], 1ull << 32);
        }
    }
}

// Cold events of the row (bit j of rec: event j) -> the warp's chunk of the cold-record stream:
// one warp scan of the per-lane counts gives each lane its run of slots, the records (the events'
// meta words) are staged in the warp's own 4-KiB slice of the TMA box it just read (its rows are in
// registers now; at most 256 records) and copied out with lane-contiguous stores (whole sectors).
// A new chunk is taken from the pool when the current one cannot hold the row's records (the rest
// of it is left unused; its fill is written when the warp leaves it).  When the pool is exhausted
// the records are returned for the direct L2 path.  Sets `staged` when the slice was written (the
// async proxy's next TMA write must be ordered after it: fence.proxy.async before the box is
// released).  (Measured alternatives on config 3: lane-scattered stores from registers and a bulk
// copy of the slice, within 2 %; 4-B records (site - kWarm : 16 | kind : 1 | size : 15) halve the
// record traffic but their encoding and the L2 path of the larger sizes cost the issue-bound compute
// warps more: +6 % on the stream pass.)
struct ColdCursor { unsigned long long base; unsigned fill; };   // base ~0: no chunk (pool exhausted)

__device__ __forceinline__ unsigned cold_records(const ReplayParams& p, ColdCursor& cc, const unsigned long long* meta,
                                                 unsigned rec, uint32_t slice_s, int lane, bool& staged)
{
#ifdef SCL_COLD_L2
    return rec;                                       // (A/B: every cold event through two L2 reductions)
#endif
    const unsigned nc = __popc(rec);
    unsigned incl = nc;
    #pragma unroll
    for (int d = 1; d < 32; d <<= 1) { const unsigned o = __shfl_up_sync(kFull, incl, d); if (lane >= d) incl += o; }
    const unsigned tot = __shfl_sync(kFull, incl, 31);
    if (tot == 0) return 0u;
    if (cc.fill + tot > (unsigned)kRecChunk) {
        unsigned long long nb = 0;
        if (lane == 0) {
            if (cc.base != ~0ull) p.crec_fill[cc.base / kRecChunk] = cc.fill;
            nb = atomicAdd(p.cctr, (unsigned long long)kRecChunk);
            if (nb + kRecChunk > p.crec_cap) { nb = ~0ull; if (p.covf) *p.covf = 1ull; }   // pool exhausted
        }
        cc.base = __shfl_sync(kFull, nb, 0); cc.fill = 0;
    }
    if (cc.base == ~0ull) return rec;                 // -> direct L2 reductions
    __syncwarp();                                     // every lane's row is in registers
    uint32_t a = slice_s + 8u * (incl - nc);
    #pragma unroll
    for (int j = 0; j < kEpt; ++j)
        if ((rec >> j) & 1u) { asm volatile("st.shared.u64 [%0], %1;" :: "r"(a), "l"(meta[j]) : "memory"); a += 8u; }
    __syncwarp();
    SCL_CHECK(cc.base + cc.fill + tot <= p.crec_cap);
    unsigned long long* dst = p.crec + cc.base + cc.fill;
    for (unsigned k = (unsigned)lane; k < tot; k += 32) {
        unsigned long long v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(slice_s + 8u * k) : "memory");
        dst[k] = v;
    }
    cc.fill += tot;
    staged = true;
    return 0u;
}

// Two groups of 8 warps alternate boxes (group 0: boxes 0 and 2 of a unit, group 1: 1 and 3);
// warp w8 of a group takes rows 32*w8 .. 32*w8+31 of its box = chunk g*8 + w8 of the unit.
__device__ void compute_role(const ReplayParams& p, Smem& s, unsigned char* stage, int grp, int w8, int lane)
{
    const uint32_t cnt_s = smem_u32(s.cnt);
    const uint32_t dslot = (uint32_t)(kTabSlots + (grp * 8 + w8) * 32 + lane) * 4u;   // this lane's sink slot
    const bool all_hot = p.n_sites <= (unsigned)kHot;       // no cold site: no record stream
    ColdCursor cc{~0ull, (unsigned)kRecChunk};              // no chunk yet (taken at the first cold record)
    // this lane's row r = 32*w8 + lane of every box: its 8 swizzled 16-B chunks (chunk j at j ^ (r & 7))
    const int r = w8 * 32 + lane;
    unsigned rofs[kEpt];
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) rofs[j] = (unsigned)r * 128u + (unsigned)((j ^ (r & 7)) << 4);
    int sl = kSlots - 1;                                    // unit slot (itu % kSlots) and its phase,
    unsigned sph = 1u, cur_itu = ~0u;                       // advanced incrementally (no division)
    PROF_DECL
    for (unsigned it = grp;; it += 2) {
        const int st = it % kStages;
        PROF_MARK(3)
        mbar_wait(&s.full[st], (it / kStages) & 1u);
        PROF_MARK(0)
        const SegInfo inf = s.info[st];
        const unsigned g = s.sub[st];
        const unsigned itu = it / kSub;                   // unit iteration of this CTA
        if (itu != cur_itu) { cur_itu = itu; if (++sl == kSlots) { sl = 0; sph ^= 1u; } }
        if (inf.u == kInvalid) {
            if (lane == 0 && cc.base != ~0ull) p.crec_fill[cc.base / kRecChunk] = cc.fill;   // the last chunk's fill
            // the publisher stops once all `itu` units of this CTA are published
            if (grp == 0 && w8 == 0 && lane == 0) atomicExch(&s.n_units, itu);
            PROF_FLUSH(0)
            return;
        }
        if (g == (unsigned)grp) mbar_wait(&s.sempty[sl], sph ^ 1u);   // group's first box of the unit
        PROF_MARK(1)
        Slot& S = s.slot[sl];
        const int c = g * 8 + w8;                         // chunk index within the unit
        #pragma unroll
        for (int q = 0; q < kBloomWords; q += 32) if (q + lane < kBloomWords) S.bloom[c][q + lane] = 0u;
        if (g == 0 && w8 == 0 && lane == 0) S.info = inf;
        __syncwarp();
        const uint32_t bl_s = smem_u32(&S.bloom[c][0]);

        long long run = 0, tmx = kNeg, tmn = kPos;
        int r32 = 0, mx32 = 0, mn32 = 0;                  // the lane's max / min include its start value
                                                          // (an earlier F: harmless for M and the band)
        bool small = true;                                // 32-bit chunk summary is exact for this lane
        bool staged = false;                              // cold records staged in this warp's slice of the box
        if (g < inf.nbox) {
            // ---- the 8 events of row r of the box
            const unsigned char* boxp = stage + (size_t)st * kSegBytes;
            unsigned long long ptr[kEpt], meta[kEpt];
            #pragma unroll
            for (int j = 0; j < kEpt; ++j) {
                ulonglong2 v = *reinterpret_cast<const ulonglong2*>(boxp + rofs[j]);
                ptr[j] = v.x; meta[j] = v.y;
            }
            const long long e0 = (inf.row_base + (long long)g * kThreads + r) * kEpt - inf.off_t;
            unsigned big = 0;                                 // any size >= 2^27 in the row?
            #pragma unroll
            for (int j = 0; j < kEpt; ++j) big |= ((unsigned)meta[j] >> 27) | ((unsigned)(meta[j] >> 32) & 0xffu);
            unsigned cold = 0, rec = 0;                       // events for the L2 path / the record stream
            if (e0 >= 0 && e0 + kEpt <= inf.n_t && big == 0) {
                // fast path: the whole row is in the trace and |partial sums| < 2^30: 32-bit running
                // sum / max / min (a copy's d = 0 repeats an F already seen: harmless)
                if (all_hot) fast_row<true>(ptr, meta, cnt_s, bl_s, dslot, p.table, r32, mx32, mn32, rec);
                else         fast_row<false>(ptr, meta, cnt_s, bl_s, dslot, p.table, r32, mx32, mn32, rec);
                run = r32;
                tmx = mx32; tmn = mn32;
                small = r32 > -(1 << 25) && r32 < (1 << 25) && mx32 < (1 << 25) && mn32 > -(1 << 25);
            } else {
                // exact 64-bit path: rows crossing a trace boundary or holding a size >= 2^27
                small = false;
                #pragma unroll
                for (int j = 0; j < kEpt; ++j) {
                    const long long ie = e0 + j;
                    const unsigned kind = ev_kind(meta[j]);
                    const bool af = ie >= 0 && ie < inf.n_t && kind < 2;
                    const unsigned long long size = ev_size(meta[j]);
                    run += af ? (kind == 0 ? (long long)size : -(long long)size) : 0;     // a1: signed size
                    if (af) {
                        tmx = llmax(tmx, run); tmn = llmin(tmn, run);
                        const unsigned site = ev_site(meta[j]);
                        if (site < (unsigned)(all_hot ? kHot : kWarm) && size < (1ull << 32)) {
                            const int x = (int)kind * (all_hot ? kHot : kWarm) + (int)site;
                            atomicAdd(&s.cnt[x], 1u);
                            const unsigned old = atomicAdd(&s.blo[x], (unsigned)size);
                            if (old + (unsigned)size < old)
                                atomicAdd(&p.table[(size_t)site * SCL_NCOL + SCL_COL_MALLOC_BYTES + kind], 1ull << 32);
                        } else {
                            cold |= 1u << j;
                        }
                        if (kind == 1) atomicOr(&S.bloom[c][bloom_word(ptr[j], size >= kBloomBig)], bloom_mask(ptr[j]));
                    }
                }
            }
            if (!all_hot)                                     // (warp-collective; fallback -> L2)
                cold |= cold_records(p, cc, meta, rec, smem_u32(boxp) + (uint32_t)w8 * 32u * 128u, lane, staged);
            if (__any_sync(kFull, cold != 0u)) {              // cold site / huge size: L2 reductions (rare)
                #pragma unroll
                for (int j = 0; j < kEpt; ++j) {
                    if ((cold >> j) & 1u) {
                        const unsigned kind = ev_kind(meta[j]);
                        SCL_CHECK(ev_site(meta[j]) < p.n_sites);
                        unsigned long long* row = p.table + (size_t)ev_site(meta[j]) * SCL_NCOL;
                        atomicAdd(&row[SCL_COL_N_MALLOC + kind], 1ull);
                        atomicAdd(&row[SCL_COL_MALLOC_BYTES + kind], ev_size(meta[j]));
                    }
                }
            }
        }
        PROF_MARK(4)
        // ---- chunk summary: sum, max / min prefix relative to the chunk start
        long long csum, cmx, cmn;
        if (__all_sync(kFull, small)) {                       // 32-bit scan + REDUX
            const int tot = __reduce_add_sync(kFull, r32);      // (off the scan's dependency chain)
            int incl = r32;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { int o = __shfl_up_sync(kFull, incl, d); if (lane >= d) incl += o; }
            const int am = __reduce_max_sync(kFull, incl - r32 + mx32), bm = __reduce_min_sync(kFull, incl - r32 + mn32);
            csum = tot; cmx = am; cmn = bm;
        } else {
            long long incl = run;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { long long o = shfl_up_ll(incl, d); if (lane >= d) incl += o; }
            const long long Pl = incl - run;
            cmx = warp_max(Pl + tmx); cmn = warp_min(Pl + tmn);
            csum = shfl_ll(incl, 31);
        }
        if (lane == 0) { S.Pc[c] = csum; S.ax[c] = cmx; S.an[c] = cmn; }   // composed in place below
        if (staged) fence_proxy_async_shared();            // generic writes before the next TMA write of the box
        __syncwarp();
        mbar_arrive(&s.empty[st]);                        // box consumed
        PROF_MARK(2)
        if (lane == 0) mbar_arrive(&s.sdone[sl]);         // chunk summarised: the 32nd arrival completes the unit
    }
}

// ============================================================================ producer warp
__device__ void producer_role(const ReplayParams& p, const CUtensorMap* tmap, Smem& s, unsigned char* stage, int lane)
{
    if (lane != 0) return;
    // the events are streamed once: evict them first, keeping the unit records, samples and the
    // site table (which the runners and the post pass re-read) in L2
    const uint64_t pol = l2_policy_evict_first();
    wait_prepared(p);                                     // ticket counter zeroed by CTA 0
    PROF_DECL
    auto resolve = [&](unsigned u) {
        SegInfo inf; inf.u = kInvalid; inf.nbox = 0;
        if (u < p.n_segs) {
            const TicketInfo ti = p.tk[u];
            inf.u = u; inf.t = ti.t; inf.kraw = ti.kraw; inf.slot = ti.slot; inf.nbox = ti.nbox;
            inf.off_t = ti.off_t; inf.n_t = ti.n_t;
            inf.row_base = (ti.off_t >> 3) + (long long)(ti.kraw & 0x7fffffffu) * kUnitRows;
        }
        return inf;
    };
    // two tickets in flight: the atomic for unit i+2 and the record load for unit i+1
    // are issued before unit i's boxes, and consumed after them
    SegInfo cur = resolve(atomicAdd(p.ticket, 1u));
    unsigned u_next = cur.u == kInvalid ? kInvalid : atomicAdd(p.ticket, 1u);
    unsigned it = 0;
    for (;;) {
        const SegInfo nxt = resolve(u_next);
        const unsigned u_after = nxt.u == kInvalid ? kInvalid : atomicAdd(p.ticket, 1u);
        for (unsigned g = 0; g < (unsigned)kSub; ++g, ++it) {
            const int st = it % kStages;
            PROF_MARK(1)
            mbar_wait(&s.empty[st], ((it / kStages) & 1u) ^ 1u);
            PROF_MARK(0)
            s.info[st] = cur; s.sub[st] = g;
            if (cur.u == kInvalid || g >= cur.nbox) {
                mbar_arrive(&s.full[st]);                  // sentinel / box outside the trace
                if (cur.u == kInvalid && g == 0) continue; // the sentinel goes to both compute groups
            } else {
                mbar_expect_tx(&s.full[st], kSegBytes);
                tma_load_2d_hint(stage + (size_t)st * kSegBytes, tmap, 0, (int)(cur.row_base + (long long)g * kThreads),
                                 &s.full[st], pol);
            }
            if (cur.u == kInvalid) { PROF_FLUSH(8) return; }
        }
        cur = nxt;
        u_next = u_after;
    }
}

// ============================================================================ runner warps
// Each trace has one RUNNER lane (static assignment) that advances it strictly in order over
// every published unit, with the exact sequential state in registers.  Units without a sample
// are composed 32 at a time from their aggregates (sampler band test, HWM); only units in
// which a sample fires are resolved chunk by chunk.  The runner does no pointer matching: it
// records the state entering each unit (UnitEntry) and the reclaim pass settles every episode
// afterwards, all units in parallel -- the chain carries only what the sampler needs.
struct RState { long long F, M, B; unsigned long long n, nep, ep1, eptr; long long Ms; unsigned next; };

__device__ __forceinline__ RState load_rstate(const RunState* rs, int lane) {
    const unsigned long long* w = reinterpret_cast<const unsigned long long*>(rs);
    unsigned long long v = lane < 9 ? __ldcg(w + lane) : 0ull;      // F M B n nep ep1 eptr Ms {next,pad}
    RState x;
    x.F = (long long)__shfl_sync(kFull, v, 0); x.M = (long long)__shfl_sync(kFull, v, 1);
    x.B = (long long)__shfl_sync(kFull, v, 2); x.n = __shfl_sync(kFull, v, 3);
    x.nep = __shfl_sync(kFull, v, 4); x.ep1 = __shfl_sync(kFull, v, 5); x.eptr = __shfl_sync(kFull, v, 6);
    x.Ms = (long long)__shfl_sync(kFull, v, 7);
    x.next = (unsigned)__shfl_sync(kFull, v, 8);      // low word: next
    return x;
}
__device__ __forceinline__ void store_rstate(RunState* rs, const RState& x, int lane) {
    if (lane == 0) {
        rs->F = x.F; rs->M = x.M; rs->B = x.B; rs->n = x.n; rs->nep = x.nep; rs->ep1 = x.ep1; rs->eptr = x.eptr;
        rs->Ms = x.Ms; rs->next = x.next;
    }
}

// A unit in which a sample fires: resolve it chunk by chunk (a3).  x: state before the unit
// -> state after it.  Only chunks whose F range leaves (B-T, B+T) are read (lane l <-> row
// 32c+l, 8 events); one combined warp scan gives each lane the footprint and the running
// high-water mark before its first event, and the lane holding the first exit of the band
// walks its own events sequentially (successive samples included), then broadcasts the state.
// One candidate chunk of resolve_unit in 32-bit arithmetic: every prefix of the chunk (relative to
// its start Fc) is within +-2^29, so event sizes, lane sums and their combined scan fit in int32.  A
// lane's running max / min include its start value (the F of an earlier event, inside the band and
// <= Mc), so no sentinel is needed; the band limits are taken relative to Fc and clamped to int32.
__device__ __forceinline__ int clamp_i32(long long v) {
    return (int)llmax(llmin(v, (long long)INT_MAX), (long long)INT_MIN);
}
__device__ __forceinline__ void resolve_chunk32(const ReplayParams& p, const unsigned long long* rp,
                                             const unsigned long long* rm, long long e0, long long n_t, long long Fc,
                                             long long Mc, long long& B, unsigned long long& n, unsigned long long& nep,
                                             unsigned long long& ep1, unsigned long long& eptr, long long& Ms,
                                             unsigned long long sb, int lane)
{
#ifdef SCL_PROFILE
    const long long t_0 = clock64();
    { unsigned long long v = rm[0] ^ rm[7]; PROF_TOUCH(v) }
    const long long t_1 = clock64(); RPROF_ADD(9, t_1 - t_0)
#endif
    int fe[kEpt], run = 0, lmx = 0, lmn = 0;                 // relative to the lane's start
    unsigned live = 0;
    // events of the row inside the trace: [jlo, jhi)
    const int jlo = (int)llmin(llmax(-e0, 0ll), (long long)kEpt), jhi = (int)llmax(llmin(n_t - e0, (long long)kEpt), 0ll);
    const unsigned inr = ((1u << jhi) - 1u) & ~((1u << jlo) - 1u);
    #pragma unroll
    for (int jj = 0; jj < kEpt; ++jj) {
        const unsigned kind = ev_kind(rm[jj]);
        const bool af = ((inr >> jj) & 1u) && kind < 2;
        const int sz = (int)(unsigned)rm[jj];                 // < 2^30 for a counted event here
        run += af ? (kind == 0 ? sz : -sz) : 0;
        fe[jj] = run;
        lmx = max(lmx, run); lmn = min(lmn, run);
        live |= (af ? 1u : 0u) << jj;
    }
    int ssum = run, smax = lmx;                               // combined inclusive scan, relative to Fc
    #pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
        const int os = __shfl_up_sync(kFull, ssum, dd), om = __shfl_up_sync(kFull, smax, dd);
        if (lane >= dd) { smax = max(om, os + smax); ssum = os + ssum; }
    }
    const int xl = ssum - run;                                // F before the lane, relative to Fc
    const int mprev = __shfl_up_sync(kFull, smax, 1);
    const long long Ml = lane == 0 ? Mc : llmax(Mc, Fc + mprev);   // max F before the lane's events
#ifdef SCL_PROFILE
    { long long v = Ml; PROF_TOUCH(v) }
    const long long t_2 = clock64(); RPROF_ADD(10, t_2 - t_1)
#endif
    int cur = 0;
    for (;;) {
        const int hi = clamp_i32(B + p.T - Fc), lo = clamp_i32(B - p.T - Fc);
        const unsigned cm = __ballot_sync(kFull, lane >= cur && (xl + lmx >= hi || xl + lmn <= lo));
        if (!cm) break;
        const int l0 = __ffs(cm) - 1;
        if (lane == l0) {                                     // this lane's exits, in order
            unsigned from = 0;
            int h2 = hi, l2 = lo;
            for (;;) {
                unsigned ex = 0;
                #pragma unroll
                for (int jj = 0; jj < kEpt; ++jj) { const int v = xl + fe[jj]; ex |= (v >= h2 || v <= l2 ? 1u : 0u) << jj; }
                ex &= live & ~((1u << from) - 1u);
                if (!ex) break;
                const int js = __ffs(ex) - 1;
                int vf = 0, mp = INT_MIN;
                unsigned long long ms = 0, ps = 0;
                #pragma unroll
                for (int jj = 0; jj < kEpt; ++jj) {
                    if (jj < js) mp = max(mp, xl + fe[jj]);
                    if (jj == js) { vf = xl + fe[jj]; ms = rm[jj]; ps = rp[jj]; }
                }
                const long long F = Fc + vf, Mp = mp == INT_MIN ? Ml : llmax(Ml, Fc + mp);
                const long long net = F - B;                  // the |A - F| counter
                const bool growth = net > 0;
                const bool nm = growth && F > (p.hwm_sample ? Ms : Mp);   // new high-water mark (Q3, Q4)
                const unsigned long long slot_s = sb + n;
                scl_sample smp;
                smp.idx = (unsigned long long)(e0 + js); smp.net = net; smp.footprint = F;
                smp.site = ev_site(ms); smp.kind = growth ? 0 : 1; smp.new_max = nm ? 1 : 0; smp.pad = 0;
                SCL_CHECK(slot_s < p.sample_cap);
                p.samples[slot_s] = smp;
                sample_counters(p, smp.site, growth, net, nm);
                if (nm) { p.ep_flag[slot_s] = ev_size(ms) >= kBloomBig ? 2u : 0u; ep1 = slot_s + 1; eptr = ps; ++nep; }   // bit 0 set by the reclaim pass
                ++n; B = F; Ms = llmax(Ms, F);            // "resets the counters"
                h2 = clamp_i32(B + p.T - Fc); l2 = clamp_i32(B - p.T - Fc);
                from = (unsigned)js + 1;
            }
        }
        B = shfl_ll(B, l0); n = __shfl_sync(kFull, n, l0);
        nep = __shfl_sync(kFull, nep, l0); ep1 = __shfl_sync(kFull, ep1, l0); eptr = __shfl_sync(kFull, eptr, l0);
        Ms = shfl_ll(Ms, l0);
        cur = l0 + 1;
    }
#ifdef SCL_PROFILE
    { long long v = B; PROF_TOUCH(v) }
    RPROF_ADD(12, clock64() - t_2)
#endif
}

__device__ void resolve_unit(const ReplayParams& p, const Slot& S, RState& x, unsigned long long sb, int lane)
{
    const SegInfo inf = S.info;
    const long long F0 = x.F, M0 = x.M;
    const long long sPc = S.Pc[lane], sax = S.ax[lane], san = S.an[lane], susum = S.usum, sumx = S.umx;
    long long B = x.B;
    unsigned long long n = x.n, nep = x.nep, ep1 = x.ep1, eptr = x.eptr;
    long long Ms = x.Ms;                                     // max sample footprint (hwm_mode SAMPLE)
    const long long hiL = F0 + sax, loL = F0 + san;          // F range of chunk `lane`
#ifdef SCL_PROFILE
    const long long t_a = clock64();
    { long long v0 = sPc, v1 = sax, v2 = san, v3 = susum; PROF_TOUCH(v0) PROF_TOUCH(v1) PROF_TOUCH(v2) PROF_TOUCH(v3) }
    const long long t_b = clock64(); RPROF_ADD(8, t_b - t_a)          /* record wait */
    long long t_rows = 0, t_scan = 0, t_walk = 0;
#endif
    // chunks whose footprint stays within +-2^29 of their start: resolved in 32-bit arithmetic
    const unsigned small = __ballot_sync(kFull, sax - sPc < (1ll << 29) && sax - sPc > -(1ll << 29) &&
                                                san - sPc < (1ll << 29) && san - sPc > -(1ll << 29));
    const bool ufit = __all_sync(kFull, sax < (1ll << 31) && sax > -(1ll << 31));   // chunk maxima fit int32
    int cnext = 0;                                           // chunks < cnext are resolved
    for (;;) {
        const unsigned ccm = __ballot_sync(kFull, lane >= cnext && (hiL >= B + p.T || loL <= B - p.T));
        if (!ccm) break;
        const int c = __ffs(ccm) - 1;
        RPROF_ADD(11, 1)
        const long long row = inf.row_base + (long long)c * 32 + lane;
        unsigned long long rp[kEpt], rm[kEpt];
#ifdef SCL_PROFILE
        long long t_l = clock64();
#endif
        load_row_global(p.ev, row, rp, rm);
        // while the rows are in flight: F and the high-water mark before chunk c
        const long long Fc = F0 + shfl_ll(sPc, c);
        long long Mc;                                           // max F before chunk c
        if (ufit) { const int m = __reduce_max_sync(kFull, lane < c ? (int)sax : INT_MIN); Mc = c ? llmax(M0, F0 + m) : M0; }
        else      Mc = llmax(M0, warp_max(lane < c ? hiL : kNeg));
#ifdef SCL_PROFILE
        #pragma unroll
        for (int jj = 0; jj < kEpt; ++jj) { long long v = (long long)rm[jj]; PROF_TOUCH(v) rm[jj] = (unsigned long long)v; }
        const long long t_r = clock64(); t_rows += t_r - t_l;
#endif
        const long long e0 = row * kEpt - inf.off_t;           // trace index of the lane's first event
        if ((small >> c) & 1u) {
            resolve_chunk32(p, rp, rm, e0, inf.n_t, Fc, Mc, B, n, nep, ep1, eptr, Ms, sb, lane);
            cnext = c + 1;
            continue;
        }
        long long fe[kEpt], run = 0, lmx = kNeg, lmn = kPos;   // fe[jj]: F after event jj - F before the lane
        unsigned live = 0;                                      // events that move F (alloc/free in the trace)
        #pragma unroll
        for (int jj = 0; jj < kEpt; ++jj) {
            const long long ie = e0 + jj;
            const unsigned kind = ev_kind(rm[jj]);
            const bool af = ie >= 0 && ie < inf.n_t && kind < 2;
            const long long sz = (long long)ev_size(rm[jj]);
            run += af ? (kind == 0 ? sz : -sz) : 0;
            fe[jj] = run;
            if (af) { lmx = llmax(lmx, run); lmn = llmin(lmn, run); live |= 1u << jj; }
        }
        // combined exclusive scan over lanes of (sum, max prefix): (s1,m1).(s2,m2) = (s1+s2, max(m1, s1+m2))
        long long ssum = run, smax = lmx;                       // inclusive, relative to the chunk start
        #pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
            const long long os = shfl_up_ll(ssum, dd), om = shfl_up_ll(smax, dd);
            if (lane >= dd) { smax = llmax(om, os + smax); ssum = os + ssum; }
        }
        const long long Fl = Fc + ssum - run;                  // F before the lane's first event
        long long Ml = shfl_up_ll(smax, 1);                     // max F over the events of lanes < lane
        Ml = lane == 0 ? Mc : llmax(Mc, Fc + Ml);
#ifdef SCL_PROFILE
        { long long v = Ml; PROF_TOUCH(v) Ml = v; }
        const long long t_s = clock64(); t_scan += t_s - t_r;
#endif
        int cur = 0;
        for (;;) {
            const unsigned cm = __ballot_sync(kFull, lane >= cur && (Fl + lmx >= B + p.T || Fl + lmn <= B - p.T));
            if (!cm) break;
            const int l0 = __ffs(cm) - 1;
            if (lane == l0) {           // this lane's events: exits of the band found in parallel, in order
                unsigned from = 0;                              // events < from are settled
                for (;;) {
                    unsigned ex = 0;
                    #pragma unroll
                    for (int jj = 0; jj < kEpt; ++jj) {
                        const long long F = Fl + fe[jj];
                        ex |= (F >= B + p.T || F <= B - p.T ? 1u : 0u) << jj;
                    }
                    ex &= live & ~((1u << from) - 1u);
                    if (!ex) break;
                    const int js = __ffs(ex) - 1;
                    long long F = 0, Mp = Ml;                   // F at the event, max F before it (M_{i-1})
                    unsigned long long ms = 0, ps = 0;
                    #pragma unroll
                    for (int jj = 0; jj < kEpt; ++jj) {
                        if (jj < js) Mp = llmax(Mp, Fl + fe[jj]);
                        if (jj == js) { F = Fl + fe[jj]; ms = rm[jj]; ps = rp[jj]; }
                    }
                    const long long net = F - B;              // the |A - F| counter
                    const bool growth = net > 0;
                    const bool nm = growth && F > (p.hwm_sample ? Ms : Mp);   // new high-water mark (Q3, Q4)
                    const unsigned long long slot_s = sb + n;
                    scl_sample smp;
                    smp.idx = (unsigned long long)(e0 + js); smp.net = net; smp.footprint = F;
                    smp.site = ev_site(ms); smp.kind = growth ? 0 : 1; smp.new_max = nm ? 1 : 0; smp.pad = 0;
                    SCL_CHECK(slot_s < p.sample_cap);
                p.samples[slot_s] = smp;
                    sample_counters(p, smp.site, growth, net, nm);
                    if (nm) { p.ep_flag[slot_s] = ev_size(ms) >= kBloomBig ? 2u : 0u; ep1 = slot_s + 1; eptr = ps; ++nep; }   // bit 0 set by the reclaim pass
                    ++n; B = F; Ms = llmax(Ms, F);            // "resets the counters"
                    from = (unsigned)js + 1;
                }
            }
            B = shfl_ll(B, l0); n = __shfl_sync(kFull, n, l0);
            nep = __shfl_sync(kFull, nep, l0); ep1 = __shfl_sync(kFull, ep1, l0); eptr = __shfl_sync(kFull, eptr, l0);
            Ms = shfl_ll(Ms, l0);
            cur = l0 + 1;
        }
#ifdef SCL_PROFILE
        { long long v = B; PROF_TOUCH(v) B = v; }
        t_walk += clock64() - t_s;
#endif
        cnext = c + 1;
    }
    x.F = F0 + susum; x.M = llmax(M0, F0 + sumx); x.B = B;
    x.n = n; x.nep = nep; x.ep1 = ep1; x.eptr = eptr; x.Ms = Ms;
#ifdef SCL_PROFILE
    RPROF_ADD(9, t_rows) RPROF_ADD(10, t_scan) RPROF_ADD(12, t_walk) RPROF_ADD(13, clock64() - t_b - t_rows - t_scan - t_walk)
#endif
    __syncwarp();
}

// Advance a trace as far as its units are published (the caller is the trace's runner).
__device__ void run_trace(const ReplayParams& p, RState& x, unsigned t, unsigned base, unsigned nseg,
                          unsigned long long sb, unsigned ep_tag, int lane)
{
    const Slot* rec = reinterpret_cast<const Slot*>(p.urec);
    RPROF_ADD(0, 1)
    while (x.next < nseg) {
        // ready prefix of the next 32 units (lane i <-> unit next+i)
        // the unit's tagged aggregate words are its ready flag: one load gives both
        const unsigned ui = x.next + (unsigned)lane;
        long long us = 0, ux = kNeg, un = kPos;
        bool rdy = false;
        if (ui < nseg) {
            const unsigned long long* w = p.uagg + (size_t)(base + ui) * 4;
            unsigned long long w0, w1, w2;
            ld_relaxed_v2(w, w0, w1);
            w2 = ld_relaxed_u64(w + 2);
            const unsigned long long tag = ep_tag & 0xffffu;
            rdy = (w0 & 0xffffu) == tag && (w1 & 0xffffu) == tag && (w2 & 0xffffu) == tag;
            us = (long long)w0 >> 16; ux = (long long)w1 >> 16; un = (long long)w2 >> 16;
        }
        const unsigned nr = ~__ballot_sync(kFull, rdy);
        const int m = nr ? __ffs(nr) - 1 : 32;               // units next .. next+m-1 are ready
        if (m == 0) return;
        fence_acquire();
        RPROF_ADD(1, 1) RPROF_ADD(2, m)
#ifdef SCL_PROFILE
        if (lane < m) PROF_UNIT_T(base + x.next + lane, 2)
        const long long t_bat = clock64();
        long long t_res = 0;
#endif
        const Slot* R = rec + base + x.next;
        SCL_CHECK(base + x.next + (unsigned)m <= p.n_segs);
        UnitEntry* ue = p.uent + base + x.next;
        if (lane >= m) { us = 0; ux = kNeg; un = kPos; }
        if (__any_sync(kFull, lane < m && us == kAggBig)) {   // a value beyond 48 bits: from the records
            if (lane < m) { us = R[lane].usum; ux = R[lane].umx; un = R[lane].umn; }
        }
        // footprint and high-water mark do not depend on the samples: one combined scan gives F and
        // M at the start of every unit of the batch ((s1,m1).(s2,m2) = (s1+s2, max(m1, s1+m2)))
        long long ps, pm;                                     // inclusive, relative to the batch start
        const bool bfit = __all_sync(kFull, lane >= m || (us < (1ll << 25) && us > -(1ll << 25) &&
                                                            ux < (1ll << 25) && un > -(1ll << 25)));
        if (bfit) {                                           // 32-bit scan; a unit's max includes its start
            int ps32 = lane < m ? (int)us : 0, pm32 = lane < m ? (int)llmax(ux, 0ll) : 0;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int os = __shfl_up_sync(kFull, ps32, d), om = __shfl_up_sync(kFull, pm32, d);
                if (lane >= d) { pm32 = max(om, os + pm32); ps32 = os + ps32; }
            }
            ps = ps32; pm = pm32;
        } else {
            ps = us; pm = ux;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const long long os = shfl_up_ll(ps, d), om = shfl_up_ll(pm, d);
                if (lane >= d) { pm = llmax(om, os + pm); ps = os + ps; }
            }
        }
        const long long Pe = ps - us;                         // F at the unit start - F at the batch start
        long long Me = shfl_up_ll(pm, 1);                      // max F (rel.) over the units before
        if (lane == 0) Me = kNeg;
        const long long Fb = x.F, Mb = x.M;
        int j = 0;
        for (;;) {
            // jf = first unit (>= j) whose F range leaves (B-T, B+T): a sample fires in it
            const long long c0 = Fb + Pe - x.B;
            const unsigned bm = __ballot_sync(kFull, lane >= j && lane < m && (c0 + ux >= p.T || c0 + un <= -p.T));
            const int jf = bm ? __ffs(bm) - 1 : m;
            // units j .. jf-1 take no sample: same episode, empty sample range
            if (lane >= j && lane < jf) { UnitEntry e; e.ep1 = x.ep1; e.eptr = x.eptr; e.s_in = sb + x.n; e.s_out = e.s_in; ue[lane] = e; }
            if (jf == m) break;
            UnitEntry ef; ef.ep1 = x.ep1; ef.eptr = x.eptr; ef.s_in = sb + x.n;   // unit jf, before its samples
            x.F = Fb + shfl_ll(Pe, jf);
            x.M = llmax(Mb, Fb + shfl_ll(Me, jf));
#ifdef SCL_PROFILE
            const long long t_r = clock64();
#endif
            resolve_unit(p, R[jf], x, sb, lane);
            if (lane == 0) { ef.s_out = sb + x.n; ue[jf] = ef; }
            RPROF_ADD(3, 1) RPROF_ADD(4, clock64() - t_r)
#ifdef SCL_PROFILE
            if (p.prof && lane == 0) p.prof[48 + 4 * (size_t)(base + x.next + jf) + 3] = clock64() - t_r;
            t_res += clock64() - t_r;
#endif
            j = jf + 1;
        }
        x.F = Fb + shfl_ll(ps, m - 1);
        x.M = llmax(Mb, Fb + shfl_ll(pm, m - 1));
#ifdef SCL_PROFILE
        if (lane < m) PROF_UNIT_T(base + x.next + lane, 1)
        RPROF_ADD(14, clock64() - t_bat - t_res)
#endif
        x.next += (unsigned)m;
        if (x.next == nseg && lane == 0) {          // trace done: summary, trend end points, gate sums (Q10)
            scl_trace_summary* sm = &p.summ[t];
            sm->f_final = x.F; sm->hwm = x.M; sm->n_samples = x.n; sm->n_episodes = x.nep;
            const long long ff = x.n ? __ldcg(&p.samples[sb].footprint) : 0, fl = x.n ? x.B : 0;
            sm->f_first_sample = ff; sm->f_last_sample = fl;
            if (x.n >= 2) {
                unsigned long long* gate = p.table + (size_t)p.n_sites * SCL_NCOL;
                atomicAdd(&gate[0], (unsigned long long)(fl - ff));
                atomicAdd(&gate[1], (unsigned long long)(ff > 1 ? ff : 1));
                atomicAdd(&gate[2], 1ull);
            }
        }
    }
}

// Publisher warp (one per CTA): copies each finished unit's summary from its shared-memory
// slot to the unit's global record, frees the slot, publishes the tagged aggregate words.
__device__ void publisher_role(const ReplayParams& p, Smem& s, int lane)
{
    const unsigned ep_tag = p.epoch;
    Slot* urec = reinterpret_cast<Slot*>(p.urec);
    PROF_DECL
    unsigned j = 0;                                      // this CTA's next unit (slot j % kSlots)
    for (;;) {
        // units complete in order (almost): wait for unit j, take every complete unit after it,
        // copy each to its unit record and hand the shared-memory slot back right away (the copy
        // is in flight from registers), then ONE device-scope fence before the aggregate words
        if (!mbar_try_hint(&s.sdone[j % kSlots], (j / kSlots) & 1u, 2000u)) {
            const unsigned nu = ((volatile unsigned*)&s.n_units)[0];
            if (nu != kInvalid && j >= nu) { PROF_FLUSH(16) return; }
            PROF_MARK(0)
            continue;
        }
        unsigned nb = 1;
        while (nb < (unsigned)kSlots && mbar_test(&s.sdone[(j + nb) % kSlots], ((j + nb) / kSlots) & 1u)) ++nb;
        unsigned fm = 0;
        for (unsigned b = 0; b < nb; ++b) fm |= 1u << ((j + b) % kSlots);
        j += nb;
        const bool mine = (fm >> lane) & 1u;                 // lane q <-> slot q: its unit id and aggregate
        const unsigned uq = mine ? ((volatile unsigned*)&s.slot[lane].info.slot)[0] : 0u;
        long long a3[3] = {0, 0, 0};                         // the aggregate of slot `lane` (composed below)
        for (unsigned m = fm; m; m &= m - 1) {
            const int q = __ffs(m) - 1;
            Slot& S = s.slot[q];
            {   // compose the unit's 32 chunk summaries (lane = chunk): prefixes, max / min, aggregate
                const long long cs = S.Pc[lane], cx = S.ax[lane], cn = S.an[lane];
                long long ci = cs;
                #pragma unroll
                for (int d = 1; d < 32; d <<= 1) { long long o = shfl_up_ll(ci, d); if (lane >= d) ci += o; }
                const long long Pc = ci - cs, ax = Pc + cx, an = Pc + cn;
                S.Pc[lane] = Pc; S.ax[lane] = ax; S.an[lane] = an;
                const long long usum = shfl_ll(ci, 31), umx = warp_max(ax), umn = warp_min(an);
                if (lane == 0) { S.usum = usum; S.umx = umx; S.umn = umn; PROF_UNIT_T(S.info.slot, 0) }
                if (lane == q) { a3[0] = usum; a3[1] = umx; a3[2] = umn; }
            }
            // the record goes out through the TMA engine (one bulk copy of the slot)
            fence_proxy_async_shared();                      // the compose's writes before the async-proxy read
            __syncwarp();
            const unsigned u = __shfl_sync(kFull, uq, q);
            if (lane == 0) bulk_s2g(urec + u, &S, (uint32_t)sizeof(Slot));
        }
        if (lane == 0) {
            bulk_commit();
            bulk_wait_read();                                // every slot of the batch read: hand them back
            for (unsigned m = fm; m; m &= m - 1) mbar_arrive(&s.sempty[__ffs(m) - 1]);
            bulk_wait_all();                                 // the records written
            fence_proxy_async_global();
        }
        __syncwarp();
        __threadfence();                                     // the records before their aggregate words
        if (mine) {
            const unsigned long long tag = ep_tag & 0xffffu;
            const bool fit = a3[0] > kAggBig && a3[0] < -kAggBig && a3[1] > kAggBig && a3[1] < -kAggBig &&
                             a3[2] > kAggBig && a3[2] < -kAggBig;
            unsigned long long* w = p.uagg + (size_t)uq * 4;
            #pragma unroll
            for (int i = 0; i < 3; ++i) st_relaxed_u64(w + i, ((unsigned long long)(fit ? a3[i] : kAggBig) << 16) | tag);
        }
        __syncwarp();
        PROF_MARK(1)
    }
}

// Runner warp ri of nr (= p.n_runners): owns traces ri, ri + nr, ...  (lane i <-> its i-th
// trace, whose next unit index it keeps) and advances whichever of them has its next unit
// published, with the exact sequential state (kept in p.run between visits).
__device__ void runner_role(const ReplayParams& p, unsigned ri, int lane)
{
    if (p.no_chain) return;                               // the chains run in the pchain kernels
    const unsigned ep_tag = p.epoch;
    const unsigned nr = p.n_runners;
    if (!p.rechain) wait_prepared(p);                     // runner states, sample bases: CTA 0
    const unsigned cnt = ri < p.n_traces ? (p.n_traces - ri + nr - 1) / nr : 0u;
    const unsigned my_t = ri + (unsigned)lane * nr;
    unsigned my_base = 0, my_nseg = 0, my_next = 0;
    unsigned long long my_sb = 0;
    if ((unsigned)lane < cnt) { my_nseg = __ldg(p.tr_nseg + my_t); my_base = __ldg(p.tr_base + my_t); my_sb = p.sbase[my_t]; }
    PROF_DECL
    unsigned nap = 64;                                    // polling back-off (ns): units are published every
    for (;;) {                                            //   few us per CTA; the polls cost the stream issue slots
        const bool alive = (unsigned)lane < cnt && my_next < my_nseg;
        if (!__any_sync(kFull, alive)) break;
        const bool ready = alive && (ld_relaxed_u64(p.uagg + (size_t)(my_base + my_next) * 4 + 2) & 0xffffu) == (ep_tag & 0xffffu);
        unsigned rm = __ballot_sync(kFull, ready);
        if (!rm) { PROF_MARK(0) __nanosleep(nap); nap = min(nap * 2u, (unsigned)SCL_RUNNER_NAP); continue; }
        nap = 64;
        fence_acquire();
        PROF_MARK(0)
        while (rm) {
            const int i = __ffs(rm) - 1;
            rm &= rm - 1;
            const unsigned t = ri + (unsigned)i * nr;
            RunState* rs = p.run + t;
            RState x = load_rstate(rs, lane);
            x.next = __shfl_sync(kFull, my_next, i);
            run_trace(p, x, t, __shfl_sync(kFull, my_base, i), __shfl_sync(kFull, my_nseg, i), __shfl_sync(kFull, my_sb, i),
                      ep_tag, lane);
            store_rstate(rs, x, lane);
            if (lane == i) my_next = x.next;
        }
        PROF_MARK(2)
    }
    PROF_FLUSH(16)
}

// ============================================================================ post pass: reclaim (a4) + per-sample reduce (+ a6)
// One persistent cooperative launch (every block resident):
//  A. units (strided over the warps): a warp settles each unit that carries an episode or
//     samples -- the leak tracker's free-pointer comparison for every episode segment
//     inside the unit: the episode entering it up to the first episode started in it, then each
//     episode started in it up to the next (an episode is reclaimed iff its pointer is freed
//     anywhere in its span, so units are independent): Bloom query per chunk (lane <-> chunk),
//     each positive chunk queued as an exact re-check task;
//     traces: the per-sample reduce, one warp per trace;
//  -- grid barrier --
//  B. the re-check tasks, spread over all warps (one chunk each, through L2).  The first re-check
//     that finds the free of an episode flips its ep_flag and counts the episode's frees;
//  C. with fuse_report: a6 (report.cuh) over all blocks: flags per 32-site word, grid barrier,
//     ranks and rows.
// ep_flag was zeroed by the runner at each episode's start.
__device__ __forceinline__ bool chunk_has_free(const ReplayParams& p, long long row0, long long off_t, long long n_t,
                                               unsigned pos0, unsigned long long ptr, unsigned sbeg, unsigned send, int lane)
{
    // the chunk's 256 events with coalesced loads: lane l reads events 32k + l (no row order needed)
    const ulonglong2* cev = reinterpret_cast<const ulonglong2*>(p.ev + row0 * kEpt);
    ulonglong2 v[kEpt];
    #pragma unroll
    for (int k = 0; k < kEpt; ++k) v[k] = __ldcg(cev + k * 32 + lane);
    bool hit = false;
    #pragma unroll
    for (int k = 0; k < kEpt; ++k) {
        const unsigned e = (unsigned)(k * 32 + lane);
        const long long ie = row0 * kEpt + e - off_t;
        const unsigned q = pos0 + e;
        hit |= v[k].x == ptr && q >= sbeg && q < send && ie >= 0 && ie < n_t && ev_kind(v[k].y) == 1;
    }
    return __any_sync(kFull, hit);
}

// The episode whose tracked object is freed: once, ep_flag 0 -> 1 and one free for its site.
__device__ __forceinline__ void reclaimed(const ReplayParams& p, unsigned long long ep1, unsigned site) {
    SCL_CHECK(ep1 >= 1 && ep1 <= p.sample_cap && site < p.n_sites);
    if ((atomicOr(&p.ep_flag[ep1 - 1], 1u) & 1u) == 0u)
        atomicAdd(&p.table[(size_t)site * SCL_NCOL + SCL_COL_LEAK_FREES], 1ull);
}

struct UnitCtx { long long row_base, off_t, n_t; unsigned long long ep1, eptr, s_in, s_out; };

constexpr int kBloomRow = kBloomWords + 1;                  // staged filter row, padded: word w of the
constexpr size_t kPostBloom = 8 * 32 * kBloomRow * 4;       //   32 chunks in 32 banks; 8 warps per block

// sb: the warp's shared-memory slice for the unit's 32 chunk filters.
__device__ void reclaim_unit(const ReplayParams& p, unsigned u, const UnitCtx& x, int lane, unsigned* sb)
{
    const Slot& S = reinterpret_cast<const Slot*>(p.urec)[u];
    const bool staged = x.s_out >= x.s_in + 8;               // many segments: stage the filters (few
    if (staged) {                                            //   segments: one word per chunk, from L2)
        // lane = chunk: its filter, one 128-B row
        const uint4* src = reinterpret_cast<const uint4*>(&S.bloom[lane][0]);
        uint4 v[kBloomWords / 4];
        #pragma unroll
        for (int k = 0; k < kBloomWords / 4; ++k) v[k] = __ldcg(src + k);
        #pragma unroll
        for (int k = 0; k < kBloomWords / 4; ++k) {
            unsigned* d = sb + lane * kBloomRow + 4 * k;
            d[0] = v[k].x; d[1] = v[k].y; d[2] = v[k].z; d[3] = v[k].w;
        }
        __syncwarp();
    }
    const long long row_base = x.row_base, off_t = x.off_t, n_t = x.n_t;
    const long long g0 = row_base * kEpt;                    // global event index of unit position 0
    unsigned long long ep1 = x.ep1, ptr = x.eptr;            // current segment: episode (slot + 1), pointer, start
    unsigned sbeg = 0, site = 0;
    bool big = false;                                        // the tracked object >= kBloomBig (ep_flag bit 1)
    const bool in_ep = ep1 != 0;
    if (in_ep) { site = __ldcg(&p.samples[ep1 - 1].site); big = (__ldcg(&p.ep_flag[ep1 - 1]) & 2u) != 0; }
    auto segment = [&](unsigned send) {                      // [sbeg, send) of the current episode
        if (!ep1 || send <= sbeg) return;
        const unsigned w = bloom_word(ptr, big), msk = bloom_mask(ptr);
        const unsigned cb = (unsigned)lane * 32 * kEpt;
        const unsigned bw = staged ? sb[lane * kBloomRow + w] : __ldcg(&S.bloom[lane][w]);
        const bool pos = cb < send && cb + 32 * kEpt > sbeg && (bw & msk) == msk;
        const unsigned cm = __ballot_sync(kFull, pos);
        if (!cm) return;
#ifdef SCL_POST_INLINE
        {                                                    // the exact re-checks here, in order
            bool found = false;
            for (unsigned c = cm; c && !found; c &= c - 1) {
                const int ch = __ffs(c) - 1;
                found = chunk_has_free(p, row_base + (long long)ch * 32, off_t, n_t, (unsigned)ch * 32 * kEpt, ptr, sbeg, send, lane);
            }
            if (found && lane == 0) reclaimed(p, ep1, site);
            return;
        }
#endif
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(&p.ticket[2], (unsigned)__popc(cm));
        base = __shfl_sync(kFull, base, 0);
        if (base + (unsigned)__popc(cm) <= p.rtask_cap) {   // queue one re-check per positive chunk
            if (pos) {
                RTask tk;
                tk.ep1 = ep1; tk.ptr = ptr; tk.row0 = row_base + (long long)lane * 32; tk.off_t = off_t; tk.n_t = n_t;
                tk.pos0 = cb; tk.sbeg = sbeg; tk.send = send; tk.site = site;
                p.rtask[base + __popc(cm & ((1u << lane) - 1u))] = tk;
            }
        } else {                                             // queue full: re-check here, in order
            bool found = false;
            for (unsigned c = cm; c && !found; c &= c - 1) {
                const int ch = __ffs(c) - 1;
                found = chunk_has_free(p, row_base + (long long)ch * 32, off_t, n_t, (unsigned)ch * 32 * kEpt, ptr, sbeg, send, lane);
            }
            if (found && lane == 0) reclaimed(p, ep1, site);
        }
    };
    for (unsigned long long s0 = x.s_in; s0 < x.s_out; s0 += 32) {         // samples taken in this unit
        const unsigned long long si = s0 + (unsigned long long)lane;
        bool nm = false; long long idx = 0; unsigned st = 0;
        SCL_CHECK(x.s_out <= p.sample_cap);
        if (si < x.s_out) { const scl_sample smp = p.samples[si]; nm = smp.new_max != 0; idx = (long long)smp.idx; st = smp.site; }
        ulonglong2 evl = make_ulonglong2(0, 0);              // every episode's tracked object, loaded at once
        if (nm) evl = __ldcg(reinterpret_cast<const ulonglong2*>(p.ev + off_t + idx));
        unsigned em = __ballot_sync(kFull, nm);
        while (em) {
            const int e = __ffs(em) - 1;
            em &= em - 1;
            const long long ie = shfl_ll(idx, e);
            const unsigned pos = (unsigned)(off_t + ie - g0);
            segment(pos);
            ep1 = s0 + (unsigned long long)e + 1;
            ptr = __shfl_sync(kFull, evl.x, e);
            big = ev_size(__shfl_sync(kFull, evl.y, e)) >= kBloomBig;
            site = __shfl_sync(kFull, st, e);
            sbeg = pos;
        }
    }
    segment((unsigned)kUnit);
}

// Grid-wide barrier on counter ctr (zeroed per run): one arrival and one spinning thread per block.
__device__ __forceinline__ void grid_barrier(unsigned* ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (ld_relaxed(ctr) < gridDim.x) __nanosleep(32);
        fence_acquire();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256, 3) post_kernel(const __grid_constant__ ReplayParams p)
{
    extern __shared__ __align__(16) unsigned char post_smem[];            // a6 row staging (fuse_report)
    const int lane = threadIdx.x & 31;
    const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
#ifdef SCL_PROFILE
#define POST_T(i, op) if (p.prof && lane == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); op(&p.prof[40 + (i)], t_); }
    POST_T(0, atomicMin)
#else
#define POST_T(i, op)
#endif
    for (unsigned k0 = 0; wid + k0 * nw < p.n_segs; k0 += 32) {                           // phase A
        // this warp's units wid + k*nw: lane k loads unit k's entry and placement at once
        const unsigned u = wid + (k0 + (unsigned)lane) * nw;
        UnitCtx c{0, 0, 0, 0, 0, 0, 0};
        if (u < p.n_segs) {
            const UnitEntry e = p.uent[u];
            const SegInfo& inf = reinterpret_cast<const Slot*>(p.urec)[u].info;
            c.row_base = inf.row_base; c.off_t = inf.off_t; c.n_t = inf.n_t;
            c.ep1 = e.ep1; c.eptr = e.eptr; c.s_in = e.s_in; c.s_out = e.s_out;
        }
        unsigned todo = __ballot_sync(kFull, u < p.n_segs && (c.ep1 != 0 || c.s_in != c.s_out));
        while (todo) {
            const int i = __ffs(todo) - 1;
            todo &= todo - 1;
            UnitCtx x;
            x.row_base = shfl_ll(c.row_base, i); x.off_t = shfl_ll(c.off_t, i); x.n_t = shfl_ll(c.n_t, i);
            x.ep1 = __shfl_sync(kFull, c.ep1, i); x.eptr = __shfl_sync(kFull, c.eptr, i);
            x.s_in = __shfl_sync(kFull, c.s_in, i); x.s_out = __shfl_sync(kFull, c.s_out, i);
            reclaim_unit(p, wid + (k0 + (unsigned)i) * nw, x, lane,
                         reinterpret_cast<unsigned*>(post_smem) + (threadIdx.x >> 5) * 32 * kBloomRow);
        }
    }
    if (p.tierE && !p.rechain) {                        // Tier E of this stream pass, kept for re-thresholds
        const size_t n4 = (size_t)p.n_sites * 4;
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
            p.tierE[i] = __ldcg(&p.table[(i >> 2) * SCL_NCOL + (i & 3)]);
    }
    POST_T(1, atomicMax)
#ifndef SCL_POST_INLINE
    grid_barrier(&p.ticket[1]);
    POST_T(2, atomicMax)
    const unsigned ntask = min(ld_acquire(&p.ticket[2]), p.rtask_cap);
#ifdef SCL_PROFILE
    if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) p.prof[39] = ld_acquire(&p.ticket[2]);
#endif
    for (unsigned h = wid; h < ntask; h += nw) {                                          // phase B
        const RTask tk = p.rtask[h];
        if (chunk_has_free(p, tk.row0, tk.off_t, tk.n_t, tk.pos0, tk.ptr, tk.sbeg, tk.send, lane) && lane == 0)
            reclaimed(p, tk.ep1, tk.site);
    }
#endif
    POST_T(3, atomicMax)
    if (!p.fuse_report) return;                                                           // phase C: a6
    if (p.n_sites <= kReportSites) {                        // small table: a6 in the block that finishes last
        __shared__ unsigned last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();                                // this block's leak frees before its arrival
            last = atomicAdd(&p.ticket[3], 1u) == gridDim.x - 1;
            if (last) fence_acquire();                      // every block's leak frees before the reads below
        }
        __syncthreads();
        if (!last) return;
        report_block<256>(p.fin, p.rows, *reinterpret_cast<ReportSmem<256>*>(post_smem));
        POST_T(5, atomicMax)
        return;
    }
    grid_barrier(&p.ticket[3]);                             // every re-check done: leak frees final
    POST_T(4, atomicMax)
    const ReportScratch rx{p.rbits, p.rlrate, p.rlsite, &p.ticket[5], p.rsbcnt};
    report_grid_flags(p.fin, rx, wid, nw, lane);
    grid_barrier(&p.ticket[4]);
    report_grid_rows(p.fin, p.rows, rx, reinterpret_cast<unsigned long long*>(post_smem) + (threadIdx.x >> 5) * 32 * kRowWords,
                     wid, nw, lane);
    POST_T(5, atomicMax)
}

constexpr size_t kPostStage = std::max<size_t>(std::max<size_t>(8 * 32 * kRowWords * 8,   // a6 row staging: 8 warps x 32
                                                                report_smem_bytes<256>()),  // rows, or report_block in the
                                               kPostBloom);                                 // last block; phase A's filters

cudaError_t launch_post(const ReplayParams& p, cudaStream_t st)
{
    static int occ = 0, nsm = 0;
    const size_t smem = p.fuse_report ? kPostStage : kPostBloom;
    static int occ_fused = 0;
    if (!occ) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaFuncSetAttribute(post_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kPostStage);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, post_kernel, 256, kPostBloom);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_fused, post_kernel, 256, kPostStage);
        if (e != cudaSuccess) return e;
        occ = std::max(occ, 1); occ_fused = std::max(occ_fused, 1);
    }
    // every block resident (the phases wait for all warps): a cooperative launch of at most
    // occupancy x SMs blocks
    const unsigned need = std::max<unsigned>((std::max(p.n_segs, p.n_traces) + 7) / 8, 1u);
    const unsigned grid = std::min<unsigned>(need, (unsigned)((p.fuse_report ? occ_fused : occ) * nsm));
    void* args[] = {const_cast<ReplayParams*>(&p)};
    return cudaLaunchCooperativeKernel((const void*)post_kernel, dim3(grid), dim3(256), args, smem, st);
}

// ============================================================================ kernel
__global__ void __maxnreg__(96)
replay_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ ReplayParams p)
{
    // Pointers into dynamic shared memory are derived by pointer arithmetic only (never through
    // an integer), so that ptxas keeps the shared state space: LDS / ATOMS, not generic LD / ATOM.
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* stage = smem_raw;                                 // kStages x 32 KiB, 1024-aligned (swizzle)
    Smem& s = *reinterpret_cast<Smem*>(smem_raw + (size_t)kStages * kSegBytes);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0 && (smem_u32(smem_raw) & 1023u) != 0) __trap();     // the 128-B swizzle needs 1024-B alignment

    for (int x = tid; x < kTabSlots; x += kCtaThreads) { s.cnt[x] = 0; s.blo[x] = 0; }
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], 8 * 32); }
        for (int i = 0; i < kSlots; ++i) { mbar_init(&s.sempty[i], 1); mbar_init(&s.sdone[i], kChunks); }
        s.n_units = kInvalid;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"((uint64_t)&tmap) : "memory");
    }
    __syncthreads();
    zero_slice(p);
    if (blockIdx.x == 0) prepare_run(p, reinterpret_cast<unsigned long long*>(stage));   // stage: not in use yet

    // register rebalancing per warpgroup (launch: 96/thread): the four compute warpgroups give 16
    // each, the producer + publisher + runners warpgroup takes them (no spills in the resolver)
    if (warp < kComputeWarps) asm volatile("setmaxnreg.dec.sync.aligned.u32 80;\n" ::: "memory");
    else                      asm volatile("setmaxnreg.inc.sync.aligned.u32 160;\n" ::: "memory");
    if (warp < kComputeWarps) {
        compute_role(p, s, stage, warp / 8, warp % 8, lane);
        named_bar(1, kComputeWarps * 32);                            // all compute warps done
        const int cap = p.n_sites <= (unsigned)kHot ? kHot : kWarm;
        for (int x = tid; x < 2 * cap; x += kComputeWarps * 32) {    // flush Tier-E counters (allocs, frees)
            const int kind = x / cap, site = x % cap;
            const unsigned c = s.cnt[x];
            if (c && (unsigned)site < p.n_sites) {                   // (an invalid site id is dropped)
                unsigned long long* row = p.table + (size_t)site * SCL_NCOL;
                atomicAdd(&row[SCL_COL_N_MALLOC + kind], (unsigned long long)c);
                atomicAdd(&row[SCL_COL_MALLOC_BYTES + kind], (unsigned long long)s.blo[x]);
            }
        }
    } else if (warp == kProducerWarp) {
        producer_role(p, &tmap, s, stage, lane);
    } else if (warp == kProducerWarp + 1) {
        publisher_role(p, s, lane);
    } else {                                                          // 2 runner warps per CTA
        runner_role(p, blockIdx.x * kEmbeddedRunners + (warp - kProducerWarp - 2), lane);
    }
}

// Another threshold over the handle's last stream pass: the runners alone, reading the published
// unit records and aggregate words (tagged with that pass's epoch) and re-reading only the rows
// where a sample fires.
__global__ void __launch_bounds__(128) rechain_kernel(const __grid_constant__ ReplayParams p)
{
    runner_role(p, blockIdx.x * 4 + (threadIdx.x >> 5), threadIdx.x & 31);
}

cudaError_t launch_rechain(const ReplayParams& p, cudaStream_t st)
{
    if (p.n_segs == 0) return cudaSuccess;
    rechain_kernel<<<(p.n_runners + 3) / 4, 128, 0, st>>>(p);
    return cudaGetLastError();
}

int replay_occupancy(int* grid)
{
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    *grid = nsm;
    return 1;
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
    replay_kernel<<<grid, kCtaThreads, replay_smem_bytes(), st>>>(*tmap, p);
    return cudaGetLastError();
}

}  // namespace scl
