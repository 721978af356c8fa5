// replay_kernel.cu -- the streaming hot path a1..a5 in one pass over the events.
//
// Paper (PAPER.md lines): threshold sampler P:429-438 ("|A - F| >= T ... resets
// the counters"), footprint P:430-431 / P:490-494, high-water mark P:24-25,
// leak tracker with the free-pointer comparison P:20-39, per-line statistics
// P:488-494.  Readings Q1-Q16: DESIGN.md §3.
//
// One persistent CTA per SM, warp-specialised:
//   producer warp   one ticket per 8192-event unit (tickets ordered (unit index,
//                   trace), so the units of one trace are spread over time);
//                   issues the unit's 2-D TMA boxes (32 KiB, 128-B swizzle)
//                   into a kStages-deep shared-memory ring;
//   8 compute warps one 256-event chunk per box each: signed sizes, chunk sum
//                   and max/min prefix, Tier-E site counters (32-bit shared
//                   atomics + carry word), a 2048-bit Bloom filter of freed
//                   pointers; the last warp to finish a unit composes the 32
//                   chunk summaries and publishes the unit aggregate at once;
//   3 look-back warps take whole units round-robin: find the incoming state by
//                   a decoupled look-back over the trace's earlier units
//                   (aggregates are composed while the sampler band provably
//                   stays closed; the warp waits only at the first unit where
//                   a sample could fire), resolve the samples (re-reading only
//                   the chunks whose range leaves the band, through L2),
//                   publish the inclusive state, then check the frees against
//                   the tracked pointer (Bloom query per chunk, exact re-check
//                   of positives).
#include <climits>
#include "scl_internal.cuh"
#include "ptx.cuh"

namespace scl {

struct SegInfo {                     // one unit ticket, as the producer resolved it
    unsigned u, t, kraw, slot;       // ticket, trace, unit index (| last << 31), state slot
    long long off_t, n_t, row_base;  // trace start, trace length, first global row of the unit
    unsigned nbox, pad;              // boxes of this unit that overlap the trace
};
struct __align__(16) Slot {          // compute -> look-back summary of one unit
    SegInfo info;
    long long csum[kChunks], cmx[kChunks], cmn[kChunks];   // per chunk, relative to the chunk start
    long long Pc[kChunks], ax[kChunks], an[kChunks];       // chunk prefix; max/min relative to the unit start
    long long usum, umx, umn;                              // unit aggregate
    unsigned done, itu;                                    // chunks finished; CTA unit iteration
    unsigned bloom[kChunks][kBloomWords];
};
struct __align__(16) Smem {
    unsigned cnt[2 * kHot];          // Tier-E per (kind, hot site): event count
    unsigned blo[2 * kHot];          //   bytes, low 32 bits
    unsigned bhi[2 * kHot];          //   carries out of blo
    Slot slot[kSlots];
    SegInfo info[kStages];
    unsigned sub[kStages];           // box index within the unit
    uint64_t full[kStages], empty[kStages], sempty[kSlots];
    unsigned sstate[kSlots];         // 0 compute-owned, 1 full (ready for look-back), 2 claimed
    unsigned situ[kSlots];           // priority of a full slot (unit iteration; + 10^6 after a failed try)
    unsigned n_units;                // units handed to this CTA (known at the end of the tickets)
    unsigned n_done;                 // units finished by the look-back warps
};

size_t replay_park_bytes() { return sizeof(Slot); }
size_t replay_smem_bytes() { return 1024 + (size_t)kStages * kSegBytes + sizeof(Smem); }

// Blocked Bloom filter of freed pointers, 64 words (2048 bits) per 256-event chunk: one
// word per pointer, two bits in it (one shared-memory OR per free; ~1.4 % false positives
// at ~128 frees per chunk).
__device__ __forceinline__ unsigned bloom_word(unsigned long long ptr) {
    return ((unsigned)(ptr >> 4) * 0x9E3779B1u) >> 26;
}
__device__ __forceinline__ unsigned bloom_mask(unsigned long long ptr) {
    const unsigned h = (unsigned)(ptr >> 4) * 0x85EBCA77u;
    return (1u << (h >> 27)) | (1u << ((h >> 22) & 31u));
}

// Optional per-role cycle accounting (debug build with -DSCL_PROFILE only).
#ifdef SCL_PROFILE
#define PROF_DECL unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long pt = clock64();
#define PROF_MARK(i) { const long long now_ = clock64(); pacc[i] += now_ - pt; pt = now_; }
#define PROF_FLUSH(base) if (lane == 0 && p.prof) { for (int q_ = 0; q_ < 8; ++q_) atomicAdd(&p.prof[(base) + q_], pacc[q_]); }
#define PROF_UNIT_T(u, which) if (p.prof) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); p.prof[32 + 2 * (size_t)(u) + (which)] = t_; }
#else
#define PROF_DECL
#define PROF_MARK(i)
#define PROF_FLUSH(base)
#define PROF_UNIT_T(u, which)
#endif

// The 8 events of one global row, through L2 (re-read path).
__device__ __forceinline__ void load_row_global(const scl_event* ev, long long row, unsigned long long* ptr,
                                                unsigned long long* meta) {
    const ulonglong2* q = reinterpret_cast<const ulonglong2*>(ev + row * kEpt);
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) { ulonglong2 v = __ldcg(q + j); ptr[j] = v.x; meta[j] = v.y; }
}

// ============================================================================ compute warps
// Two groups of 8 warps alternate boxes (group 0: boxes 0 and 2 of a unit, group 1: 1 and 3);
// warp w8 of a group takes rows 32*w8 .. 32*w8+31 of its box = chunk g*8 + w8 of the unit.
__device__ void compute_role(const ReplayParams& p, Smem& s, unsigned char* stage, int grp, int w8, int lane)
{
    const unsigned want = p.epoch * 4u;
    const uint32_t cnt_s = smem_u32(s.cnt), blo_s = smem_u32(s.blo), bhi_s = smem_u32(s.bhi);
    PROF_DECL
    for (unsigned it = grp;; it += 2) {
        const int st = it % kStages;
        PROF_MARK(3)
        mbar_wait(&s.full[st], (it / kStages) & 1u);
        PROF_MARK(0)
        const SegInfo inf = s.info[st];
        const unsigned g = s.sub[st];
        const unsigned itu = it / kSub;                   // unit iteration of this CTA
        const int sl = itu % kSlots;
        if (inf.u == kInvalid) {
            // the look-back warps stop once all `itu` units of this CTA are published
            if (grp == 0 && w8 == 0 && lane == 0) atomicExch(&s.n_units, itu);
            PROF_FLUSH(0)
            return;
        }
        if (g == (unsigned)grp) mbar_wait(&s.sempty[sl], ((itu / kSlots) & 1u) ^ 1u);   // group's first box of the unit
        PROF_MARK(1)
        Slot& S = s.slot[sl];
        const int c = g * 8 + w8;                         // chunk index within the unit
        S.bloom[c][lane] = 0u; S.bloom[c][lane + 32] = 0u;
        if (g == 0 && w8 == 0 && lane == 0) S.info = inf;
        __syncwarp();
        const uint32_t bl_s = smem_u32(&S.bloom[c][0]);

        long long run = 0, tmx = kNeg, tmn = kPos;
        int r32 = 0, mx32 = INT_MIN, mn32 = INT_MAX;
        bool small = true;                                // 32-bit chunk summary is exact for this lane
        if (g < inf.nbox) {
            // ---- the 8 events of row 32*w8+lane (16-B chunk j of row r sits at j ^ (r & 7))
            const int r = w8 * 32 + lane;
            const unsigned char* rowp = stage + (size_t)st * kSegBytes + (size_t)r * 128;
            unsigned long long ptr[kEpt], meta[kEpt];
            #pragma unroll
            for (int j = 0; j < kEpt; ++j) {
                ulonglong2 v = *reinterpret_cast<const ulonglong2*>(rowp + ((j ^ (r & 7)) << 4));
                ptr[j] = v.x; meta[j] = v.y;
            }
            const long long e0 = (inf.row_base + (long long)g * kThreads + r) * kEpt - inf.off_t;
            unsigned big = 0;                                 // any size >= 2^27 in the row?
            #pragma unroll
            for (int j = 0; j < kEpt; ++j) big |= ((unsigned)meta[j] >> 27) | ((unsigned)(meta[j] >> 32) & 0xffu);
            unsigned cold = 0;                                // events for the L2 (cold site) path
            if (e0 >= 0 && e0 + kEpt <= inf.n_t && big == 0) {
                // fast path: the whole row is in the trace and |partial sums| < 2^30: 32-bit running
                // sum / max / min (a copy's d = 0 repeats an F already seen: harmless), predicated
                // shared atomics issued back to back, carries checked after all of them
                unsigned old[kEpt];
                #pragma unroll
                for (int j = 0; j < kEpt; ++j) {
                    const unsigned hi = (unsigned)(meta[j] >> 32), lo = (unsigned)meta[j];
                    const unsigned kind = (hi >> 8) & 3u, site = hi >> 11;
                    r32 += kind == 0 ? (int)lo : (kind == 1 ? -(int)lo : 0);          // a1: signed size
                    mx32 = max(mx32, r32); mn32 = min(mn32, r32);
                    const bool h = kind < 2 && site < (unsigned)kHot;
                    cold |= (kind < 2 && !h ? 1u : 0u) << j;
                    const uint32_t x = ((kind & 1u) * kHot + (h ? site : 0u)) * 4u;
                    red_add_if(cnt_s + x, 1u, h);                                     // a5 Tier E
                    old[j] = atom_add_if(blo_s + x, lo, h);
                    red_or_if(bl_s + bloom_word(ptr[j]) * 4u, bloom_mask(ptr[j]), kind == 1);   // freed ptr -> Bloom
                }
                #pragma unroll
                for (int j = 0; j < kEpt; ++j) {
                    const unsigned hi = (unsigned)(meta[j] >> 32), lo = (unsigned)meta[j];
                    const unsigned kind = (hi >> 8) & 3u, site = hi >> 11;
                    const bool h = kind < 2 && site < (unsigned)kHot;
                    red_add_if(bhi_s + ((kind & 1u) * kHot + (h ? site : 0u)) * 4u, 1u, h && old[j] + lo < old[j]);
                }
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
                        if (site < (unsigned)kHot && size < (1ull << 32)) {
                            const int x = kind * kHot + site;
                            atomicAdd(&s.cnt[x], 1u);
                            const unsigned old = atomicAdd(&s.blo[x], (unsigned)size);
                            if (old + (unsigned)size < old) atomicAdd(&s.bhi[x], 1u);
                        } else {
                            cold |= 1u << j;
                        }
                        if (kind == 1) atomicOr(&S.bloom[c][bloom_word(ptr[j])], bloom_mask(ptr[j]));
                    }
                }
            }
            while (cold) {                                    // cold site / huge size: L2 reductions
                const int j = __ffs(cold) - 1;
                cold &= cold - 1;
                unsigned long long mj = 0;
                #pragma unroll
                for (int q = 0; q < kEpt; ++q) if (q == j) mj = meta[q];
                const unsigned kind = ev_kind(mj);
                unsigned long long* row = p.table + (size_t)ev_site(mj) * SCL_NCOL;
                atomicAdd(&row[SCL_COL_N_MALLOC + kind], 1ull);
                atomicAdd(&row[SCL_COL_MALLOC_BYTES + kind], ev_size(mj));
            }
        }
        PROF_MARK(4)
        // ---- chunk summary: sum, max / min prefix relative to the chunk start
        long long csum, cmx, cmn;
        if (__all_sync(kFull, small)) {                       // 32-bit scan + REDUX
            int incl = r32;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { int o = __shfl_up_sync(kFull, incl, d); if (lane >= d) incl += o; }
            const int a = mx32 == INT_MIN ? INT_MIN : incl - r32 + mx32;
            const int b = mn32 == INT_MAX ? INT_MAX : incl - r32 + mn32;
            const int am = __reduce_max_sync(kFull, a), bm = __reduce_min_sync(kFull, b);
            csum = __shfl_sync(kFull, incl, 31);
            cmx = am == INT_MIN ? kNeg : am; cmn = bm == INT_MAX ? kPos : bm;
        } else {
            long long incl = run;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { long long o = shfl_up_ll(incl, d); if (lane >= d) incl += o; }
            const long long Pl = incl - run;
            cmx = warp_max(Pl + tmx); cmn = warp_min(Pl + tmn);
            csum = shfl_ll(incl, 31);
        }
        if (lane == 0) { S.csum[c] = csum; S.cmx[c] = cmx; S.cmn[c] = cmn; }
        __syncwarp();
        mbar_arrive(&s.empty[st]);                        // box consumed
        PROF_MARK(2)
        unsigned old = 0;
        if (lane == 0) { __threadfence_block(); old = atomicAdd(&S.done, 1u); __threadfence_block(); }
        old = __shfl_sync(kFull, old, 0);
        if (old == kChunks - 1) {
            // last chunk of the unit: compose the 32 chunk summaries (lane = chunk) and publish
            const long long cs = S.csum[lane], cx = S.cmx[lane], cn = S.cmn[lane];
            long long ci = cs;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { long long o = shfl_up_ll(ci, d); if (lane >= d) ci += o; }
            const long long Pc = ci - cs, ax = Pc + cx, an = Pc + cn;
            S.Pc[lane] = Pc; S.ax[lane] = ax; S.an[lane] = an;
            const long long usum = shfl_ll(ci, 31), umx = warp_max(ax), umn = warp_min(an);
            if (lane == 0) {
                S.usum = usum; S.umx = umx; S.umn = umn;
                SegState* my = &p.state[S.info.slot];
                my->sum = usum; my->mx = umx; my->mn = umn;
                st_release(&my->flag, want + 1);
                PROF_UNIT_T(S.info.slot, 0)
            }
            __syncwarp();
            if (lane == 0) { S.itu = itu; ((volatile unsigned*)s.situ)[sl] = itu; __threadfence_block(); atomicExch(&s.sstate[sl], 1u); }
        }
    }
}

// ============================================================================ producer warp
__device__ void producer_role(const ReplayParams& p, const CUtensorMap* tmap, Smem& s, unsigned char* stage, int lane)
{
    if (lane != 0) return;
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
                tma_load_2d(stage + (size_t)st * kSegBytes, tmap, 0, (int)(cur.row_base + (long long)g * kThreads),
                            &s.full[st]);
            }
            if (cur.u == kInvalid) { PROF_FLUSH(8) return; }
        }
        cur = nxt;
        u_next = u_after;
    }
}

// ============================================================================ look-back warps
struct InState { long long F, M, B; unsigned long long n, nep, ep, eptr; };

// The 7 inclusive words of a SegState (F, M, B, n, nep, ep, ep_ptr are consecutive):
// lanes 0..6 load one word each, then broadcast.
__device__ __forceinline__ InState load_inclusive_warp(const SegState* q, int lane) {
    const unsigned long long* w = reinterpret_cast<const unsigned long long*>(&q->F);
    unsigned long long v = lane < 7 ? __ldcg(w + lane) : 0ull;
    InState x;
    x.F = (long long)__shfl_sync(kFull, v, 0); x.M = (long long)__shfl_sync(kFull, v, 1);
    x.B = (long long)__shfl_sync(kFull, v, 2); x.n = __shfl_sync(kFull, v, 3);
    x.nep = __shfl_sync(kFull, v, 4); x.ep = __shfl_sync(kFull, v, 5); x.eptr = __shfl_sync(kFull, v, 6);
    return x;
}

// State before unit k of a trace (a1-a4 carries), NON-BLOCKING: returns false (with the
// flag it waits for) if a state it needs is not published yet.  Backward: windows of 32
// units (lane i <-> unit j-i) until the nearest inclusive state (the "base"; or the trace
// start), checking that every unit after it has its aggregate.  Forward: from the base,
// units are composed 32 at a time (lane i <-> unit start+i) while the sampler provably
// does not fire (every prefix of the carry stays in (-T, T)); at the first unit where it
// could fire, that unit's inclusive state is needed and becomes the new base.
__device__ bool look_back(const ReplayParams& p, const SegState* ts, unsigned k, unsigned want, int lane, InState& b,
                          const unsigned*& blk, unsigned& need, int resume = -1)
{
    b = InState{0, 0, 0, 0, 0, kNoEp, 0};
    blk = nullptr; need = 0;
    if (k == 0) return true;
    int base = resume;                                     // unit holding the base state (-1: trace start)
    // resume: a parked unit re-tried because the inclusive state it waited for (unit `resume`)
    // is published -- start the forward walk there (aggregates after it were checked before)
    if (resume < 0) for (int j = (int)k - 1;; j -= 32) {
        const int idx = j - lane;
        const unsigned fl = idx >= 0 ? ld_acquire(&ts[idx].flag) : 0u;
        const unsigned im = __ballot_sync(kFull, idx >= 0 && fl >= want + 2);
        const int stop = im ? __ffs(im) - 1 : 32;
        const unsigned lowmask = stop >= 32 ? kFull : ((1u << stop) - 1u);
        const unsigned miss = __ballot_sync(kFull, idx >= 0 && fl < want + 1) & lowmask;
        if (miss) { blk = &ts[j - (__ffs(miss) - 1)].flag; need = want + 1; return false; }   // an aggregate is missing
        if (im) { base = j - stop; break; }
        if (j - 31 <= 0) break;                            // reached unit 0: base = trace start
    }
    if (base >= 0) b = load_inclusive_warp(&ts[base], lane);
    for (int start = base + 1; start < (int)k;) {
        const int idx = start + lane;
        const bool in = idx < (int)k;
        long long a_s = 0, a_x = kNeg, a_n = kPos;
        if (in) { const SegState* q = &ts[idx]; a_s = __ldcg(&q->sum); a_x = __ldcg(&q->mx); a_n = __ldcg(&q->mn); }
        long long inc = a_s;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) { long long o = shfl_up_ll(inc, d); if (lane >= d) inc += o; }
        const long long E = inc - a_s;                     // sum of the earlier units of the window
        const long long c = b.F - b.B + E;
        const unsigned bm = __ballot_sync(kFull, in && (c + a_x >= p.T || c + a_n <= -p.T));
        if (!bm) {
            const long long mx = warp_max(in ? E + a_x : kNeg);
            b.M = llmax(b.M, b.F + mx);
            b.F += shfl_ll(inc, 31);
            start += 32;
            continue;
        }
        const int jf = __ffs(bm) - 1;                      // earliest unit where a sample may fire
        const SegState* q = &ts[start + jf];
        unsigned f = lane == 0 ? ld_acquire(&q->flag) : 0u;
        if (__shfl_sync(kFull, f, 0) < want + 2) { blk = &q->flag; need = want + 2; return false; }
        b = load_inclusive_warp(q, lane);
        start += jf + 1;
    }
    return true;
}

// Finish unit S (smem slot or its parked global copy) once its incoming state is known:
// samples, inclusive state, free-pointer match.
__device__ void finish_unit(const ReplayParams& p, const Slot* Sp, const InState& in, unsigned want,
                            EpStart* eplist, int lane)
{
    const Slot& S = *Sp;
    const SegInfo inf = S.info;
    const bool last = (inf.kraw >> 31) != 0;
    SegState* my = &p.state[inf.slot];
    const long long usum = S.usum, umx = S.umx, umn = S.umn;
    {
        // ---- a3/a4: samples of this unit (band test per chunk; exact re-scan only where needed)
        long long B = in.B;
        unsigned long long n = in.n, nep = in.nep, ep = in.ep, eptr = in.eptr;
        unsigned nl = 0;
        const long long F0 = in.F;
        if (F0 - B + umx >= p.T || F0 - B + umn <= -p.T) {
            const unsigned long long sb = __ldg(p.sbase + inf.t);
            const long long myax = S.ax[lane], myan = S.an[lane], myPc = S.Pc[lane];
            long long Mrun = in.M;                             // max F over events before the chunk
            for (int c = 0; c < kChunks; ++c) {
                const long long Pw = shfl_ll(myPc, c), hi = F0 + shfl_ll(myax, c), lo = F0 + shfl_ll(myan, c);
                if (!(hi >= B + p.T || lo <= B - p.T)) { Mrun = llmax(Mrun, hi); continue; }
                // re-read the chunk: lane l <-> row 32c+l of the unit (8 events)
                const long long row = inf.row_base + (long long)c * 32 + lane;
                unsigned long long rp[kEpt], rm[kEpt];
                load_row_global(p.ev, row, rp, rm);
                const long long e0 = row * kEpt - inf.off_t;
                long long d[kEpt], run = 0, lmx = kNeg, lmn = kPos;
                #pragma unroll
                for (int jj = 0; jj < kEpt; ++jj) {
                    const long long ie = e0 + jj;
                    const unsigned kind = ev_kind(rm[jj]);
                    const bool af = ie >= 0 && ie < inf.n_t && kind < 2;
                    const long long sz = (long long)ev_size(rm[jj]);
                    d[jj] = af ? (kind == 0 ? sz : -sz) : 0;
                    run += d[jj];
                    if (af) { lmx = llmax(lmx, run); lmn = llmin(lmn, run); }
                }
                long long li = run;
                #pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) { long long o = shfl_up_ll(li, dd); if (lane >= dd) li += o; }
                const long long Fl = F0 + Pw + (li - run);          // F before this lane's first event
                long long pmx = Fl + lmx;                             // max F over lanes <= lane
                #pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) { long long o = shfl_up_ll(pmx, dd); if (lane >= dd) pmx = llmax(pmx, o); }
                long long PMl = shfl_up_ll(pmx, 1);
                if (lane == 0) PMl = kNeg;
                int cur = 0;
                for (;;) {
                    const bool cand = lane >= cur && (Fl + lmx >= B + p.T || Fl + lmn <= B - p.T);
                    const unsigned cm = __ballot_sync(kFull, cand);
                    if (!cm) break;
                    const int l0 = __ffs(cm) - 1;
                    // lanes 0..7 take the 8 events of lane l0
                    long long de = 0; unsigned long long pe = 0, me = 0;
                    #pragma unroll
                    for (int jj = 0; jj < kEpt; ++jj) {
                        const long long v = shfl_ll(d[jj], l0);
                        const unsigned long long pv = __shfl_sync(kFull, rp[jj], l0), mv = __shfl_sync(kFull, rm[jj], l0);
                        if (lane == jj) { de = v; pe = pv; me = mv; }
                    }
                    const long long iev = shfl_ll(e0, l0) + lane;
                    const bool af = lane < kEpt && iev >= 0 && iev < inf.n_t && ev_kind(me) < 2;
                    long long L = de;
                    #pragma unroll
                    for (int dd = 1; dd < kEpt; dd <<= 1) { long long o = shfl_up_ll(L, dd); if (lane >= dd) L += o; }
                    const long long Fe = shfl_ll(Fl, l0) + L;
                    const long long Mbase = llmax(Mrun, shfl_ll(PMl, l0));
                    int ef = 0;
                    for (;;) {                                      // successive first exits of (B-T, B+T)
                        const bool ex = af && lane >= ef && (Fe >= B + p.T || Fe <= B - p.T);
                        const unsigned em = __ballot_sync(kFull, ex);
                        if (!em) break;
                        const int e = __ffs(em) - 1;
                        const long long Fs = shfl_ll(Fe, e);
                        const long long Mprev = llmax(Mbase, warp_max((af && lane < e) ? Fe : kNeg));   // M_{i-1}
                        const long long net = Fs - B;              // the |A - F| counter
                        const bool growth = net > 0;
                        const bool nm = growth && Fs > Mprev;      // new high-water mark (Q3, Q4)
                        const unsigned long long slot_s = sb + n;
                        if (lane == e) {
                            scl_sample smp;
                            smp.idx = (unsigned long long)iev; smp.net = net; smp.footprint = Fs;
                            smp.site = ev_site(me); smp.kind = growth ? 0 : 1; smp.new_max = nm ? 1 : 0; smp.pad = 0;
                            p.samples[slot_s] = smp;
                            if (nm) {
                                p.ep_flag[slot_s] = 0u;
                                EpStart es; es.ep = slot_s; es.ptr = pe; es.pos = (unsigned)((c * 32 + l0) * kEpt + e); es.pad = 0;
                                eplist[nl] = es;
                            }
                        }
                        if (nm) { ep = slot_s; eptr = __shfl_sync(kFull, pe, e); ++nep; ++nl; }
                        ++n; B = Fs; ef = e + 1;                   // "resets the counters"
                    }
                    cur = l0 + 1;
                }
                Mrun = llmax(Mrun, hi);
            }
        }
        // ---- publish the inclusive state (the end of the chain's critical path)
        if (lane == 0) {
            my->F = F0 + usum; my->M = llmax(in.M, F0 + umx); my->B = B;
            my->n = n; my->nep = nep; my->ep = ep; my->ep_ptr = eptr;
            st_release(&my->flag, want + 2);
            PROF_UNIT_T(inf.slot, 1)
            if (last) {
                scl_trace_summary* sm = &p.summ[inf.t];
                sm->f_final = F0 + usum; sm->hwm = llmax(in.M, F0 + umx);
                sm->n_samples = n; sm->n_episodes = nep;
            }
        }
        __syncwarp();

        // ---- a4 free-pointer match, "a pointer comparison that is almost always false":
        // lane c decides whether chunk c may hold a free of an active tracked pointer (Bloom)
        if (in.ep != kNoEp || nl > 0) {
            const unsigned cbeg = (unsigned)lane * 32 * kEpt, cend = cbeg + 32 * kEpt;
            unsigned li = 0;
            unsigned long long cptr = in.eptr; bool cval = in.ep != kNoEp;
            while (li < nl && eplist[li].pos < cbeg) { cptr = eplist[li].ptr; cval = true; ++li; }
            bool need = false;
            for (;;) {
                if (cval) { const unsigned m = bloom_mask(cptr); if ((S.bloom[lane][bloom_word(cptr)] & m) == m) need = true; }
                if (li < nl && eplist[li].pos < cend) { cptr = eplist[li].ptr; cval = true; ++li; } else break;
            }
            unsigned nm = __ballot_sync(kFull, need);
            if (nm && in.ep != kNoEp && nl == 0) {
                // the incoming episode may already be known reclaimed: nothing left to learn
                unsigned f0 = lane == 0 ? __ldcg(&p.ep_flag[in.ep]) : 0u;
                if (__shfl_sync(kFull, f0, 0)) nm = 0;
            }
            while (nm) {
                const int c = __ffs(nm) - 1;
                nm &= nm - 1;
                const long long row = inf.row_base + (long long)c * 32 + lane;
                unsigned long long rp[kEpt], rm[kEpt];
                load_row_global(p.ev, row, rp, rm);
                const long long e0 = row * kEpt - inf.off_t;
                const unsigned pos0 = (unsigned)(c * 32 + lane) * kEpt;
                unsigned lk = 0;
                unsigned long long aep = in.ep, aptr = in.eptr;
                while (lk < nl && eplist[lk].pos < pos0) { aep = eplist[lk].ep; aptr = eplist[lk].ptr; ++lk; }
                #pragma unroll
                for (int jj = 0; jj < kEpt; ++jj) {
                    while (lk < nl && eplist[lk].pos <= pos0 + jj) { aep = eplist[lk].ep; aptr = eplist[lk].ptr; ++lk; }
                    const long long ie = e0 + jj;
                    if (aep != kNoEp && ie >= 0 && ie < inf.n_t && ev_kind(rm[jj]) == 1 && rp[jj] == aptr)
                        atomicOr(&p.ep_flag[aep], 1u);
                }
            }
        }
    }
    __syncwarp();
}

// Look-back warp: claims full slots (oldest first).  A unit whose incoming state is
// available is finished from shared memory; otherwise its slot is copied to a global
// "park" record, released at once (compute never waits on a trace's chain), and the
// unit is finished later, when the flag it waits for has moved.  Lane i of the warp
// tracks parked unit i.
__device__ void lookback_role(const ReplayParams& p, Smem& s, int lbw, int lane)
{
    const unsigned want = p.epoch * 4u;
    const size_t wid = (size_t)blockIdx.x * kLBWarps + lbw;
    EpStart* eplist = p.ep_scratch + wid * kUnit;
    Slot* park = reinterpret_cast<Slot*>(p.park) + wid * kPark;
    unsigned pk_itu = kInvalid, pk_need = 0;           // lane i: parked unit i (CTA unit iteration), flag value needed
    const unsigned* pk_blk = nullptr;
    PROF_DECL
    for (;;) {
        // ---- 1. a parked unit whose blocker moved (oldest first)
        unsigned prio = kInvalid;
        if (pk_itu != kInvalid && ld_acquire(pk_blk) >= pk_need) prio = pk_itu;
        #pragma unroll
        for (int d = 16; d > 0; d >>= 1) prio = min(prio, __shfl_xor_sync(kFull, prio, d));
        if (prio != kInvalid) {
            const int i = __ffs(__ballot_sync(kFull, pk_itu == prio)) - 1;
            const Slot* G = park + i;
            const SegInfo inf = G->info;
            const unsigned k = inf.kraw & 0x7fffffffu;
            const SegState* ts = &p.state[inf.slot - k];
            // the blocker was an inclusive state of this trace: resume the forward walk from it
            const unsigned* bptr = (const unsigned*)__shfl_sync(kFull, (unsigned long long)pk_blk, i);
            const unsigned bneed = __shfl_sync(kFull, pk_need, i);
            const int resume = bneed == want + 2 ? (int)(((const char*)bptr - (const char*)&ts[0].flag) / sizeof(SegState)) : -1;
            InState in; const unsigned* blk; unsigned need;
            if (look_back(p, ts, k, want, lane, in, blk, need, resume)) {
                finish_unit(p, G, in, want, eplist, lane);
                if (lane == i) pk_itu = kInvalid;
                if (lane == 0) atomicAdd(&s.n_done, 1u);
            } else if (lane == i) {
                pk_blk = blk; pk_need = need;
            }
            __syncwarp();
            PROF_MARK(2)
            continue;
        }
        // ---- 2. the oldest full slot (only if a park lane is free)
        const unsigned freelanes = __ballot_sync(kFull, lane < kPark && pk_itu == kInvalid);
        unsigned best = kInvalid;
        if (freelanes && lane < kSlots && ((volatile unsigned*)s.sstate)[lane] == 1) best = ((volatile unsigned*)s.situ)[lane];
        #pragma unroll
        for (int d = 16; d > 0; d >>= 1) best = min(best, __shfl_xor_sync(kFull, best, d));
        if (best == kInvalid) {
            const unsigned nu = ((volatile unsigned*)&s.n_units)[0], nd = ((volatile unsigned*)&s.n_done)[0];
            if (nu != kInvalid && nd >= nu) { PROF_FLUSH(16) return; }
            PROF_MARK(0)
            __nanosleep(64);
            continue;
        }
        const bool mine = lane < kSlots && ((volatile unsigned*)s.sstate)[lane] == 1 && ((volatile unsigned*)s.situ)[lane] == best;
        const unsigned cand = __ballot_sync(kFull, mine);
        if (!cand) continue;
        const int q = __ffs(cand) - 1;
        unsigned got = 0;
        if (lane == 0) got = atomicCAS(&s.sstate[q], 1u, 2u);
        if (__shfl_sync(kFull, got, 0) != 1u) continue;
        __threadfence_block();
        PROF_MARK(0)
        Slot& S = s.slot[q];
        const SegInfo inf = S.info;
        const unsigned k = inf.kraw & 0x7fffffffu;
        InState in; const unsigned* blk; unsigned need;
        const bool ready = look_back(p, &p.state[inf.slot - k], k, want, lane, in, blk, need);
        PROF_MARK(1)
        if (ready) {
            finish_unit(p, &S, in, want, eplist, lane);
        } else {
            // park: copy the slot to global memory, remember what it waits for
            const int i = __ffs(freelanes) - 1;
            const uint4* src = reinterpret_cast<const uint4*>(&S);
            uint4* dst = reinterpret_cast<uint4*>(park + i);
            for (int o = lane; o < (int)(sizeof(Slot) / 16); o += 32) dst[o] = src[o];
            if (lane == i) { pk_itu = S.itu; pk_blk = blk; pk_need = need; }
        }
        __syncwarp();
        if (lane == 0) {
            S.done = 0; __threadfence_block();
            atomicExch(&s.sstate[q], 0u); mbar_arrive(&s.sempty[q]);
            if (ready) atomicAdd(&s.n_done, 1u);
        }
        __syncwarp();
        PROF_MARK(3)
    }
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

    for (int x = tid; x < 2 * kHot; x += kCtaThreads) { s.cnt[x] = 0; s.blo[x] = 0; s.bhi[x] = 0; }
    for (int x = tid; x < kSlots; x += kCtaThreads) s.slot[x].done = 0;
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], 8 * 32); }
        for (int i = 0; i < kSlots; ++i) { mbar_init(&s.sempty[i], 1); s.sstate[i] = 0; s.situ[i] = 0; }
        s.n_units = kInvalid; s.n_done = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"((uint64_t)&tmap) : "memory");
    }
    __syncthreads();

    if (warp < kComputeWarps) {
        compute_role(p, s, stage, warp / 8, warp % 8, lane);
        named_bar(1, kComputeWarps * 32);                            // all compute warps done
        for (int x = tid; x < 2 * kHot; x += kComputeWarps * 32) {   // flush Tier-E counters
            const unsigned c = s.cnt[x];
            if (c) {
                const int kind = x / kHot, site = x % kHot;
                unsigned long long* row = p.table + (size_t)site * SCL_NCOL;
                atomicAdd(&row[SCL_COL_N_MALLOC + kind], (unsigned long long)c);
                atomicAdd(&row[SCL_COL_MALLOC_BYTES + kind], ((unsigned long long)s.bhi[x] << 32) | s.blo[x]);
            }
        }
    } else if (warp == kProducerWarp) {
        producer_role(p, &tmap, s, stage, lane);
    } else {
        lookback_role(p, s, warp - kProducerWarp - 1, lane);
    }
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
