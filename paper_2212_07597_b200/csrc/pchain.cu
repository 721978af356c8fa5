// pchain.cu -- the threshold sampler's chain cut at sync events (a3 with hwm_mode PREFIX), so that
// one trace's samples are found by many warps at once (dense thresholds, few traces per GPU).
//
// The sampler "resets the counters" after every sample (reading Q2): its state between
// events is B, the footprint at the last sample, and a sample fires at the first event whose F leaves
// (B - T, B + T).  An event with |d| >= 2T - 1 leaves that band from ANY state (|F - B| < T before
// it), so it always takes a sample and the state after it is B = F there, whatever came before
// (SURVEY §7.3, Appendix A W5).  Every other quantity of the chain is associative: F and the prefix
// maximum M (so the new-maximum test F_i > M_(i-1) of PREFIX mode, reading Q3), the sample count and
// the last episode start.  So each trace splits into independent PIECES: one from the trace start,
// and one after the first sync event of every unit that has one, each ending at the first sync event
// of a later unit (included) or at the trace end.  Four stream-ordered launches:
//   pc_scan     = pc_prefix (warp per trace: F at every unit start and the max F before it, from the
//               unit aggregates) and, in the other blocks of the same launch, pc_sync (warp per unit:
//               its first sync event -- chunks whose F range spans >= 2T - 1 are read -- and F through
//               it relative to the unit start);
//   pc_run      warp per piece: the exact chain over the piece; its samples go to scratch blocks in
//               the order found (their slots are not known yet), Tier S (a5) to the site table, and
//               the piece-local sample count and last episode start at each unit's ends;
//   pc_combine  warp per trace: scan of the pieces' counts -> each piece's first sample slot and the
//               episode entering it; the trace summary, trend end points and gate sums (Q10);
//   pc_place    warp per piece: the samples copied to their slots, episode flags, and the unit entries
//               the reclaim pass reads (a4).
// The walk inside a unit is replay_kernel.cu's resolve_unit with an event window (the piece's part of
// the unit); its results are identical to the sequential runners' (checked against the oracle).
#include <algorithm>
#include "scl_internal.cuh"
#include "ptx.cuh"


namespace scl {

// ---------------------------------------------------------------------------- pc_prefix
// (blocks [0, nb) of the pc_scan launch)
__device__ void pc_prefix(const ReplayParams& p, unsigned blk, unsigned nb)
{
    const int lane = threadIdx.x & 31;
    const unsigned w = (blk * blockDim.x + threadIdx.x) >> 5, nw = (nb * blockDim.x) >> 5;
    const Slot* rec = reinterpret_cast<const Slot*>(p.urec);
    if (blk == 0 && threadIdx.x < 2) p.pctr[threadIdx.x] = 0;            // pc_run's scratch blocks and pieces
    for (unsigned t = w; t < p.n_traces; t += nw) {
        const unsigned base = __ldg(p.tr_base + t), nseg = __ldg(p.tr_nseg + t);
        long long F = 0, M = 0;                              // F before the next unit; max F so far (M_-1 = 0)
        for (unsigned k0 = 0; k0 < nseg; k0 += 32) {
            const unsigned k = k0 + (unsigned)lane;
            long long us = 0, ux = kNeg;
            if (k < nseg) { us = __ldcg(&rec[base + k].usum); ux = __ldcg(&rec[base + k].umx); }
            long long ps = us, pm = ux;                      // combined inclusive scan (s1+s2, max(m1, s1+m2))
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const long long os = shfl_up_ll(ps, d), om = shfl_up_ll(pm, d);
                if (lane >= d) { pm = llmax(om, os + pm); ps = os + ps; }
            }
            const long long pe = ps - us;                    // F at the unit start, relative to F
            long long me = shfl_up_ll(pm, 1);
            if (lane == 0) me = kNeg;
            if (k < nseg) { UnitStart x; x.F0 = F + pe; x.M0 = llmax(M, me == kNeg ? kNeg : F + me); p.ust[base + k] = x; }
            const long long ls = shfl_ll(ps, 31), lm = shfl_ll(pm, 31);
            M = llmax(M, F + lm);
            F += ls;
        }
    }
}

// ---------------------------------------------------------------------------- pc_sync
// The unit's first event with |d| >= 2T - 1 (kind alloc / free, inside its trace) and F there,
// relative to the unit start (pc_run adds the unit's F0: this pass does not wait for pc_prefix).  A
// chunk can hold one only if its F range, chunk start included, spans at least 2T - 1.
// (blocks [nb0, gridDim.x) of the pc_scan launch)
__device__ void pc_sync(const ReplayParams& p, unsigned blk, unsigned nb, unsigned long long (*tb)[33])
{
    const int lane = threadIdx.x & 31;
    const unsigned w = (blk * blockDim.x + threadIdx.x) >> 5, nw = (nb * blockDim.x) >> 5;
    const Slot* rec = reinterpret_cast<const Slot*>(p.urec);
    const unsigned long long thr = 2ull * (unsigned long long)p.T - 1ull;
    for (unsigned u = w; u < p.n_segs; u += nw) {
        const Slot& S = rec[u];
        const long long sPc = __ldcg(&S.Pc[lane]), sax = __ldcg(&S.ax[lane]), san = __ldcg(&S.an[lane]);
        const long long row_base = __ldcg(&S.info.row_base), off_t = __ldcg(&S.info.off_t), n_t = __ldcg(&S.info.n_t);
        const long long span = llmax(sax, sPc) - llmin(san, sPc);
        unsigned cand = __ballot_sync(kFull, span >= (long long)thr);
        SyncInfo out; out.pos = -1; out.pad0 = 0; out.Fs = 0; out.pad1 = 0; out.pad2 = 0;
        while (cand) {
            const int c = __ffs(cand) - 1;
            cand &= cand - 1;
            const long long row = row_base + (long long)c * 32 + lane;
            unsigned long long rm[kEpt];
            {   // coalesced loads of the chunk's meta words, transposed to rows (as in pc_run)
                const scl_event* cev = p.ev + (row_base + (long long)c * 32) * kEpt;
                unsigned long long v[kEpt];
                #pragma unroll
                for (int k = 0; k < kEpt; ++k) v[k] = __ldcg(&cev[k * 32 + lane].meta);
                __syncwarp();
                #pragma unroll
                for (int k = 0; k < kEpt; ++k) tb[lane & 7][4 * k + (lane >> 3)] = v[k];
                __syncwarp();
                #pragma unroll
                for (int jj = 0; jj < kEpt; ++jj) rm[jj] = tb[jj][lane];
            }
            const long long e0 = row * kEpt - off_t;
            long long run = 0;
            unsigned sy = 0;
            #pragma unroll
            for (int j = 0; j < kEpt; ++j) {
                const long long ie = e0 + j;
                const unsigned kind = ev_kind(rm[j]);
                const bool af = ie >= 0 && ie < n_t && kind < 2;
                const unsigned long long sz = ev_size(rm[j]);
                run += af ? (kind == 0 ? (long long)sz : -(long long)sz) : 0;
                sy |= (af && sz >= thr ? 1u : 0u) << j;
            }
            const unsigned lm = __ballot_sync(kFull, sy != 0);
            if (!lm) continue;
            const int l0 = __ffs(lm) - 1;
            // F before lane l0's row, relative to the unit start: scan of the row sums
            long long ssum = run;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { const long long os = shfl_up_ll(ssum, d); if (lane >= d) ssum += os; }
            const long long Fl = shfl_ll(sPc, c) + ssum - run;
            if (lane == l0) {
                const int j0 = __ffs(sy) - 1;
                long long F = Fl;
                #pragma unroll
                for (int j = 0; j < kEpt; ++j) {
                    if (j <= j0) {
                        const long long ie = e0 + j;
                        const unsigned kind = ev_kind(rm[j]);
                        if (ie >= 0 && ie < n_t && kind < 2) {
                            const long long sz = (long long)ev_size(rm[j]);
                            F += kind == 0 ? sz : -sz;
                        }
                    }
                }
                out.pos = c * 256 + l0 * kEpt + j0; out.Fs = F;
            }
            out.pos = __shfl_sync(kFull, out.pos, l0); out.Fs = shfl_ll(out.Fs, l0);
            break;
        }
        if (lane == 0) p.sync[u] = out;
    }
}

__global__ void __launch_bounds__(128) pc_scan_kernel(const __grid_constant__ ReplayParams p, unsigned nbp)
{
    __shared__ unsigned long long tb[4][kEpt][33];           // pc_sync: per-warp transposition buffer
    if (blockIdx.x < nbp) pc_prefix(p, blockIdx.x, nbp);
    else pc_sync(p, blockIdx.x - nbp, gridDim.x - nbp, tb[threadIdx.x >> 5]);
}

// ---------------------------------------------------------------------------- pc_run
struct PState {
    long long B;                                  // footprint at the last sample (the counter's origin)
    unsigned long long n, nep, lep, lep_ptr;      // samples, episode starts, last start (local index + 1), its ptr
    long long ffirst;                             // footprint at the first sample
    unsigned blk, first_blk;                      // the scratch block being filled, the piece's first
};

// Per warp of pc_run: the current row's absolute F after each event, the max F before it relative
// to the row start, and the meta words, event-major ([j][lane]) so that a dynamic event index is one shared-memory load.
struct RowStage {
    long long F[kEpt][32], P[kEpt][32];
    unsigned long long meta[kEpt][33];                   // (padded: the transposing stores below)
};

// Bits j of [a, b) within [0, kEpt).
__device__ __forceinline__ unsigned bit_range(long long a, long long b)
{
    const unsigned aa = (unsigned)llmin(llmax(a, 0), kEpt), bb = (unsigned)llmin(llmax(b, 0), kEpt);
    return bb > aa ? ((1u << bb) - 1u) & ~((1u << aa) - 1u) : 0u;
}

constexpr long long kI32Min = -2147483648ll, kI32Max = 2147483647ll;

// Lane mask of the events j of a row whose F (as f[j] relative to the row start) leaves the band:
// f >= hi or f <= lo.
template <typename V>
__device__ __forceinline__ unsigned band_exits(const V (&f)[kEpt], V hi, V lo)
{
    unsigned ex = 0;
    #pragma unroll
    for (int j = 0; j < kEpt; ++j) ex |= (f[j] >= hi || f[j] <= lo ? 1u : 0u) << j;
    return ex;
}

// The samples of one unit inside a piece's window [wlo, whi) (unit positions).  Fu: F before the
// unit's first event, Mu: max F before it.  The chunks whose F range leaves (B - T, B + T) and meet
// the window are read (lane <-> row); one combined scan gives every lane F and the running maximum
// before its row.  Then, per chunk:
//   (1) the sample positions, in order: every lane tests its row's events against the band around
//       B, the first lane with an exit holds the next sample, B becomes F there (the only state that
//       crosses lanes; ~60 warp instructions per sample, the 32-bit compare when the rows allow);
//   (2) the samples' records, lane-parallel: slot = an exclusive scan of the lanes' counts, the
//       counter before each one = F at the sample before it (reading Q2), the new-maximum test
//       against the max F before the event (Q3).
// Events outside the window move F and M but take no sample.
__device__ void piece_unit(const ReplayParams& p, const Slot& S, long long Fu, long long Mu, unsigned wlo, unsigned whi,
                           PState& x, int lane, RowStage& st)
{
    const long long sPc = __ldcg(&S.Pc[lane]), sax = __ldcg(&S.ax[lane]), san = __ldcg(&S.an[lane]);
    const long long row_base = __ldcg(&S.info.row_base), off_t = __ldcg(&S.info.off_t), n_t = __ldcg(&S.info.n_t);
    const long long hiL = Fu + llmax(sax, sPc), loL = Fu + llmin(san, sPc);
    const long long T = (long long)p.T;
    const unsigned cb = (unsigned)lane * 256u;
    const bool inwin = cb < whi && cb + 256u > wlo;
    long long cmx = Fu + sax;                                // max F through each chunk (inclusive scan)
    #pragma unroll
    for (int d = 1; d < 32; d <<= 1) { const long long o = shfl_up_ll(cmx, d); if (lane >= d) cmx = llmax(cmx, o); }
    int cnext = 0;
    for (;;) {
        const unsigned ccm = __ballot_sync(kFull, lane >= cnext && inwin && (hiL >= x.B + T || loL <= x.B - T));
        if (!ccm) break;
        const int c = __ffs(ccm) - 1;
        const long long row = row_base + (long long)c * 32 + lane;
        unsigned long long rm[kEpt];
        {   // the chunk's 256 meta words with coalesced loads (lane l: events 32k + l), transposed to
            // rows through the stage (event 32k + l is event l % 8 of row 4k + l / 8)
            const scl_event* cev = p.ev + (row_base + (long long)c * 32) * kEpt;
            unsigned long long v[kEpt];
            #pragma unroll
            for (int k = 0; k < kEpt; ++k) v[k] = __ldcg(&cev[k * 32 + lane].meta);
            #pragma unroll
            for (int k = 0; k < kEpt; ++k) st.meta[lane & 7][4 * k + (lane >> 3)] = v[k];
            __syncwarp();
            #pragma unroll
            for (int jj = 0; jj < kEpt; ++jj) rm[jj] = st.meta[jj][lane];
        }
        const long long Fc = Fu + shfl_ll(sPc, c);
        const long long cm1 = shfl_ll(cmx, c > 0 ? c - 1 : 0);
        const long long Mc = c > 0 ? llmax(Mu, cm1) : Mu;                             // max F before chunk c
        const long long e0 = row * kEpt - off_t;                                     // trace index of the row
        const unsigned q0 = (unsigned)c * 256u + (unsigned)lane * kEpt;              // unit position of the row
        // the row's events inside the trace and inside the window, as bit masks (bit j: event j)
        const unsigned tm = e0 >= 0 && e0 + kEpt <= n_t ? 0xFFu : bit_range(-e0, n_t - e0);
        const unsigned wm = q0 >= wlo && q0 + kEpt <= whi ? 0xFFu
                          : bit_range((long long)wlo - (long long)q0, (long long)whi - (long long)q0);
        long long fe[kEpt], run = 0;                             // F after event j relative to the row start
        unsigned live = 0, big = 0;
        #pragma unroll
        for (int jj = 0; jj < kEpt; ++jj) {
            const unsigned mh = (unsigned)(rm[jj] >> 32);
            const unsigned kind = (mh >> 8) & 3u;
            const bool af = ((tm >> jj) & 1u) && kind < 2;
            const long long sz = (long long)ev_size(rm[jj]);
            const long long neg = kind == 1 ? -1ll : 0ll;
            run += af ? (sz ^ neg) - neg : 0ll;
            fe[jj] = run;
            big |= (mh & 0xFFu) | ((unsigned)rm[jj] >> 22);      // a size >= 2^22
            live |= (af ? 1u : 0u) << jj;
        }
        live &= wm;
        // with every size of the chunk < 2^22, |fe| < 2^25 and the chunk's prefix sums < 2^30: int32 sums,
        // maxima and band compares (the band edges clamped to the int32 range) are exact
        const bool n32 = __all_sync(kFull, big == 0);
        // the max of fe before each event, from 0 (the F before the row, which is <= the max F before
        // it; a non-alloc/free event repeats the F before it: neither changes a maximum) -> st.P
        long long lmx;
        if (n32) {
            int m = 0;
            #pragma unroll
            for (int jj = 0; jj < kEpt; ++jj) { st.P[jj][lane] = m; m = max(m, (int)fe[jj]); }
            lmx = m;
        } else {
            long long m = 0;
            #pragma unroll
            for (int jj = 0; jj < kEpt; ++jj) { st.P[jj][lane] = m; m = llmax(m, fe[jj]); }
            lmx = m;
        }
        long long ssum, smax;                                    // combined scan of the rows: (sum, max prefix)
        if (n32) {
            int s32 = (int)run, m32 = (int)lmx;
            #pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const int os = __shfl_up_sync(kFull, s32, dd), om = __shfl_up_sync(kFull, m32, dd);
                if (lane >= dd) { m32 = max(om, os + m32); s32 = os + s32; }
            }
            ssum = s32; smax = __shfl_up_sync(kFull, m32, 1);
        } else {
            ssum = run; smax = lmx;
            #pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const long long os = shfl_up_ll(ssum, dd), om = shfl_up_ll(smax, dd);
                if (lane >= dd) { smax = llmax(om, os + smax); ssum = os + ssum; }
            }
            smax = shfl_up_ll(smax, 1);
        }
        const long long Fl = Fc + ssum - run;                                         // F before the lane's row
        const long long Ml = lane == 0 ? Mc : llmax(Mc, Fc + smax);                   // max F before it
        // stage the row: F after each event (the meta words are staged already)
        #pragma unroll
        for (int jj = 0; jj < kEpt; ++jj) st.F[jj][lane] = Fl + fe[jj];
        __syncwarp();
        // ---- (1) the sample positions, in order
        unsigned smask = 0;
        {
            int f32[kEpt];
            #pragma unroll
            for (int jj = 0; jj < kEpt; ++jj) f32[jj] = (int)fe[jj];
            long long B = x.B;
            int cl = 0;
            unsigned cfrom = 0;
            for (;;) {
                const long long hi = B + T - Fl, lo = B - T - Fl;
                unsigned ex;
                if (n32) ex = band_exits(f32, (int)llmin(llmax(hi, kI32Min), kI32Max), (int)llmin(llmax(lo, kI32Min), kI32Max));
                else ex = band_exits(fe, hi, lo);
                ex &= live & (lane > cl ? ~0u : lane == cl ? ~0u << cfrom : 0u);
                const unsigned m = __ballot_sync(kFull, ex != 0);
                if (!m) break;
                const int l0 = __ffs(m) - 1;
                const int js = __shfl_sync(kFull, __ffs(ex) - 1, l0);
                B = st.F[js][l0];                                                     // "resets the counters"
                if (lane == l0) smask |= 1u << js;
                cl = l0; cfrom = (unsigned)js + 1u;
            }
        }
        // ---- (2) the samples' records, lane-parallel
        const unsigned cnt = __popc(smask);
        unsigned incl = cnt;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) { const unsigned o = __shfl_up_sync(kFull, incl, d); if (lane >= d) incl += o; }
        const unsigned tot = __shfl_sync(kFull, incl, 31);
        if (tot) {
            const unsigned long long n0 = x.n;
            const unsigned long long have = (n0 + kPBlock - 1) / kPBlock, need = (n0 + tot + kPBlock - 1) / kPBlock;
            unsigned nb0 = 0;
            if (need > have) {                                       // new scratch blocks, contiguous and linked
                if (lane == 0) {
                    nb0 = atomicAdd(p.pctr, (unsigned)(need - have));
                    if (n0 == 0) x.first_blk = nb0; else if (x.blk < p.pblocks) p.pnext[x.blk] = nb0;
                    for (unsigned k = 1; k < (unsigned)(need - have); ++k)
                        if (nb0 + k - 1 < p.pblocks) p.pnext[nb0 + k - 1] = nb0 + k;
                }
                nb0 = __shfl_sync(kFull, nb0, 0);
                x.first_blk = __shfl_sync(kFull, x.first_blk, 0);
            }
            // the counter's origin before this lane's first sample: F at the last sample of an earlier
            // lane, else the state entering the chunk
            int last = smask ? lane : -1;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { const int o = __shfl_up_sync(kFull, last, d); if (lane >= d) last = max(last, o); }
            int prev = __shfl_up_sync(kFull, last, 1);
            if (lane == 0) prev = -1;
            const long long myLastF = st.F[smask ? 31 - __clz(smask) : 0][lane];
            const long long myFirstF = st.F[smask ? __ffs(smask) - 1 : 0][lane];
            long long Bp = shfl_ll(myLastF, prev < 0 ? 0 : prev);
            if (prev < 0) Bp = x.B;
            unsigned long long n = n0 + incl - cnt;
            unsigned long long nep = 0, lep = 0, lep_ptr = 0;
            for (unsigned sm = smask; sm; sm &= sm - 1) {
                const int j = __ffs(sm) - 1;
                const long long F = st.F[j][lane], Mp = llmax(Ml, Fl + st.P[j][lane]);   // max F before it
                const unsigned long long ms = st.meta[j][lane];
                const long long net = F - Bp;                                         // the |A - F| counter
                const bool growth = net > 0;
                const bool nm = growth && F > Mp;                                     // new high-water mark (Q3)
                scl_sample smp;
                smp.idx = (unsigned long long)(e0 + j); smp.net = net; smp.footprint = F;
                smp.site = ev_site(ms); smp.kind = growth ? 0 : 1; smp.new_max = nm ? 1 : 0;
                smp.pad = nm && ev_size(ms) >= kBloomBig ? 1 : 0;                     // (pc_place: episode flag bit 1)
                const unsigned long long bi = n / kPBlock;
                const unsigned blk = bi < have ? x.blk : nb0 + (unsigned)(bi - have);
                if (blk < p.pblocks) p.pscr[(size_t)blk * kPBlock + n % kPBlock] = smp;
                sample_counters(p, smp.site, growth, net, nm);
                if (nm) { ++nep; lep = n + 1; lep_ptr = __ldcg(&p.ev[row * kEpt + j].ptr); }
                Bp = F; ++n;
            }
            x.nep += (unsigned long long)warp_sum((long long)nep);
            const unsigned lm = __ballot_sync(kFull, lep != 0);
            if (lm) { const int ll = 31 - __clz(lm); x.lep = __shfl_sync(kFull, lep, ll); x.lep_ptr = __shfl_sync(kFull, lep_ptr, ll); }
            const unsigned sl = __ballot_sync(kFull, smask != 0);
            if (n0 == 0) x.ffirst = shfl_ll(myFirstF, __ffs(sl) - 1);
            x.B = shfl_ll(myLastF, 31 - __clz(sl));
            const unsigned long long bl = (n0 + tot - 1) / kPBlock;
            x.blk = bl < have ? x.blk : nb0 + (unsigned)(bl - have);
            x.n = n0 + tot;
        }
        __syncwarp();                                                                 // (st is rewritten next chunk)
        cnext = c + 1;
    }
}

#ifndef SCL_PCRUN_MINB
#define SCL_PCRUN_MINB 1
#endif
__global__ void __launch_bounds__(128, SCL_PCRUN_MINB) pc_run_kernel(const __grid_constant__ ReplayParams p)
{
    const int lane = threadIdx.x & 31;
    const Slot* rec = reinterpret_cast<const Slot*>(p.urec);
    const unsigned npieces = p.n_traces + p.n_segs;
    __shared__ RowStage stage[4];
    // pieces are taken one at a time from a counter (their lengths vary; a resident grid)
    for (;;) {
        unsigned id = 0;
        if (lane == 0) id = atomicAdd(p.pctr + 1, 1u);
        id = __shfl_sync(kFull, id, 0);
        if (id >= npieces) break;
        const bool tfirst = id < p.n_traces;
        unsigned t, u0, wlo0;
        long long B0;
        if (tfirst) {
            t = id;
            if (__ldg(p.tr_nseg + t) == 0) { if (lane == 0) p.pc[id].active = 0; continue; }
            u0 = __ldg(p.tr_base + t); wlo0 = 0; B0 = 0;
        } else {
            u0 = id - p.n_traces;
            const SyncInfo sy = p.sync[u0];
            if (sy.pos < 0) { if (lane == 0) p.pc[id].active = 0; continue; }
            t = __ldcg(&rec[u0].info.t); wlo0 = (unsigned)sy.pos + 1; B0 = p.ust[u0].F0 + sy.Fs;
        }
        const unsigned uend = __ldg(p.tr_base + t) + __ldg(p.tr_nseg + t);
        PState x{B0, 0, 0, 0, 0, 0, ~0u, ~0u};
        unsigned end_sync = 0, ulast = uend - 1;
        // the piece's units 32 at a time (lane = unit): one load of their start F, F range and first sync
        // event; a unit whose range stays inside the band around B (and holds no sync event, and is not
        // the piece's first unit after a sync event) passes the state through unchanged and is not walked
        for (unsigned u = u0; u < uend && !end_sync; u += 32) {
            const unsigned ub = u + (unsigned)lane;
            const bool valid = ub < uend;
            long long hiU = kNeg, loU = kPos;
            int sp = -1;
            if (valid) {
                const long long F0 = p.ust[ub].F0;
                hiU = F0 + __ldcg(&rec[ub].umx); loU = F0 + __ldcg(&rec[ub].umn);
                if (ub != u0 || tfirst) sp = p.sync[ub].pos;  // the piece ends at this unit's first sync event
            }
            const bool opener = ub == u0 && !tfirst;          // starts after the sync event: window [wlo0, ...)
            unsigned k = 0;                                   // lanes of the batch handled
            for (;;) {
                const bool need = valid && (unsigned)lane >= k &&
                                  (sp >= 0 || opener || hiU >= x.B + p.T || loU <= x.B - p.T);
                const unsigned nmask = __ballot_sync(kFull, need);
                const unsigned kn = nmask ? (unsigned)(__ffs(nmask) - 1) : 32u;
                if (valid && (unsigned)lane >= k && (unsigned)lane < kn) {   // passed through
                    UnitLocal* l = p.ul + ub;
                    l->n_start = x.n; l->lep_start = x.lep; l->lep_ptr_start = x.lep_ptr; l->n_end = x.n;
                }
                if (kn == 32u) break;
                const unsigned uw = u + kn;
                const unsigned wlo = uw == u0 ? wlo0 : 0u;
                const int spk = __shfl_sync(kFull, sp, (int)kn);
                unsigned whi = (unsigned)kUnit;
                if (spk >= 0) { whi = (unsigned)spk + 1; end_sync = 1; }
                if (wlo == 0 && lane == 0) {                  // the state entering the unit
                    UnitLocal* l = p.ul + uw;
                    l->n_start = x.n; l->lep_start = x.lep; l->lep_ptr_start = x.lep_ptr;
                }
                const UnitStart us = p.ust[uw];
                piece_unit(p, rec[uw], us.F0, us.M0, wlo, whi, x, lane, stage[threadIdx.x >> 5]);
                if (whi == (unsigned)kUnit && lane == 0) p.ul[uw].n_end = x.n;
                if (end_sync) { ulast = uw; break; }
                k = kn + 1;
            }
        }
        const unsigned u = ulast;
        if (lane == 0) {
            PieceCount c;
            c.n = x.n; c.nep = x.nep; c.lep = x.lep; c.lep_ptr = x.lep_ptr; c.ffirst = x.ffirst; c.flast = x.B;
            c.active = 1; c.first_blk = x.first_blk; c.u_first = u0; c.u_last = u; c.end_sync = end_sync; c.pad = 0;
            p.pc[id] = c;
        }
    }
}

// ---------------------------------------------------------------------------- pc_place
// Each piece's samples from its scratch blocks to their slots (and the episode flags the reclaim
// pass sets), and the unit entries of its units: the episode entering the unit (the piece's last
// start before it, else the one entering the piece), the slots of the unit's samples.
__global__ void __launch_bounds__(128) pc_place_kernel(const __grid_constant__ ReplayParams p)
{
    const int lane = threadIdx.x & 31;
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const unsigned npieces = p.n_traces + p.n_segs;
    for (unsigned id = w; id < npieces; id += nw) {
        const PieceCount c = p.pc[id];
        if (!c.active) continue;
        const PieceRun r = p.pr[id];
        unsigned b = c.first_blk;
        for (unsigned long long k0 = 0; k0 < c.n; k0 += kPBlock) {
            #pragma unroll
            for (int h = 0; h < kPBlock / 32; ++h) {
                const unsigned long long k = k0 + (unsigned long long)(h * 32 + lane);
                if (k < c.n && b < p.pblocks) {
                    scl_sample smp = p.pscr[(size_t)b * kPBlock + h * 32 + lane];
                    SCL_CHECK(r.base + k < p.sample_cap);
                    if (smp.new_max) p.ep_flag[r.base + k] = smp.pad ? 2u : 0u;   // the tracked object >= kBloomBig
                    smp.pad = 0;
                    p.samples[r.base + k] = smp;
                }
            }
            if (k0 + kPBlock < c.n) b = b < p.pblocks ? __ldcg(p.pnext + b) : ~0u;
        }
        const bool tfirst = id < p.n_traces;
        for (unsigned u = c.u_first + (unsigned)lane; u <= c.u_last; u += 32) {
            const UnitLocal l = p.ul[u];
            SCL_CHECK(u < p.n_segs);
            UnitEntry* e = p.uent + u;
            if (u != c.u_first || tfirst) {                  // the piece holds the unit's start
                e->ep1 = l.lep_start ? r.base + l.lep_start : r.ep1;
                e->eptr = l.lep_start ? l.lep_ptr_start : r.eptr;
                e->s_in = r.base + l.n_start;
            }
            if (u != c.u_last || !c.end_sync) e->s_out = r.base + l.n_end;   // ... and its end
        }
    }
}

// ---------------------------------------------------------------------------- pc_combine
// Per trace, its pieces in order (the trace-first piece, then one per unit with a sync event): first
// sample slot = sbase + the samples of the pieces before; the episode entering a piece = the last
// episode start of the pieces before (slot + 1, pointer); the summary (f_final, hwm, n_samples,
// n_episodes, trend end points) and the gate sums (reading Q10).
__global__ void __launch_bounds__(128) pc_combine_kernel(const __grid_constant__ ReplayParams p)
{
    const int lane = threadIdx.x & 31;
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const Slot* rec = reinterpret_cast<const Slot*>(p.urec);
    for (unsigned t = w; t < p.n_traces; t += nw) {
        const unsigned base = __ldg(p.tr_base + t), nseg = __ldg(p.tr_nseg + t);
        if (nseg == 0) continue;                             // summary zeroed by the preparation
        const unsigned long long sb = p.sbase[t];
        const PieceCount f = p.pc[t];
        if (lane == 0) { PieceRun r; r.base = sb; r.ep1 = 0; r.eptr = 0; r.pad = 0; p.pr[t] = r; }
        unsigned long long slot = sb + f.n, ep1 = f.lep ? sb + f.lep : 0, eptr = f.lep ? f.lep_ptr : 0, nep = f.nep;
        long long ffirst = f.ffirst, flast = f.flast;
        bool any = f.n > 0;
        for (unsigned k0 = 0; k0 < nseg; k0 += 32) {
            const unsigned u = base + k0 + (unsigned)lane;
            const bool act = k0 + (unsigned)lane < nseg && p.sync[u].pos >= 0;
            PieceCount c{};
            if (act) c = p.pc[p.n_traces + u];
            unsigned long long ns = act ? c.n : 0;
            unsigned long long incl = ns;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { const unsigned long long o = __shfl_up_sync(kFull, incl, d); if (lane >= d) incl += o; }
            const unsigned long long pbase = slot + incl - ns;
            // the episode entering this lane's piece: the last episode start among the earlier lanes
            const bool hep = act && c.lep != 0;
            const unsigned long long my_ep1 = hep ? pbase + c.lep : 0, my_ptr = hep ? c.lep_ptr : 0;
            int last = hep ? lane : -1;                      // inclusive max scan of the lanes with a start
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) { const int o = __shfl_up_sync(kFull, last, d); if (lane >= d) last = max(last, o); }
            int prev = __shfl_up_sync(kFull, last, 1);
            if (lane == 0) prev = -1;
            const unsigned long long pe1 = __shfl_sync(kFull, my_ep1, prev < 0 ? 0 : prev);
            const unsigned long long pep = __shfl_sync(kFull, my_ptr, prev < 0 ? 0 : prev);
            if (act) {
                PieceRun r; r.base = pbase; r.ep1 = prev < 0 ? ep1 : pe1; r.eptr = prev < 0 ? eptr : pep; r.pad = 0;
                p.pr[p.n_traces + u] = r;
            }
            const int lastall = __shfl_sync(kFull, last, 31);
            if (lastall >= 0) { ep1 = __shfl_sync(kFull, my_ep1, lastall); eptr = __shfl_sync(kFull, my_ptr, lastall); }
            nep += (unsigned long long)warp_sum((long long)(act ? c.nep : 0));
            // trend end points: the first / last piece (in order) that took a sample
            const unsigned hs = __ballot_sync(kFull, act && c.n > 0);
            if (hs) {
                const long long ff = shfl_ll(c.ffirst, __ffs(hs) - 1), fl = shfl_ll(c.flast, 31 - __clz(hs));
                if (!any) ffirst = ff;
                flast = fl;
                any = true;
            }
            slot = __shfl_sync(kFull, slot + incl, 31);
        }
        if (lane == 0) {
            const unsigned ul = base + nseg - 1;
            const UnitStart us = p.ust[ul];
            scl_trace_summary* sm = &p.summ[t];
            sm->f_final = us.F0 + __ldcg(&rec[ul].usum);
            sm->hwm = llmax(us.M0, us.F0 + __ldcg(&rec[ul].umx));
            const unsigned long long n = slot - sb;
            sm->n_samples = n; sm->n_episodes = nep;
            const long long ff = any ? ffirst : 0, fl = any ? flast : 0;
            sm->f_first_sample = ff; sm->f_last_sample = fl;
            if (n >= 2) {
                unsigned long long* gate = p.table + (size_t)p.n_sites * SCL_NCOL;
                atomicAdd(&gate[0], (unsigned long long)(fl - ff));
                atomicAdd(&gate[1], (unsigned long long)(ff > 1 ? ff : 1));
                atomicAdd(&gate[2], 1ull);
            }
        }
    }
}

// ---------------------------------------------------------------------------- launch
cudaError_t launch_pchain(const ReplayParams& p, cudaStream_t st)
{
    if (p.n_segs == 0) return cudaSuccess;
    auto grid = [](unsigned warps) { return std::max(1u, std::min((warps + 3) / 4, 148u * 16)); };
    const unsigned nbp = grid(p.n_traces);                   // pc_prefix and pc_sync are independent: one launch
    pc_scan_kernel<<<nbp + grid(p.n_segs), 128, 0, st>>>(p, nbp);
    static int run_blocks = 0;                               // resident pc_run blocks (it takes pieces from a counter)
    if (!run_blocks) {
        int dev = 0, nsm = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pc_run_kernel, 128, 0);
        if (e != cudaSuccess) return e;
        run_blocks = std::max(1, occ) * nsm;
    }
    pc_run_kernel<<<std::min(grid(p.n_traces + p.n_segs), (unsigned)run_blocks), 128, 0, st>>>(p);
    pc_combine_kernel<<<grid(p.n_traces), 128, 0, st>>>(p);
    pc_place_kernel<<<grid(p.n_traces + p.n_segs), 128, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace scl
