// api.cu -- host side of the C-ABI declared in include/scl.h.
//
// Owns the device copies of the traces (padded to whole 128-B rows so that a
// 2-D TMA tensor map with the 128-byte swizzle can stage 2048-event segments),
// the segment plan (ticket order interleaves traces so that one trace's
// segments are spread over time and its look-back chain rarely waits), and
// the per-run result buffers.  Every compute step runs in the kernels of
// replay.cu; this file only plans, allocates, launches and copies.
#include "scl_internal.cuh"
#include "report.cuh"
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <unordered_map>
#include <dlfcn.h>
#include <nccl.h>                              // types only: the functions come from dlsym
#include <algorithm>

using namespace scl;

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;
static scl_status fail(scl_status st, const std::string& msg) { g_err = msg; return st; }
#define CU(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return fail(SCL_ECUDA, std::string(#x ": ") + cudaGetErrorString(_e)); } while (0)

extern "C" const char* scl_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- handles
struct scl_traces {
    int device = 0;
    uint32_t n_traces = 0, n_sites = 0;
    uint64_t n_events = 0, max_len = 0, tick_ns = 1000;
    // device buffers, reused by scl_trace_reload while the new traces fit (cap_*)
    scl_event* d_ev = nullptr;                 // padded_rows * 8 events
    size_t cap_rows = 0;
    unsigned long long* d_off = nullptr;       // n_traces + 1
    unsigned long long* d_sabs = nullptr;      // per trace: sum |d| (sample-capacity bound)
    unsigned int* d_tr_nseg = nullptr;         // per trace: number of units
    unsigned int* d_tr_base = nullptr;         // per trace: first unit id
    RunState* d_run = nullptr;                 // per trace: runner state (zeroed per run)
    size_t cap_tr = 0;
    TicketInfo* d_tk = nullptr;
    void* d_urec = nullptr;                    // per unit: published summary record
    unsigned long long* d_uagg = nullptr;      // per unit: tagged aggregate words (published flag)
    UnitEntry* d_uent = nullptr;               // per unit: state entering it (runner -> reclaim pass)
    size_t cap_segs = 0;
    unsigned long long* d_err = nullptr;       // [1 + 64] first invalid event (load check), then the log2-size
                                               // histogram of the alloc / free events (chain-split heuristic)
    std::vector<uint64_t> h_shist;
    // site ids by frequency (n_sites > kHot): internal id = rank of the site in a strided sample of the
    // events, so that the hottest sites land in the shared-memory Tier-E table whatever the caller's
    // numbering; every output is mapped back to the caller's ids
    unsigned* d_remap = nullptr;               // [n_sites] caller id -> internal id
    std::vector<uint32_t> h_inv;               // internal id -> caller id (empty: identity)
    bool remapped = false;
    unsigned int* d_ticket = nullptr;
    std::vector<uint64_t> h_off, h_sabs;
    uint32_t n_segs = 0;
    mutable unsigned int epoch = 0;
    mutable uint32_t zc_arrivals = 0;          // CTAs of the replay launches since ticket[8] was zeroed
    CUtensorMap tmap;
    // rate sampler (lazy, per loaded traces): alloc / free / copy bytes per unit, before each unit, per trace
    mutable unsigned long long *d_usum = nullptr, *d_ustart = nullptr, *d_ttot = nullptr;
    mutable size_t cap_usum = 0, cap_ttot = 0;
    mutable bool usum_valid = false;
    // cold-record stream of the sites beyond the shared-memory table (n_sites > kWarm), per stream pass
    mutable unsigned long long* d_crec = nullptr;
    mutable unsigned* d_crec_fill = nullptr;
    mutable unsigned long long* d_cctr = nullptr;       // [2] records allocated, exhausted
    mutable unsigned long long crec_cap = 0;         // records (of the current record size)
    mutable size_t crec_bytes = 0, crec_fills = 0;
    mutable unsigned long long* h_covf = nullptr;       // pinned: the last exhausted pool (grow it)
    mutable unsigned* d_cpart = nullptr;                // cold_hist's partial tables
    mutable size_t cap_cpart = 0;
    // Tier-E columns of the last stream pass (written by its post pass; a re-threshold copies them)
    mutable unsigned long long* d_tierE = nullptr;
    mutable size_t cap_tierE = 0;
    // chain split at sync events (pchain.cu): per unit and per piece, sized with the unit plan
    mutable UnitStart* d_ust = nullptr;
    mutable SyncInfo* d_sync = nullptr;
    mutable PieceCount* d_pc = nullptr;
    mutable PieceRun* d_pr = nullptr;
    mutable UnitLocal* d_ul = nullptr;
    mutable size_t cap_pieces = 0;
    mutable scl_sample* d_pscr = nullptr;              // scratch blocks of the pieces' samples
    mutable unsigned* d_pnext = nullptr;
    mutable unsigned* d_pctr = nullptr;
    mutable size_t cap_pblocks = 0;
};

constexpr int kRing = 128;
constexpr unsigned kRTaskCap = 1u << 16;      // reclaim re-check queue (overflow: re-checked in place)                     // replay-kernel timing event pairs kept per result

struct scl_result {
    const scl_traces* tr = nullptr;
    unsigned long long* d_el = nullptr;        // nccl_comm runs: the elapsed time being MAX-reduced
    unsigned long long h_el = 0;
    uint64_t T = 0;
    unsigned epoch = 0;                        // the handle's stream pass this result belongs to
    int formula = 0;
    uint64_t elapsed_ns = 0;
    cudaStream_t stream = nullptr;
    // device
    unsigned long long* d_table = nullptr;     // n_sites*NCOL + 3, in the caller's site ids
    unsigned long long* d_table_int = nullptr; // the same in internal ids (remapped handles; else == d_table)
    scl_sample* d_samples = nullptr; unsigned int* d_epflag = nullptr; size_t cap = 0;
    unsigned long long* d_sbase = nullptr;
    scl_trace_summary* d_summ = nullptr;
    size_t cap_sites = 0, cap_tr = 0;
    int grid = 0;
    scl_site_row* d_rows = nullptr;
    RTask* d_rtask = nullptr;                  // reclaim pass re-check queue
    unsigned* d_rbits = nullptr; double* d_rlrate = nullptr; unsigned* d_rlsite = nullptr;   // a6 scratch
    unsigned* d_rsb = nullptr;                 // [n_sb + 1]: a6 superblock flag counts, then the flagged count
    unsigned n_sb = 0;
    unsigned nlaunch = 0;                      // kernels launched by the last run (+ its finalize)
    unsigned long long* d_P = nullptr;         // per-sample (alloc, managed) prefixes (NEXT-2, lazy)
    scl_sample_domain* d_dom = nullptr;
    size_t cap_dom = 0;
    bool dom_valid = false;
    unsigned long long* d_recon = nullptr;     // per-trace max reconstruction error (NEXT-4, lazy)
    size_t cap_recon = 0;
    bool recon_valid = false;
    // host
    std::vector<unsigned long long> h_sbase;
    std::vector<scl_trace_summary> h_summ;
    unsigned long long* h_gate = nullptr;      // pinned, written by the a6 kernel (gate sums)
    bool summ_valid = false;
    bool finalized = false;
    bool timed = false;                        // the last run recorded its phase events
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};   // run begin/end, finalize begin/end
    cudaEvent_t kev[3 * kRing] = {};           // per run (ring): replay kernel begin, its end, the end of the
                                               // stream pass's other kernels (cold_hist, pchain)
    uint64_t nrun = 0, nread = 0, nread_pass = 0;
    unsigned long long* d_prof = nullptr;     // SCL_PROFILE builds only
};

// ---------------------------------------------------------------- helpers
static bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// Validity of one host trace (reading Q16): frees match a live prior alloc of
// the same size, live pointers are unique.  Returns -1 or the first bad index.
static int64_t validate_trace(const scl_event* ev, uint64_t n) {
    std::unordered_map<uint64_t, uint64_t> live;
    live.reserve(1024);
    for (uint64_t i = 0; i < n; ++i) {
        const unsigned kind = ev_kind(ev[i].meta);
        if (kind == 2) continue;
        const uint64_t size = ev_size(ev[i].meta);
        if (kind == 0) {
            if (!live.emplace(ev[i].ptr, size).second) return (int64_t)i;
        } else {
            auto it = live.find(ev[i].ptr);
            if (it == live.end() || it->second != size) return (int64_t)i;
            live.erase(it);
        }
    }
    return -1;
}

static scl_status read_file(const char* path, std::vector<scl_event>& ev, std::vector<uint64_t>& off,
                            uint32_t& n_traces, uint32_t& n_sites, uint64_t& tick) {
    FILE* f = fopen(path, "rb");
    if (!f) return fail(SCL_EIO, std::string("cannot open ") + path);
    char magic[8]; uint32_t hdr[4]; uint64_t tk;
    bool ok = fread(magic, 1, 8, f) == 8 && memcmp(magic, "SCLTRC01", 8) == 0 &&
              fread(hdr, 4, 4, f) == 4 && fread(&tk, 8, 1, f) == 1 && hdr[0] == 1;
    if (ok) {
        n_traces = hdr[1]; n_sites = hdr[2]; tick = tk ? tk : 1000;
        off.resize((size_t)n_traces + 1);
        ok = fread(off.data(), 8, off.size(), f) == off.size() && off[0] == 0;
        for (uint32_t t = 0; ok && t < n_traces; ++t) ok = off[t] <= off[t + 1];
        if (ok) {
            ev.resize(off[n_traces]);
            ok = fread(ev.data(), sizeof(scl_event), ev.size(), f) == ev.size();
        }
    }
    fclose(f);
    if (!ok) return fail(SCL_EIO, std::string("malformed trace file ") + path);
    return SCL_OK;
}

// ---------------------------------------------------------------- load
template <class T> static bool grow(T*& p, size_t n) {
    cudaFree(p); p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) { cudaGetLastError(); p = nullptr; return false; }
    return true;
}

// Host offsets (from host or device memory) with their argument checks.
static scl_status read_offsets(const uint64_t* offsets, uint32_t n_traces, std::vector<uint64_t>& h_off) {
    h_off.resize((size_t)n_traces + 1);
    if (is_device_ptr(offsets)) CU(cudaMemcpy(h_off.data(), offsets, h_off.size() * 8, cudaMemcpyDeviceToHost));
    else memcpy(h_off.data(), offsets, h_off.size() * 8);
    if (h_off[0] != 0) return fail(SCL_EINVAL, "offsets[0] != 0");
    for (uint32_t t = 0; t < n_traces; ++t)
        if (h_off[t + 1] < h_off[t]) return fail(SCL_EINVAL, "offsets not non-decreasing at trace " + std::to_string(t));
    return SCL_OK;
}

static scl_status validate_host(const scl_event* src, bool src_dev, const std::vector<uint64_t>& h_off, uint32_t n_traces) {
    const uint64_t n = h_off[n_traces];
    if (n == 0) return SCL_OK;
    std::vector<scl_event> tmp;
    const scl_event* hv = src;
    if (src_dev) { tmp.resize(n); CU(cudaMemcpy(tmp.data(), src, n * sizeof(scl_event), cudaMemcpyDeviceToHost)); hv = tmp.data(); }
    for (uint32_t t = 0; t < n_traces; ++t) {
        int64_t bad = validate_trace(hv + h_off[t], h_off[t + 1] - h_off[t]);
        if (bad >= 0) return fail(SCL_ETRACE, "trace " + std::to_string(t) + " event " + std::to_string(bad) +
                                                  ": free of a non-live pointer, size mismatch or live pointer reused");
    }
    return SCL_OK;
}

// Site ids by frequency (n_sites > kHot): count the sites of a strided sample of up to 2^21 alloc /
// free events (host memory read in place, device memory through one strided copy), order the sites
// by (sampled count desc, id asc) and upload caller -> internal.  No remap when that order is the
// identity on the shared-memory table's range.  The remap is a permutation: every result is exact
// whatever it is; it only decides which sites take the fast Tier-E path.
static scl_status site_remap(scl_traces* tr, const scl_event* src, bool src_dev, uint64_t n, uint32_t n_sites,
                             cudaStream_t st, bool& changed)
{
    tr->remapped = false; tr->h_inv.clear(); changed = false;
    if (n_sites <= (uint32_t)kHot || n == 0) return SCL_OK;
    const uint64_t want = 1ull << 21, stride = std::max<uint64_t>(1, n / want), m = (n + stride - 1) / stride;
    std::vector<uint32_t> cnt(n_sites, 0);
    if (src_dev) {                                    // counted on the device, n_sites words back
        unsigned* d_cnt = nullptr;
        if (cudaMallocAsync(&d_cnt, (size_t)n_sites * 4, st) != cudaSuccess) { cudaGetLastError(); return SCL_OK; }
        CU(cudaMemsetAsync(d_cnt, 0, (size_t)n_sites * 4, st));
        CU(launch_site_sample(src, stride, m, n_sites, d_cnt, st));
        CU(cudaMemcpyAsync(cnt.data(), d_cnt, (size_t)n_sites * 4, cudaMemcpyDeviceToHost, st));
        CU(cudaFreeAsync(d_cnt, st));
        CU(cudaStreamSynchronize(st));
    } else {
        for (uint64_t i = 0; i < m; ++i) {
            const uint64_t meta = src[i * stride].meta;
            const uint32_t site = ev_site(meta);
            if (site < n_sites && ev_kind(meta) < 2) ++cnt[site];
        }
    }
    std::vector<uint32_t> order(n_sites);
    for (uint32_t i = 0; i < n_sites; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cnt[a] > cnt[b]; });
    // keep the caller's ids when the table's id range already holds (nearly) the sampled mass of the
    // hottest sites: a remap costs a permute of the table and an unfused a6 per run
    const uint32_t lim = std::min<uint32_t>(n_sites, (uint32_t)kWarm);
    uint64_t top = 0, low = 0;
    for (uint32_t i = 0; i < lim; ++i) { top += cnt[order[i]]; low += cnt[i]; }
    if (low * 100 >= top * 98) return SCL_OK;
    std::vector<uint32_t> remap(n_sites);
    for (uint32_t i = 0; i < n_sites; ++i) remap[order[i]] = i;
    cudaFree(tr->d_remap); tr->d_remap = nullptr;
    if (cudaMalloc(&tr->d_remap, (size_t)n_sites * 4) != cudaSuccess) { cudaGetLastError(); tr->d_remap = nullptr; return SCL_OK; }
    CU(cudaMemcpyAsync(tr->d_remap, remap.data(), (size_t)n_sites * 4, cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));                    // (remap is a local vector)
    tr->h_inv = std::move(order);
    tr->remapped = true; changed = true;
    return SCL_OK;
}

// Copy the events into the handle's device buffers (growing them if needed), run the load
// statistics and build the unit plan.  Stream-ordered on st; one synchronisation at the end
// (the host needs the per-trace sum |d| to size the sample buffer of each run).
static scl_status upload(scl_traces* tr, const scl_event* src, bool src_dev, std::vector<uint64_t>&& h_off,
                         uint32_t n_traces, uint32_t n_sites, cudaStream_t st)
{
    const uint64_t n = h_off[n_traces];
    {   // every trace needs a runner lane: n_traces <= grid * kEmbeddedRunners * 32
        int grid = 0;
        replay_occupancy(&grid);
        const uint64_t cap = (uint64_t)grid * kEmbeddedRunners * 32;
        if ((uint64_t)n_traces > cap)
            return fail(SCL_EOVERFLOW, "too many traces for one launch (max " + std::to_string(cap) +
                                       "): load them in waves");
    }
    const uint64_t rows_alloc = std::max<uint64_t>((n + 7) / 8, 1);
    // After a failed allocation the handle holds no traces (its buffers may already be replaced):
    // every count is 0 and earlier results are stale, so no later run reads freed memory.
    auto nomem = [&](const char* what) {
        tr->n_traces = 0; tr->n_events = 0; tr->n_segs = 0; tr->max_len = 0; tr->epoch += 1;
        return fail(SCL_ENOMEM, std::string("out of device memory: ") + what + " (the handle now holds no traces)");
    };
    // + kPadRows zeroed rows: a candidate chunk's lanes past the last event of the last trace
    // re-read up to 31 rows beyond it (load_row_global); they land here, not past the mapping.
    constexpr uint64_t kPadRows = 32;
    if (rows_alloc > tr->cap_rows) {
        cudaFree(tr->d_ev); tr->d_ev = nullptr; tr->cap_rows = 0;
        if (cudaMalloc(&tr->d_ev, (rows_alloc + kPadRows) * 128) != cudaSuccess) { cudaGetLastError(); tr->d_ev = nullptr; return nomem("events"); }
        tr->cap_rows = rows_alloc;
    }
    const size_t nt1 = std::max<uint32_t>(n_traces, 1);
    if (nt1 > tr->cap_tr) {
        tr->cap_tr = 0;
        if (!grow(tr->d_off, nt1 + 1) || !grow(tr->d_sabs, nt1) || !grow(tr->d_tr_nseg, nt1) ||
            !grow(tr->d_tr_base, nt1) || !grow(tr->d_run, nt1))
            return nomem("per-trace buffers");
        tr->cap_tr = nt1;
    }
    if (!tr->d_err) {
        if (!grow(tr->d_err, 65) || !grow(tr->d_ticket, 10)) { cudaFree(tr->d_err); tr->d_err = nullptr; return nomem("counters"); }
        // ticket[7] is the "run prepared" flag compared with the run's epoch: a fresh block may hold
        // a freed handle's epoch (fuzzing found producers starting before CTA 0 had prepared)
        CU(cudaMemsetAsync(tr->d_ticket, 0, 10 * sizeof(unsigned), st));
    }
    // A device source is copied by the statistics pass itself (one read of the source, one write to
    // HBM -- the events are not read back).  Host memory takes the DMA copy, then the statistics pass
    // reads the events from HBM: a zero-copy kernel reading pinned host memory measured 22 GB/s against
    // the DMA engine's ~50 GB/s, and the extra HBM pass costs < 1 % of the H2D time.
    const scl_event* csrc = n == 0 ? nullptr : src_dev ? src : nullptr;
    if (csrc && (reinterpret_cast<uintptr_t>(csrc) & 15u)) csrc = nullptr;
    if (n > 0 && !csrc) CU(cudaMemcpyAsync(tr->d_ev, src, n * sizeof(scl_event), src_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(tr->d_ev + n, 0, ((rows_alloc + kPadRows) * 8 - n) * sizeof(scl_event), st));
    CU(cudaMemcpyAsync(tr->d_off, h_off.data(), h_off.size() * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(tr->d_sabs, 0, nt1 * 8, st));
    CU(cudaMemsetAsync(tr->d_err, 0xff, 8, st));
    CU(cudaMemsetAsync(tr->d_err + 1, 0, 64 * 8, st));
    {
        bool changed = false;
        scl_status rs = site_remap(tr, src, src_dev, n, n_sites, st, changed);
        if (rs != SCL_OK) { tr->n_traces = 0; tr->n_events = 0; tr->n_segs = 0; return rs; }
    }
    CU(launch_load_stats(csrc ? csrc : tr->d_ev, tr->d_off, n_traces, n, n_sites, tr->d_sabs, tr->d_err,
                         csrc ? tr->d_ev : nullptr, tr->d_err + 1, tr->remapped ? tr->d_remap : nullptr, st));

    // unit plan (while the copy runs): unit k of trace t covers rows (off_t/8) + 1024k ...;
    // tickets ordered (k, t) so that one trace's units are spread over the run
    std::vector<uint32_t> nseg(n_traces), seg_base(n_traces);
    uint32_t total = 0, maxk = 0;
    uint64_t max_len = 0;
    for (uint32_t t = 0; t < n_traces; ++t) {
        const uint64_t a = h_off[t], b = h_off[t + 1];
        max_len = std::max<uint64_t>(max_len, b - a);
        uint32_t ns = 0;
        if (b > a) { uint64_t r = (b + 7) / 8 - a / 8; ns = (uint32_t)((r + kUnitRows - 1) / kUnitRows); }
        nseg[t] = ns; seg_base[t] = total; total += ns; maxk = std::max(maxk, ns);
    }
    std::vector<TicketInfo> tk;
    tk.reserve(total);
    for (uint32_t k = 0; k < maxk; ++k)
        for (uint32_t t = 0; t < n_traces; ++t)
            if (k < nseg[t]) {
                TicketInfo ti;
                ti.off_t = (long long)h_off[t]; ti.n_t = (long long)(h_off[t + 1] - h_off[t]);
                ti.t = t; ti.kraw = k | (k + 1 == nseg[t] ? 0x80000000u : 0u); ti.slot = seg_base[t] + k;
                const uint64_t row_base = h_off[t] / 8 + (uint64_t)k * kUnitRows;
                const uint64_t rows_left = (h_off[t + 1] + 7) / 8 - row_base;
                ti.nbox = (unsigned)std::min<uint64_t>((rows_left + kThreads - 1) / kThreads, kSub);
                tk.push_back(ti);
            }
    const size_t nn = std::max<size_t>(total, 1);
    if (nn > tr->cap_segs) {
        tr->cap_segs = 0;
        cudaFree(tr->d_urec); tr->d_urec = nullptr;
        if (!grow(tr->d_tk, nn) || !grow(tr->d_uagg, nn * 4) || !grow(tr->d_uent, nn) ||
            cudaMalloc(&tr->d_urec, nn * replay_urec_bytes()) != cudaSuccess)
            { cudaGetLastError(); tr->d_urec = nullptr; return nomem("unit plan"); }
        tr->cap_segs = nn;
    }
    // no aggregate word of an earlier trace set survives a (re)load: a unit index unused for a
    // while could otherwise hold a tag that a later run reuses (tags are the epoch's low 16 bits)
    CU(cudaMemsetAsync(tr->d_uagg, 0, tr->cap_segs * 32, st));
    if (total) CU(cudaMemcpyAsync(tr->d_tk, tk.data(), total * sizeof(TicketInfo), cudaMemcpyHostToDevice, st));
    if (n_traces) {
        CU(cudaMemcpyAsync(tr->d_tr_nseg, nseg.data(), n_traces * 4, cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(tr->d_tr_base, seg_base.data(), n_traces * 4, cudaMemcpyHostToDevice, st));
    }
    unsigned long long err = 0;
    tr->h_sabs.resize(n_traces);
    CU(cudaMemcpyAsync(&err, tr->d_err, 8, cudaMemcpyDeviceToHost, st));
    tr->h_shist.assign(64, 0);
    CU(cudaMemcpyAsync(tr->h_shist.data(), tr->d_err + 1, 64 * 8, cudaMemcpyDeviceToHost, st));
    if (n_traces) CU(cudaMemcpyAsync(tr->h_sabs.data(), tr->d_sabs, n_traces * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    tr->n_traces = n_traces; tr->n_sites = n_sites; tr->n_events = n; tr->max_len = max_len; tr->n_segs = total;
    tr->usum_valid = false;
    tr->h_off = std::move(h_off);
    if (err != ~0ull) {
        uint32_t t = (uint32_t)(std::upper_bound(tr->h_off.begin(), tr->h_off.end(), err) - tr->h_off.begin()) - 1;
        tr->n_traces = 0; tr->n_events = 0; tr->n_segs = 0;     // the handle holds no valid traces
        return fail(SCL_EINVAL, "trace " + std::to_string(t) + " event " + std::to_string(err - tr->h_off[t]) +
                                ": size 0, kind 3 or site >= n_sites");
    }

    // TMA descriptor: rows of 32 x u32 (128 B), box 32 x 256 rows, 128-B swizzle
    auto enc = get_encode();
    if (!enc) return fail(SCL_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t gdim[2] = {32, (cuuint64_t)rows_alloc};
    cuuint64_t gstride[1] = {128};
    cuuint32_t box[2] = {32, (cuuint32_t)kThreads};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&tr->tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void*)tr->d_ev, gdim, gstride, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(SCL_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
    return SCL_OK;
}

extern "C" scl_status scl_trace_load(const char* path, const scl_event* events, const uint64_t* offsets,
                                     uint32_t n_traces, uint32_t n_sites, int device, int validate,
                                     scl_traces** out)
{
    if (!out) return fail(SCL_EINVAL, "out is NULL");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { cudaGetLastError(); return fail(SCL_ECUDA, "no CUDA device"); }
    if (device < 0 || device >= ndev) return fail(SCL_EINVAL, "bad device ordinal");
    CU(cudaSetDevice(device));

    std::vector<scl_event> file_ev;
    std::vector<uint64_t> h_off;
    uint64_t tick = 1000;
    const scl_event* src = events;
    if (path) {
        scl_status st = read_file(path, file_ev, h_off, n_traces, n_sites, tick);
        if (st != SCL_OK) return st;
        src = file_ev.data();
    } else {
        if (!offsets || (n_traces > 0 && !events)) return fail(SCL_EINVAL, "events/offsets is NULL");
        scl_status st = read_offsets(offsets, n_traces, h_off);
        if (st != SCL_OK) return st;
    }
    if (n_sites == 0 || n_sites > (1u << 21)) return fail(SCL_EINVAL, "n_sites must be in 1..2^21");
    const uint64_t n = h_off[n_traces];
    const bool src_dev = n > 0 && !path && is_device_ptr(src);
    if (validate) { scl_status st = validate_host(src, src_dev, h_off, n_traces); if (st != SCL_OK) return st; }

    scl_traces* tr = new scl_traces();
    tr->device = device; tr->tick_ns = tick;
    scl_status st = upload(tr, src, src_dev, std::move(h_off), n_traces, n_sites, 0);
    if (st != SCL_OK) { scl_traces_free(tr); return st; }
    *out = tr;
    return SCL_OK;
}

extern "C" scl_status scl_trace_reload(scl_traces* tr, const scl_event* events, const uint64_t* offsets,
                                       uint32_t n_traces, uint32_t n_sites, int validate, void* cuda_stream)
{
    if (!tr || !offsets || (n_traces > 0 && !events)) return fail(SCL_EINVAL, "NULL argument");
    if (n_sites == 0 || n_sites > (1u << 21)) return fail(SCL_EINVAL, "n_sites must be in 1..2^21");
    CU(cudaSetDevice(tr->device));
    std::vector<uint64_t> h_off;
    scl_status st = read_offsets(offsets, n_traces, h_off);
    if (st != SCL_OK) return st;
    const uint64_t n = h_off[n_traces];
    const bool src_dev = n > 0 && is_device_ptr(events);
    if (validate) { st = validate_host(events, src_dev, h_off, n_traces); if (st != SCL_OK) return st; }
    tr->epoch += 1;                            // no earlier result is of this handle's stream pass any more
    return upload(tr, events, src_dev, std::move(h_off), n_traces, n_sites, (cudaStream_t)cuda_stream);
}

extern "C" void scl_traces_free(scl_traces* t) {
    if (!t) return;
    cudaFree(t->d_ev); cudaFree(t->d_off); cudaFree(t->d_sabs); cudaFree(t->d_tk); cudaFree(t->d_urec); cudaFree(t->d_uagg);
    cudaFree(t->d_tr_nseg); cudaFree(t->d_tr_base); cudaFree(t->d_run); cudaFree(t->d_uent); cudaFree(t->d_ticket);
    cudaFree(t->d_err); cudaFree(t->d_usum); cudaFree(t->d_ustart); cudaFree(t->d_ttot);
    cudaFree(t->d_crec); cudaFree(t->d_crec_fill); cudaFree(t->d_cctr); cudaFree(t->d_tierE); cudaFree(t->d_cpart);
    cudaFree(t->d_ust); cudaFree(t->d_sync); cudaFree(t->d_pc); cudaFree(t->d_pr); cudaFree(t->d_ul); cudaFree(t->d_remap);
    cudaFree(t->d_pscr); cudaFree(t->d_pnext); cudaFree(t->d_pctr);
    if (t->h_covf) cudaFreeHost(t->h_covf);
    delete t;
}

extern "C" scl_status scl_traces_info(const scl_traces* t, uint64_t* n_events, uint32_t* n_traces, uint32_t* n_sites) {
    if (!t) return fail(SCL_EINVAL, "NULL handle");
    if (n_events) *n_events = t->n_events;
    if (n_traces) *n_traces = t->n_traces;
    if (n_sites) *n_sites = t->n_sites;
    return SCL_OK;
}

// ---------------------------------------------------------------- run
static void free_result_buffers(scl_result* r) {
    if (r->d_table_int != r->d_table) cudaFree(r->d_table_int);
    r->d_table_int = nullptr;
    cudaFree(r->d_table); cudaFree(r->d_sbase); cudaFree(r->d_summ); cudaFree(r->d_rows);
    cudaFree(r->d_rbits); cudaFree(r->d_rsb);
    r->d_table = nullptr; r->d_sbase = nullptr; r->d_summ = nullptr; r->d_rows = nullptr;
    r->d_rbits = nullptr; r->d_rsb = nullptr;
    r->cap_sites = 0; r->cap_tr = 0;
}

extern "C" void scl_result_free(scl_result* r) {
    if (!r) return;
    free_result_buffers(r);
    cudaFree(r->d_samples); cudaFree(r->d_epflag); cudaFree(r->d_prof); cudaFree(r->d_rtask);
    cudaFree(r->d_rlrate); cudaFree(r->d_rlsite);
    cudaFree(r->d_P); cudaFree(r->d_dom); cudaFree(r->d_recon); cudaFree(r->d_el);
    if (r->h_gate) cudaFreeHost(r->h_gate);
    for (auto& e : r->ev) if (e) cudaEventDestroy(e);
    for (auto& e : r->kev) if (e) cudaEventDestroy(e);
    delete r;
}

// Per-site and per-trace buffers, sized for the handle (re-sized when a reloaded handle outgrows them).
static scl_status alloc_result(scl_result* r, const scl_traces* tr) {
    const size_t S = tr->n_sites, nt = std::max<uint32_t>(tr->n_traces, 1);
    if (!r->ev[0]) {
        for (auto& e : r->ev) CU(cudaEventCreate(&e));
        for (auto& e : r->kev) CU(cudaEventCreate(&e));
        CU(cudaMallocHost(&r->h_gate, 32));
        CU(cudaMalloc(&r->d_rtask, (size_t)kRTaskCap * sizeof(RTask)));
        CU(cudaMalloc(&r->d_rlrate, kReportList * 8)); CU(cudaMalloc(&r->d_rlsite, kReportList * 4));
        int grid = 0;
        replay_occupancy(&grid);
        r->grid = grid;
    }
    if (S <= r->cap_sites && nt <= r->cap_tr) return SCL_OK;
    free_result_buffers(r);
    CU(cudaMalloc(&r->d_table, (S * SCL_NCOL + 3) * 8));
    CU(cudaMalloc(&r->d_table_int, (S * SCL_NCOL + 3) * 8));
    CU(cudaMalloc(&r->d_sbase, nt * 8));
    CU(cudaMalloc(&r->d_summ, nt * sizeof(scl_trace_summary)));
    const size_t nwd = (std::max<size_t>(S, kReportSites) + 31) / 32;
    CU(cudaMalloc(&r->d_rbits, nwd * 4));
    r->n_sb = (unsigned)((nwd + kSuper - 1) / kSuper);
    CU(cudaMalloc(&r->d_rsb, (r->n_sb + 1) * 4));
    CU(cudaMalloc(&r->d_rows, S * sizeof(scl_site_row)));
    r->cap_sites = S; r->cap_tr = nt;
    return SCL_OK;
}

static FinalParams final_params(scl_result* r) {
    FinalParams f{};
    f.table = r->d_table; f.n_sites = r->tr->n_sites; f.formula = r->formula;
    f.elapsed_ns = (double)(r->elapsed_ns ? r->elapsed_ns : 1);
    f.gate_out = r->h_gate;                    // pinned host memory, device-accessible (unified addressing)
    f.prof = r->d_prof;
    return f;
}

// NCCL through the process's libnccl.so.2 (torch's, when loaded) or the system's, resolved once.
using AllReduceFn = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
static AllReduceFn nccl_allreduce() {
    static AllReduceFn fn = []() -> AllReduceFn {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        return h ? (AllReduceFn)dlsym(h, "ncclAllReduce") : nullptr;
    }();
    return fn;
}

// Cold-record pool of a stream pass (n_sites > kWarm): room for 5/16 of the events plus one partial
// chunk per compute warp; a pass that exhausts it is still exact (the rest of its cold events take
// the direct L2 path) and the next pass gets twice the room.  Best effort: no pool = all L2.
static void ensure_cold_pool(const scl_traces* tr) {
    if (tr->n_sites <= (uint32_t)kWarm) return;
    if (!tr->d_cctr) {
        if (cudaMalloc(&tr->d_cctr, 16) != cudaSuccess) { cudaGetLastError(); tr->d_cctr = nullptr; return; }
        cudaMemset(tr->d_cctr, 0, 16);
        if (cudaHostAlloc(&tr->h_covf, 8, cudaHostAllocMapped) != cudaSuccess) { cudaGetLastError(); tr->h_covf = nullptr; }
        else *tr->h_covf = 0;
    }
    {   // cold_hist's partial tables: one per CTA (R ranges x G groups <= max(SMs, R))
        int grid = 0;
        replay_occupancy(&grid);
        const size_t np = std::max<size_t>((size_t)grid, cold_ranges(tr->n_sites)) * 2 * kColdSites;
        if (np > tr->cap_cpart) {
            cudaFree(tr->d_cpart); tr->d_cpart = nullptr; tr->cap_cpart = 0;
            if (cudaMalloc(&tr->d_cpart, np * 4) != cudaSuccess) { cudaGetLastError(); tr->d_cpart = nullptr; }
            else tr->cap_cpart = np;
        }
    }
    const size_t rs = 8;
    unsigned long long want = tr->n_events / 16 * 5 + 4096ull * kRecChunk;
    if (tr->h_covf && *tr->h_covf) { want = std::max(want, 2 * tr->crec_cap); *tr->h_covf = 0; }
    want = std::min<unsigned long long>(want, tr->n_events + 4096ull * kRecChunk);
    want = (want + kRecChunk - 1) / kRecChunk * kRecChunk;
    if (want * rs <= tr->crec_bytes && want / kRecChunk <= tr->crec_fills) {   // (a reload may change the record size)
        tr->crec_cap = std::min<unsigned long long>(tr->crec_bytes / rs / kRecChunk, tr->crec_fills) * kRecChunk;
        return;
    }
    cudaFree(tr->d_crec); cudaFree(tr->d_crec_fill); tr->d_crec = nullptr; tr->d_crec_fill = nullptr;
    tr->crec_cap = 0; tr->crec_bytes = 0; tr->crec_fills = 0;
    if (cudaMalloc(&tr->d_crec, want * rs) != cudaSuccess ||
        cudaMalloc(&tr->d_crec_fill, want / kRecChunk * 4) != cudaSuccess) {
        cudaGetLastError(); cudaFree(tr->d_crec); tr->d_crec = nullptr; tr->d_crec_fill = nullptr; return;
    }
    tr->crec_cap = want; tr->crec_bytes = want * rs; tr->crec_fills = want / kRecChunk;
}

// SCL_CHAIN_AUTO: split the chains at sync events when the runners' sequential chains would outlast
// the stream pass they overlap AND the traces have enough sync events to cut them into many pieces.
// Chain estimate: the longest trace's sum|d| / T samples, about one in 16 of which survives the
// cancellation of allocs and frees in our workloads, at ~3 us per resolve; stream: ~5 TB/s of 16-B
// events; sync events per trace from the load-time log2-size histogram.  (Fitted on config 2 at
// T = 2^20 .. 10 MiB, 8 and 64 traces, config 3, config 5: profiles/r02_chain_split.txt.)
static bool split_pays(const scl_traces* tr, uint64_t T) {
    if (tr->n_traces == 0) return false;
    uint64_t smax = 0;
    for (uint32_t t = 0; t < tr->n_traces; ++t) smax = std::max<uint64_t>(smax, tr->h_sabs[t] / T);
    const double chain_us = (double)smax / 16.0 * 3.0;
    const double stream_us = (double)tr->n_events * 16.0 / 5.0e6;
    uint64_t sync = 0;                                 // events with size >= 2T - 1, about (whole log2 bins
    for (int k = 0; k < 64 && k < (int)tr->h_shist.size(); ++k)   //  from the one holding 2T - 1)
        if (k >= 62 || (2ull << k) > 2 * T - 1) sync += tr->h_shist[k];
    return chain_us > 2.0 * stream_us && (double)sync / tr->n_traces >= 32.0;
}

static scl_status replay_impl(uint64_t threshold, const scl_traces* tr, const scl_run_opts* opts, scl_result** out,
                              const scl_result* base)
{
    if (!tr || !out) return fail(SCL_EINVAL, "NULL argument");
    if (base && (base->tr != tr || base->epoch != tr->epoch || !base->epoch))
        return fail(SCL_EINVAL, "base is not a result of the handle's last stream pass");
    if (base && *out == base) return fail(SCL_EINVAL, "*out must not be the base result");
    if (threshold == 0) return fail(SCL_EINVAL, "threshold must be >= 1");
    if (threshold > (1ull << 62)) return fail(SCL_EINVAL, "threshold too large");
    scl_run_opts o{};
    if (opts) o = *opts;
    if (o.hwm_mode != SCL_HWM_PREFIX && o.hwm_mode != SCL_HWM_SAMPLE) return fail(SCL_EINVAL, "bad hwm_mode");
    if (o.formula != SCL_FORMULA_PAPER && o.formula != SCL_FORMULA_TEXTBOOK) return fail(SCL_EINVAL, "bad formula");
    CU(cudaSetDevice(tr->device));
    cudaStream_t st = (cudaStream_t)o.cuda_stream;

    scl_result* r = *out;
    const bool fresh = (r == nullptr);
    if (fresh) r = new scl_result();
    else if (r->tr != tr) return fail(SCL_EINVAL, "*out is a result of another traces handle");
    {
        scl_status s2 = alloc_result(r, tr);
        if (s2 != SCL_OK) { if (fresh) scl_result_free(r); return s2; }
    }
    r->tr = tr; r->T = threshold; r->formula = o.formula; r->stream = st;
    const uint64_t tick = o.tick_ns ? o.tick_ns : tr->tick_ns;
    r->elapsed_ns = o.elapsed_ns ? o.elapsed_ns : tr->max_len * tick;
    r->summ_valid = false; r->finalized = false; r->dom_valid = false; r->recon_valid = false;
    r->nlaunch = 0;

    // sample capacity per trace: min(n_t, floor(sum|d| / T)) -- every sample consumes |net| >= T
    // (CTA 0 of the replay kernel computes the same bases on the device; the host copy serves scl_samples)
    const uint32_t NT = tr->n_traces;
    unsigned long long tot = 0;
    r->h_sbase.resize((size_t)NT + 1);
    for (uint32_t t = 0; t < NT; ++t) {
        r->h_sbase[t] = tot;
        tot += std::min<uint64_t>(tr->h_off[t + 1] - tr->h_off[t], tr->h_sabs[t] / threshold);
    }
    r->h_sbase[NT] = tot;
    if (tot > r->cap || !r->d_samples) {
        cudaFree(r->d_samples); cudaFree(r->d_epflag);
        r->d_samples = nullptr; r->d_epflag = nullptr; r->cap = 0;
        const size_t c = std::max<size_t>(tot, 1);
        if (cudaMalloc(&r->d_samples, c * sizeof(scl_sample)) != cudaSuccess ||
            cudaMalloc(&r->d_epflag, c * 4) != cudaSuccess) { cudaGetLastError(); if (fresh) scl_result_free(r); return fail(SCL_ENOMEM, "samples"); }
        r->cap = c;
    }

    // epoch-tagged unit aggregate words: no per-run clear
    // (the aggregate words carry the low 16 bits: cleared, and tag 0 skipped, once per 2^16 runs)
    if (!base) {                               // a new stream pass (a re-threshold reads the last one)
        if (tr->epoch >= (1u << 30)) { tr->epoch = 0; tr->zc_arrivals = 0; CU(cudaMemsetAsync(tr->d_ticket, 0, 10 * 4, st)); }   // no stale "prepared"
        if (((tr->epoch + 1) & 0xffffu) == 0) { CU(cudaMemsetAsync(tr->d_uagg, 0, tr->cap_segs * 32, st)); tr->epoch += 1; }
        if (tr->epoch == 0) CU(cudaMemsetAsync(tr->d_uagg, 0, tr->cap_segs * 32, st));
        tr->epoch += 1;
    }
    r->epoch = tr->epoch;

    const bool tm = o.timing != 0;                 // phase / kernel events only when asked for
    r->timed = tm;
    if (tm) CU(cudaEventRecord(r->ev[0], st));

    ReplayParams p{};
    p.ev = tr->d_ev; p.off = tr->d_off; p.tk = tr->d_tk;
    p.urec = tr->d_urec; p.uagg = tr->d_uagg; p.run = tr->d_run; p.tr_nseg = tr->d_tr_nseg; p.tr_base = tr->d_tr_base;
    p.ticket = tr->d_ticket; p.n_segs = tr->n_segs; p.epoch = tr->epoch;
    p.n_runners = (unsigned)r->grid * kEmbeddedRunners;    // 2 runner warps in every CTA
    p.n_sites = tr->n_sites; p.n_traces = NT; p.T = (long long)threshold; p.hwm_sample = o.hwm_mode == SCL_HWM_SAMPLE;
    unsigned long long* tab = tr->remapped ? r->d_table_int : r->d_table;   // the kernels' table (internal ids)
    p.table = tab; p.samples = r->d_samples; p.ep_flag = r->d_epflag; p.sbase = r->d_sbase;
    p.sample_cap = r->cap;
    p.summ = r->d_summ; p.uent = tr->d_uent;
    if (!base) ensure_cold_pool(tr);
    p.crec = tr->d_crec; p.crec_cap = tr->crec_cap; p.cctr = tr->d_cctr; p.crec_fill = tr->d_crec_fill;
    p.cpart = tr->d_cpart;
    p.covf = tr->h_covf;

    if (tr->n_sites > tr->cap_tierE) {
        cudaFree(tr->d_tierE); tr->d_tierE = nullptr; tr->cap_tierE = 0;
        if (cudaMalloc(&tr->d_tierE, (size_t)tr->n_sites * 32) != cudaSuccess) { cudaGetLastError(); if (fresh) scl_result_free(r); return fail(SCL_ENOMEM, "tier E"); }
        tr->cap_tierE = tr->n_sites;
    }
    p.tierE = tr->d_tierE;
    if (o.chain_mode < SCL_CHAIN_AUTO || o.chain_mode > SCL_CHAIN_SPLIT) { if (fresh) scl_result_free(r); return fail(SCL_EINVAL, "bad chain_mode"); }
    const bool split = o.hwm_mode == SCL_HWM_PREFIX && tr->n_segs > 0 &&
                       (o.chain_mode == SCL_CHAIN_SPLIT || (o.chain_mode == SCL_CHAIN_AUTO && split_pays(tr, threshold)));
    if (split) {
        const size_t np = (size_t)tr->n_segs + tr->n_traces;
        if (np > tr->cap_pieces) {
            cudaFree(tr->d_ust); cudaFree(tr->d_sync); cudaFree(tr->d_pc); cudaFree(tr->d_pr); cudaFree(tr->d_ul);
            tr->d_ust = nullptr; tr->d_sync = nullptr; tr->d_pc = nullptr; tr->d_pr = nullptr; tr->d_ul = nullptr;
            tr->cap_pieces = 0;
            if (cudaMalloc(&tr->d_ust, np * sizeof(UnitStart)) != cudaSuccess || cudaMalloc(&tr->d_sync, np * sizeof(SyncInfo)) != cudaSuccess ||
                cudaMalloc(&tr->d_pc, np * sizeof(PieceCount)) != cudaSuccess || cudaMalloc(&tr->d_pr, np * sizeof(PieceRun)) != cudaSuccess ||
                cudaMalloc(&tr->d_ul, np * sizeof(UnitLocal)) != cudaSuccess)
                { cudaGetLastError(); if (fresh) scl_result_free(r); return fail(SCL_ENOMEM, "chain pieces"); }
            tr->cap_pieces = np;
        }
        // scratch: every piece's samples in blocks of kPBlock (at most the run's sample capacity
        // plus one partly filled block per piece)
        const size_t nb = (size_t)(tot + kPBlock - 1) / kPBlock + np + 1;
        if (nb > tr->cap_pblocks) {
            cudaFree(tr->d_pscr); cudaFree(tr->d_pnext); tr->d_pscr = nullptr; tr->d_pnext = nullptr; tr->cap_pblocks = 0;
            if (!tr->d_pctr && cudaMalloc(&tr->d_pctr, 8) != cudaSuccess) { cudaGetLastError(); tr->d_pctr = nullptr; }
            if (!tr->d_pctr || cudaMalloc(&tr->d_pscr, nb * kPBlock * sizeof(scl_sample)) != cudaSuccess ||
                cudaMalloc(&tr->d_pnext, nb * 4) != cudaSuccess)
                { cudaGetLastError(); if (fresh) scl_result_free(r); return fail(SCL_ENOMEM, "chain piece samples"); }
            tr->cap_pblocks = nb;
        }
        p.no_chain = 1; p.ust = tr->d_ust; p.sync = tr->d_sync; p.pc = tr->d_pc; p.pr = tr->d_pr; p.ul = tr->d_ul;
        p.pscr = tr->d_pscr; p.pnext = tr->d_pnext; p.pctr = tr->d_pctr; p.pblocks = (unsigned)std::min<size_t>(tr->cap_pblocks, 0xffffffffu);
    }
    PrepParams& pp = p.prep;                   // done by CTA 0 of the replay kernel
    pp.table = tab; pp.table_words = (size_t)tr->n_sites * SCL_NCOL + 3;
    pp.summ = reinterpret_cast<unsigned long long*>(r->d_summ); pp.summ_words = (size_t)NT * sizeof(scl_trace_summary) / 8;
    pp.run = reinterpret_cast<unsigned long long*>(tr->d_run); pp.run_words = (size_t)NT * sizeof(RunState) / 8;
    pp.ticket = tr->d_ticket; pp.sbase = r->d_sbase; pp.off = tr->d_off; pp.sabs = tr->d_sabs;
    pp.rsbcnt = r->d_rsb; pp.n_sb = r->n_sb;
    pp.n_traces = NT; pp.T = threshold; p.rtask = r->d_rtask; p.rtask_cap = kRTaskCap;
#ifdef SCL_PROFILE
    if (!r->d_prof) CU(cudaMalloc(&r->d_prof, (48 + 4 * (size_t)tr->cap_segs) * 8));
    CU(cudaMemsetAsync(r->d_prof, 0, (48 + 4 * (size_t)tr->n_segs) * 8, st));
    CU(cudaMemsetAsync(r->d_prof + 40, 0xff, 8, st));          // post pass start: atomicMin
    p.prof = r->d_prof;
#endif
    const int ks = (int)(r->nrun % kRing);
    if (tm) CU(cudaEventRecord(r->kev[3 * ks], st));
    if (tr->n_segs == 0 || base) {             // no replay launch: prepare here
        CU(cudaMemsetAsync(pp.table, 0, pp.table_words * 8, st));
        CU(cudaMemsetAsync(pp.summ, 0, pp.summ_words * 8, st));
        CU(cudaMemsetAsync(tr->d_ticket, 0, 7 * 4, st));
        CU(cudaMemsetAsync(r->d_rsb, 0, r->n_sb * 4, st));
        if (NT) CU(cudaMemcpyAsync(r->d_sbase, r->h_sbase.data(), (size_t)NT * 8, cudaMemcpyHostToDevice, st));
    }
    if (base) {                                // the per-event columns (Tier E) of the stream pass, as its
                                               // post pass kept them (base's own table may be reduced since)
        CU(cudaMemsetAsync(pp.run, 0, pp.run_words * 8, st));
        if (tr->n_sites)
            CU(cudaMemcpy2DAsync(tab, SCL_NCOL * 8, tr->d_tierE, 4 * 8, 4 * 8, tr->n_sites,
                                 cudaMemcpyDeviceToDevice, st));
        p.rechain = 1;
        p.n_runners = std::min<unsigned>(NT, (unsigned)r->grid * 8);
        if (split) { CU(launch_pchain(p, st)); r->nlaunch += 4; }
        else { CU(launch_rechain(p, st)); r->nlaunch += tr->n_segs ? 1 : 0; }
    } else {
        p.zc_target = tr->zc_arrivals + (uint32_t)r->grid;      // every CTA of every launch arrives once
        CU(launch_replay(&tr->tmap, p, r->grid, st));
        if (tr->n_segs) tr->zc_arrivals += (uint32_t)r->grid;
        if (tm) CU(cudaEventRecord(r->kev[3 * ks + 1], st));
        CU(launch_cold_hist(p, st));           // Tier E of the sites beyond the shared-memory table
        r->nlaunch += (tr->n_segs ? 1 : 0) + cold_hist_launches(p);
        if (split) { CU(launch_pchain(p, st)); r->nlaunch += 4; }
    }
    if (tm) {
        if (base) CU(cudaEventRecord(r->kev[3 * ks + 1], st));   // (no replay kernel: the re-chain)
        CU(cudaEventRecord(r->kev[3 * ks + 2], st));
        r->nrun += 1;
    }
    // a6 fused into the post pass when the run finalizes at once on a small table (not when the
    // table is first reduced across ranks)
    const bool reduce = o.nccl_comm != nullptr;
    const bool fuse = !o.defer_finalize && !reduce && !tr->remapped;   // (remapped: a6 after the permute)
    if (fuse) {
        p.fuse_report = 1; p.fin = final_params(r); p.rows = r->d_rows;
        p.rbits = r->d_rbits; p.rlrate = r->d_rlrate; p.rlsite = r->d_rlsite; p.rsbcnt = r->d_rsb;
    }
    CU(launch_post(p, st));
    r->nlaunch += 1;
    if (tr->remapped) {                        // the table in the caller's site order (a6, the all-reduce)
        CU(launch_permute_table(tab, r->d_table, tr->d_remap, tr->n_sites, st));
        r->nlaunch += 1;
    }
    if (tm) CU(cudaEventRecord(r->ev[1], st));
    if (fuse) {
        if (tm) CU(cudaEventRecord(r->ev[2], st));
        CU(cudaEventRecord(r->ev[3], st));
        r->finalized = true;
        *out = r;
        return SCL_OK;
    }
    *out = r;
    if (reduce) {                              // one int64 SUM all-reduce of the table
        AllReduceFn ar = nccl_allreduce();
        if (!ar) return fail(SCL_ENCCL, "libnccl.so.2 not found");
        ncclComm_t comm = (ncclComm_t)o.nccl_comm;
        if (ar(r->d_table, r->d_table, (size_t)tr->n_sites * SCL_NCOL + 3, ncclInt64, ncclSum, comm, st) != ncclSuccess)
            return fail(SCL_ENCCL, "ncclAllReduce (site table) failed");
        if (!o.elapsed_ns) {                   // Q11 over every rank's traces: MAX of max_t n_t * tick
            if (!r->d_el) CU(cudaMalloc(&r->d_el, 8));
            r->h_el = r->elapsed_ns;
            CU(cudaMemcpyAsync(r->d_el, &r->h_el, 8, cudaMemcpyHostToDevice, st));
            if (ar(r->d_el, r->d_el, 1, ncclUint64, ncclMax, comm, st) != ncclSuccess)
                return fail(SCL_ENCCL, "ncclAllReduce (elapsed) failed");
            CU(cudaMemcpyAsync(&r->h_el, r->d_el, 8, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            r->elapsed_ns = r->h_el;
        }
    }
    if (!o.defer_finalize) {
        scl_status s3 = scl_finalize(r, 0);
        if (s3 != SCL_OK) return s3;
    }
    return SCL_OK;
}

extern "C" scl_status scl_replay_run(uint64_t threshold, const scl_traces* tr, const scl_run_opts* opts, scl_result** out)
{
    return replay_impl(threshold, tr, opts, out, nullptr);
}

extern "C" scl_status scl_replay_rethreshold(uint64_t threshold, const scl_traces* tr, const scl_result* base,
                                             const scl_run_opts* opts, scl_result** out)
{
    if (!base) return fail(SCL_EINVAL, "NULL base");
    return replay_impl(threshold, tr, opts, out, base);
}

extern "C" scl_status scl_result_device_table(scl_result* r, int64_t** dev_ptr, size_t* n_int64) {
    if (!r || !dev_ptr || !n_int64) return fail(SCL_EINVAL, "NULL argument");
    *dev_ptr = (int64_t*)r->d_table;
    *n_int64 = (size_t)r->tr->n_sites * SCL_NCOL + 3;
    return SCL_OK;
}

extern "C" scl_status scl_finalize(scl_result* r, uint64_t elapsed_ns) {
    if (!r) return fail(SCL_EINVAL, "NULL result");
    const scl_traces* tr = r->tr;
    CU(cudaSetDevice(tr->device));
    cudaStream_t st = r->stream;
    if (elapsed_ns) r->elapsed_ns = elapsed_ns;
    const unsigned S = tr->n_sites;
    if (r->timed) CU(cudaEventRecord(r->ev[2], st));
    const FinalParams f = final_params(r);
    if (report_fused(S)) {
        CU(launch_report(f, r->d_rows, st));
        r->nlaunch += 1;
    } else {                                   // larger tables: the grid a6 of report.cuh in two kernels
        CU(cudaMemsetAsync(r->d_rsb, 0, (r->n_sb + 1) * 4, st));
        const ReportScratch x{r->d_rbits, r->d_rlrate, r->d_rlsite, r->d_rsb + r->n_sb, r->d_rsb};
        CU(launch_report_grid(f, x, r->d_rows, st));
        r->nlaunch += 2;
    }
    CU(cudaEventRecord(r->ev[3], st));
    r->finalized = true;
    return SCL_OK;
}

// ---------------------------------------------------------------- accessors (wait for the run)
static scl_status ensure_summ(const scl_result* rc) {
    scl_result* r = const_cast<scl_result*>(rc);
    if (r->summ_valid) return SCL_OK;
    const uint32_t NT = r->tr->n_traces;
    r->h_summ.resize(NT);
    if (NT) {
        CU(cudaMemcpyAsync(r->h_summ.data(), r->d_summ, NT * sizeof(scl_trace_summary), cudaMemcpyDeviceToHost, r->stream));
        CU(cudaStreamSynchronize(r->stream));
    }
    r->summ_valid = true;
    return SCL_OK;
}

extern "C" scl_status scl_site_report(const scl_result* r, scl_site_row* rows, size_t cap, size_t* n_rows) {
    if (!r || !n_rows) return fail(SCL_EINVAL, "NULL argument");
    if (!r->finalized) return fail(SCL_EINVAL, "result not finalized (call scl_finalize)");
    const size_t S = r->tr->n_sites;
    *n_rows = S;
    if (cap == 0) return SCL_OK;
    if (!rows) return fail(SCL_EINVAL, "rows is NULL");
    CU(cudaSetDevice(r->tr->device));
    CU(cudaMemcpyAsync(rows, r->d_rows, std::min(cap, S) * sizeof(scl_site_row), cudaMemcpyDeviceToHost, r->stream));
    CU(cudaStreamSynchronize(r->stream));
    return SCL_OK;
}

extern "C" scl_status scl_samples(const scl_result* r, uint32_t trace, scl_sample* out, size_t cap, size_t* n) {
    if (!r || !n) return fail(SCL_EINVAL, "NULL argument");
    if (trace >= r->tr->n_traces) return fail(SCL_EINVAL, "trace out of range");
    CU(cudaSetDevice(r->tr->device));
    scl_status s = ensure_summ(r);
    if (s != SCL_OK) return s;
    const size_t cnt = r->h_summ[trace].n_samples;
    *n = cnt;
    if (cap == 0 || cnt == 0) return SCL_OK;
    if (!out) return fail(SCL_EINVAL, "out is NULL");
    const size_t k = std::min(cap, cnt);
    CU(cudaMemcpyAsync(out, r->d_samples + r->h_sbase[trace], k * sizeof(scl_sample), cudaMemcpyDeviceToHost, r->stream));
    CU(cudaStreamSynchronize(r->stream));
    if (r->tr->remapped)                       // internal site ids -> the caller's
        for (size_t i = 0; i < k; ++i) out[i].site = r->tr->h_inv[out[i].site];
    return SCL_OK;
}

extern "C" scl_status scl_trace_summaries(const scl_result* r, scl_trace_summary* out, size_t cap, size_t* n) {
    if (!r || !n) return fail(SCL_EINVAL, "NULL argument");
    CU(cudaSetDevice(r->tr->device));
    scl_status s = ensure_summ(r);
    if (s != SCL_OK) return s;
    *n = r->tr->n_traces;
    if (cap == 0) return SCL_OK;
    if (!out) return fail(SCL_EINVAL, "out is NULL");
    memcpy(out, r->h_summ.data(), std::min(cap, (size_t)*n) * sizeof(scl_trace_summary));
    return SCL_OK;
}

extern "C" scl_status scl_trace_summary_of(const scl_result* r, uint32_t trace, int64_t* f_final, int64_t* hwm,
                                        uint64_t* n_samples, uint64_t* n_episodes) {
    if (!r) return fail(SCL_EINVAL, "NULL result");
    if (trace >= r->tr->n_traces) return fail(SCL_EINVAL, "trace out of range");
    CU(cudaSetDevice(r->tr->device));
    scl_status s = ensure_summ(r);
    if (s != SCL_OK) return s;
    const scl_trace_summary& m = r->h_summ[trace];
    if (f_final) *f_final = m.f_final;
    if (hwm) *hwm = m.hwm;
    if (n_samples) *n_samples = m.n_samples;
    if (n_episodes) *n_episodes = m.n_episodes;
    return SCL_OK;
}

extern "C" scl_status scl_gate(const scl_result* r, int64_t* num, int64_t* den, int* open) {
    if (!r) return fail(SCL_EINVAL, "NULL result");
    if (!r->finalized) return fail(SCL_EINVAL, "result not finalized");
    CU(cudaEventSynchronize(r->ev[3]));
    const long long gn = (long long)r->h_gate[0], gd = (long long)r->h_gate[1];
    if (num) *num = gn;
    if (den) *den = gd;
    if (open) *open = r->h_gate[2] > 0 && (__int128)100 * (__int128)gn >= (__int128)gd;
    return SCL_OK;
}

extern "C" scl_status scl_result_timing(const scl_result* r, float* replay_kernel_ms, float* run_ms, float* finalize_ms) {
    if (!r) return fail(SCL_EINVAL, "NULL result");
    float k = -1, a = -1, f = -1;
    if (r->timed) {
        CU(cudaEventSynchronize(r->finalized ? r->ev[3] : r->ev[1]));
        if (r->nrun) {
            const int ks = (int)((r->nrun - 1) % kRing);
            CU(cudaEventElapsedTime(&k, r->kev[3 * ks], r->kev[3 * ks + 1]));
        }
        CU(cudaEventElapsedTime(&a, r->ev[0], r->ev[1]));
        if (r->finalized) CU(cudaEventElapsedTime(&f, r->ev[2], r->ev[3]));
    }
    if (replay_kernel_ms) *replay_kernel_ms = k;
    if (run_ms) *run_ms = a;
    if (finalize_ms) *finalize_ms = f;
    return SCL_OK;
}

extern "C" scl_status scl_result_launches(const scl_result* r, uint32_t* n) {
    if (!r || !n) return fail(SCL_EINVAL, "NULL argument");
    *n = r->nlaunch;
    return SCL_OK;
}

// Durations (ms) of the runs enqueued since the previous read: the replay kernel (what = 0), or the
// whole stream pass -- the replay kernel and the kernels after it up to the post pass (what = 1).
static scl_status run_times(const scl_result* rc, int what, float* ms, size_t cap, size_t* n) {
    if (!rc || !n) return fail(SCL_EINVAL, "NULL argument");
    scl_result* r = const_cast<scl_result*>(rc);
    uint64_t& nread = what ? r->nread_pass : r->nread;
    const uint64_t avail = std::min<uint64_t>(r->nrun - nread, kRing);
    const uint64_t cnt = std::min<uint64_t>(avail, cap);
    *n = (size_t)cnt;
    if (cnt == 0) return SCL_OK;
    if (!ms) return fail(SCL_EINVAL, "ms is NULL");
    const uint64_t first = r->nrun - avail;
    for (uint64_t i = 0; i < cnt; ++i) {
        const int ks = (int)((first + i) % kRing);
        CU(cudaEventSynchronize(r->kev[3 * ks + 2]));
        CU(cudaEventElapsedTime(&ms[i], r->kev[3 * ks], r->kev[3 * ks + (what ? 2 : 1)]));
    }
    nread = r->nrun;
    return SCL_OK;
}

extern "C" scl_status scl_result_kernel_times(const scl_result* rc, float* ms, size_t cap, size_t* n) {
    return run_times(rc, 0, ms, cap, n);
}

extern "C" scl_status scl_result_pass_times(const scl_result* rc, float* ms, size_t cap, size_t* n) {
    return run_times(rc, 1, ms, cap, n);
}

#ifdef SCL_PROFILE
// Debug build only: per-role cycle sums of the last run (compute 0..7, producer 8..15, publisher + runners 16..23).
extern "C" scl_status scl_debug_prof(const scl_result* r, unsigned long long* out) {
    if (!r || !r->d_prof) return fail(SCL_EINVAL, "no profile");
    CU(cudaMemcpy(out, r->d_prof, (48 + 4 * (size_t)r->tr->n_segs) * 8, cudaMemcpyDeviceToHost));
    return SCL_OK;
}
#endif

// Per-unit alloc / free / copy / managed-alloc byte sums and their prefix within each trace (lazy,
// once per loaded traces; the rate sampler and the per-sample domain split use them).
static scl_status ensure_unit_sums(const scl_traces* tr, cudaStream_t st) {
    if (tr->usum_valid) return SCL_OK;
    const size_t nt1 = std::max<uint32_t>(tr->n_traces, 1), ns1 = std::max<uint32_t>(tr->n_segs, 1);
    if (ns1 > tr->cap_usum) {
        cudaFree(tr->d_usum); cudaFree(tr->d_ustart); tr->d_usum = tr->d_ustart = nullptr; tr->cap_usum = 0;
        CU(cudaMalloc(&tr->d_usum, ns1 * kUCols * 8)); CU(cudaMalloc(&tr->d_ustart, ns1 * kUCols * 8));
        tr->cap_usum = ns1;
    }
    if (nt1 > tr->cap_ttot) {
        cudaFree(tr->d_ttot); tr->d_ttot = nullptr; tr->cap_ttot = 0;
        CU(cudaMalloc(&tr->d_ttot, nt1 * kUCols * 8));
        tr->cap_ttot = nt1;
    }
    CU(cudaMemsetAsync(tr->d_ttot, 0, nt1 * kUCols * 8, st));
    CU(launch_unit_sums(tr->d_ev, tr->d_tk, tr->n_segs, tr->d_usum, tr->d_tr_base, tr->d_tr_nseg, tr->n_traces,
                        tr->d_ustart, tr->d_ttot, st));
    tr->usum_valid = true;
    return SCL_OK;
}

extern "C" scl_status scl_sample_domains(const scl_result* rc, uint32_t trace, scl_sample_domain* out, size_t cap, size_t* n) {
    if (!rc || !n) return fail(SCL_EINVAL, "NULL argument");
    scl_result* r = const_cast<scl_result*>(rc);
    const scl_traces* tr = r->tr;
    if (trace >= tr->n_traces) return fail(SCL_EINVAL, "trace out of range");
    CU(cudaSetDevice(tr->device));
    scl_status s = ensure_summ(r);
    if (s != SCL_OK) return s;
    if (!r->dom_valid) {
        s = ensure_unit_sums(tr, r->stream);
        if (s != SCL_OK) return s;
        if (r->cap_dom < r->cap || !r->d_dom) {
            cudaFree(r->d_P); cudaFree(r->d_dom); cudaFree(r->d_recon); r->d_P = nullptr; r->d_dom = nullptr; r->cap_dom = 0;
            if (cudaMalloc(&r->d_P, r->cap * 16) != cudaSuccess || cudaMalloc(&r->d_dom, r->cap * sizeof(scl_sample_domain)) != cudaSuccess)
                { cudaGetLastError(); return fail(SCL_ENOMEM, "sample domains"); }
            r->cap_dom = r->cap;
        }
        DomainParams p{};
        p.ev = tr->d_ev; p.tk = tr->d_tk; p.n_segs = tr->n_segs; p.n_traces = tr->n_traces; p.ustart = tr->d_ustart;
        p.samples = r->d_samples; p.sbase = r->d_sbase; p.summ = r->d_summ; p.P = r->d_P; p.dom = r->d_dom;
        CU(launch_domains(p, r->stream));
        r->dom_valid = true;
    }
    const size_t cnt = r->h_summ[trace].n_samples;
    *n = cnt;
    if (cap == 0 || cnt == 0) return SCL_OK;
    if (!out) return fail(SCL_EINVAL, "out is NULL");
    CU(cudaMemcpyAsync(out, r->d_dom + r->h_sbase[trace], std::min(cap, cnt) * sizeof(scl_sample_domain),
                       cudaMemcpyDeviceToHost, r->stream));
    CU(cudaStreamSynchronize(r->stream));
    return SCL_OK;
}

extern "C" scl_status scl_trace_recon_error(const scl_result* rc, uint64_t* err, size_t cap, size_t* n) {
    if (!rc || !n) return fail(SCL_EINVAL, "NULL argument");
    scl_result* r = const_cast<scl_result*>(rc);
    const scl_traces* tr = r->tr;
    *n = tr->n_traces;
    if (cap == 0) return SCL_OK;
    if (!err) return fail(SCL_EINVAL, "err is NULL");
    CU(cudaSetDevice(tr->device));
    if (!r->recon_valid) {
        scl_status s = ensure_unit_sums(tr, r->stream);
        if (s != SCL_OK) return s;
        const size_t nt1 = std::max<uint32_t>(tr->n_traces, 1);
        if (r->cap_recon < nt1) {
            cudaFree(r->d_recon); r->d_recon = nullptr; r->cap_recon = 0;
            if (cudaMalloc(&r->d_recon, nt1 * 8) != cudaSuccess) { cudaGetLastError(); return fail(SCL_ENOMEM, "recon"); }
            r->cap_recon = nt1;
        }
        CU(cudaMemsetAsync(r->d_recon, 0, nt1 * 8, r->stream));
        DomainParams p{};
        p.ev = tr->d_ev; p.tk = tr->d_tk; p.n_segs = tr->n_segs; p.n_traces = tr->n_traces; p.ustart = tr->d_ustart;
        p.samples = r->d_samples; p.sbase = r->d_sbase; p.summ = r->d_summ;
        CU(launch_recon(p, r->d_recon, r->stream));
        r->recon_valid = true;
    }
    CU(cudaMemcpyAsync(err, r->d_recon, std::min(cap, (size_t)*n) * 8, cudaMemcpyDeviceToHost, r->stream));
    CU(cudaStreamSynchronize(r->stream));
    return SCL_OK;
}

// ---------------------------------------------------------------- rate-based sampler (rate.cu)
struct scl_rate_result {
    const scl_traces* tr = nullptr;
    cudaStream_t st = nullptr;
    unsigned long long *d_count = nullptr, *d_sbase = nullptr, *d_S = nullptr, *d_site = nullptr, *d_kfirst = nullptr;
    scl_rate_sample* d_samples = nullptr;
    size_t cap = 0, cap_sites = 0, cap_tr = 0, cap_segs = 0;
    std::vector<unsigned long long> h_count, h_sbase;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

extern "C" void scl_rate_free(scl_rate_result* r) {
    if (!r) return;
    cudaFree(r->d_count); cudaFree(r->d_sbase); cudaFree(r->d_S); cudaFree(r->d_site); cudaFree(r->d_samples);
    cudaFree(r->d_kfirst);
    for (auto& e : r->ev) if (e) cudaEventDestroy(e);
    delete r;
}

extern "C" scl_status scl_rate_run(uint64_t R, uint64_t seed, unsigned kinds, const scl_traces* tr, void* cuda_stream,
                                   scl_rate_result** out)
{
    if (!tr || !out) return fail(SCL_EINVAL, "NULL argument");
    if (R == 0) return fail(SCL_EINVAL, "rate_bytes must be >= 1");
    if (kinds == 0 || (kinds & ~7u)) return fail(SCL_EINVAL, "kinds: a nonzero mask of 1 alloc, 2 free, 4 copy");
    CU(cudaSetDevice(tr->device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const uint32_t NT = tr->n_traces;
    const size_t nt1 = std::max<uint32_t>(NT, 1), ns1 = std::max<uint32_t>(tr->n_segs, 1);
    {
        scl_status s0 = ensure_unit_sums(tr, st);
        if (s0 != SCL_OK) return s0;
    }
    scl_rate_result* r = *out;
    const bool fresh = r == nullptr;
    if (fresh) {
        r = new scl_rate_result();
        for (auto& e : r->ev) if (cudaEventCreate(&e) != cudaSuccess) { scl_rate_free(r); return fail(SCL_ECUDA, "event"); }
    } else if (r->tr != tr) {
        return fail(SCL_EINVAL, "*out is a result of another traces handle");
    }
    r->tr = tr; r->st = st;
    auto fail_free = [&](scl_status s2, const std::string& m) { if (fresh) scl_rate_free(r); return fail(s2, m); };
    if (nt1 > r->cap_tr) {
        cudaFree(r->d_count); cudaFree(r->d_sbase); r->d_count = r->d_sbase = nullptr; r->cap_tr = 0;
        if (cudaMalloc(&r->d_count, nt1 * 8) != cudaSuccess || cudaMalloc(&r->d_sbase, nt1 * 8) != cudaSuccess)
            { cudaGetLastError(); return fail_free(SCL_ENOMEM, "rate counts"); }
        r->cap_tr = nt1;
    }
    if (ns1 > r->cap_segs) {
        cudaFree(r->d_kfirst); r->d_kfirst = nullptr; r->cap_segs = 0;
        if (cudaMalloc(&r->d_kfirst, ns1 * 8) != cudaSuccess) { cudaGetLastError(); return fail_free(SCL_ENOMEM, "rate ranges"); }
        r->cap_segs = ns1;
    }
    if (tr->n_sites > r->cap_sites) {
        cudaFree(r->d_site); r->d_site = nullptr; r->cap_sites = 0;
        if (cudaMalloc(&r->d_site, (size_t)tr->n_sites * 8) != cudaSuccess) { cudaGetLastError(); return fail_free(SCL_ENOMEM, "rate sites"); }
        r->cap_sites = tr->n_sites;
    }
    RateParams p{};
    p.ev = tr->d_ev; p.tk = tr->d_tk; p.n_segs = tr->n_segs; p.n_traces = NT; p.R = R; p.seed = seed; p.kinds = kinds;
    p.ttot = tr->d_ttot; p.ustart = tr->d_ustart; p.count = r->d_count; p.sbase = r->d_sbase; p.site_count = r->d_site;
    p.kfirst = r->d_kfirst;
    CU(cudaEventRecord(r->ev[0], st));
    CU(launch_rate(p, 0, st));                         // samples per trace
    CU(cudaEventRecord(r->ev[1], st));
    r->h_count.resize(NT); r->h_sbase.resize((size_t)NT + 1);
    if (NT) CU(cudaMemcpyAsync(r->h_count.data(), r->d_count, NT * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    unsigned long long tot = 0;
    for (uint32_t t = 0; t < NT; ++t) { r->h_sbase[t] = tot; tot += r->h_count[t]; }
    r->h_sbase[NT] = tot;
    if (tot > (1ull << 32)) return fail_free(SCL_EOVERFLOW, "more than 2^32 rate samples: raise rate_bytes");
    if (tot > r->cap || !r->d_S) {
        cudaFree(r->d_S); cudaFree(r->d_samples); r->d_S = nullptr; r->d_samples = nullptr; r->cap = 0;
        const size_t c = std::max<unsigned long long>(tot, 1);
        if (cudaMalloc(&r->d_S, c * 8) != cudaSuccess || cudaMalloc(&r->d_samples, c * sizeof(scl_rate_sample)) != cudaSuccess)
            { cudaGetLastError(); return fail_free(SCL_ENOMEM, "rate samples"); }
        r->cap = c;
    }
    p.S = r->d_S; p.samples = r->d_samples;
    if (NT) CU(cudaMemcpyAsync(r->d_sbase, r->h_sbase.data(), NT * 8, cudaMemcpyHostToDevice, st));
    CU(cudaEventRecord(r->ev[2], st));
    CU(cudaMemsetAsync(r->d_site, 0, (size_t)tr->n_sites * 8, st));
    CU(launch_rate(p, 1, st));                         // S_k
    CU(launch_rate(p, 2, st));                         // placement
    CU(cudaEventRecord(r->ev[3], st));
    *out = r;
    return SCL_OK;
}

extern "C" scl_status scl_rate_counts(const scl_rate_result* r, uint64_t* counts, size_t cap, size_t* n) {
    if (!r || !n) return fail(SCL_EINVAL, "NULL argument");
    *n = r->h_count.size();
    if (cap == 0) return SCL_OK;
    if (!counts) return fail(SCL_EINVAL, "counts is NULL");
    memcpy(counts, r->h_count.data(), std::min(cap, *n) * 8);
    return SCL_OK;
}

extern "C" scl_status scl_rate_samples(const scl_rate_result* r, uint32_t trace, scl_rate_sample* out, size_t cap, size_t* n) {
    if (!r || !n) return fail(SCL_EINVAL, "NULL argument");
    if (trace >= r->h_count.size()) return fail(SCL_EINVAL, "trace out of range");
    *n = r->h_count[trace];
    if (cap == 0 || *n == 0) return SCL_OK;
    if (!out) return fail(SCL_EINVAL, "out is NULL");
    CU(cudaSetDevice(r->tr->device));
    const size_t k = std::min(cap, (size_t)*n);
    CU(cudaMemcpyAsync(out, r->d_samples + r->h_sbase[trace], k * sizeof(scl_rate_sample), cudaMemcpyDeviceToHost, r->st));
    CU(cudaStreamSynchronize(r->st));
    if (r->tr->remapped)                       // internal site ids -> the caller's
        for (size_t i = 0; i < k; ++i) out[i].site = r->tr->h_inv[out[i].site];
    return SCL_OK;
}

extern "C" scl_status scl_rate_site_counts(const scl_rate_result* r, uint64_t* counts, size_t cap, size_t* n) {
    if (!r || !n) return fail(SCL_EINVAL, "NULL argument");
    *n = r->tr->n_sites;
    if (cap == 0) return SCL_OK;
    if (!counts) return fail(SCL_EINVAL, "counts is NULL");
    CU(cudaSetDevice(r->tr->device));
    if (r->tr->remapped) {                     // per internal site -> per caller site
        std::vector<uint64_t> tmp(*n);
        CU(cudaMemcpyAsync(tmp.data(), r->d_site, *n * 8, cudaMemcpyDeviceToHost, r->st));
        CU(cudaStreamSynchronize(r->st));
        for (size_t i = 0; i < *n; ++i) if (r->tr->h_inv[i] < cap) counts[r->tr->h_inv[i]] = tmp[i];
        return SCL_OK;
    }
    CU(cudaMemcpyAsync(counts, r->d_site, std::min(cap, *n) * 8, cudaMemcpyDeviceToHost, r->st));
    CU(cudaStreamSynchronize(r->st));
    return SCL_OK;
}

extern "C" scl_status scl_rate_timing(const scl_rate_result* r, float* ms) {
    if (!r || !ms) return fail(SCL_EINVAL, "NULL argument");
    CU(cudaEventSynchronize(r->ev[3]));
    float a = 0, b = 0;
    CU(cudaEventElapsedTime(&a, r->ev[0], r->ev[1]));
    CU(cudaEventElapsedTime(&b, r->ev[2], r->ev[3]));
    *ms = a + b;
    return SCL_OK;
}

// "a prime number slightly above 10MB" -- smallest prime >= base (trial division)
extern "C" uint64_t scl_next_prime(uint64_t base) {
    for (uint64_t x = base < 2 ? 2 : base;; ++x) {
        bool prime = true;
        for (uint64_t q = 2; q * q <= x; ++q) if (x % q == 0) { prime = false; break; }
        if (prime) return x;
    }
}
