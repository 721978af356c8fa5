// api.cu -- host side of the C-ABI declared in include/scl.h.
//
// Owns the device copies of the traces (padded to whole 128-B rows so that a
// 2-D TMA tensor map with the 128-byte swizzle can stage 2048-event segments),
// the segment plan (ticket order interleaves traces so that one trace's
// segments are spread over time and its look-back chain rarely waits), and
// the per-run result buffers.  Every compute step runs in the kernels of
// replay.cu; this file only plans, allocates, launches and copies.
#include "scl_internal.cuh"
#include <cudaTypedefs.h>
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <unordered_map>
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
    scl_event* d_ev = nullptr;                 // padded_rows * 8 events
    unsigned long long* d_off = nullptr;       // n_traces + 1
    std::vector<uint64_t> h_off, h_sabs;
    uint32_t n_segs = 0;
    TicketInfo* d_tk = nullptr;
    void* d_urec = nullptr;                    // per unit: published summary record
    unsigned int* d_uready = nullptr;          // per unit: run epoch when published
    unsigned int* d_tr_nseg = nullptr;         // per trace: number of units
    unsigned int* d_tr_base = nullptr;         // per trace: first unit id
    RunState* d_run = nullptr;                 // per trace: runner state (zeroed per run)
    UnitEntry* d_uent = nullptr;               // per unit: state entering it (runner -> reclaim pass)
    unsigned int* d_ticket = nullptr;
    mutable unsigned int epoch = 0;
    CUtensorMap tmap;
};

struct scl_result {
    const scl_traces* tr = nullptr;
    uint64_t T = 0;
    int formula = 0;
    uint64_t elapsed_ns = 0;
    cudaStream_t stream = nullptr;
    // device
    unsigned long long* d_table = nullptr;     // n_sites*NCOL + 3
    scl_sample* d_samples = nullptr; unsigned int* d_epflag = nullptr; size_t cap = 0;
    unsigned long long* d_sbase = nullptr;
    scl_trace_summary* d_summ = nullptr;
    int grid = 0;
    double* d_prob = nullptr; double* d_rate = nullptr; unsigned char* d_flag = nullptr;
    unsigned long long *d_key = nullptr, *d_key2 = nullptr; unsigned int *d_val = nullptr, *d_order = nullptr;
    void* d_cub = nullptr; size_t cub_bytes = 0;
    scl_site_row* d_rows = nullptr;
    // host
    std::vector<unsigned long long> h_sbase;
    std::vector<scl_trace_summary> h_summ;
    bool summ_valid = false;
    long long gate_num = 0, gate_den = 0; unsigned long long gate_cnt = 0;
    bool finalized = false;
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    float kern_ms = 0;
    unsigned long long* d_prof = nullptr;     // SCL_PROFILE builds only
    float run_ms = 0, fin_ms = 0;
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
        h_off.resize((size_t)n_traces + 1);
        if (is_device_ptr(offsets)) CU(cudaMemcpy(h_off.data(), offsets, h_off.size() * 8, cudaMemcpyDeviceToHost));
        else memcpy(h_off.data(), offsets, h_off.size() * 8);
        if (h_off[0] != 0) return fail(SCL_EINVAL, "offsets[0] != 0");
        for (uint32_t t = 0; t < n_traces; ++t)
            if (h_off[t + 1] < h_off[t]) return fail(SCL_EINVAL, "offsets not non-decreasing at trace " + std::to_string(t));
    }
    if (n_sites == 0 || n_sites > (1u << 21)) return fail(SCL_EINVAL, "n_sites must be in 1..2^21");
    const uint64_t n = h_off[n_traces];
    const bool src_dev = n > 0 && !path && is_device_ptr(src);

    if (validate && n > 0) {
        std::vector<scl_event> tmp;
        const scl_event* hv = src;
        if (src_dev) { tmp.resize(n); CU(cudaMemcpy(tmp.data(), src, n * sizeof(scl_event), cudaMemcpyDeviceToHost)); hv = tmp.data(); }
        for (uint32_t t = 0; t < n_traces; ++t) {
            int64_t bad = validate_trace(hv + h_off[t], h_off[t + 1] - h_off[t]);
            if (bad >= 0) return fail(SCL_ETRACE, "trace " + std::to_string(t) + " event " + std::to_string(bad) +
                                                      ": free of a non-live pointer, size mismatch or live pointer reused");
        }
    }

    scl_traces* tr = new scl_traces();
    tr->device = device; tr->n_traces = n_traces; tr->n_sites = n_sites; tr->n_events = n; tr->tick_ns = tick;
    tr->h_off = h_off;
    auto cleanup = [&](scl_status st) { scl_traces_free(tr); return st; };

    const uint64_t rows = (n + 7) / 8;
    const uint64_t rows_alloc = rows > 0 ? rows : 1;
    if (cudaMalloc(&tr->d_ev, rows_alloc * 128) != cudaSuccess) { cudaGetLastError(); return cleanup(fail(SCL_ENOMEM, "events")); }
    if (n > 0 && cudaMemcpy(tr->d_ev, src, n * sizeof(scl_event), src_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice) != cudaSuccess)
        return cleanup(fail(SCL_ECUDA, "event copy failed"));
    if (rows_alloc * 8 > n && cudaMemset(tr->d_ev + n, 0, (rows_alloc * 8 - n) * sizeof(scl_event)) != cudaSuccess)
        return cleanup(fail(SCL_ECUDA, "pad"));
    if (cudaMalloc(&tr->d_off, h_off.size() * 8) != cudaSuccess) return cleanup(fail(SCL_ENOMEM, "offsets"));
    if (cudaMemcpy(tr->d_off, h_off.data(), h_off.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) return cleanup(fail(SCL_ECUDA, "off copy"));

    // per-trace sum |d| (sample capacity bound) and argument check, on the device
    unsigned long long *d_sabs = nullptr, *d_err = nullptr;
    if (cudaMalloc(&d_sabs, std::max<size_t>(n_traces, 1) * 8) != cudaSuccess || cudaMalloc(&d_err, 8) != cudaSuccess)
        { cudaFree(d_sabs); return cleanup(fail(SCL_ENOMEM, "stats")); }
    cudaMemset(d_err, 0xff, 8);
    launch_load_stats(tr->d_ev, tr->d_off, n_traces, n_sites, d_sabs, d_err, 0);
    unsigned long long err = 0;
    tr->h_sabs.resize(n_traces);
    cudaError_t ce = cudaMemcpy(&err, d_err, 8, cudaMemcpyDeviceToHost);
    if (ce == cudaSuccess && n_traces) ce = cudaMemcpy(tr->h_sabs.data(), d_sabs, n_traces * 8, cudaMemcpyDeviceToHost);
    cudaFree(d_sabs); cudaFree(d_err);
    if (ce != cudaSuccess) return cleanup(fail(SCL_ECUDA, std::string("load stats: ") + cudaGetErrorString(ce)));
    if (err != ~0ull) {
        uint32_t t = (uint32_t)(std::upper_bound(h_off.begin(), h_off.end(), err) - h_off.begin()) - 1;
        return cleanup(fail(SCL_EINVAL, "trace " + std::to_string(t) + " event " + std::to_string(err - h_off[t]) +
                                        ": size 0, kind 3 or site >= n_sites"));
    }

    // segment plan: segment k of trace t covers rows (off_t/8) + 256k ... ; tickets ordered (k, t)
    std::vector<uint32_t> nseg(n_traces), seg_base(n_traces);
    uint32_t total = 0, maxk = 0;
    for (uint32_t t = 0; t < n_traces; ++t) {
        const uint64_t a = h_off[t], b = h_off[t + 1];
        tr->max_len = std::max<uint64_t>(tr->max_len, b - a);
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
    tr->n_segs = total;
    const size_t nn = std::max<size_t>(total, 1);
    if (cudaMalloc(&tr->d_tk, nn * sizeof(TicketInfo)) != cudaSuccess ||
        cudaMalloc(&tr->d_urec, nn * replay_urec_bytes()) != cudaSuccess || cudaMalloc(&tr->d_uready, nn * 4) != cudaSuccess ||
        cudaMalloc(&tr->d_tr_nseg, std::max<size_t>(n_traces, 1) * 4) != cudaSuccess ||
        cudaMalloc(&tr->d_tr_base, std::max<size_t>(n_traces, 1) * 4) != cudaSuccess ||
        cudaMalloc(&tr->d_run, std::max<size_t>(n_traces, 1) * sizeof(RunState)) != cudaSuccess ||
        cudaMalloc(&tr->d_uent, nn * sizeof(UnitEntry)) != cudaSuccess ||
        cudaMalloc(&tr->d_ticket, 4) != cudaSuccess)
        { cudaGetLastError(); return cleanup(fail(SCL_ENOMEM, "segment plan")); }
    if (total) cudaMemcpy(tr->d_tk, tk.data(), total * sizeof(TicketInfo), cudaMemcpyHostToDevice);
    cudaMemset(tr->d_uready, 0, nn * 4);
    {   // every trace needs a runner lane: n_traces <= grid * kRunners * 32
        int grid = 0;
        replay_occupancy(&grid);
        if ((uint64_t)n_traces > (uint64_t)grid * kRunners * 32)
            return cleanup(fail(SCL_EOVERFLOW, "too many traces for one launch (max " +
                                std::to_string((uint64_t)grid * kRunners * 32) + "): load them in waves"));
    }
    if (n_traces) {
        cudaMemcpy(tr->d_tr_nseg, nseg.data(), n_traces * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(tr->d_tr_base, seg_base.data(), n_traces * 4, cudaMemcpyHostToDevice);
    }

    // TMA descriptor: rows of 32 x u32 (128 B), box 32 x 256 rows, 128-B swizzle
    auto enc = get_encode();
    if (!enc) return cleanup(fail(SCL_ECUDA, "cuTensorMapEncodeTiled unavailable"));
    cuuint64_t gdim[2] = {32, (cuuint64_t)rows_alloc};
    cuuint64_t gstride[1] = {128};
    cuuint32_t box[2] = {32, (cuuint32_t)kThreads};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&tr->tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void*)tr->d_ev, gdim, gstride, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cleanup(fail(SCL_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr)));
    if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(fail(SCL_ECUDA, "load sync"));
    *out = tr;
    return SCL_OK;
}

extern "C" void scl_traces_free(scl_traces* t) {
    if (!t) return;
    cudaFree(t->d_ev); cudaFree(t->d_off); cudaFree(t->d_tk); cudaFree(t->d_urec); cudaFree(t->d_uready);
    cudaFree(t->d_tr_nseg); cudaFree(t->d_tr_base); cudaFree(t->d_run); cudaFree(t->d_uent); cudaFree(t->d_ticket);
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
extern "C" void scl_result_free(scl_result* r) {
    if (!r) return;
    cudaFree(r->d_table); cudaFree(r->d_samples); cudaFree(r->d_epflag); cudaFree(r->d_sbase);
    cudaFree(r->d_summ); cudaFree(r->d_prob); cudaFree(r->d_rate); cudaFree(r->d_flag);
    cudaFree(r->d_prof); cudaFree(r->d_key); cudaFree(r->d_key2); cudaFree(r->d_val); cudaFree(r->d_order); cudaFree(r->d_cub); cudaFree(r->d_rows);
    for (auto& e : r->ev) if (e) cudaEventDestroy(e);
    delete r;
}

static scl_status alloc_result(scl_result* r, const scl_traces* tr) {
    const size_t S = tr->n_sites, nt = std::max<uint32_t>(tr->n_traces, 1);
    int grid = 0;
    replay_occupancy(&grid);
    r->grid = grid;
    CU(cudaMalloc(&r->d_table, (S * SCL_NCOL + 3) * 8));
    CU(cudaMalloc(&r->d_sbase, nt * 8));
    CU(cudaMalloc(&r->d_summ, nt * sizeof(scl_trace_summary)));
    CU(cudaMalloc(&r->d_prob, S * 8)); CU(cudaMalloc(&r->d_rate, S * 8)); CU(cudaMalloc(&r->d_flag, S));
    CU(cudaMalloc(&r->d_key, S * 8)); CU(cudaMalloc(&r->d_key2, S * 8));
    CU(cudaMalloc(&r->d_val, S * 4)); CU(cudaMalloc(&r->d_order, S * 4));
    CU(cudaMalloc(&r->d_rows, S * sizeof(scl_site_row)));
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, r->d_key, r->d_key2, r->d_val, r->d_order, (int)S);
    r->cub_bytes = std::max<size_t>(tb, 1);
    CU(cudaMalloc(&r->d_cub, r->cub_bytes));
    for (auto& e : r->ev) CU(cudaEventCreate(&e));
    r->h_sbase.resize(nt + 1);
    return SCL_OK;
}

extern "C" scl_status scl_replay_run(uint64_t threshold, const scl_traces* tr, const scl_run_opts* opts, scl_result** out)
{
    if (!tr || !out) return fail(SCL_EINVAL, "NULL argument");
    if (threshold == 0) return fail(SCL_EINVAL, "threshold must be >= 1");
    if (threshold > (1ull << 62)) return fail(SCL_EINVAL, "threshold too large");
    scl_run_opts o{};
    if (opts) o = *opts;
    if (o.hwm_mode != SCL_HWM_PREFIX) return fail(SCL_EINVAL, "only hwm_mode PREFIX is implemented on the GPU");
    if (o.formula != SCL_FORMULA_PAPER && o.formula != SCL_FORMULA_TEXTBOOK) return fail(SCL_EINVAL, "bad formula");
    CU(cudaSetDevice(tr->device));
    cudaStream_t st = (cudaStream_t)o.cuda_stream;

    scl_result* r = *out;
    const bool fresh = (r == nullptr);
    if (fresh) {
        r = new scl_result();
        scl_status s2 = alloc_result(r, tr);
        if (s2 != SCL_OK) { scl_result_free(r); return s2; }
    } else if (r->tr != tr) {
        return fail(SCL_EINVAL, "*out is a result of another traces handle");
    }
    r->tr = tr; r->T = threshold; r->formula = o.formula; r->stream = st;
    const uint64_t tick = o.tick_ns ? o.tick_ns : tr->tick_ns;
    r->elapsed_ns = o.elapsed_ns ? o.elapsed_ns : tr->max_len * tick;
    r->summ_valid = false; r->finalized = false;

    // sample capacity per trace: min(n_t, floor(sum|d| / T)) -- every sample consumes |net| >= T
    const uint32_t NT = tr->n_traces;
    unsigned long long tot = 0;
    for (uint32_t t = 0; t < NT; ++t) {
        r->h_sbase[t] = tot;
        tot += std::min<uint64_t>(tr->h_off[t + 1] - tr->h_off[t], tr->h_sabs[t] / threshold);
    }
    r->h_sbase[NT] = tot;
    if (tot > r->cap || !r->d_samples) {
        cudaFree(r->d_samples); cudaFree(r->d_epflag);
        r->d_samples = nullptr; r->d_epflag = nullptr;
        const size_t c = std::max<size_t>(tot, 1);
        if (cudaMalloc(&r->d_samples, c * sizeof(scl_sample)) != cudaSuccess ||
            cudaMalloc(&r->d_epflag, c * 4) != cudaSuccess) { cudaGetLastError(); if (fresh) scl_result_free(r); return fail(SCL_ENOMEM, "samples"); }
        r->cap = c;
    }

    // epoch-tagged look-back flags: no per-run clear of the state array
    if (tr->epoch >= (1u << 30)) { CU(cudaMemsetAsync(tr->d_uready, 0, (size_t)std::max<uint32_t>(tr->n_segs, 1) * 4, st)); tr->epoch = 0; }
    tr->epoch += 1;

    CU(cudaEventRecord(r->ev[0], st));
    CU(cudaMemcpyAsync(r->d_sbase, r->h_sbase.data(), (size_t)std::max<uint32_t>(NT, 1) * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(r->d_table, 0, ((size_t)tr->n_sites * SCL_NCOL + 3) * 8, st));
    CU(cudaMemsetAsync(r->d_summ, 0, (size_t)std::max<uint32_t>(NT, 1) * sizeof(scl_trace_summary), st));
    CU(cudaMemsetAsync(tr->d_ticket, 0, 4, st));
    CU(cudaMemsetAsync(tr->d_run, 0, (size_t)std::max<uint32_t>(NT, 1) * sizeof(RunState), st));

    ReplayParams p{};
    p.ev = tr->d_ev; p.off = tr->d_off; p.tk = tr->d_tk;
    p.urec = tr->d_urec; p.uready = tr->d_uready; p.run = tr->d_run; p.tr_nseg = tr->d_tr_nseg; p.tr_base = tr->d_tr_base;
    p.ticket = tr->d_ticket; p.n_segs = tr->n_segs; p.epoch = tr->epoch;
    p.n_sites = tr->n_sites; p.n_traces = NT; p.T = (long long)threshold;
    p.table = r->d_table; p.samples = r->d_samples; p.ep_flag = r->d_epflag; p.sbase = r->d_sbase;
    p.summ = r->d_summ; p.uent = tr->d_uent;
#ifdef SCL_PROFILE
    if (!r->d_prof) CU(cudaMalloc(&r->d_prof, (48 + 4 * (size_t)tr->n_segs) * 8));
    CU(cudaMemsetAsync(r->d_prof, 0, (48 + 4 * (size_t)tr->n_segs) * 8, st));
    p.prof = r->d_prof;
#endif
    CU(cudaEventRecord(r->ev[4], st));
    CU(launch_replay(&tr->tmap, p, r->grid, st));
    CU(cudaEventRecord(r->ev[5], st));
    CU(launch_reclaim(p, st));
    CU(launch_samples(p, st));
    CU(cudaEventRecord(r->ev[1], st));
    *out = r;
    if (!o.defer_finalize) {
        scl_status s3 = scl_finalize(r, 0);
        if (s3 != SCL_OK) return s3;
    } else {
        CU(cudaStreamSynchronize(st));
        cudaEventElapsedTime(&r->run_ms, r->ev[0], r->ev[1]);
        cudaEventElapsedTime(&r->kern_ms, r->ev[4], r->ev[5]);
    }
    return SCL_OK;
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
    CU(cudaEventRecord(r->ev[2], st));
    FinalParams f{};
    f.table = r->d_table; f.n_sites = S; f.formula = r->formula;
    f.elapsed_ns = (double)(r->elapsed_ns ? r->elapsed_ns : 1);
    f.prob = r->d_prob; f.rate = r->d_rate; f.flag = r->d_flag; f.key1 = r->d_key; f.val = r->d_val;
    CU(launch_finalize(f, st));
    size_t tb = r->cub_bytes;
    CU(cub::DeviceRadixSort::SortPairs(r->d_cub, tb, r->d_key, r->d_key2, r->d_val, r->d_order, (int)S, 0, 64, st));
    CU(launch_rows(r->d_table, r->d_prob, r->d_rate, r->d_flag, r->d_order, S, r->d_rows, st));
    unsigned long long g[3];
    CU(cudaMemcpyAsync(g, r->d_table + (size_t)S * SCL_NCOL, 24, cudaMemcpyDeviceToHost, st));
    CU(cudaEventRecord(r->ev[3], st));
    CU(cudaStreamSynchronize(st));
    r->gate_num = (long long)g[0]; r->gate_den = (long long)g[1]; r->gate_cnt = g[2];
    cudaEventElapsedTime(&r->run_ms, r->ev[0], r->ev[1]);
    cudaEventElapsedTime(&r->kern_ms, r->ev[4], r->ev[5]);
    cudaEventElapsedTime(&r->fin_ms, r->ev[2], r->ev[3]);
    r->finalized = true;
    return SCL_OK;
}

// ---------------------------------------------------------------- accessors
static scl_status ensure_summ(const scl_result* rc) {
    scl_result* r = const_cast<scl_result*>(rc);
    if (r->summ_valid) return SCL_OK;
    const uint32_t NT = r->tr->n_traces;
    r->h_summ.resize(NT);
    if (NT) CU(cudaMemcpy(r->h_summ.data(), r->d_summ, NT * sizeof(scl_trace_summary), cudaMemcpyDeviceToHost));
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
    CU(cudaMemcpy(rows, r->d_rows, std::min(cap, S) * sizeof(scl_site_row), cudaMemcpyDeviceToHost));
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
    CU(cudaMemcpy(out, r->d_samples + r->h_sbase[trace], std::min(cap, cnt) * sizeof(scl_sample), cudaMemcpyDeviceToHost));
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

extern "C" scl_status scl_gate(const scl_result* r, int64_t* num, int64_t* den, int* open) {
    if (!r) return fail(SCL_EINVAL, "NULL result");
    if (!r->finalized) return fail(SCL_EINVAL, "result not finalized");
    if (num) *num = r->gate_num;
    if (den) *den = r->gate_den;
    if (open) *open = r->gate_cnt > 0 && (__int128)100 * (__int128)r->gate_num >= (__int128)r->gate_den;
    return SCL_OK;
}

extern "C" scl_status scl_result_timing(const scl_result* r, float* replay_kernel_ms, float* run_ms, float* finalize_ms) {
    if (!r) return fail(SCL_EINVAL, "NULL result");
    if (replay_kernel_ms) *replay_kernel_ms = r->kern_ms;
    if (run_ms) *run_ms = r->run_ms;
    if (finalize_ms) *finalize_ms = r->fin_ms;
    return SCL_OK;
}

#ifdef SCL_PROFILE
// Debug build only: per-role cycle sums of the last run (compute 0..7, producer 8..15, look-back 16..23).
extern "C" scl_status scl_debug_prof(const scl_result* r, unsigned long long* out) {
    if (!r || !r->d_prof) return fail(SCL_EINVAL, "no profile");
    CU(cudaMemcpy(out, r->d_prof, (48 + 4 * (size_t)r->tr->n_segs) * 8, cudaMemcpyDeviceToHost));
    return SCL_OK;
}
#endif

// "a prime number slightly above 10MB" -- smallest prime >= base (trial division)
extern "C" uint64_t scl_next_prime(uint64_t base) {
    for (uint64_t x = base < 2 ? 2 : base;; ++x) {
        bool prime = true;
        for (uint64_t q = 2; q * q <= x; ++q) if (x % q == 0) { prime = false; break; }
        if (prime) return x;
    }
}
