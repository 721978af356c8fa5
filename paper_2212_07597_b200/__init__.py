"""B200-native batched replay of malloc/free traces through Scalene's memory
profiling method (arXiv 2212.07597): footprint / high-water mark, threshold
sampler, leak tracker and per-site leak report.

This package is a thin ctypes binding over ``libscl.so`` (C-ABI in
``include/scl.h``); it only marshals arguments.  Every step of the hot path runs
in the sm_100a kernels of ``csrc/``.  There is no CPU fallback: if the library
cannot be loaded, importing this package raises, and without a CUDA device
every compute call raises ``SclError`` (SCL_ECUDA).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

__all__ = ["SclError", "Traces", "Result", "scl_trace_load", "scl_trace_reload", "scl_replay_run", "scl_replay_rethreshold", "scl_replay_sweep", "scl_finalize",
           "scl_site_report", "scl_samples", "scl_trace_summaries", "scl_gate", "scl_result_device_table",
           "scl_result_timing", "scl_result_kernel_times", "scl_result_pass_times", "scl_result_launches", "scl_next_prime", "scl_traces_info", "EVENT_DTYPE", "SAMPLE_DTYPE",
           "SUMMARY_DTYPE", "SITE_ROW_DTYPE", "COLS", "device_table_tensor", "write_trace_file",
           "DOMAIN_DTYPE", "scl_sample_domains", "scl_trace_recon_error", "RATE_SAMPLE_DTYPE", "RATE_ALLOC_FREE", "RATE_COPY", "RateResult", "scl_rate_run", "scl_rate_counts",
           "scl_rate_samples", "scl_rate_site_counts", "scl_rate_timing"]

EVENT_DTYPE = np.dtype([("ptr", "<u8"), ("meta", "<u8")])
SAMPLE_DTYPE = np.dtype([("idx", "<u8"), ("net", "<i8"), ("footprint", "<i8"), ("site", "<u4"),
                         ("kind", "u1"), ("new_max", "u1"), ("pad", "<u2")])
SUMMARY_DTYPE = np.dtype([("f_final", "<i8"), ("hwm", "<i8"), ("n_samples", "<u8"), ("n_episodes", "<u8"),
                          ("f_first_sample", "<i8"), ("f_last_sample", "<i8")])
RATE_SAMPLE_DTYPE = np.dtype([("idx", "<u8"), ("draw_sum", "<u8"), ("site", "<u4"), ("kind", "<u4")])
DOMAIN_DTYPE = np.dtype([("alloc_bytes", "<u8"), ("managed_bytes", "<u8")])
RATE_ALLOC_FREE, RATE_COPY = 3, 4
SITE_ROW_DTYPE = np.dtype([("site", "<u4"), ("leak_flag", "<u4"), ("col", "<u8", (10,)),
                           ("leak_prob", "<f8"), ("leak_rate_mbps", "<f8")])
COLS = ("n_malloc", "n_free", "malloc_bytes", "free_bytes", "n_growth", "n_decline",
        "growth_bytes", "decline_bytes", "leak_mallocs", "leak_frees")
STATUS = {0: "SCL_OK", -1: "SCL_EINVAL", -2: "SCL_ENOMEM", -3: "SCL_ECUDA", -4: "SCL_ETRACE",
          -5: "SCL_EOVERFLOW", -6: "SCL_EIO", -7: "SCL_ENCCL"}
assert SAMPLE_DTYPE.itemsize == 32 and SUMMARY_DTYPE.itemsize == 48 and SITE_ROW_DTYPE.itemsize == 104


class SclError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _RunOpts(ctypes.Structure):
    _fields_ = [("tick_ns", ctypes.c_uint64), ("hwm_mode", ctypes.c_int), ("formula", ctypes.c_int),
                ("defer_finalize", ctypes.c_int), ("timing", ctypes.c_int), ("elapsed_ns", ctypes.c_uint64),
                ("cuda_stream", ctypes.c_void_p), ("nccl_comm", ctypes.c_void_p), ("chain_mode", ctypes.c_int)]


def _load():
    path = os.environ.get("SCL_LIB", _build.LIB)     # SCL_LIB: the debug build (libscl_prof.so)
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() (nvcc for sm_100a)")
    lib = ctypes.CDLL(path)
    P, U64, U32, I32, SZ = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_size_t
    sig = {
        "scl_trace_load": [ctypes.c_char_p, P, P, U32, U32, I32, I32, P],
        "scl_trace_reload": [P, P, P, U32, U32, I32, P],
        "scl_result_kernel_times": [P, P, SZ, P],
        "scl_result_launches": [P, P],
        "scl_result_pass_times": [P, P, SZ, P],
        "scl_rate_run": [U64, U64, U32, P, P, P],
        "scl_sample_domains": [P, U32, P, SZ, P],
        "scl_trace_recon_error": [P, P, SZ, P],
        "scl_rate_counts": [P, P, SZ, P],
        "scl_rate_samples": [P, U32, P, SZ, P],
        "scl_rate_site_counts": [P, P, SZ, P],
        "scl_rate_timing": [P, P],
        "scl_replay_run": [U64, P, P, P],
        "scl_replay_rethreshold": [U64, P, P, P, P],
        "scl_trace_summary_of": [P, U32, P, P, P, P],
        "scl_result_device_table": [P, P, P],
        "scl_finalize": [P, U64],
        "scl_site_report": [P, P, SZ, P],
        "scl_samples": [P, U32, P, SZ, P],
        "scl_trace_summaries": [P, P, SZ, P],
        "scl_gate": [P, P, P, P],
        "scl_result_timing": [P, P, P, P],
        "scl_traces_info": [P, P, P, P],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.scl_traces_free.argtypes = [P]
    lib.scl_traces_free.restype = None
    lib.scl_result_free.argtypes = [P]
    lib.scl_result_free.restype = None
    lib.scl_rate_free.argtypes = [P]
    lib.scl_rate_free.restype = None
    lib.scl_last_error.restype = ctypes.c_char_p
    lib.scl_next_prime.argtypes = [U64]
    lib.scl_next_prime.restype = U64
    return lib


lib = _load()


def _check(st: int):
    if st != 0:
        raise SclError(st, (lib.scl_last_error() or b"").decode())


def _addr(x):
    """Host numpy array or CUDA tensor -> raw address."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


class Traces:
    """Owning handle of scl_traces (device copy of events + offsets + segment plan)."""

    def __init__(self, handle, n_traces, n_sites):
        self._h = ctypes.c_void_p(handle)
        self.n_traces, self.n_sites = n_traces, n_sites

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h:
            lib.scl_traces_free(self._h)
            self._h = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Result:
    """Owning handle of scl_result."""

    def __init__(self, traces: Traces):
        self._h = ctypes.c_void_p(None)
        self.traces = traces

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h:
            lib.scl_result_free(self._h)
            self._h = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def scl_trace_load(events=None, offsets=None, n_sites: int = 0, device: int = 0, validate: bool = False,
                   path: str | None = None) -> Traces:
    """events: host EVENT_DTYPE array or CUDA tensor (int64 / uint8 view of 16-B events);
    offsets: uint64 [n_traces+1] (host or CUDA)."""
    out = ctypes.c_void_p()
    if path is not None:
        _check(lib.scl_trace_load(path.encode(), None, None, 0, 0, device, int(validate), ctypes.byref(out)))
    else:
        if isinstance(offsets, np.ndarray):
            offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        if isinstance(events, np.ndarray):
            events = np.ascontiguousarray(events)
        n_traces = len(offsets) - 1
        _check(lib.scl_trace_load(None, _addr(events), _addr(offsets), n_traces, n_sites, device,
                                  int(validate), ctypes.byref(out)))
    nev, nt, ns = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint32()
    _check(lib.scl_traces_info(out, ctypes.byref(nev), ctypes.byref(nt), ctypes.byref(ns)))
    t = Traces(out.value, nt.value, ns.value)
    t.n_events = nev.value
    return t


def scl_trace_reload(traces: Traces, events, offsets, n_sites: int, validate: bool = False, stream=None) -> Traces:
    """Refill ``traces`` with new events (host or CUDA), reusing its device buffers while
    they fit; stream-ordered on ``stream`` (torch.cuda.Stream / raw handle / None)."""
    if isinstance(offsets, np.ndarray):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    if isinstance(events, np.ndarray):
        events = np.ascontiguousarray(events)
    st = getattr(stream, "cuda_stream", stream) if stream is not None else None
    _check(lib.scl_trace_reload(traces.handle, _addr(events), _addr(offsets), len(offsets) - 1, n_sites,
                                int(validate), st))
    nev, nt, ns = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint32()
    _check(lib.scl_traces_info(traces.handle, ctypes.byref(nev), ctypes.byref(nt), ctypes.byref(ns)))
    traces.n_traces, traces.n_sites, traces.n_events = nt.value, ns.value, nev.value
    return traces


HWM_PREFIX, HWM_SAMPLE = 0, 1
CHAIN_AUTO, CHAIN_RUNNERS, CHAIN_SPLIT = 0, 1, 2
FORMULA_PAPER, FORMULA_TEXTBOOK = 0, 1


def scl_replay_run(threshold: int, traces: Traces, tick_ns: int = 0, formula: int = 0,
                   defer_finalize: bool = False, elapsed_ns: int = 0, stream=None,
                   out: Result | None = None, timing: bool = False, hwm_mode: int = HWM_PREFIX,
                   nccl_comm: int | None = None, chain_mode: int = 0) -> Result:
    """Replay all traces at threshold T; ``out`` (a previous Result of the same
    traces) is reused in place.  stream: torch.cuda.Stream / raw handle / None.
    timing: record CUDA events for scl_result_timing / scl_result_kernel_times."""
    o = _RunOpts()
    o.tick_ns, o.hwm_mode, o.formula = tick_ns, hwm_mode, formula
    o.defer_finalize, o.elapsed_ns, o.timing = int(defer_finalize), elapsed_ns, int(timing)
    o.chain_mode = chain_mode
    if stream is not None:
        o.cuda_stream = getattr(stream, "cuda_stream", stream)
    if nccl_comm is not None:
        o.nccl_comm = nccl_comm                     # raw ncclComm_t: table SUM / elapsed MAX in the library
    r = out if out is not None else Result(traces)
    h = ctypes.c_void_p(r._h.value)
    _check(lib.scl_replay_run(threshold, traces.handle, ctypes.byref(o), ctypes.byref(h)))
    r._h = h
    return r


def scl_replay_rethreshold(threshold: int, traces: Traces, base: Result, tick_ns: int = 0, formula: int = 0,
                           defer_finalize: bool = False, elapsed_ns: int = 0, stream=None,
                           out: Result | None = None, timing: bool = False, hwm_mode: int = HWM_PREFIX,
                           chain_mode: int = 0) -> Result:
    """The replay at another threshold over the handle's last stream pass (the run that gave
    ``base``): the events are not streamed again (K5, several thresholds in one read)."""
    o = _RunOpts()
    o.tick_ns, o.hwm_mode, o.formula = tick_ns, hwm_mode, formula
    o.defer_finalize, o.elapsed_ns, o.timing = int(defer_finalize), elapsed_ns, int(timing)
    o.chain_mode = chain_mode
    if stream is not None:
        o.cuda_stream = getattr(stream, "cuda_stream", stream)
    r = out if out is not None else Result(traces)
    h = ctypes.c_void_p(r._h.value)
    _check(lib.scl_replay_rethreshold(threshold, traces.handle, base.handle, ctypes.byref(o), ctypes.byref(h)))
    r._h = h
    return r


def scl_replay_sweep(thresholds, traces: Traces, **kw) -> list:
    """One stream pass at thresholds[0], every other threshold re-chained over it."""
    rs = [scl_replay_run(int(thresholds[0]), traces, **kw)]
    for T in thresholds[1:]:
        rs.append(scl_replay_rethreshold(int(T), traces, rs[0], **kw))
    return rs


def scl_result_device_table(r: Result):
    ptr, n = ctypes.c_void_p(), ctypes.c_size_t()
    _check(lib.scl_result_device_table(r.handle, ctypes.byref(ptr), ctypes.byref(n)))
    return ptr.value, n.value


def device_table_tensor(r: Result):
    """torch.int64 CUDA view of the summable table (site table + 3 gate sums),
    for an all-reduce across ranks before scl_finalize."""
    import torch
    ptr, n = scl_result_device_table(r)

    class _Iface:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False), "version": 2}
    # no device argument: the tensor stays on the pointer's own device (never a copy on the
    # current device, which an all-reduce would update instead of the library's table)
    t = torch.as_tensor(_Iface())
    assert t.data_ptr() == ptr, "device_table_tensor must alias the library's table"
    return t


def scl_finalize(r: Result, elapsed_ns: int = 0):
    _check(lib.scl_finalize(r.handle, elapsed_ns))


def scl_site_report(r: Result) -> np.ndarray:
    n = ctypes.c_size_t()
    _check(lib.scl_site_report(r.handle, None, 0, ctypes.byref(n)))
    rows = np.zeros(n.value, dtype=SITE_ROW_DTYPE)
    _check(lib.scl_site_report(r.handle, rows.ctypes.data, n.value, ctypes.byref(n)))
    return rows


def scl_samples(r: Result, trace: int) -> np.ndarray:
    n = ctypes.c_size_t()
    _check(lib.scl_samples(r.handle, trace, None, 0, ctypes.byref(n)))
    out = np.zeros(n.value, dtype=SAMPLE_DTYPE)
    if n.value:
        _check(lib.scl_samples(r.handle, trace, out.ctypes.data, n.value, ctypes.byref(n)))
    return out


def scl_sample_domains(r: Result, trace: int) -> np.ndarray:
    """Per sample of the trace: bytes allocated since the previous sample and the managed-domain
    part of them (NEXT-2); managed fraction = managed_bytes / max(alloc_bytes, 1)."""
    n = ctypes.c_size_t()
    _check(lib.scl_sample_domains(r.handle, trace, None, 0, ctypes.byref(n)))
    out = np.zeros(n.value, dtype=DOMAIN_DTYPE)
    if n.value:
        _check(lib.scl_sample_domains(r.handle, trace, out.ctypes.data, n.value, ctypes.byref(n)))
    return out


def scl_trace_recon_error(r: Result) -> np.ndarray:
    """Per trace: max |F_i - latest sample footprint| over events (NEXT-4 trend; < T)."""
    n = ctypes.c_size_t()
    _check(lib.scl_trace_recon_error(r.handle, None, 0, ctypes.byref(n)))
    out = np.zeros(n.value, dtype=np.uint64)
    if n.value:
        _check(lib.scl_trace_recon_error(r.handle, out.ctypes.data, n.value, ctypes.byref(n)))
    return out


def scl_trace_summaries(r: Result) -> np.ndarray:
    n = ctypes.c_size_t()
    _check(lib.scl_trace_summaries(r.handle, None, 0, ctypes.byref(n)))
    out = np.zeros(n.value, dtype=SUMMARY_DTYPE)
    if n.value:
        _check(lib.scl_trace_summaries(r.handle, out.ctypes.data, n.value, ctypes.byref(n)))
    return out


def scl_trace_summary_of(r: Result, trace: int):
    """(f_final, hwm, n_samples, n_episodes) of one trace."""
    f, h, n, e = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib.scl_trace_summary_of(r.handle, trace, ctypes.byref(f), ctypes.byref(h), ctypes.byref(n), ctypes.byref(e)))
    return f.value, h.value, n.value, e.value


def scl_gate(r: Result):
    num, den, op = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    _check(lib.scl_gate(r.handle, ctypes.byref(num), ctypes.byref(den), ctypes.byref(op)))
    return num.value, den.value, bool(op.value)


def scl_result_timing(r: Result):
    """(replay_kernel_ms, run_ms, finalize_ms) of the last run (CUDA events; -1 without timing=True)."""
    a, b, c = ctypes.c_float(), ctypes.c_float(), ctypes.c_float()
    _check(lib.scl_result_timing(r.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def scl_result_kernel_times(r: Result) -> list:
    """Replay-kernel durations (ms) of the runs enqueued since the previous call (<= 128)."""
    buf = (ctypes.c_float * 128)()
    n = ctypes.c_size_t()
    _check(lib.scl_result_kernel_times(r.handle, buf, 128, ctypes.byref(n)))
    return [buf[i] for i in range(n.value)]


def scl_result_pass_times(r: Result) -> list:
    """Stream-pass durations (ms: replay kernel + the kernels completing a1-a5 after it) of the runs
    enqueued with timing=True since the previous call (<= 128)."""
    buf = (ctypes.c_float * 128)()
    n = ctypes.c_size_t()
    _check(lib.scl_result_pass_times(r.handle, buf, 128, ctypes.byref(n)))
    return [buf[i] for i in range(n.value)]


def scl_result_launches(r: Result) -> int:
    """Kernels the library launched for the result's last run (+ its finalize)."""
    n = ctypes.c_uint32()
    _check(lib.scl_result_launches(r.handle, ctypes.byref(n)))
    return n.value


def scl_next_prime(base: int) -> int:
    return int(lib.scl_next_prime(base))


def scl_traces_info(t: Traces):
    nev, nt, ns = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint32()
    _check(lib.scl_traces_info(t.handle, ctypes.byref(nev), ctypes.byref(nt), ctypes.byref(ns)))
    return nev.value, nt.value, ns.value


def write_trace_file(path: str, events: np.ndarray, offsets: np.ndarray, n_sites: int, tick_ns: int = 1000,
                     site_names=None):
    """Binary trace file: "SCLTRC01", u32 version=1, u32 n_traces,
    u32 n_sites, u32 0, u64 tick_ns, u64 offsets[n+1], 16-B events, then an
    optional site table of "file\\tline\\n" strings (ignored by the loader)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    with open(path, "wb") as f:
        f.write(b"SCLTRC01")
        f.write(np.array([1, len(offsets) - 1, n_sites, 0], dtype=np.uint32).tobytes())
        f.write(np.array([tick_ns], dtype=np.uint64).tobytes())
        f.write(offsets.tobytes())
        f.write(np.ascontiguousarray(events).tobytes())
        if site_names:
            f.write("".join(f"{a}\t{b}\n" for a, b in site_names).encode())


class RateResult:
    """Owning handle of scl_rate_result (the rate-based sampler, NEXT-1 / NEXT-3)."""

    def __init__(self, traces: Traces):
        self._h = ctypes.c_void_p(None)
        self.traces = traces

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h:
            lib.scl_rate_free(self._h)
            self._h = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def scl_rate_run(rate_bytes: int, traces: Traces, seed: int = 1, kinds: int = RATE_ALLOC_FREE, stream=None,
                 out: RateResult | None = None) -> RateResult:
    """Rate-based byte sampler over every trace: mean rate_bytes between samples, counted kinds
    (RATE_ALLOC_FREE: the paper's baseline; RATE_COPY: copy volume); seed 0 = deterministic."""
    st = getattr(stream, "cuda_stream", stream) if stream is not None else None
    r = out if out is not None else RateResult(traces)
    h = ctypes.c_void_p(r._h.value)
    _check(lib.scl_rate_run(rate_bytes, seed, kinds, traces.handle, st, ctypes.byref(h)))
    r._h = h
    return r


def scl_rate_counts(r: RateResult) -> np.ndarray:
    n = ctypes.c_size_t()
    _check(lib.scl_rate_counts(r.handle, None, 0, ctypes.byref(n)))
    out = np.zeros(n.value, dtype=np.uint64)
    if n.value:
        _check(lib.scl_rate_counts(r.handle, out.ctypes.data, n.value, ctypes.byref(n)))
    return out


def scl_rate_samples(r: RateResult, trace: int) -> np.ndarray:
    n = ctypes.c_size_t()
    _check(lib.scl_rate_samples(r.handle, trace, None, 0, ctypes.byref(n)))
    out = np.zeros(n.value, dtype=RATE_SAMPLE_DTYPE)
    if n.value:
        _check(lib.scl_rate_samples(r.handle, trace, out.ctypes.data, n.value, ctypes.byref(n)))
    return out


def scl_rate_site_counts(r: RateResult) -> np.ndarray:
    n = ctypes.c_size_t()
    _check(lib.scl_rate_site_counts(r.handle, None, 0, ctypes.byref(n)))
    out = np.zeros(n.value, dtype=np.uint64)
    if n.value:
        _check(lib.scl_rate_site_counts(r.handle, out.ctypes.data, n.value, ctypes.byref(n)))
    return out


def scl_rate_timing(r: RateResult) -> float:
    ms = ctypes.c_float()
    _check(lib.scl_rate_timing(r.handle, ctypes.byref(ms)))
    return ms.value
