"""CPU oracle for the Scalene trace-replay hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2212_07597_b200``): it links only ``oracle/liboracle.so``
built from ``oracle/oracle.c`` (plain C, ``-ffp-contract=off``), and the tiny
pure-Python ``oracle.mini`` used to cross-check it on small inputs.

Paper passages followed (PAPER.md lines): sampler P:429-438, footprint/HWM
P:24-25 and P:490-494, leak tracker P:20-39, probability P:49-57, filter and
rate P:59-71.  Readings where the paper is silent: DESIGN.md section 3.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
except the growth gate (reading Q10), which the paper does not define
precisely -- "parity unpinned" for the gate's exact denominator.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

EVENT_DTYPE = np.dtype([("ptr", "<u8"), ("meta", "<u8")])
SAMPLE_DTYPE = np.dtype([("idx", "<u8"), ("net", "<i8"), ("footprint", "<i8"),
                         ("site", "<u4"), ("kind", "u1"), ("new_max", "u1"), ("pad", "<u2")])
DOMAIN_DTYPE = np.dtype([("alloc_bytes", "<u8"), ("managed_bytes", "<u8")])   # per sample (NEXT-2)
SUMMARY_DTYPE = np.dtype([("f_final", "<i8"), ("hwm", "<i8"), ("n_samples", "<u8"),
                          ("n_episodes", "<u8"), ("f_first_sample", "<i8"), ("f_last_sample", "<i8")])
assert EVENT_DTYPE.itemsize == 16 and SAMPLE_DTYPE.itemsize == 32 and SUMMARY_DTYPE.itemsize == 48

NCOL = 10
COLS = ("n_malloc", "n_free", "malloc_bytes", "free_bytes", "n_growth", "n_decline",
        "growth_bytes", "decline_bytes", "leak_mallocs", "leak_frees")
HWM_PREFIX, HWM_SAMPLE = 0, 1
FORMULA_PAPER, FORMULA_TEXTBOOK = 0, 1
SIZE_MASK = (1 << 40) - 1

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain C; no FMA contraction)."""
    src = os.path.join(_HERE, "oracle.c")
    src2 = os.path.join(_HERE, "rate.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(src2), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        cmd = (f"gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread "
               f"-o {_LIB_PATH}.tmp {src} {src2} -lm")
        if os.system(cmd) != 0:
            raise RuntimeError("oracle build failed: " + cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P, U64, U32, I32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        lib.orc_replay_trace.argtypes = [P, U64, U64, I32, P, U64, P, P, U32, P]
        lib.orc_replay_all.argtypes = [P, P, U32, U32, U64, I32, I32, P, P, P, P, P]
        lib.orc_gate.argtypes = [P, U32, P, P, P]
        lib.orc_finalize.argtypes = [P, U32, I32, U64, I32, P, P, P]
        lib.orc_report_order.argtypes = [P, P, U32, P]
        lib.orc_next_prime.argtypes = [U64]
        lib.orc_next_prime.restype = U64
        lib.orc_validate_trace.argtypes = [P, U64, U32]
        lib.orc_validate_trace.restype = ctypes.c_int64
        lib.orc_soft_log.argtypes = [ctypes.c_double]
        lib.orc_soft_log.restype = ctypes.c_double
        lib.orc_rate_draw.argtypes = [U64, U64, U32, U64]
        lib.orc_rate_draw.restype = U64
        lib.orc_rate_trace.argtypes = [P, U64, U64, U64, U32, U32, P, U64, P]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class OracleResult:
    samples: np.ndarray          # SAMPLE_DTYPE, all traces concatenated
    sample_off: np.ndarray       # uint64 [n_traces+1] (offsets into samples after trimming)
    summaries: np.ndarray        # SUMMARY_DTYPE [n_traces]
    site_table: np.ndarray       # uint64 [n_sites, 10]
    domains: np.ndarray = None   # DOMAIN_DTYPE parallel to samples (NEXT-2)

    def trace_samples(self, t: int) -> np.ndarray:
        return self.samples[int(self.sample_off[t]):int(self.sample_off[t + 1])]


def sample_bound(events: np.ndarray, offsets: np.ndarray, T: int) -> np.ndarray:
    """Per-trace capacity min(n_t, floor(sum|d|/T)) -- an upper bound on the
    number of samples, since every sample consumes |net| >= T of sum|d|."""
    meta = np.ascontiguousarray(events).view(np.uint64)[1::2]
    sizes = meta & np.uint64(SIZE_MASK)
    sizes[((meta >> np.uint64(40)) & np.uint64(3)) == 2] = 0          # copies do not count
    off = np.asarray(offsets, dtype=np.int64)
    n = off[1:] - off[:-1]
    tot = np.zeros(len(n), dtype=np.uint64)
    nz = n > 0
    if nz.any():
        tot[nz] = np.add.reduceat(sizes, off[:-1][nz], dtype=np.uint64)
    return np.minimum(n.astype(np.uint64), tot // np.uint64(T))


def replay(events: np.ndarray, offsets, n_sites: int, T: int, hwm_mode: int = HWM_PREFIX,
           n_threads: int = 1) -> OracleResult:
    lib = _load()
    events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n_traces = len(offsets) - 1
    cap = sample_bound(events, offsets, T)
    soff = np.zeros(n_traces + 1, dtype=np.uint64)
    soff[1:] = np.cumsum(cap)
    # slot buffers sized by the sample bound; only the slots the replay writes are read back (`keep`
    # below), so they are not zero-filled (at dense thresholds the bound is many GB, the samples few)
    samples = np.empty(max(int(soff[-1]), 1), dtype=SAMPLE_DTYPE)
    summ = np.zeros(n_traces, dtype=SUMMARY_DTYPE)
    table = np.zeros((n_sites, NCOL), dtype=np.uint64)
    dom = np.empty(len(samples), dtype=DOMAIN_DTYPE)
    rc = lib.orc_replay_all(_ptr(events), _ptr(offsets), n_traces, n_sites, T, hwm_mode,
                            n_threads, _ptr(samples), _ptr(soff), _ptr(summ), _ptr(table), _ptr(dom))
    if rc != 0:
        raise ValueError("oracle: invalid event (site >= n_sites or kind 3)")
    ns = summ["n_samples"].astype(np.uint64)
    assert np.all(ns <= cap), "sample bound violated"
    keep = np.concatenate([np.arange(int(soff[t]), int(soff[t] + ns[t])) for t in range(n_traces)]) \
        if n_traces else np.zeros(0, dtype=np.int64)
    out_off = np.zeros(n_traces + 1, dtype=np.uint64)
    out_off[1:] = np.cumsum(ns)
    return OracleResult(samples[keep.astype(np.int64)], out_off, summ, table, dom[keep.astype(np.int64)])


def gate(summaries: np.ndarray):
    lib = _load()
    s = np.ascontiguousarray(summaries, dtype=SUMMARY_DTYPE)
    num, den, op = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    lib.orc_gate(_ptr(s), len(s), ctypes.byref(num), ctypes.byref(den), ctypes.byref(op))
    return num.value, den.value, bool(op.value)


def finalize(site_table: np.ndarray, gate_open: bool, elapsed_ns: int,
             formula: int = FORMULA_PAPER):
    lib = _load()
    t = np.ascontiguousarray(site_table, dtype=np.uint64)
    n = t.shape[0]
    prob = np.zeros(n, dtype=np.float64)
    rate = np.zeros(n, dtype=np.float64)
    flag = np.zeros(n, dtype=np.uint8)
    lib.orc_finalize(_ptr(t), n, int(gate_open), elapsed_ns, formula, _ptr(prob), _ptr(rate), _ptr(flag))
    return prob, rate, flag


def report_order(rate: np.ndarray, flag: np.ndarray) -> np.ndarray:
    lib = _load()
    r = np.ascontiguousarray(rate, dtype=np.float64)
    f = np.ascontiguousarray(flag, dtype=np.uint8)
    order = np.zeros(len(r), dtype=np.uint32)
    lib.orc_report_order(_ptr(r), _ptr(f), len(r), _ptr(order))
    return order


def next_prime(base: int) -> int:
    return int(_load().orc_next_prime(base))


def validate(events: np.ndarray, offsets, n_sites: int):
    """Returns None if every trace is valid, else (trace, event index)."""
    lib = _load()
    events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    for t in range(len(offsets) - 1):
        b, e = int(offsets[t]), int(offsets[t + 1])
        sub = events[b:e]
        bad = lib.orc_validate_trace(_ptr(sub), e - b, n_sites)
        if bad >= 0:
            return t, int(bad)
    return None


def elapsed_ns(offsets, tick_ns: int = 1000) -> int:
    """Synthetic elapsed time (reading Q11): t_i = (i+1) * tick_ns, so the run
    lasts max_t n_t * tick_ns."""
    off = np.asarray(offsets, dtype=np.int64)
    return int((off[1:] - off[:-1]).max()) * tick_ns if len(off) > 1 else 0


def full(events, offsets, n_sites, T, hwm_mode=HWM_PREFIX, formula=FORMULA_PAPER,
         tick_ns=1000, n_threads=1):
    """Whole path a1..a6 -> dict (for tests and bench)."""
    r = replay(events, offsets, n_sites, T, hwm_mode, n_threads)
    num, den, op = gate(r.summaries)
    el = elapsed_ns(offsets, tick_ns)
    prob, rate, flag = finalize(r.site_table, op, el, formula)
    order = report_order(rate, flag)
    return dict(result=r, gate=(num, den, op), elapsed_ns=el, prob=prob, rate=rate,
                flag=flag, order=order)


# ---- rate-based byte sampler (NEXT-1 baseline, NEXT-3 copy volume; oracle/rate.c) ----
RATE_SAMPLE_DTYPE = np.dtype([("idx", "<u8"), ("draw_sum", "<u8"), ("site", "<u4"), ("kind", "<u4")])
KINDS_ALLOC_FREE, KINDS_COPY = 0b011, 0b100


def soft_log(x: float) -> float:
    return float(_load().orc_soft_log(x))


def rate_draw(R: int, seed: int, trace: int, k: int) -> int:
    return int(_load().orc_rate_draw(R, seed, trace, k))


def rate_replay(events: np.ndarray, offsets, R: int, seed: int, kinds: int = KINDS_ALLOC_FREE):
    """Per trace: the rate sampler's samples (RATE_SAMPLE_DTYPE) -> (samples, sample_off)."""
    lib = _load()
    offsets = np.asarray(offsets, dtype=np.uint64)
    events = np.ascontiguousarray(events)
    n_traces = len(offsets) - 1
    per, counts = [], np.zeros(n_traces, dtype=np.uint64)
    for t in range(n_traces):
        b, e = int(offsets[t]), int(offsets[t + 1])
        sub = events[b:e]
        cap = 1024
        while True:
            out = np.zeros(cap, dtype=RATE_SAMPLE_DTYPE)
            ns = ctypes.c_uint64()
            rc = lib.orc_rate_trace(_ptr(sub) if e > b else None, e - b, R, seed, t, kinds, _ptr(out), cap,
                                    ctypes.byref(ns))
            if rc != 0:
                raise ValueError(f"trace {t}: invalid event")
            if ns.value <= cap:
                break
            cap = int(ns.value)
        per.append(out[:ns.value]); counts[t] = ns.value
    off = np.zeros(n_traces + 1, dtype=np.uint64)
    off[1:] = np.cumsum(counts)
    return (np.concatenate(per) if per else np.zeros(0, dtype=RATE_SAMPLE_DTYPE)), off
