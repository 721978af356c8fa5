"""Seeded synthetic trace generator (inputs only -- none of the method's arithmetic).

Shared by the oracle tests, the GPU parity tests and bench.py.  The five
configurations are BASELINE.json ``configs`` as read in SURVEY.md §8(d);
``T`` is the threshold each config is run at, ``scl_next_prime``/
``oracle.next_prime`` of a MiB base, written out as constants
here so that this module needs neither side.

The event record is the 16-byte trace format of include/scl.h:
``ptr`` u64, ``meta`` u64 = size (bits 0..39) | kind << 40 | domain << 42 | site << 43.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtracegen.so")
EVENT_DTYPE = np.dtype([("ptr", "<u8"), ("meta", "<u8")])


class _Cfg(ctypes.Structure):
    _fields_ = [("n_traces", ctypes.c_uint32), ("n_sites", ctypes.c_uint32),
                ("events_per_trace", ctypes.c_uint64), ("zipf_s", ctypes.c_double),
                ("n_planted", ctypes.c_uint32), ("heavy_tailed", ctypes.c_uint32),
                ("leak_T", ctypes.c_uint64), ("leak_lambda", ctypes.c_double),
                ("leak_rate_spread", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("copy_lambda", ctypes.c_double)]


@dataclass(frozen=True)
class Config:
    name: str
    n_traces: int
    events_per_trace: int
    n_sites: int
    zipf_s: float
    n_planted: int
    T: int                       # threshold (prime) the config is replayed at
    leak_lambda: float           # per-step probability of a planted-leak allocation
    leak_rate_spread: float = 0.0
    heavy_tailed: bool = False
    seed: int = 0
    t_sweep: tuple = ()          # config 5: thresholds of the sweep
    copy_lambda: float = 0.0     # per-step probability of a copy event (NEXT-3 copy volume); 0: none
    leak_T: int = 0              # planted leak sizes U[leak_T/4, leak_T]; 0: the config's T

    @property
    def n_events(self) -> int:
        return self.n_traces * self.events_per_trace

    def with_traces(self, n: int) -> "Config":
        return replace(self, n_traces=n)

    def ctype(self) -> _Cfg:
        return _Cfg(self.n_traces, self.n_sites, self.events_per_trace, self.zipf_s,
                    self.n_planted, int(self.heavy_tailed), self.leak_T or self.T, self.leak_lambda,
                    self.leak_rate_spread, self.seed, self.copy_lambda)


# smallest primes >= the bases (pinned against trial division
# in tests/test_oracle_pins.py::test_next_prime_table)
P_1MIB = 1048583
P_10MIB = 10485767
SWEEP = (65537, 131101, 262147, 524309, 1048583, 2097169, 4194319, 8388617,
         16777259, 33554467, 67108879)

CONFIGS = {
    1: Config("cfg1", 1, 10_000, 16, 0.8, 1, P_1MIB, 0.01, seed=20221215 + 1),
    2: Config("cfg2", 64, 1_000_000, 1_000, 0.8, 4, P_10MIB, 5.0e-5, seed=20221215 + 2),
    3: Config("cfg3", 1024, 1_000_000, 50_000, 1.0, 16, P_10MIB, 1.6e-4, 100.0, seed=20221215 + 3),
    4: Config("cfg4", 8192, 4_000_000, 200_000, 1.2, 32, P_10MIB, 1.0e-5, seed=20221215 + 4),
    5: Config("cfg5", 256, 100_000_000, 10_000, 1.0, 8, 65537, 8.0e-6, heavy_tailed=True, leak_T=1 << 26,
              seed=20221215 + 5, t_sweep=SWEEP),
}

# NEXT-3 (copy volume): config 2 with 2 % copy events (memcpy of an object-sized
# buffer at the current line); copies leave the footprint, samples and leak tracker unchanged.
COPY_CFG = replace(CONFIGS[2], name="cfg2-copy", copy_lambda=0.02, seed=20221215 + 26)

_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "tracegen.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        cmd = f"g++ -O2 -std=c++17 -fPIC -shared -pthread -o {_LIB_PATH}.tmp {src}"
        if os.system(cmd) != 0:
            raise RuntimeError("tracegen build failed: " + cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.tg_generate.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint32, ctypes.c_uint32,
                                    ctypes.c_void_p, ctypes.c_int]
        lib.tg_site_classes.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_void_p]
        _lib = lib
    return _lib


def generate(cfg: Config, t0: int = 0, t1: int | None = None, n_threads: int | None = None,
             out: np.ndarray | None = None):
    """Traces [t0, t1) of ``cfg`` -> (events[EVENT_DTYPE], offsets[uint64])."""
    lib = _load()
    t1 = cfg.n_traces if t1 is None else t1
    n = (t1 - t0) * cfg.events_per_trace
    if out is None:
        out = np.empty(n, dtype=EVENT_DTYPE)
    assert out.dtype == EVENT_DTYPE and out.size >= n and out.flags.c_contiguous
    c = cfg.ctype()
    lib.tg_generate(ctypes.byref(c), t0, t1, out.ctypes.data_as(ctypes.c_void_p),
                    n_threads or os.cpu_count() or 1)
    offsets = np.arange(t1 - t0 + 1, dtype=np.uint64) * np.uint64(cfg.events_per_trace)
    return out[:n], offsets


def site_classes(cfg: Config) -> np.ndarray:
    lib = _load()
    out = np.zeros(cfg.n_sites, dtype=np.uint8)
    c = cfg.ctype()
    lib.tg_site_classes(ctypes.byref(c), out.ctypes.data_as(ctypes.c_void_p))
    return out


def planted_sites(cfg: Config) -> np.ndarray:
    return np.nonzero(site_classes(cfg) == 3)[0].astype(np.uint32)


def pack(kind: int, size: int, site: int, domain: int = 0) -> int:
    """meta word of one event (kind 0 alloc, 1 free, 2 copy)."""
    return (size & ((1 << 40) - 1)) | (kind << 40) | (domain << 42) | (site << 43)


def from_tuples(events) -> np.ndarray:
    """[(kind 'a'|'f'|'c', ptr, size, site[, domain]), ...] -> EVENT_DTYPE array (hand-written
    traces; domain 1 = managed / Python, 0 = native, NEXT-2)."""
    k = {"a": 0, "f": 1, "c": 2}
    arr = np.zeros(len(events), dtype=EVENT_DTYPE)
    for i, e in enumerate(events):
        kind, ptr, size, site = e[:4]
        arr[i] = (ptr, pack(k[kind], size, site, e[4] if len(e) > 4 else 0))
    return arr


def random_small_trace(rng: np.random.Generator, n: int, n_sites: int = 4,
                       max_size: int = 8, p_free: float = 0.45, max_ptrs: int = 6):
    """Small valid random trace with pointer reuse (for exhaustive-style tests):
    list of (kind, ptr, size, site)."""
    live = {}
    free_ptrs = list(range(1, max_ptrs + 1))
    out = []
    for _ in range(n):
        if live and (rng.random() < p_free or not free_ptrs):
            p = list(live)[int(rng.integers(len(live)))]
            out.append(("f", p, live.pop(p), int(rng.integers(n_sites))))
            free_ptrs.append(p)
        else:
            p = free_ptrs.pop(int(rng.integers(len(free_ptrs))))
            s = int(rng.integers(1, max_size + 1))
            live[p] = s
            out.append(("a", p, s, int(rng.integers(n_sites))))
    return out
