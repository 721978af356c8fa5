"""CPU-side checks of the C-ABI boundary: libscl.so loads, exports every
function include/scl.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes

import oracle
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2212_07597_b200 as scl
from paper_2212_07597_b200 import _build

HEADER = os.path.join(os.path.dirname(_build.HERE), "include", "scl.h")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(scl_[a-z_0-9]+)\s*\(", txt)))


def test_header_symbols_exported():
    names = declared()
    assert len(names) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (scl_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(_build.LIB)
    for n in names:
        assert getattr(lib, n) is not None


def test_library_built_for_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_next_prime_host_only():
    assert [scl.scl_next_prime(b) for b in (2**20, 10 * 2**20, 2**16, 0, 13)] == [1048583, 10485767, 65537, 2, 13]


def test_struct_sizes():
    assert scl.SAMPLE_DTYPE.itemsize == 32 and scl.SITE_ROW_DTYPE.itemsize == 104
    assert scl.SUMMARY_DTYPE.itemsize == 48 and ctypes.sizeof(scl._RunOpts) == 56
    assert scl.RATE_SAMPLE_DTYPE.itemsize == 24 and oracle.RATE_SAMPLE_DTYPE.itemsize == 24


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    ev = np.zeros(1, dtype=scl.EVENT_DTYPE)
    ev["meta"] = 8
    with pytest.raises(scl.SclError) as e:
        scl.scl_trace_load(ev, np.array([0, 1], dtype=np.uint64), 1)
    assert e.value.status == -3
