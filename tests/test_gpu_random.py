"""Randomised GPU-vs-oracle parity (a short, fixed-seed slice of tools/fuzz.py): random trace
counts, lengths on and around the 8-event row / 256-event chunk / 8192-event unit boundaries,
site counts on and around the shared-memory table sizes (1,024 / 2,048), sizes up to 2^40 - 1,
thresholds from 1 to past 2^40, both hwm modes and both leak formulas (DESIGN.md §3 readings),
then a re-threshold over the same stream pass -- each compared element by element."""
import numpy as np
import pytest

import paper_2212_07597_b200 as scl
import tracegen
from parity import compare

pytestmark = pytest.mark.gpu


def _case(rng):
    n_traces = int(rng.integers(1, 40))
    n_sites = int(rng.choice([1, 7, 300, 1024, 1025, 2048, 2049, 5000, 1 << 21]))
    max_size = int(rng.choice([8, 300, 5000, 1 << 20, 1 << 27, (1 << 40) - 1]))
    traces = []
    for _ in range(n_traces):
        n = int(rng.choice([0, 1, 7, 8, 9, 255, 256, 257, 2047, 2048, 8191, 8192, 8193, 16385,
                            int(rng.integers(1, 60000))]))
        traces.append(tracegen.random_small_trace(rng, n, n_sites=n_sites, max_size=max_size,
                                                  max_ptrs=int(rng.integers(1, 200))))
    ev = tracegen.from_tuples([e for t in traces for e in t])
    off = np.zeros(n_traces + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in traces])
    T = int(rng.choice([1, 2, 17, 257, 4099, 65537, 1048583, (1 << 40) + 15, int(rng.integers(1, 1 << 24))]))
    return ev, off, n_sites, T, int(rng.integers(0, 2)), int(rng.integers(0, 2)), int(rng.choice([3, 1031, 1048583]))


@pytest.mark.parametrize("seed", [5, 6])
def test_random_cases(seed):
    rng = np.random.default_rng(seed)
    keep = None      # the previous case's re-threshold result stays alive: varies the allocation layout
    for case in range(20):
        ev, off, n_sites, T, hwm, formula, T2 = _case(rng)
        tr = scl.scl_trace_load(ev, off, n_sites)
        r = scl.scl_replay_run(T, tr, tick_ns=1000, hwm_mode=hwm, formula=formula)
        compare(ev, off, n_sites, T, r, hwm_mode=hwm, formula=formula)
        r2 = scl.scl_replay_rethreshold(T2, tr, r, tick_ns=1000, hwm_mode=hwm, formula=formula)
        compare(ev, off, n_sites, T2, r2, hwm_mode=hwm, formula=formula)
        keep = r2
        del tr, r
    del keep
