"""Resident waves (configs 4/5 at 1/2/4 GPUs do not fit in HBM): a shard replayed
in waves of whole traces through one refilled device buffer, the waves' tables summed on the
device and a6 run once, against the oracle on the whole shard, element by element."""
import numpy as np
import pytest

import oracle
import tracegen
from paper_2212_07597_b200 import dist as sdist
import paper_2212_07597_b200 as scl
from parity import REL_TOL

pytestmark = pytest.mark.gpu


def _check(ev, off, n_sites, T, wave_events):
    r, summ, samples, _ = sdist.replay_waves(ev, off, n_sites, T, wave_events)
    ref = oracle.full(ev, off, n_sites, T, n_threads=8)
    res = ref["result"]
    for f in ("f_final", "hwm", "n_samples", "n_episodes", "f_first_sample", "f_last_sample"):
        assert np.array_equal(summ[f], res.summaries[f]), f
    for t in range(len(off) - 1):
        g, o = samples[t], res.trace_samples(t)
        assert len(g) == len(o), t
        for f in ("idx", "net", "footprint", "site", "kind", "new_max"):
            assert np.array_equal(g[f], o[f]), (t, f)
    rows = scl.scl_site_report(r)
    order = ref["order"]
    assert np.array_equal(rows["site"], order)
    assert np.array_equal(rows["col"], res.site_table[order].astype(rows["col"].dtype))
    assert np.array_equal(rows["leak_flag"], ref["flag"][order].astype(np.uint32))
    for name, key in (("leak_prob", "prob"), ("leak_rate_mbps", "rate")):
        a, b = rows[name], ref[key][order]
        assert np.all((a == b) | (np.abs(a - b) <= REL_TOL * np.abs(b))), name
    assert scl.scl_gate(r) == ref["gate"]
    return r


def test_waves_config2_subset_match_oracle():
    cfg = tracegen.CONFIGS[2].with_traces(10)
    ev, off = tracegen.generate(cfg)
    waves = sdist.plan_waves(off, 2_500_000)
    assert len(waves) == 5                                    # two 10^6-event traces per wave
    _check(ev, off, cfg.n_sites, cfg.T, 2_500_000)


def test_waves_ragged_one_trace_per_wave_and_long_trace():
    rng = np.random.default_rng(7)
    traces = []
    for n in (0, 1, 9000, 120000, 3, 70000, 0, 8193):
        traces.append(tracegen.random_small_trace(rng, n, n_sites=2000, max_size=int(rng.integers(1, 5000)),
                                                  max_ptrs=64))
    ev = tracegen.from_tuples([e for tr in traces for e in tr])
    off = np.zeros(len(traces) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in traces])
    for wave_events in (1, 50_000, 10 ** 9):                  # one trace per wave .. one wave
        _check(ev, off, 2000, 65537, wave_events)
