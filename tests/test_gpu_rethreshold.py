"""Re-threshold over the last stream pass (scl_replay_rethreshold: several thresholds
with one read of the events): every re-chained result against the oracle at its own threshold,
element by element, plus the stale-base errors."""
import numpy as np
import pytest

import oracle
import paper_2212_07597_b200 as scl
import tracegen
from parity import compare

pytestmark = pytest.mark.gpu


def test_rethreshold_config2_subset_matches_oracle():
    cfg = tracegen.CONFIGS[2].with_traces(8)
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    Ts = [cfg.T, 1048583, 65537, 104857601, cfg.T]
    rs = scl.scl_replay_sweep(Ts, tr, tick_ns=1000)
    for T, r in zip(Ts, rs):
        compare(ev, off, cfg.n_sites, T, r)


def test_rethreshold_ragged_cold_sites_and_variants():
    rng = np.random.default_rng(21)
    traces = [tracegen.random_small_trace(rng, int(rng.choice([0, 1, 9, 8193, int(rng.integers(1, 30000))])),
                                          n_sites=3000, max_size=int(rng.integers(1, 4000)), max_ptrs=40)
              for _ in range(40)]
    ev = tracegen.from_tuples([e for t in traces for e in t])
    off = np.zeros(len(traces) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in traces])
    tr = scl.scl_trace_load(ev, off, 3000)
    base = scl.scl_replay_run(4099, tr, tick_ns=1000)
    compare(ev, off, 3000, 4099, base)
    out = None
    for T, hwm, formula in ((257, scl.HWM_PREFIX, 0), (65537, scl.HWM_SAMPLE, 0), (1, scl.HWM_PREFIX, 1)):
        out = scl.scl_replay_rethreshold(T, tr, base, tick_ns=1000, hwm_mode=hwm, formula=formula, out=out)
        compare(ev, off, 3000, T, out, hwm_mode=hwm, formula=formula)


def test_rethreshold_stale_base_errors():
    cfg = tracegen.CONFIGS[1]
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    base = scl.scl_replay_run(cfg.T, tr)
    r2 = scl.scl_replay_rethreshold(cfg.T * 2 + 1, tr, base)
    with pytest.raises(scl.SclError):
        scl.scl_replay_rethreshold(7, tr, base, out=base)          # *out is the base
    scl.scl_replay_run(cfg.T, tr, out=r2)                            # a new stream pass: base is stale
    with pytest.raises(scl.SclError):
        scl.scl_replay_rethreshold(7, tr, base)
    b2 = scl.scl_replay_run(cfg.T, tr)
    scl.scl_trace_reload(tr, ev, off, cfg.n_sites)                   # a reload: b2 is stale
    with pytest.raises(scl.SclError):
        scl.scl_replay_rethreshold(7, tr, b2)


def test_rethreshold_all_empty_and_deferred_finalize():
    ev = tracegen.from_tuples([])
    off = np.zeros(4, dtype=np.uint64)
    tr = scl.scl_trace_load(ev, off, 5)
    base = scl.scl_replay_run(101, tr)
    r = scl.scl_replay_rethreshold(7, tr, base)
    compare(ev, off, 5, 7, r)
    cfg = tracegen.CONFIGS[1]
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    base = scl.scl_replay_run(cfg.T, tr)
    r = scl.scl_replay_rethreshold(65537, tr, base, defer_finalize=True, tick_ns=1000)
    scl.scl_finalize(r, oracle.elapsed_ns(off, 1000))
    compare(ev, off, cfg.n_sites, 65537, r)


def test_rethreshold_after_an_all_reduced_base():
    """a base whose table was all-reduced (here: two identical 'ranks', the table
    doubled in place as a SUM all-reduce would) must not leak the other rank's Tier E into a
    re-threshold: the re-chained result is this rank's alone until it is reduced itself."""
    cfg = tracegen.CONFIGS[2].with_traces(4)
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    el = cfg.events_per_trace * 1000
    base = scl.scl_replay_run(cfg.T, tr, defer_finalize=True)
    tab = scl.device_table_tensor(base)
    tab.add_(tab.clone())                                  # the SUM all-reduce of two equal shards
    scl.scl_finalize(base, el)
    ref1 = oracle.replay(ev, off, cfg.n_sites, cfg.T).site_table
    assert np.array_equal(scl.device_table_tensor(base).cpu().numpy()[:cfg.n_sites * 10].reshape(-1, 10)
                          .astype(np.uint64), 2 * ref1)
    T2 = 1048583
    r2 = scl.scl_replay_rethreshold(T2, tr, base, defer_finalize=True)
    ref2 = oracle.replay(ev, off, cfg.n_sites, T2).site_table
    t2 = scl.device_table_tensor(r2)
    assert np.array_equal(t2.cpu().numpy()[:cfg.n_sites * 10].reshape(-1, 10).astype(np.uint64), ref2)
    t2.add_(t2.clone())
    scl.scl_finalize(r2, el)
    rows = scl.scl_site_report(r2)
    assert np.array_equal(rows["col"][np.argsort(rows["site"])], 2 * ref2)
