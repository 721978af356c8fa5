"""GPU parity of the rate-based byte sampler (NEXT-1 baseline, NEXT-3 copy volume) against the
oracle (oracle/rate.c): every sample (event index, draw prefix sum, site, kind), per-trace counts
and per-site counts, bit-exact, on ragged random traces with copies and on config-2 traces."""
import numpy as np
import pytest

import oracle
import paper_2212_07597_b200 as scl
import tracegen

pytestmark = pytest.mark.gpu


def _concat(traces):
    ev = tracegen.from_tuples([e for tr in traces for e in tr])
    off = np.zeros(len(traces) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in traces])
    return ev, off


def _check(ev, off, n_sites, R, seed, kinds, r):
    ref, roff = oracle.rate_replay(ev, off, R, seed, kinds)
    counts = scl.scl_rate_counts(r)
    assert np.array_equal(counts, np.diff(roff)), "per-trace sample counts"
    for t in range(len(off) - 1):
        got = scl.scl_rate_samples(r, t)
        exp = ref[int(roff[t]):int(roff[t + 1])]
        for f in ("idx", "draw_sum", "site", "kind"):
            bad = np.nonzero(got[f] != exp[f])[0]
            assert len(bad) == 0, f"trace {t} field {f} differs at {bad[:5]}"
    sites = scl.scl_rate_site_counts(r)
    assert np.array_equal(sites, np.bincount(ref["site"].astype(np.int64), minlength=n_sites).astype(np.uint64))
    return ref


def _random_traces(rng, n_traces, n_sites):
    traces = []
    for _ in range(n_traces):
        n = int(rng.choice([0, 1, 7, 8, 9, 255, 257, 2048, 8191, 8193, 20000, int(rng.integers(1, 9000))]))
        tr = tracegen.random_small_trace(rng, n, n_sites=n_sites, max_size=int(rng.integers(1, 5000)),
                                         max_ptrs=int(rng.integers(2, 40)))
        traces.append([e if rng.random() > 0.15 else ("c", 0, int(rng.integers(1, 9000)), e[3]) for e in tr])
    return traces


def test_rate_random_ragged():
    rng = np.random.default_rng(17)
    ev, off = _concat(_random_traces(rng, 150, 31))
    tr = scl.scl_trace_load(ev, off, 31)
    r = None
    for R, seed, kinds in ((1000, 5, scl.RATE_ALLOC_FREE), (97, 123456789, scl.RATE_ALLOC_FREE), (4096, 0, scl.RATE_ALLOC_FREE),
                           (2000, 77, scl.RATE_COPY), (1, 3, 1), (333, 9, 7)):
        r = scl.scl_rate_run(R, tr, seed=seed, kinds=kinds, out=r)
        _check(ev, off, 31, R, seed, kinds, r)
    assert scl.scl_rate_timing(r) > 0


def test_rate_config2_vs_threshold():
    """Config-2 traces at R = T: the paper's comparison (tab:sampling-comparison): the rate
    sampler takes many times more samples than the threshold sampler on the same traces."""
    cfg = tracegen.CONFIGS[2].with_traces(8)
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    rr = scl.scl_rate_run(cfg.T, tr, seed=2022)
    ref = _check(ev, off, cfg.n_sites, cfg.T, 2022, scl.RATE_ALLOC_FREE, rr)
    thr = scl.scl_replay_run(cfg.T, tr)
    n_thr = int(scl.scl_trace_summaries(thr)["n_samples"].sum())
    assert len(ref) > 5 * n_thr


def test_rate_reload_and_errors():
    rng = np.random.default_rng(4)
    ev, off = _concat(_random_traces(rng, 20, 5))
    tr = scl.scl_trace_load(ev, off, 5)
    r = scl.scl_rate_run(500, tr, seed=1)
    _check(ev, off, 5, 500, 1, scl.RATE_ALLOC_FREE, r)
    ev2, off2 = _concat(_random_traces(rng, 33, 5))               # unit sums recomputed after a reload
    scl.scl_trace_reload(tr, ev2, off2, 5)
    r2 = scl.scl_rate_run(500, tr, seed=1)
    _check(ev2, off2, 5, 500, 1, scl.RATE_ALLOC_FREE, r2)
    for bad in ((0, 1, 3), (10, 1, 0), (10, 1, 8)):
        with pytest.raises(scl.SclError):
            scl.scl_rate_run(bad[0], tr, seed=bad[1], kinds=bad[2])


def test_copy_volume():
    """NEXT-3: copy volume by rate sampling of the copied bytes at
    R = 2 T (copy_rate_multiple 2); each sample credits R bytes to its site.  GPU = oracle
    sample by sample; the credited bytes estimate every site's true copy bytes (binomial
    tolerance); the threshold sampler ignores the copies (oracle parity on the same traces)."""
    from parity import compare
    cfg = tracegen.COPY_CFG.with_traces(6)
    ev, off = tracegen.generate(cfg)
    kind = ((ev["meta"] >> np.uint64(40)) & np.uint64(3)).astype(np.int64)
    assert (kind == 2).sum() > 0.01 * len(ev)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    R = 2 * cfg.T
    r = scl.scl_rate_run(R, tr, seed=31, kinds=scl.RATE_COPY)
    _check(ev, off, cfg.n_sites, R, 31, scl.RATE_COPY, r)
    site = (ev["meta"] >> np.uint64(43)).astype(np.int64)
    size = (ev["meta"] & np.uint64((1 << 40) - 1)).astype(np.float64)
    true = np.bincount(site[kind == 2], weights=size[kind == 2], minlength=cfg.n_sites)
    est = scl.scl_rate_site_counts(r).astype(np.float64) * R
    assert abs(est.sum() - true.sum()) < 4 * np.sqrt(true.sum() * R) + R
    top = np.argsort(true)[-5:]                              # the heaviest copy sites
    for s_ in top:
        assert abs(est[s_] - true[s_]) < 5 * np.sqrt(true[s_] * R) + 2 * R
    thr = scl.scl_replay_run(cfg.T, tr)
    compare(ev, off, cfg.n_sites, cfg.T, thr)
