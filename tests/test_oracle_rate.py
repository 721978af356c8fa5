"""Pins of the rate-based byte sampler oracle (oracle/rate.c; SURVEY §8(f) NEXT-1 baseline and
NEXT-3 copy volume).  Each pin is something other than the oracle's own code: the C library's
log, SPEC's worked examples, closed forms of the deterministic mode, an independent
prefix-sum formulation of the sample positions, and the geometric distribution's moments."""
import math

import numpy as np

import oracle
import tracegen


def _events(tuples):
    return tracegen.from_tuples(tuples)


def test_soft_log_matches_libm():
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.random(20000), rng.random(2000) ** 30, [1.0, 0.5, 2.0 ** -53, 1 - 1e-7, 0.75]])
    xs = xs[xs > 0]
    for x in xs:
        got, ref = oracle.soft_log(float(x)), math.log(float(x))
        assert abs(got - ref) <= 2 * math.ulp(ref) + 1e-300, (x, got, ref)
    assert oracle.soft_log(1.0) == 0.0


def test_spec_deterministic_examples():
    # deterministic rate=100, record 250 bytes -> 2 samples, counter 50 afterwards
    s, off = oracle.rate_replay(_events([("a", 1, 250, 3)]), [0, 1], 100, 0)
    assert len(s) == 2 and list(s["idx"]) == [0, 0] and list(s["draw_sum"]) == [100, 200]
    assert list(s["site"]) == [3, 3]
    # 0 counted bytes -> 0 samples (copies do not count for the alloc/free sampler)
    s, _ = oracle.rate_replay(_events([("c", 0, 500, 0), ("c", 0, 900, 1)]), [0, 2], 100, 0)
    assert len(s) == 0


def test_deterministic_count_closed_form_and_split_invariance():
    """Counter = R after every sample: over B counted bytes the count is floor((B - 1) / R)
    ("drops below 0" is strict: B = 200, R = 100 gives 1), whatever the split into events."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        R = int(rng.integers(1, 500))
        sizes = rng.integers(1, 3 * R + 2, size=int(rng.integers(1, 30)))
        B = int(sizes.sum())
        ev = _events([("a", 16 * (i + 1), int(z), 0) for i, z in enumerate(sizes)])
        s, _ = oracle.rate_replay(ev, [0, len(sizes)], R, 0)
        assert len(s) == (B - 1) // R
        ev1 = _events([("a", 16, B, 0)])                         # the same bytes in one event
        s1, _ = oracle.rate_replay(ev1, [0, 1], R, 0)
        assert len(s1) == len(s)
    s, _ = oracle.rate_replay(_events([("a", 1, 200, 0)]), [0, 1], 100, 0)
    assert len(s) == 1


def test_positions_match_prefix_formulation():
    """Sample k fires at the first event j with A_j > S_k (A: counted-byte prefix sum, S: draw
    prefix sum) -- the countdown of P:421-427 restated without a counter."""
    rng = np.random.default_rng(11)
    for trial in range(40):
        n = int(rng.integers(1, 3000))
        tr = tracegen.random_small_trace(rng, n, n_sites=9, max_size=int(rng.integers(1, 5000)), max_ptrs=20)
        tr = [e if rng.random() > 0.1 else ("c", 0, int(rng.integers(1, 4000)), e[3]) for e in tr]
        ev = _events(tr)
        R, seed, t = int(rng.integers(1, 3000)), int(rng.integers(1, 2**40)), trial
        for kinds in (oracle.KINDS_ALLOC_FREE, oracle.KINDS_COPY):
            s = _as_trace(ev, n, R, seed, kinds, t)
            kind = (ev["meta"] >> np.uint64(40)) & np.uint64(3)
            counted = np.isin(kind.astype(np.int64), [k for k in range(3) if (kinds >> k) & 1])
            size = np.where(counted, ev["meta"] & np.uint64((1 << 40) - 1), 0).astype(np.int64)
            A = np.cumsum(size)
            K = len(s)
            S = np.cumsum([oracle.rate_draw(R, seed, t, k) for k in range(1, K + 2)])
            assert K == int(np.searchsorted(S, A[-1], side="left")) if n else K == 0   # S_k < A_n
            for k in range(K):
                j = int(np.searchsorted(A, S[k], side="right"))                      # first A_j > S_k
                assert s["idx"][k] == j and s["draw_sum"][k] == S[k]


def _as_trace(ev, n, R, seed, kinds, t):
    """The rate samples of `ev` replayed as trace t of a batch (draws are keyed by the trace id;
    traces 0..t-1 are one copy event each)."""
    pad = _events([("c", 0, 1, 0)])
    evs = np.concatenate([pad] * t + [ev])
    off = list(range(t + 1)) + [t + n]
    s, so = oracle.rate_replay(evs, off, R, seed, kinds)
    return s[int(so[t]):int(so[t + 1])]


def test_rate_one_samples_every_byte_but_the_first():
    s, _ = oracle.rate_replay(_events([("a", 1, 5, 0), ("f", 1, 5, 1)]), [0, 2], 1, 99)
    assert len(s) == 9 and list(s["idx"]) == [0] * 4 + [1] * 5


def test_geometric_draws_moments():
    """G ~ geometric(1/R) on {1, 2, ...}: mean R, P(G <= x) = 1 - (1 - 1/R)^x."""
    for R in (4, 1000, 10485767):
        g = np.array([oracle.rate_draw(R, 12345, 7, k) for k in range(1, 60001)], dtype=np.float64)
        sd = math.sqrt(R * (R - 1)) if R > 1 else 0
        assert abs(g.mean() - R) < 5 * sd / math.sqrt(len(g))
        for q in (0.1, 0.5, 0.9):
            x = math.log(1 - q) / math.log(1 - 1 / R)
            frac = float((g <= x).mean())
            assert abs(frac - (1 - (1 - 1 / R) ** math.floor(x))) < 0.015
    assert {oracle.rate_draw(R, 0, 5, 9) for R in (1, 7, 10**9)} == {1, 7, 10**9}
    assert oracle.rate_draw(1, 77, 0, 1) == 1


def test_threshold_vs_rate_on_config1():
    """The paper's comparison (Table tab:sampling-comparison): on a trace the rate sampler at
    R = T takes several times more samples than the threshold sampler."""
    cfg = tracegen.CONFIGS[1]
    ev, off = tracegen.generate(cfg)
    thr = oracle.replay(ev, off, cfg.n_sites, cfg.T)
    rs, _ = oracle.rate_replay(ev, off, cfg.T, 2022)
    assert len(rs) > 2 * len(thr.samples)
