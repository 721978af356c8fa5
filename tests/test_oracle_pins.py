"""Pins for the CPU oracle (``-m "not gpu"``): the oracle is checked against
things other than itself -- hand-worked traces (tests/golden, each citing
PAPER.md), a brute-force first-exit formulation of the sampler, a death-time
formulation of the leak tracker, closed forms, invariants, exact rational
arithmetic and trial division.  A dropped term, wrong sign/index or swapped
operand anywhere in oracle.c fails at least one of these.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import tracegen
from oracle import mini
import _golden

SIZE_MASK = (1 << 40) - 1


# ----------------------------------------------------------------------------- helpers
def run_oracle(events, T, hwm_mode=oracle.HWM_PREFIX, n_sites=None):
    ev = tracegen.from_tuples(events)
    n_sites = n_sites or (max((e[3] for e in events), default=0) + 1)
    off = np.array([0, len(events)], dtype=np.uint64)
    return oracle.replay(ev, off, n_sites, T, hwm_mode)


def as_tuples(samples):
    return [(int(s["idx"]), "G" if s["kind"] == 0 else "D", int(s["net"]), int(s["footprint"]),
             int(s["site"]), bool(s["new_max"])) for s in samples]


def signed(events):
    return [(s if k == "a" else -s) for k, _, s, _ in events]


def first_exit_samples(events, T):
    """Independent formulation of the threshold sampler:
    s_1 = min{j : |F_j| >= T}, s_{k+1} = min{j > s_k : |F_j - F_{s_k}| >= T}.
    O(n^2); returns [(j, net)]."""
    F = list(itertools.accumulate(signed(events)))
    out, B, j0 = [], 0, -1
    while True:
        nxt = next((j for j in range(j0 + 1, len(F)) if abs(F[j] - B) >= T), None)
        if nxt is None:
            return out
        out.append((nxt, F[nxt] - B))
        B, j0 = F[nxt], nxt


def leak_scores_by_death(events, samples):
    """Independent formulation of the leak score (readings Q5-Q7):
    episode e starts at a new-max growth sample (the tracked object is that
    alloc) and ends at the next one or at trace end; reclaimed_e iff the
    tracked object's own free (its death: the first later free of the same
    pointer) comes before the episode ends."""
    starts = [s[0] for s in samples if s[5]]
    ends = starts[1:] + [len(events)]
    m, f = {}, {}
    for a, b in zip(starts, ends):
        ptr, site = events[a][1], events[a][3]
        death = next((j for j in range(a + 1, len(events)) if events[j][0] == "f" and events[j][1] == ptr),
                     math.inf)
        m[site] = m.get(site, 0) + 1
        f[site] = f.get(site, 0) + (1 if death < b else 0)
    return m, f


def enumerate_traces(max_len, sizes=(1, 2, 3)):
    """All traces up to max_len: an alloc of each size (at the smallest
    pointer id not live, so addresses are reused) or a free of any live
    object; the site of event i is i % 3."""
    out = []

    def rec(prefix, live):
        if prefix:
            out.append(list(prefix))
        if len(prefix) == max_len:
            return
        i = len(prefix)
        p = min(set(range(1, len(live) + 2)) - set(live))
        for s in sizes:
            rec(prefix + [("a", p, s, i % 3)], {**live, p: s})
        for q, s in sorted(live.items()):
            nl = dict(live)
            del nl[q]
            rec(prefix + [("f", q, s, i % 3)], nl)

    rec([], {})
    return out


# ----------------------------------------------------------------------------- golden (hand-worked)
@pytest.mark.parametrize("name", _golden.all_names())
def test_golden_c_oracle(name):
    g = _golden.load(name)
    mode = oracle.HWM_SAMPLE if g["hwm"] == "sample" else oracle.HWM_PREFIX
    n_sites = max(max(e[3] for e in g["events"]) + 1, max(g["sites"], default=0) + 1)
    r = run_oracle(g["events"], g["T"], mode, n_sites)
    assert as_tuples(r.trace_samples(0)) == g["samples"]
    for k, v in g["summary"].items():
        assert int(r.summaries[0][k]) == v, k
    for s, cols in g["sites"].items():
        for k, v in cols.items():
            assert int(r.site_table[s, oracle.COLS.index(k)]) == v, (s, k)
    if g["gate"]:
        num, den, op = oracle.gate(r.summaries)
        assert (num, den, int(op)) == (g["gate"]["num"], g["gate"]["den"], g["gate"]["open"])
    if g["probs"]:
        prob, _, _ = oracle.finalize(r.site_table, True, 10**9)
        for s, p in g["probs"].items():
            assert prob[s] == p


@pytest.mark.parametrize("name", _golden.all_names())
def test_golden_mini_oracle(name):
    g = _golden.load(name)
    samples, summ, cols = mini.replay_trace(g["events"], g["T"], g["hwm"])
    assert samples == g["samples"]
    for k, v in g["summary"].items():
        assert summ[k] == v, k
    for s, c in g["sites"].items():
        for k, v in c.items():
            assert cols[s][k] == v, (s, k)


# ----------------------------------------------------------------------------- SPEC examples
def test_spec_sampler_examples():
    # T=8: alloc 5 then alloc 4 -> one growth sample, net 9
    r = run_oracle([("a", 1, 5, 0), ("a", 2, 4, 0)], 8)
    assert as_tuples(r.trace_samples(0)) == [(1, "G", 9, 9, 0, True)]
    # (alloc 3, free 3) x 1000 -> 0 samples (P:440-447 churn filtering)
    ev = []
    for i in range(1000):
        ev += [("a", 7, 3, 0), ("f", 7, 3, 1)]
    r = run_oracle(ev, 8)
    assert int(r.summaries[0]["n_samples"]) == 0 and int(r.summaries[0]["hwm"]) == 3
    # one 512 MB alloc at T = 1 MiB -> exactly one sample, peak exact
    r = run_oracle([("a", 1, 512 << 20, 0)], tracegen.P_1MIB)
    assert as_tuples(r.trace_samples(0)) == [(0, "G", 512 << 20, 512 << 20, 0, True)]
    assert int(r.summaries[0]["hwm"]) == 512 << 20
    # staircase of k allocs of T -> footprints T, 2T, ..., kT, all new maxima
    T, k = 1009, 25
    r = run_oracle([("a", i + 1, T, 0) for i in range(k)], T)
    s = r.trace_samples(0)
    assert list(s["footprint"]) == [T * (i + 1) for i in range(k)]
    assert all(s["new_max"]) and int(r.site_table[0, oracle.COLS.index("leak_mallocs")]) == k


def test_staircase_closed_form():
    """Staircase of s < T: samples at j = r*ceil(T/s) - 1 with net ceil(T/s)*s (W4)."""
    for s, T, k in [(3, 10, 40), (7, 50, 300), (1, 4, 33), (5, 5, 20)]:
        r = run_oracle([("a", i + 1, s, 0) for i in range(k)], T)
        q = -(-T // s)
        exp = [(r_ * q - 1, q * s) for r_ in range(1, k // q + 1)]
        got = [(int(x["idx"]), int(x["net"])) for x in r.trace_samples(0)]
        assert got == exp
    # W4: s=3, T=10, k=40 -> score (10, 0), p = 1 - 1/12
    r = run_oracle([("a", i + 1, 3, 0) for i in range(40)], 10)
    col = oracle.COLS.index
    assert (int(r.site_table[0, col("leak_mallocs")]), int(r.site_table[0, col("leak_frees")])) == (10, 0)
    prob, _, _ = oracle.finalize(r.site_table, True, 10**9)
    assert abs(Fraction(prob[0]) - Fraction(11, 12)) <= Fraction(1, 2**52)


def test_sync_event_forces_sample():
    """W5: any event with |d| >= 2T-1 samples whatever the incoming carry
    c in [-(T-1), T-1], because |c + d| >= T."""
    T = 9
    for c in range(-(T - 1), T):
        for d in (2 * T - 1, 2 * T + 5):
            for sign in (1, -1):
                if c >= 0:
                    evs = [("a", 1, d, 0)] + ([("a", 2, c, 1)] if c else [])
                else:
                    evs = [("a", 2, -c, 1), ("a", 1, d, 0), ("f", 2, -c, 1)]
                # one sample so far (at the alloc of d); the carry is now c
                evs += [("a", 3, d, 2)] if sign > 0 else [("f", 1, d, 2)]
                s = run_oracle(evs, T).trace_samples(0)
                assert len(s) == 2 and int(s["idx"][-1]) == len(evs) - 1
                assert int(s["net"][-1]) == c + sign * d


# ----------------------------------------------------------------------------- brute force
def _check_against_brute(trace, T, r_samples):
    got = [(int(x["idx"]), int(x["net"])) for x in r_samples]
    assert got == first_exit_samples(trace, T)
    F = list(itertools.accumulate(signed(trace)))
    for x in r_samples:
        j = int(x["idx"])
        assert int(x["footprint"]) == F[j]
        assert (x["kind"] == 0) == (trace[j][0] == "a")            # growth <=> alloc
        assert int(x["site"]) == trace[j][3]
        prev_max = max([0] + F[:j])
        assert bool(x["new_max"]) == (x["kind"] == 0 and F[j] > prev_max)


def test_enumerated_traces_brute_force():
    traces = enumerate_traces(6)
    assert len(traces) > 5000
    for T in (1, 2, 3, 4):
        ev = tracegen.from_tuples([e for tr in traces for e in tr])
        off = np.zeros(len(traces) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(t) for t in traces])
        r = oracle.replay(ev, off, 3, T)
        M, Fr = [0, 0, 0], [0, 0, 0]                  # death-time leak scores summed over EVERY trace
        for t, tr in enumerate(traces):
            smp = r.trace_samples(t)
            _check_against_brute(tr, T, smp)
            m, f = leak_scores_by_death(tr, as_tuples(smp))
            for s in range(3):
                M[s] += m.get(s, 0)
                Fr[s] += f.get(s, 0)
            # per-trace leak score: recompute from a single-trace replay
            rt = run_oracle(tr, T, n_sites=3) if t % 7 == 0 else None
            if rt is not None:
                for s in range(3):
                    assert int(rt.site_table[s, 8]) == m.get(s, 0)
                    assert int(rt.site_table[s, 9]) == f.get(s, 0)
        # the batched replay's leak columns are the sums of the independent per-trace scores
        assert [int(x) for x in r.site_table[:, 8]] == M and [int(x) for x in r.site_table[:, 9]] == Fr
        assert sum(M) > 0 and sum(Fr) > 0


def test_random_traces_brute_force_and_mini():
    rng = np.random.default_rng(20221215)
    for it in range(1500):
        n = int(rng.integers(1, 60))
        tr = tracegen.random_small_trace(rng, n, n_sites=4, max_size=int(rng.integers(1, 40)))
        T = int(rng.integers(1, 30))
        r = run_oracle(tr, T, n_sites=4)
        smp = r.trace_samples(0)
        _check_against_brute(tr, T, smp)
        m, f = leak_scores_by_death(tr, as_tuples(smp))
        for s in range(4):
            assert int(r.site_table[s, 8]) == m.get(s, 0)
            assert int(r.site_table[s, 9]) == f.get(s, 0)
        ms, msum, mcols = mini.replay_trace(tr, T)
        assert ms == as_tuples(smp)
        for s in range(4):
            for k, c in enumerate(oracle.COLS):
                assert mcols[s][c] == int(r.site_table[s, k]), (s, c)
        # SAMPLE reading cross-check between the two transcriptions
        r2 = run_oracle(tr, T, oracle.HWM_SAMPLE, n_sites=4)
        ms2, _, _ = mini.replay_trace(tr, T, "sample")
        assert ms2 == as_tuples(r2.trace_samples(0))


# ----------------------------------------------------------------------------- invariants on generated traces
@pytest.fixture(scope="module")
def gen_small():
    cfg = tracegen.CONFIGS[2].with_traces(3)
    ev, off = tracegen.generate(cfg)
    ev1, off1 = tracegen.generate(tracegen.CONFIGS[1])
    return [(cfg, ev, off), (tracegen.CONFIGS[1], ev1, off1)]


def test_invariants_generated(gen_small):
    for cfg, ev, off in gen_small:
        assert oracle.validate(ev, off, cfg.n_sites) is None
        for T in (cfg.T, 65537, 4099):
            r = oracle.replay(ev, off, cfg.n_sites, T, n_threads=4)
            meta = ev["meta"]
            size = (meta & np.uint64(SIZE_MASK)).astype(np.int64)
            kind = ((meta >> np.uint64(40)) & np.uint64(3)).astype(np.int64)
            site = (meta >> np.uint64(43)).astype(np.int64)
            d = np.where(kind == 0, size, -size)
            tab = np.zeros((cfg.n_sites, 10), dtype=np.int64)
            for t in range(len(off) - 1):
                b, e = int(off[t]), int(off[t + 1])
                F = np.cumsum(d[b:e])
                s = r.trace_samples(t)
                sm = r.summaries[t]
                assert int(sm["f_final"]) == int(d[b:e].sum())                 # final footprint = sum d
                assert int(sm["hwm"]) == max(0, int(F.max()))                   # prefix max
                assert len(s) <= int(np.abs(d[b:e]).sum()) // T                 # sample bound
                net = s["net"].astype(np.int64)
                idx = s["idx"].astype(np.int64)
                assert np.all(np.abs(net) >= T)
                assert np.all(np.abs(net) <= T - 1 + np.abs(d[b:e][idx]))
                assert int(net.sum()) == (int(s["footprint"][-1]) if len(s) else 0)
                assert np.all(s["footprint"] == F[idx])
                if len(s):
                    assert abs(int(sm["f_final"]) - int(s["footprint"][-1])) < T  # reconstruction
                    assert s["kind"][0] == 0 and s["new_max"][0] == 1
                assert np.all((s["kind"] == 0) == (kind[b:e][idx] == 0))
                assert int(s["new_max"].sum()) == int(sm["n_episodes"])
                # Tier S recomputed from the samples
                g = s["kind"] == 0
                tab[:, 4] += np.bincount(s["site"][g], minlength=cfg.n_sites)
                tab[:, 5] += np.bincount(s["site"][~g], minlength=cfg.n_sites)
                tab[:, 6] += np.bincount(s["site"][g], weights=net[g], minlength=cfg.n_sites).astype(np.int64)
                tab[:, 7] += np.bincount(s["site"][~g], weights=-net[~g], minlength=cfg.n_sites).astype(np.int64)
            # Tier E by bincount over all events
            a, f = kind == 0, kind == 1
            tab[:, 0] = np.bincount(site[a], minlength=cfg.n_sites)
            tab[:, 1] = np.bincount(site[f], minlength=cfg.n_sites)
            tab[:, 2] = np.bincount(site[a], weights=size[a], minlength=cfg.n_sites).astype(np.int64)
            tab[:, 3] = np.bincount(site[f], weights=size[f], minlength=cfg.n_sites).astype(np.int64)
            assert np.array_equal(tab[:, :8], r.site_table[:, :8].astype(np.int64))
            lm, lf = r.site_table[:, 8], r.site_table[:, 9]
            assert np.all(lf <= lm)
            assert int(lm.sum()) == int(r.summaries["n_episodes"].sum())


def test_planted_leaks_flagged():
    """North star: every planted leak reaches probability > 0.95 (generator
    calibration, checked with the oracle) on configs 1 and 2."""
    for cid, nt in ((1, None), (2, None)):
        cfg = tracegen.CONFIGS[cid]
        if nt:
            cfg = cfg.with_traces(nt)
        ev, off = tracegen.generate(cfg)
        out = oracle.full(ev, off, cfg.n_sites, cfg.T, n_threads=8)
        pl = tracegen.planted_sites(cfg)
        assert len(pl) == cfg.n_planted
        assert out["gate"][2]
        assert np.all(out["flag"][pl] == 1), (cid, out["result"].site_table[pl, 8:])
        assert np.all(out["prob"][pl] > 0.95)


def test_generator_deterministic_subsets():
    cfg = tracegen.CONFIGS[2].with_traces(6)
    ev, _ = tracegen.generate(cfg, n_threads=3)
    ev2, _ = tracegen.generate(cfg, 4, 6, n_threads=1)
    assert np.array_equal(ev[4 * cfg.events_per_trace:], ev2)


# ----------------------------------------------------------------------------- formula, flag, rate, gate, order
def _exact_p(m, f):
    return 1 - Fraction(f + 1, m - f + 2)


def test_formula_closed_form():
    tab = np.zeros((4, 10), dtype=np.uint64)
    for s, (m, f) in enumerate([(1, 0), (19, 0), (18, 0), (2, 2)]):
        tab[s, 8], tab[s, 9] = m, f
    prob, _, flag = oracle.finalize(tab, True, 10**9)
    ulp = Fraction(1, 2**52)
    assert abs(Fraction(prob[0]) - Fraction(2, 3)) <= ulp          # (1,0) -> 2/3
    assert abs(Fraction(prob[1]) - Fraction(20, 21)) <= ulp        # (19,0) -> 20/21
    assert abs(Fraction(prob[2]) - Fraction(19, 20)) <= ulp and flag[2] == 0   # (18,0): 0.95, excluded
    assert flag[1] == 1 and flag[0] == 0
    assert prob[3] == -0.5                                          # unclamped (reading Q8)
    _, _, flag_closed = oracle.finalize(tab, False, 10**9)
    assert not flag_closed.any()                                    # gate closed -> nothing reported


def test_rate_closed_form_and_zero_elapsed():
    """Rate (Q11): malloc bytes in MB over elapsed seconds; 3 MiB over 2 s = 1.5 MB/s.
    Elapsed 0 only happens with every trace empty (no bytes anywhere): rate 0 (reading Q20)."""
    tab = np.zeros((2, 10), dtype=np.uint64)
    tab[0, 2] = 3 << 20
    _, rate, _ = oracle.finalize(tab, True, 2 * 10**9)
    assert rate[0] == 1.5 and rate[1] == 0.0
    _, rate0, _ = oracle.finalize(np.zeros((2, 10), dtype=np.uint64), True, 0)
    assert np.array_equal(rate0, [0.0, 0.0])


def test_formula_grid_exact():
    pairs = [(m, f) for m in range(0, 101) for f in range(0, m + 1)]
    tab = np.zeros((len(pairs), 10), dtype=np.uint64)
    tab[:, 8] = [m for m, _ in pairs]
    tab[:, 9] = [f for _, f in pairs]
    prob, _, flag = oracle.finalize(tab, True, 10**9)
    _, _, flag_tb = oracle.finalize(tab, True, 10**9, oracle.FORMULA_TEXTBOOK)
    ptb, _, _ = oracle.finalize(tab, True, 10**9, oracle.FORMULA_TEXTBOOK)
    for k, (m, f) in enumerate(pairs):
        ex = _exact_p(m, f)
        # two IEEE roundings (a/b, then 1 - q): error <= (|q| + |p|) 2^-53
        assert abs(Fraction(prob[k]) - ex) <= Fraction(1, 2**51) * max(1, abs(ex))
        assert bool(flag[k]) == (ex > Fraction(95, 100))
        tb = 1 - Fraction(f + 1, m + 2)
        assert abs(Fraction(ptb[k]) - tb) <= Fraction(1, 2**51) * max(1, abs(tb))
        assert bool(flag_tb[k]) == (tb > Fraction(95, 100))
        assert prob[k] < 1.0
        assert (prob[k] < 0) == (2 * f > m + 1)
    grid = {p: prob[k] for k, p in enumerate(pairs)}
    for (m, f), p in grid.items():                                  # monotonicity
        if (m + 1, f) in grid:
            assert grid[(m + 1, f)] >= p
        if (m, f + 1) in grid:
            assert grid[(m, f + 1)] <= p


def test_flag_identity_large():
    """m > 21 f + 18 <=> exact p > 0.95, also for large counters."""
    rng = np.random.default_rng(7)
    fs = rng.integers(0, 2**40, 2000, dtype=np.int64)
    ms = fs + 21 * fs + 18 + rng.integers(-3, 4, 2000)
    ms = np.maximum(ms, fs)
    tab = np.zeros((2000, 10), dtype=np.uint64)
    tab[:, 8], tab[:, 9] = ms, fs
    _, _, flag = oracle.finalize(tab, True, 10**9)
    for k in range(2000):
        assert bool(flag[k]) == (_exact_p(int(ms[k]), int(fs[k])) > Fraction(95, 100))


def test_rate_closed_form():
    tab = np.zeros((3, 10), dtype=np.uint64)
    tab[0, 2] = 100 << 20          # 100 MiB over 10 s -> 10.0 MB/s
    tab[2, 2] = 3 << 20
    _, rate, _ = oracle.finalize(tab, True, 10 * 10**9)
    assert rate[0] == 10.0 and rate[1] == 0.0 and rate[2] == 0.3


def test_gate_rules():
    S = np.zeros(3, dtype=oracle.SUMMARY_DTYPE)
    S["n_samples"] = [5, 1, 2]
    S["f_first_sample"] = [100, 50, 200]
    S["f_last_sample"] = [101, 999, 202]
    num, den, op = oracle.gate(S)
    assert (num, den) == (1 + 2, 300) and op                       # trace 1 (<2 samples) excluded
    S["f_last_sample"] = [100, 999, 202]
    assert oracle.gate(S) == (2, 300, False)                        # 200 < 300
    S["n_samples"] = [1, 0, 1]
    assert oracle.gate(S)[2] is False                               # nothing qualifies -> closed


def test_report_order():
    rate = np.array([1.0, 5.0, 5.0, 0.5, 9.0, 2.0])
    flag = np.array([1, 1, 1, 0, 0, 1], dtype=np.uint8)
    order = oracle.report_order(rate, flag)
    assert list(order) == [1, 2, 5, 0, 3, 4]


# ----------------------------------------------------------------------------- constants, validation
def _is_prime(x):
    return x >= 2 and all(x % q for q in range(2, int(math.isqrt(x)) + 1))


def test_next_prime_table():
    table = {2**16: 65537, 2**17: 131101, 2**18: 262147, 2**19: 524309, 2**20: 1048583,
             2**21: 2097169, 2**22: 4194319, 2**23: 8388617, 2**24: 16777259, 2**25: 33554467,
             2**26: 67108879, 10 * 2**20: 10485767, 10**7: 10000019}
    for base, p in table.items():
        got = oracle.next_prime(base)
        assert got == p and _is_prime(got)
        assert not any(_is_prime(x) for x in range(base, got))
    assert tracegen.P_10MIB == table[10 * 2**20] and tracegen.P_1MIB == table[2**20]
    assert tracegen.SWEEP == tuple(table[2**k] for k in range(16, 27))
    assert [oracle.next_prime(x) for x in (0, 1, 2, 10, 13)] == [2, 2, 2, 11, 13]


def test_validation():
    good = [("a", 1, 8, 0), ("a", 2, 4, 1), ("f", 1, 8, 0), ("a", 1, 3, 0)]
    ev = tracegen.from_tuples(good)
    off = np.array([0, len(good)], dtype=np.uint64)
    assert oracle.validate(ev, off, 2) is None
    for bad, idx in [(good + [("f", 9, 8, 0)], 4),                  # free of a non-live pointer
                     (good + [("f", 2, 5, 0)], 4),                  # size mismatch
                     (good + [("a", 2, 5, 0)], 4),                  # pointer already live
                     (good[:2] + [("a", 3, 1, 5)], 2)]:             # site >= n_sites
        ev = tracegen.from_tuples(bad)
        off = np.array([0, len(bad)], dtype=np.uint64)
        assert oracle.validate(ev, off, 2) == (0, idx)
