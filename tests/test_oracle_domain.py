"""Pins of the per-sample Python/native split ("the fraction of
Python (vs. native) allocations in the total sample"; managed bytes / max(
allocated bytes, 1) since the last reset, frees excluded): a hand-worked trace, conservation of
allocated bytes, and the independent A/F-counter transcription (oracle/mini.py)."""
import numpy as np

import oracle
import tracegen
from oracle import mini


def _run(tuples, T):
    ev = tracegen.from_tuples(tuples)
    n_sites = max(e[3] for e in tuples) + 1
    return oracle.replay(ev, np.array([0, len(ev)], dtype=np.uint64), n_sites, T)


def test_hand_worked():
    # T = 8: a5(managed) a2 f2 a4(managed) -> growth at event 3 (c = 9): A = 11, managed 9;
    # f5 f4 -> decline at event 5 (c = -9): nothing allocated since the reset -> (0, 0);
    # a16 (native) -> growth at event 6: (16, 0)
    tr = [("a", 1, 5, 0, 1), ("a", 2, 2, 1, 0), ("f", 2, 2, 1), ("a", 3, 4, 0, 1),
          ("f", 1, 5, 0), ("f", 3, 4, 0), ("a", 4, 16, 2, 0)]
    r = _run(tr, 8)
    assert list(r.samples["idx"]) == [3, 5, 6]
    assert [tuple(d) for d in r.domains] == [(11, 9), (0, 0), (16, 0)]


def test_conservation_and_bounds():
    cfg = tracegen.CONFIGS[2].with_traces(3)
    ev, off = tracegen.generate(cfg)
    r = oracle.replay(ev, off, cfg.n_sites, 1048583)
    kind = ((ev["meta"] >> np.uint64(40)) & np.uint64(3)).astype(np.int64)
    dom = ((ev["meta"] >> np.uint64(42)) & np.uint64(1)).astype(bool)
    size = (ev["meta"] & np.uint64((1 << 40) - 1)).astype(np.int64)
    assert (r.domains["managed_bytes"] <= r.domains["alloc_bytes"]).all()
    for t in range(cfg.n_traces):
        b, e = int(off[t]), int(off[t + 1])
        s = r.trace_samples(t)
        d = r.domains[int(r.sample_off[t]):int(r.sample_off[t + 1])]
        last = int(s["idx"][-1])
        alloc = (kind[b:e] == 0)
        tail = slice(last + 1, e - b)
        assert int(d["alloc_bytes"].sum()) + int(size[b:e][tail][alloc[tail]].sum()) == int(size[b:e][alloc].sum())
        man = alloc & dom[b:e]
        assert int(d["managed_bytes"].sum()) + int(size[b:e][tail][man[tail]].sum()) == int(size[b:e][man].sum())
    assert 0 < r.domains["managed_bytes"].sum() < r.domains["alloc_bytes"].sum()


def test_matches_mini_transcription():
    rng = np.random.default_rng(8)
    for _ in range(300):
        n = int(rng.integers(1, 120))
        tr = tracegen.random_small_trace(rng, n, n_sites=5, max_size=int(rng.integers(1, 40)), max_ptrs=8)
        tr = [e + (int(rng.integers(0, 2)),) if e[0] == "a" else e for e in tr]
        T = int(rng.integers(1, 30))
        r = _run(tr, T)
        ms, _, _, md = mini.replay_trace(tr, T, with_domains=True)
        assert list(r.samples["idx"]) == [x[0] for x in ms]
        assert [tuple(int(v) for v in d) for d in r.domains] == md
