"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by
element, on seeded synthetic inputs shaped like the paper's workloads."""
import os
import tempfile

import numpy as np
import pytest

import _golden
import oracle
import paper_2212_07597_b200 as scl
import tracegen
from parity import compare, gpu_run

pytestmark = pytest.mark.gpu


def _concat(traces):
    """list of lists of (kind, ptr, size, site) -> events, offsets"""
    ev = tracegen.from_tuples([e for tr in traces for e in tr])
    off = np.zeros(len(traces) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in traces])
    return ev, off


@pytest.mark.parametrize("name", _golden.all_names())
def test_golden(name):
    g = _golden.load(name)
    hwm = scl.HWM_PREFIX if g["hwm"] == "prefix" else scl.HWM_SAMPLE
    n_sites = max(max(e[3] for e in g["events"]) + 1, max(g["sites"], default=0) + 1)
    ev, off = _concat([g["events"]])
    _, r = gpu_run(ev, off, n_sites, g["T"], hwm_mode=hwm)
    smp = scl.scl_samples(r, 0)
    got = [(int(s["idx"]), "G" if s["kind"] == 0 else "D", int(s["net"]), int(s["footprint"]), int(s["site"]),
            bool(s["new_max"])) for s in smp]
    assert got == g["samples"]
    compare(ev, off, n_sites, g["T"], r, hwm_mode=hwm)


def test_random_small_ragged():
    """Hundreds of small random traces of ragged lengths (incl. empty ones and
    lengths that straddle rows, threads and segments) at several T."""
    rng = np.random.default_rng(1)
    traces = []
    for i in range(400):
        n = int(rng.choice([0, 1, 3, 7, 8, 9, 31, 255, 256, 257, 2047, 2048, 2049, 5000, 8191, 8192, 8193,
                            16385, 40000, int(rng.integers(1, 9000))]))
        traces.append(tracegen.random_small_trace(rng, n, n_sites=37, max_size=int(rng.integers(1, 200)),
                                                  max_ptrs=int(rng.integers(2, 40))))
    ev, off = _concat(traces)
    tr = scl.scl_trace_load(ev, off, 37, validate=True)
    r = None
    for T in (1, 2, 7, 64, 401, 5000, 10**9):
        r = scl.scl_replay_run(T, tr, out=r)
        compare(ev, off, 37, T, r)


def test_config1():
    cfg = tracegen.CONFIGS[1]
    ev, off = tracegen.generate(cfg)
    _, r = gpu_run(ev, off, cfg.n_sites, cfg.T, validate=True)
    ref = compare(ev, off, cfg.n_sites, cfg.T, r)
    pl = tracegen.planted_sites(cfg)
    rows = scl.scl_site_report(r)
    flagged = set(rows["site"][rows["leak_flag"] == 1].tolist())
    assert set(pl.tolist()) <= flagged and ref["gate"][2]


def test_config2_full():
    """BASELINE configs[1] at full size (64 x 1M events) -- the bench workload."""
    cfg = tracegen.CONFIGS[2]
    ev, off = tracegen.generate(cfg)
    tr, r = gpu_run(ev, off, cfg.n_sites, cfg.T)
    compare(ev, off, cfg.n_sites, cfg.T, r)
    # same handle, smaller thresholds (dense samples, many episodes, P:436-438 sweep values)
    for T in (1048583, 65537):
        r = scl.scl_replay_run(T, tr, out=r)
        compare(ev, off, cfg.n_sites, T, r)


def test_config2_small_T_subset():
    cfg = tracegen.CONFIGS[2].with_traces(4)
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = None
    for T in (4099, 521, 16):
        r = scl.scl_replay_run(T, tr, out=r)
        compare(ev, off, cfg.n_sites, T, r)


def test_config3_subset_cold_sites():
    """50k sites (most beyond the shared-memory hot range) on 24 traces of config 3."""
    cfg = tracegen.CONFIGS[3].with_traces(24)
    ev, off = tracegen.generate(cfg)
    _, r = gpu_run(ev, off, cfg.n_sites, cfg.T)
    compare(ev, off, cfg.n_sites, cfg.T, r)


def test_huge_sizes_and_copies():
    """Sizes >= 2^32 (L2 reduction path), 32-bit byte-counter carries, copy events (ignored)."""
    rng = np.random.default_rng(5)
    traces = []
    for t in range(20):
        tr_ = []
        live = []
        for i in range(3000):
            if live and rng.random() < 0.4:
                p, s = live.pop(int(rng.integers(len(live))))
                tr_.append(("f", p, s, int(rng.integers(0, 3))))
            elif rng.random() < 0.1:
                tr_.append(("c", 0, int(rng.integers(1, 1 << 30)), 2))
            else:
                s = int(rng.choice([16, 4096, (1 << 31) + 17, (1 << 33) + 5, (1 << 39) + 3]))
                p = 0x1000 + 0x10000000000 * i
                live.append((p, s))
                tr_.append(("a", p, s, int(rng.integers(0, 3))))
        traces.append(tr_)
    ev, off = _concat(traces)
    for T in (1 << 20, (1 << 34) + 7):
        _, r = gpu_run(ev, off, 3, T)
        compare(ev, off, 3, T, r)


def test_reuse_and_textbook_and_ticks():
    cfg = tracegen.CONFIGS[1]
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = None
    for it in range(3):
        r = scl.scl_replay_run(cfg.T, tr, out=r)
        compare(ev, off, cfg.n_sites, cfg.T, r)
    r = scl.scl_replay_run(cfg.T, tr, out=r, formula=1, tick_ns=777)
    compare(ev, off, cfg.n_sites, cfg.T, r, formula=1, tick_ns=777)


def test_device_pointers_and_file():
    import torch
    cfg = tracegen.CONFIGS[2].with_traces(3)
    ev, off = tracegen.generate(cfg)
    dev_ev = torch.from_numpy(ev.view(np.int64).copy()).cuda()
    dev_off = torch.from_numpy(off.view(np.int64).copy()).cuda()
    tr = scl.scl_trace_load(dev_ev, dev_off, cfg.n_sites)
    r = scl.scl_replay_run(cfg.T, tr)
    ref = compare(ev, off, cfg.n_sites, cfg.T, r)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "t.scltrc")
        scl.write_trace_file(path, ev, off, cfg.n_sites)
        tr2 = scl.scl_trace_load(path=path)
        r2 = scl.scl_replay_run(cfg.T, tr2)
        compare(ev, off, cfg.n_sites, cfg.T, r2, ref=ref)


def test_errors():
    ev = tracegen.from_tuples([("a", 1, 8, 0), ("f", 2, 8, 0)])
    off = np.array([0, 2], dtype=np.uint64)
    with pytest.raises(scl.SclError) as e:
        scl.scl_trace_load(ev, off, 1, validate=True)
    assert e.value.status == -4 and "trace 0 event 1" in str(e.value)
    with pytest.raises(scl.SclError) as e:
        scl.scl_trace_load(ev, off, 1, validate=False).n_sites
        scl.scl_trace_load(tracegen.from_tuples([("a", 1, 8, 3)]), np.array([0, 1], dtype=np.uint64), 2)
    assert e.value.status == -1
    tr = scl.scl_trace_load(tracegen.from_tuples([("a", 1, 8, 0)]), np.array([0, 1], dtype=np.uint64), 1)
    with pytest.raises(scl.SclError):
        scl.scl_replay_run(0, tr)


def test_defer_finalize_table_sum():
    """Two 'ranks' (halves of the traces) on one GPU: summing their device
    tables element-wise then finalizing equals the single-run report (the
    multi-GPU reduction of SURVEY §8(e), exercised without a second GPU)."""
    import torch
    cfg = tracegen.CONFIGS[2].with_traces(8)
    ev, off = tracegen.generate(cfg)
    h = int(off[4])
    a_ev, a_off = ev[:h], off[:5]
    b_ev, b_off = ev[h:], off[4:] - off[4]
    ta = scl.scl_trace_load(a_ev, a_off, cfg.n_sites)
    tb = scl.scl_trace_load(b_ev, b_off, cfg.n_sites)
    ra = scl.scl_replay_run(cfg.T, ta, defer_finalize=True)
    rb = scl.scl_replay_run(cfg.T, tb, defer_finalize=True)
    xa, xb = scl.device_table_tensor(ra), scl.device_table_tensor(rb)
    xa += xb
    torch.cuda.synchronize()
    scl.scl_finalize(ra, elapsed_ns=oracle.elapsed_ns(off))
    ref = oracle.full(ev, off, cfg.n_sites, cfg.T)
    rows = scl.scl_site_report(ra)
    assert np.array_equal(rows["site"], ref["order"])
    assert np.array_equal(rows["col"], ref["result"].site_table[ref["order"]])
    assert np.array_equal(rows["leak_flag"], ref["flag"][ref["order"]].astype(np.uint32))
    assert np.array_equal(rows["leak_prob"], ref["prob"][ref["order"]])
    assert scl.scl_gate(ra) == ref["gate"]


def test_reload_grow_shrink_and_kernel_times():
    """scl_trace_reload: one handle refilled with larger, smaller and different-site traces
    (buffers grown and reused, results re-sized), each run checked against the oracle; the
    timing ring returns one replay-kernel duration per run enqueued."""
    rng = np.random.default_rng(11)
    batches = []
    for n_tr, n_sites in ((5, 37), (40, 37), (3, 1500), (64, 9)):
        traces = [tracegen.random_small_trace(rng, int(rng.integers(0, 30000)), n_sites=n_sites,
                                              max_size=int(rng.integers(1, 5000)), max_ptrs=30) for _ in range(n_tr)]
        batches.append((_concat(traces), n_sites))
    (ev0, off0), s0 = batches[0]
    tr = scl.scl_trace_load(ev0, off0, s0)
    r = None
    for (ev, off), n_sites in batches + batches[:1]:
        scl.scl_trace_reload(tr, ev, off, n_sites)
        assert (tr.n_traces, tr.n_sites) == (len(off) - 1, n_sites)
        for T in (97, 4001):
            r = scl.scl_replay_run(T, tr, out=r, timing=True)
            compare(ev, off, n_sites, T, r)
    assert len(scl.scl_result_kernel_times(r)) == 2 * (len(batches) + 1)
    r = scl.scl_replay_run(97, tr, out=r)                  # untimed runs record no kernel events
    assert scl.scl_result_timing(r) == (-1, -1, -1) and scl.scl_result_kernel_times(r) == []
    for _ in range(3):
        r = scl.scl_replay_run(97, tr, out=r, timing=True)
    ks = scl.scl_result_kernel_times(r)
    assert len(ks) == 3 and all(k > 0 for k in ks)
    assert scl.scl_result_kernel_times(r) == []
    # a bad event leaves the handle empty, a good reload restores it
    bad = tracegen.from_tuples([("a", 1, 8, 99)])
    with pytest.raises(scl.SclError):
        scl.scl_trace_reload(tr, bad, np.array([0, 1], dtype=np.uint64), 2)
    (ev, off), n_sites = batches[1]
    scl.scl_trace_reload(tr, ev, off, n_sites)
    r = scl.scl_replay_run(97, tr, out=r)
    compare(ev, off, n_sites, 97, r)


def test_report_many_flagged_sites():
    """a6 with more flagged sites than the fused report kernel's shared list (3000 > 2048):
    every allocation raises the high-water mark (T=1), none is freed, so each site has
    m = 20 leak mallocs, f = 0 (flagged: m > 21 f + 18); rates differ by site."""
    n_sites, reps = 3000, 20
    ev_t = []
    ptr = 0x10000
    for r_ in range(reps):
        for s_ in range(n_sites):
            ev_t.append(("a", ptr, 16 + (s_ * 7919) % 4093 + r_, s_))
            ptr += 0x1000
    ev, off = _concat([ev_t])
    _, r = gpu_run(ev, off, n_sites, 1)
    ref = compare(ev, off, n_sites, 1, r)
    assert int(ref["flag"].sum()) == n_sites


def test_hwm_mode_sample():
    """NEXT-4: hwm_mode SAMPLE (a new maximum is above every earlier sample footprint, reading
    Q3's alternative) on ragged random traces and a config-2 subset, against the oracle's SAMPLE
    mode; the two readings give different episode sets on the same traces."""
    rng = np.random.default_rng(21)
    traces = [tracegen.random_small_trace(rng, int(rng.integers(0, 20000)), n_sites=23, max_size=int(rng.integers(1, 300)),
                                          max_ptrs=int(rng.integers(2, 40))) for _ in range(120)]
    ev, off = _concat(traces)
    tr = scl.scl_trace_load(ev, off, 23)
    r = None
    for T in (3, 97, 4001):
        r = scl.scl_replay_run(T, tr, out=r, hwm_mode=scl.HWM_SAMPLE)
        compare(ev, off, 23, T, r, hwm_mode=scl.HWM_SAMPLE)
    cfg = tracegen.CONFIGS[2].with_traces(6)
    ev, off = tracegen.generate(cfg)
    _, r = gpu_run(ev, off, cfg.n_sites, 1048583, hwm_mode=scl.HWM_SAMPLE)
    a = compare(ev, off, cfg.n_sites, 1048583, r, hwm_mode=scl.HWM_SAMPLE)
    b = oracle.full(ev, off, cfg.n_sites, 1048583, hwm_mode=oracle.HWM_PREFIX)
    assert int(a["result"].summaries["n_episodes"].sum()) != int(b["result"].summaries["n_episodes"].sum())


def test_edge_many_traces_max_sites_extreme_T():
    """Edge cases: 4000 short traces (many runner lanes per warp), n_sites at the maximum 2^21
    with sites spread over it (cold-site path), sizes up to 2^40 - 1, T = 1 (every event is a
    sample) and T huge (no sample)."""
    rng = np.random.default_rng(99)
    traces = []
    for i in range(4000):
        n = int(rng.integers(0, 60))
        tr_ = []
        live = []
        for _ in range(n):
            if live and rng.random() < 0.4:
                p, z, s_ = live.pop(int(rng.integers(len(live))))
                tr_.append(("f", p, z, int(rng.integers(0, 1 << 21))))
            else:
                z = int(rng.choice([1, 16, (1 << 40) - 1, int(rng.integers(1, 1 << 30))]))
                p = 0x1000 + 16 * len(tr_) + (i << 24)
                live.append((p, z, 0))
                tr_.append(("a", p, z, int(rng.integers(0, 1 << 21))))
        traces.append(tr_)
    ev, off = _concat(traces)
    tr = scl.scl_trace_load(ev, off, 1 << 21)
    r = None
    for T in (1, 1 << 45):
        r = scl.scl_replay_run(T, tr, out=r)
        compare(ev, off, 1 << 21, T, r)


def test_sample_domains():
    """NEXT-2: per sample, allocated and managed-domain allocated bytes since the previous
    sample, against the oracle, on ragged random traces with random domain bits and on config-2
    traces (small objects managed), at several T."""
    rng = np.random.default_rng(31)
    traces = []
    for i in range(150):
        n = int(rng.choice([0, 1, 9, 255, 8191, 8193, 20000, int(rng.integers(1, 9000))]))
        tr_ = tracegen.random_small_trace(rng, n, n_sites=13, max_size=int(rng.integers(1, 400)), max_ptrs=30)
        traces.append([e + (int(rng.integers(0, 2)),) if e[0] == "a" else e for e in tr_])
    cases = [(_concat(traces), 13, (5, 97, 4001))]
    cfg = tracegen.CONFIGS[2].with_traces(4)
    cases.append((tracegen.generate(cfg), cfg.n_sites, (1048583, cfg.T)))
    for (ev, off), n_sites, Ts in cases:
        tr = scl.scl_trace_load(ev, off, n_sites)
        r = None
        for T in Ts:
            r = scl.scl_replay_run(T, tr, out=r)
            ref = oracle.replay(ev, off, n_sites, T)
            for t in range(len(off) - 1):
                got = scl.scl_sample_domains(r, t)
                exp = ref.domains[int(ref.sample_off[t]):int(ref.sample_off[t + 1])]
                assert np.array_equal(got["alloc_bytes"], exp["alloc_bytes"]), (T, t)
                assert np.array_equal(got["managed_bytes"], exp["managed_bytes"]), (T, t)


def _recon_reference(ev, off, ref):
    """Brute force from the definition on the oracle's samples: F_i by cumulative sum,
    the step function of the latest sample footprint, max |difference| per trace."""
    kind = ((ev["meta"] >> np.uint64(40)) & np.uint64(3)).astype(np.int64)
    size = (ev["meta"] & np.uint64((1 << 40) - 1)).astype(np.int64)
    d = np.where(kind == 0, size, np.where(kind == 1, -size, 0))
    out = []
    for t in range(len(off) - 1):
        b, e = int(off[t]), int(off[t + 1])
        if e == b:
            out.append(0); continue
        F = np.cumsum(d[b:e])
        s = ref.trace_samples(t)
        step = np.zeros(e - b, dtype=np.int64)
        if len(s):
            pos = np.searchsorted(s["idx"].astype(np.int64), np.arange(e - b), side="right") - 1
            step = np.where(pos >= 0, s["footprint"][np.maximum(pos, 0)], 0)
        live = kind[b:e] < 3
        out.append(int(np.abs(F - step)[live].max()))
    return np.array(out, dtype=np.uint64)


def test_trace_recon_error():
    """NEXT-4 trend: per-trace max reconstruction error equals the brute-force value on ragged
    random traces, and is below T on every trace of the full bench workload (config 2)."""
    rng = np.random.default_rng(41)
    traces = [tracegen.random_small_trace(rng, int(rng.choice([0, 1, 9, 8193, int(rng.integers(1, 20000))])), n_sites=7,
                                          max_size=int(rng.integers(1, 500)), max_ptrs=30) for _ in range(100)]
    ev, off = _concat(traces)
    tr = scl.scl_trace_load(ev, off, 7)
    r = None
    for T in (3, 211, 10**6):
        r = scl.scl_replay_run(T, tr, out=r)
        ref = oracle.replay(ev, off, 7, T)
        assert np.array_equal(scl.scl_trace_recon_error(r), _recon_reference(ev, off, ref)), T
    cfg = tracegen.CONFIGS[2]
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = scl.scl_replay_run(cfg.T, tr)
    err = scl.scl_trace_recon_error(r)
    assert len(err) == cfg.n_traces and (err < cfg.T).all() and (err > cfg.T // 2).all()


def test_all_empty_traces_after_reuse():
    """Degenerate input: every trace empty (no unit, no replay launch), on a result reused from a
    non-empty run -- the summaries, table, report and gate must be those of the empty traces."""
    rng = np.random.default_rng(5)
    full = [tracegen.random_small_trace(rng, 5000, n_sites=9, max_size=300, max_ptrs=20) for _ in range(3)]
    ev, off = _concat(full)
    tr, r = gpu_run(ev, off, 9, 257)
    compare(ev, off, 9, 257, r)
    ev0, off0 = _concat([[], [], []])
    scl.scl_trace_reload(tr, ev0, off0, 9)
    r = scl.scl_replay_run(257, tr, out=r)
    compare(ev0, off0, 9, 257, r)


def test_unit_aggregates_beyond_48_bits():
    """A unit whose footprint range exceeds 2^47 bytes (its published aggregate words cannot carry
    it, so the runner reads the unit record), among ordinary units of the same traces."""
    rng = np.random.default_rng(11)
    traces = []
    for t in range(3):
        tr_, live = [], []
        for i in range(30000):
            if 9000 <= i < 9400:                               # unit 1: 400 allocs of ~2^40 bytes
                s, p = (1 << 40) - 1 - i, 0x7000000000 + 16 * i
                live.append((p, s)); tr_.append(("a", p, s, 1))
            elif live and (i >= 20000 or rng.random() < 0.45):
                p, s = live.pop(int(rng.integers(len(live))))
                tr_.append(("f", p, s, 2))
            else:
                s, p = int(rng.integers(1, 5000)), 0x1000 + 16 * i
                live.append((p, s)); tr_.append(("a", p, s, 0))
        traces.append(tr_)
    ev, off = _concat(traces)
    for T in (1 << 20, (1 << 45) + 3):
        _, r = gpu_run(ev, off, 3, T)
        compare(ev, off, 3, T, r)


def test_hot_sites_with_high_ids():
    """n_sites > 1024 with the hot sites spread over high, colliding ids: the warm table's slots
    (site mod 2048, first claimer) and the L2 path both in play."""
    cfg = tracegen.CONFIGS[3].with_traces(12)
    ev, off = tracegen.generate(cfg)
    rng = np.random.default_rng(8)
    perm = rng.permutation(1 << 20)[:cfg.n_sites].astype(np.uint64)      # rank r -> a high random id
    site = ev["meta"] >> np.uint64(43)
    ev = ev.copy()
    ev["meta"] = (ev["meta"] & np.uint64((1 << 43) - 1)) | (perm[site.astype(np.int64)] << np.uint64(43))
    n_sites = 1 << 20
    for T in (cfg.T, 1048583):
        _, r = gpu_run(ev, off, n_sites, T)
        compare(ev, off, n_sites, T, r, traces_to_check=range(0, 12, 3))


def test_handles_created_and_freed_repeatedly():
    """Regression (found by tools/fuzz.py): a new handle's counter block may be a freed handle's
    memory, whose "run prepared" word held the same epoch; the block is now zeroed at creation.
    Create / run / check / free in a loop, one unit per trace so that every CTA races CTA 0."""
    rng = np.random.default_rng(12)
    for it in range(20):
        traces = [tracegen.random_small_trace(rng, 8191, n_sites=5000, max_size=1 << 20, max_ptrs=50), []]
        ev, off = _concat(traces)
        tr = scl.scl_trace_load(ev, off, 5000)
        r = scl.scl_replay_run(1000 + it, tr, tick_ns=1000)
        compare(ev, off, 5000, 1000 + it, r)
        r.free(); tr.free()
