"""The chain split at sync events (scl_run_opts.chain_mode = SCL_CHAIN_SPLIT, csrc/pchain.cu) gives the
same results as the sequential runners and the oracle: element by element on configs 1-3 (subsets),
config 5's heavy-tailed sizes at dense thresholds (many sync events: |d| >= 2T - 1, SURVEY Appendix A
W5), T = 1 (every event a sample), re-thresholds, and fixed-seed random traces."""
import dataclasses

import numpy as np
import pytest

import paper_2212_07597_b200 as scl
import tracegen
from parity import compare

pytestmark = pytest.mark.gpu
SPLIT = scl.CHAIN_SPLIT


def _run(cfg, Ts, n_traces=None):
    if n_traces:
        cfg = cfg.with_traces(n_traces)
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = scl.scl_replay_run(Ts[0], tr, chain_mode=SPLIT)
    compare(ev, off, cfg.n_sites, Ts[0], r)
    for T in Ts[1:]:
        r2 = scl.scl_replay_rethreshold(T, tr, r, chain_mode=SPLIT)
        compare(ev, off, cfg.n_sites, T, r2)
    return tr


def test_split_config1_and_2():
    _run(tracegen.CONFIGS[1], [tracegen.CONFIGS[1].T, 1, 257, 65537])
    _run(tracegen.CONFIGS[2], [tracegen.CONFIGS[2].T, 65537, 1048583], n_traces=8)


def test_split_config3_subset():
    _run(tracegen.CONFIGS[3], [tracegen.CONFIGS[3].T, 65537], n_traces=16)


def test_split_config5_dense():
    cfg = dataclasses.replace(tracegen.CONFIGS[5].with_traces(3), events_per_trace=3_000_000)
    _run(cfg, list(cfg.t_sweep[:4]) + [cfg.t_sweep[-1]])


def test_split_equals_runners_random():
    rng = np.random.default_rng(11)
    for case in range(30):
        n_traces = int(rng.integers(1, 20))
        n_sites = int(rng.choice([3, 300, 2049, 5000]))
        traces = [tracegen.random_small_trace(rng, int(rng.choice([0, 1, 9, 257, 8193, 16385, int(rng.integers(1, 40000))])),
                                              n_sites=n_sites, max_size=int(rng.choice([8, 300, 1 << 20, 1 << 30])),
                                              max_ptrs=int(rng.integers(1, 200))) for _ in range(n_traces)]
        ev = tracegen.from_tuples([e for t in traces for e in t])
        off = np.zeros(n_traces + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(t) for t in traces])
        T = int(rng.choice([1, 2, 17, 257, 4099, 1048583]))
        tr = scl.scl_trace_load(ev, off, n_sites)
        r = scl.scl_replay_run(T, tr, chain_mode=SPLIT)
        compare(ev, off, n_sites, T, r)
        T2 = int(rng.choice([3, 1031]))
        r2 = scl.scl_replay_rethreshold(T2, tr, r, chain_mode=SPLIT)
        compare(ev, off, n_sites, T2, r2)


def test_split_sample_mode_uses_runners():
    """hwm_mode SAMPLE depends on every earlier sample: the split request falls back to the runners."""
    cfg = tracegen.CONFIGS[1]
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = scl.scl_replay_run(cfg.T, tr, chain_mode=SPLIT, hwm_mode=scl.HWM_SAMPLE)
    compare(ev, off, cfg.n_sites, cfg.T, r, hwm_mode=scl.HWM_SAMPLE)


def test_launch_count_and_pass_times():
    """scl_result_launches counts the library's kernels of the last run; the stream-pass time covers
    the replay kernel and the kernels after it (cold-site Tier E, split chains)."""
    for cfg, mode, want in ((tracegen.CONFIGS[2].with_traces(2), 1, 2),         # replay + post
                            (tracegen.CONFIGS[3].with_traces(2), 1, 4),         # + cold_hist + cold_sum (50,000 sites)
                            (tracegen.CONFIGS[2].with_traces(2), SPLIT, 6)):    # + 4 pchain kernels
        ev, off = tracegen.generate(cfg)
        tr = scl.scl_trace_load(ev, off, cfg.n_sites)
        r = None
        for _ in range(3):
            r = scl.scl_replay_run(cfg.T, tr, out=r, timing=True, chain_mode=mode)
        # (+3 if the load renumbered the sites: the table permute and an unfused two-kernel a6)
        assert scl.scl_result_launches(r) in ((want,) if cfg.n_sites <= 1024 else (want, want + 3))
        ks, ps = scl.scl_result_kernel_times(r), scl.scl_result_pass_times(r)
        assert len(ks) == 3 and len(ps) == 3 and all(p >= k > 0 for k, p in zip(ks, ps))
        rd = scl.scl_replay_run(cfg.T, tr, defer_finalize=True, chain_mode=mode)
        scl.scl_finalize(rd, cfg.events_per_trace * 1000)
        # deferred: the post pass without a6, then a6 in its own kernel(s): report_kernel, or
        # report_flags + report_rows above 16,384 sites
        assert scl.scl_result_launches(rd) in ((want + 1,) if cfg.n_sites <= 16384 else (want + 2, want + 3))
