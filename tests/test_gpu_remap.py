"""Site ids by load-time frequency (scl_trace_load with n_sites > 1,024): the library renumbers the
sites internally so that the hottest ones take the shared-memory Tier-E table; every output stays in
the caller's ids.  Traces whose hot sites carry high, scattered ids must give exactly the oracle's
results: samples (their site field), the site table and report, the deferred / all-reduce table, the
rate sampler's samples and per-site counts."""
import numpy as np
import pytest

import oracle
import paper_2212_07597_b200 as scl
import tracegen
from parity import compare

pytestmark = pytest.mark.gpu


def _permuted(cfg, seed=5):
    ev, off = tracegen.generate(cfg)
    perm = np.random.default_rng(seed).permutation(cfg.n_sites).astype(np.uint64)
    site = ev["meta"] >> np.uint64(43)
    ev["meta"] = (ev["meta"] & np.uint64((1 << 43) - 1)) | (perm[site] << np.uint64(43))
    return ev, off


@pytest.mark.parametrize("cid,nt", [(3, 12), (4, 2)])
def test_permuted_sites_parity(cid, nt):
    cfg = tracegen.CONFIGS[cid].with_traces(nt)
    ev, off = _permuted(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = scl.scl_replay_run(cfg.T, tr)
    ref = compare(ev, off, cfg.n_sites, cfg.T, r)
    # a re-threshold over the same stream pass
    T2 = scl.scl_next_prime(1 << 20)
    compare(ev, off, cfg.n_sites, T2, scl.scl_replay_rethreshold(T2, tr, r))
    # the summable table after a deferred run is in the caller's ids (what ranks all-reduce)
    rd = scl.scl_replay_run(cfg.T, tr, defer_finalize=True)
    tab = scl.device_table_tensor(rd).cpu().numpy()
    assert np.array_equal(tab[:cfg.n_sites * 10].reshape(-1, 10).astype(np.uint64), ref["result"].site_table)
    # the split chain
    compare(ev, off, cfg.n_sites, cfg.T, scl.scl_replay_run(cfg.T, tr, chain_mode=scl.CHAIN_SPLIT))
    # rate sampler: samples and per-site counts in the caller's ids
    rr = scl.scl_rate_run(cfg.T, tr, seed=3)
    rs, _ = oracle.rate_replay(ev, off, cfg.T, 3)
    got = np.concatenate([scl.scl_rate_samples(rr, t) for t in range(nt)])
    assert np.array_equal(got["site"], rs["site"]) and np.array_equal(got["idx"], rs["idx"])
    counts = scl.scl_rate_site_counts(rr)
    assert np.array_equal(counts, np.bincount(rs["site"], minlength=cfg.n_sites).astype(np.uint64))
