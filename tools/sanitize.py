"""Workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) through the C-ABI:
config 1, a config-2 subset, a config-3 subset (cold-record stream + cold_hist + grid a6 above
16,384 sites), a re-threshold, a deferred finalize, the rate sampler, and fixed-seed fuzz cases.
    compute-sanitizer --tool memcheck python tools/sanitize.py [small]
Exit 0 with no sanitizer report = clean."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2212_07597_b200 as scl
import tracegen

small = len(sys.argv) > 1 and sys.argv[1] == "small"


def run(cfg, T=None, rethreshold=True):
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = scl.scl_replay_run(T or cfg.T, tr)
    scl.scl_site_report(r)
    scl.scl_samples(r, 0)
    if rethreshold:
        r2 = scl.scl_replay_rethreshold(scl.scl_next_prime(1 << 18), tr, r)
        scl.scl_site_report(r2)
        r2.free()
    rd = scl.scl_replay_run(T or cfg.T, tr, defer_finalize=True)
    scl.scl_finalize(rd, 0)
    scl.scl_site_report(rd)
    rr = scl.scl_rate_run(T or cfg.T, tr, seed=3)
    scl.scl_rate_counts(rr)
    scl.scl_sample_domains(r, 0)
    scl.scl_trace_recon_error(r)
    for x in (rr, rd, r, tr):
        x.free()
    print(f"{cfg.name} x{cfg.n_traces}: ok", flush=True)


run(tracegen.CONFIGS[1])
run(tracegen.CONFIGS[2].with_traces(1 if small else 3))
run(tracegen.CONFIGS[3].with_traces(1 if small else 4))
rng = np.random.default_rng(7)
for case in range(2 if small else 12):
    n_traces = int(rng.integers(1, 12))
    n_sites = int(rng.choice([1, 300, 1025, 2049, 5000, 40000]))
    traces = [tracegen.random_small_trace(rng, int(rng.choice([0, 1, 9, 257, 8193, int(rng.integers(1, 30000))])),
                                          n_sites=n_sites, max_size=int(rng.choice([300, 1 << 20, 1 << 30])),
                                          max_ptrs=int(rng.integers(1, 200))) for _ in range(n_traces)]
    ev = tracegen.from_tuples([e for t in traces for e in t])
    off = np.zeros(n_traces + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in traces])
    tr = scl.scl_trace_load(ev, off, n_sites)
    T = int(rng.choice([1, 17, 4099, 1048583]))
    r = scl.scl_replay_run(T, tr)
    scl.scl_site_report(r)
    r2 = scl.scl_replay_rethreshold(3, tr, r)
    scl.scl_site_report(r2)
    for x in (r2, r, tr):
        x.free()
print("fuzz cases: ok", flush=True)
