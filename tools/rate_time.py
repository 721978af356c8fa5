"""Rate-sampler kernel time on config 2 (R = T, seed 2022): python tools/rate_time.py"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_07597_b200 as scl, tracegen
cfg = tracegen.CONFIGS[2]
ev, off = tracegen.generate(cfg)
tr = scl.scl_trace_load(ev, off, cfg.n_sites)
rr = scl.scl_rate_run(cfg.T, tr, seed=2022)
ms = []
for _ in range(5):
    rr = scl.scl_rate_run(cfg.T, tr, seed=2022, out=rr)
    ms.append(scl.scl_rate_timing(rr))
print(f"rate sampler (draws + ranges + place): {statistics.median(ms)*1e3:.1f} us, samples {int(scl.scl_rate_counts(rr).sum())}")
