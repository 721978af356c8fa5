"""NEXT-1: the paper's Table tab:sampling-comparison ("Threshold vs. Rate-Based Sampling") and the
sample-log size comparison on the synthetic configs: per config, the threshold
sampler's and the rate-based sampler's (R = T) sample counts, their ratio (whole config and the
median over traces) and sample-log bytes (32 B per threshold sample, 24 B per rate sample).
Both samplers run on the GPU (they are checked against the oracle in tests/)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2212_07597_b200 as scl
import tracegen

rows = []
cases = [("cfg1", tracegen.CONFIGS[1]), ("cfg2", tracegen.CONFIGS[2]), ("cfg3 (128 traces)", tracegen.CONFIGS[3].with_traces(128)),
         ("cfg2-copy", tracegen.COPY_CFG)]
for name, cfg in cases:
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    for T in (cfg.T,) + ((1048583,) if name == "cfg2" else ()):
        thr = scl.scl_replay_run(T, tr)
        nt = scl.scl_trace_summaries(thr)["n_samples"].astype(np.float64)
        rr = scl.scl_rate_run(T, tr, seed=2022)
        nr = scl.scl_rate_counts(rr).astype(np.float64)
        ok = nt > 0
        med = float(np.median(nr[ok] / nt[ok])) if ok.any() else float("nan")
        rows.append((name, T, int(nt.sum()), int(nr.sum()), nr.sum() / max(nt.sum(), 1), med,
                     int(nt.sum()) * 32, int(nr.sum()) * 24, len(off) - 1))
        thr.free(); rr.free()
    tr.free()
out = ["| config | T | traces | threshold samples | rate samples (R = T) | ratio | median per-trace ratio | log bytes (threshold / rate) |",
       "|---|---|---|---|---|---|---|---|"]
for name, T, a, b, rat, med, la, lb, ntr in rows:
    out.append(f"| {name} | {T:,} | {ntr} | {a:,} | {b:,} | {rat:.1f}x | {med:.1f}x | {la:,} / {lb:,} |")
print("\n".join(out))
