"""Per-rank proxies of strong scaling on ONE B200 (only one GPU is available here): the device step
time of the shard one rank replays at N = 1, 2, 4, 8 (config 3: 1024/N traces; config 2: 64/N),
CUDA events around K back-to-back steps.  The N-GPU prediction adds an int64 all-reduce of the site
table per step (n_sites x 10 + 3 words) at an assumed NVLink 5 all-reduce time.
    python tools/scaling_proxy.py [CFG] [K]  -> one JSON line"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2212_07597_b200 as scl
import tracegen

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = tracegen.CONFIGS[cid]
st = torch.cuda.current_stream()
out = {"config": cfg.name, "n_traces": cfg.n_traces, "events_per_trace": cfg.events_per_trace, "ranks": {}}
ev_all, off_all = tracegen.generate(cfg)
for N in (1, 2, 4, 8):
    nt = cfg.n_traces // N
    ev, off = ev_all[:nt * cfg.events_per_trace], off_all[:nt + 1]
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = None
    for _ in range(3):
        r = scl.scl_replay_run(cfg.T, tr, stream=st, out=r, defer_finalize=N > 1)
        if N > 1:
            scl.scl_finalize(r, cfg.events_per_trace * 1000)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(K):
        r = scl.scl_replay_run(cfg.T, tr, stream=st, out=r, defer_finalize=N > 1)
        if N > 1:                                     # the all-reduce goes between these two
            scl.scl_finalize(r, cfg.events_per_trace * 1000)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    table_mb = (cfg.n_sites * 10 + 3) * 8 / 1e6
    ar_us = 0.0 if N == 1 else 15.0 + table_mb / 0.3 * 1e-3 * 1e3   # ~15 us latency + ~300 GB/s algbw
    pred = cfg.n_traces * cfg.events_per_trace / ((ms + ar_us / 1e3) / 1e3)
    out["ranks"][N] = {"traces_per_rank": nt, "step_ms": ms, "allreduce_us_assumed": ar_us,
                       "predicted_events_per_s": pred}
    r.free(); tr.free()
t1 = out["ranks"][1]["predicted_events_per_s"]
for N in (2, 4, 8):
    out["ranks"][N]["predicted_speedup"] = out["ranks"][N]["predicted_events_per_s"] / t1
print(json.dumps(out))
