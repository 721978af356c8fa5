"""Quick timing probe of the replay kernel on several workloads (not part of the bench)."""
import sys, os, time, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_07597_b200 as scl, tracegen

def timeit(tr, T, reps=10):
    r = None
    for _ in range(3): r = scl.scl_replay_run(T, tr, out=r, timing=True)
    ks, rs = [], []
    for _ in range(reps):
        r = scl.scl_replay_run(T, tr, out=r, timing=True); tm = scl.scl_result_timing(r); ks.append(tm[0]); rs.append(tm[1])
    s = scl.scl_trace_summaries(r)
    return statistics.median(ks), int(s["n_samples"].sum()), statistics.median(rs)

out = {}
specs = [(2, None, [10485767, 1 << 50, 1048583, 65537]), (3, 128, [10485767, 1 << 50])]
if len(sys.argv) > 1: specs = json.loads(sys.argv[1])
for cid, nt, Ts in specs:
    cfg = tracegen.CONFIGS[cid]
    if nt: cfg = cfg.with_traces(nt)
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    for T in Ts:
        ms, ns, rms = timeit(tr, T)
        n = len(ev)
        print(f"cfg{cid} traces={cfg.n_traces} T={T}: kernel {ms*1e3:.1f} us  {n/ms/1e6:.3g} Gev/s  {n*16/ms/1e6:.0f} GB/s  samples={ns}  run {rms*1e3:.1f} us", flush=True)
    del tr
