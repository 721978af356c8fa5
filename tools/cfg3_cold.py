import os, sys, dataclasses
sys.path.insert(0, "/root/repo")
import paper_2212_07597_b200 as scl, tracegen, numpy as np
for ns in (1024, 50000):
    cfg = dataclasses.replace(tracegen.CONFIGS[3].with_traces(128), n_sites=ns)
    ev, off = tracegen.generate(cfg)
    site = (ev["meta"] >> np.uint64(43)).astype(np.int64)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = None
    ks = []
    for _ in range(5):
        r = scl.scl_replay_run(1 << 50, tr, out=r, timing=True); ks.append(scl.scl_result_timing(r)[0])
    print(f"n_sites={ns}: cold events {(site >= 2048).mean():.3f}; replay kernel {sorted(ks)[2]*1e3:.1f} us", flush=True)
    del tr, r
