"""Site-id permutation sensitivity (the shared-memory Tier-E table holds the LOWEST site
ids): step time of config 2 and of a config-3 subset with the generator's site ids (Zipf rank = id)
and with a random permutation of them (the hot sites scattered over the id range); results checked
equal up to the permutation.   python tools/perm_time.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2212_07597_b200 as scl, tracegen

st = torch.cuda.current_stream()


def step_us(ev, off, cfg, K=10):
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    r = None
    for _ in range(3):
        r = scl.scl_replay_run(cfg.T, tr, stream=st, out=r)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(K):
        r = scl.scl_replay_run(cfg.T, tr, stream=st, out=r)
    b.record(st)
    torch.cuda.synchronize()
    rows = scl.scl_site_report(r)
    tab = np.zeros_like(rows["col"])
    tab[rows["site"]] = rows["col"]
    r.free(); tr.free()
    return a.elapsed_time(b) / K * 1e3, tab


for name, cfg in (("cfg2", tracegen.CONFIGS[2]), ("cfg3 x128", tracegen.CONFIGS[3].with_traces(128))):
    ev, off = tracegen.generate(cfg)
    t0, tab0 = step_us(ev, off, cfg)
    perm = np.random.default_rng(5).permutation(cfg.n_sites).astype(np.uint64)
    ev2 = ev.copy()
    site = ev2["meta"] >> np.uint64(43)
    ev2["meta"] = (ev2["meta"] & np.uint64((1 << 43) - 1)) | (perm[site] << np.uint64(43))
    t1, tab1 = step_us(ev2, off, cfg)
    assert np.array_equal(tab1[perm.astype(np.int64)], tab0), "permuted site table differs"
    print(f"{name}: step {t0:.1f} us with the generator's ids, {t1:.1f} us with permuted ids ({t1 / t0:.2f}x)", flush=True)
