"""Wall time of scl_trace_reload (device and pinned-host sources) for one config, and the remap-path
parity of a reloaded batch.   CFG=3 python tools/reload_time.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_07597_b200 as scl, tracegen
cfg = tracegen.CONFIGS[int(os.environ.get("CFG", "3"))]
ev, off = tracegen.generate(cfg)
tr = scl.scl_trace_load(ev, off, cfg.n_sites)
dev = torch.from_numpy(ev.view(np.int64)).cuda()
pin = torch.from_numpy(ev.view(np.int64)).pin_memory()
for name, src in (("device", dev), ("pinned host", pin.numpy().view(tracegen.EVENT_DTYPE))):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize(); a = time.perf_counter()
        scl.scl_trace_reload(tr, src, off, cfg.n_sites)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    print(f"{cfg.name} reload from {name}: {min(ts) * 1e3:.2f} ms (best of 4; {cfg.n_events * 16 / 1e9:.1f} GB)", flush=True)
