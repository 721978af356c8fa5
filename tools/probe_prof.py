"""Per-role cycle breakdown of replay_kernel (debug build libscl_prof.so, -DSCL_PROFILE)."""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SCL_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2212_07597_b200", "libscl_prof.so")
import numpy as np
import paper_2212_07597_b200 as scl, tracegen
lib = scl.lib
lib.scl_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
cid, nt, T = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = tracegen.CONFIGS[cid].with_traces(nt)
ev, off = tracegen.generate(cfg)
tr = scl.scl_trace_load(ev, off, cfg.n_sites)
r = None
for _ in range(4):
    r = scl.scl_replay_run(T, tr, out=r)
ms = scl.scl_result_timing(r)[0]
buf = np.zeros(32, dtype=np.uint64)
lib.scl_debug_prof(r.handle, buf.ctypes.data)
nsm = 148
cyc = ms * 1e-3 * 1.965e9
print(f"cfg{cid} traces={nt} T={T}: kernel {ms*1e3:.1f} us = {cyc:.0f} cycles @1.965GHz")
names = {0: ("compute", 16, ["wait_full", "wait_sempty", "summary", "agg+loop", "process"]),
         8: ("producer", 1, ["wait_empty", "fetch+issue"]),
         16: ("lookback", 3, ["wait_sfull", "look_back", "resolve", "publish", "ptr_match", "loop"])}
for base, (nm, nw, cats) in names.items():
    tot = buf[base:base + 8].astype(float) / (nw * nsm)
    print(f"  {nm:9s} " + "  ".join(f"{c}={tot[i]/cyc*100:5.1f}%" for i, c in enumerate(cats)))
