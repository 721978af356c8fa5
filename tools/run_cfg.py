"""Run the replay of one config a few times (for ncu captures): python tools/run_cfg.py CFG NTRACES T REPS
(EPT=n: n events per trace; CHAIN=0/1/2: chain_mode)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses
import paper_2212_07597_b200 as scl, tracegen
cid, nt, T, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = tracegen.CONFIGS[cid].with_traces(nt) if nt else tracegen.CONFIGS[cid]
if os.environ.get("EPT"):
    cfg = dataclasses.replace(cfg, events_per_trace=int(os.environ["EPT"]))
ev, off = tracegen.generate(cfg)
tr = scl.scl_trace_load(ev, off, cfg.n_sites)
r = None
for _ in range(reps):
    r = scl.scl_replay_run(T, tr, out=r, chain_mode=int(os.environ.get("CHAIN", "0")))
scl.scl_site_report(r)
print("ok")
