"""Back-to-back step time of the whole run (prep, replay, post, report) on config 2: CUDA events
around K enqueued steps (no sync in between)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_07597_b200 as scl, tracegen

cfg = tracegen.CONFIGS[int(os.environ.get("CFG", "2"))]
if os.environ.get("NT"):
    cfg = cfg.with_traces(int(os.environ["NT"]))
T = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.T
ev, off = tracegen.generate(cfg)
tr = scl.scl_trace_load(ev, off, cfg.n_sites)
st = torch.cuda.current_stream()
r = None
for _ in range(5):
    r = scl.scl_replay_run(T, tr, stream=st, out=r)
torch.cuda.synchronize()
K = 50
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(K):
    r = scl.scl_replay_run(T, tr, stream=st, out=r)
b.record(st)
torch.cuda.synchronize()
print(f"cfg{os.environ.get('CFG', '2')} nt={cfg.n_traces} T={T} step {a.elapsed_time(b) / K * 1e3:.1f} us  (events {'off' if os.environ.get('SCL_NO_EVENTS') else 'on'})")
