"""Per-kernel device times of K runs of one config (CUDA events around each kernel are not available
from outside the library: this times the whole run and the library's stream-pass events).
    CFG=3 NT=256 python tools/kt.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_07597_b200 as scl, tracegen
cfg = tracegen.CONFIGS[int(os.environ.get("CFG", "3"))]
if os.environ.get("NT"):
    cfg = cfg.with_traces(int(os.environ["NT"]))
ev, off = tracegen.generate(cfg)
tr = scl.scl_trace_load(ev, off, cfg.n_sites)
st = torch.cuda.current_stream()
r = None
for _ in range(3):
    r = scl.scl_replay_run(cfg.T, tr, stream=st, out=r)
torch.cuda.synchronize()
scl.scl_result_kernel_times(r); scl.scl_result_pass_times(r)
K = 20
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(K):
    r = scl.scl_replay_run(cfg.T, tr, stream=st, out=r, timing=True)
b.record(st)
torch.cuda.synchronize()
ks = scl.scl_result_kernel_times(r)
ps = scl.scl_result_pass_times(r)
print(f"{os.environ.get('SCL_LIB','libscl.so').split('/')[-1]} cfg{os.environ.get('CFG','3')} nt={cfg.n_traces}: "
      f"step {a.elapsed_time(b)/K*1e3:.1f} us, replay kernel {sum(ks)/len(ks)*1e3:.1f} us, stream pass {sum(ps)/len(ps)*1e3:.1f} us")
