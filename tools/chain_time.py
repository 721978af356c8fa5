"""Device step time with the runners' sequential chains vs the chains split at sync events
(chain_mode 1 vs 2) on a few workloads.  python tools/chain_time.py -> lines"""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_07597_b200 as scl, tracegen

st = torch.cuda.current_stream()
cases = [("cfg2", tracegen.CONFIGS[2], [10485767, 1048583, 65537]),
         ("cfg2 x8 traces", tracegen.CONFIGS[2].with_traces(8), [10485767, 65537]),
         ("cfg3 x256", tracegen.CONFIGS[3].with_traces(256), [10485767]),
         ("cfg5 x8 x4M", dataclasses.replace(tracegen.CONFIGS[5].with_traces(8), events_per_trace=4_000_000),
          [65537, 1048583, 67108879])]
for name, cfg, Ts in cases:
    ev, off = tracegen.generate(cfg)
    tr = scl.scl_trace_load(ev, off, cfg.n_sites)
    for T in Ts:
        res = []
        for mode in (1, 2, 0):
            r = None
            for _ in range(2):
                r = scl.scl_replay_run(T, tr, stream=st, out=r, chain_mode=mode)
            torch.cuda.synchronize()
            K = 10
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(K):
                r = scl.scl_replay_run(T, tr, stream=st, out=r, chain_mode=mode)
            b.record(st)
            torch.cuda.synchronize()
            res.append(a.elapsed_time(b) / K)
            r.free()
        print(f"{name:16s} T={T:9d}: runners {res[0]*1e3:9.1f} us  split {res[1]*1e3:9.1f} us  auto {res[2]*1e3:9.1f} us", flush=True)
    tr.free()
