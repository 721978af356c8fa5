"""Threshold sweep on config 2: 11 thresholds 1 MiB .. 1 GiB (primes above 2^k), as
11 full replays vs one stream pass + 10 re-thresholds (scl_replay_sweep).  Device time of the
whole sequence, CUDA events on one stream."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_07597_b200 as scl, tracegen

cfg = tracegen.CONFIGS[2]
ev, off = tracegen.generate(cfg)
tr = scl.scl_trace_load(ev, off, cfg.n_sites)
Ts = [scl.scl_next_prime(1 << k) for k in range(20, 31)]
st = torch.cuda.current_stream()

def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(st); out = fn(); b.record(st); torch.cuda.synchronize()
        ms = a.elapsed_time(b); best = ms if best is None else min(best, ms)
    return best, out

full = [scl.scl_replay_run(T, tr, stream=st) for T in Ts]          # results allocated once
sw = scl.scl_replay_sweep(Ts, tr, stream=st)

def run_full():
    for T, r in zip(Ts, full): scl.scl_replay_run(T, tr, stream=st, out=r)
    return full

def run_sweep():
    scl.scl_replay_run(Ts[0], tr, stream=st, out=sw[0])
    for T, r in zip(Ts[1:], sw[1:]): scl.scl_replay_rethreshold(T, tr, sw[0], stream=st, out=r)
    return sw

ms_full, full = timed(run_full)
ms_sweep, sw = timed(run_sweep)
same = all((scl.scl_trace_summaries(a) == scl.scl_trace_summaries(b)).all() for a, b in zip(full[1:], sw[1:]))
ns = [int(scl.scl_trace_summaries(r)["n_samples"].sum()) for r in sw]
print(f"11 thresholds {Ts[0]}..{Ts[-1]}: samples {ns}")
print(f"11 full replays: {ms_full:.2f} ms; 1 stream pass + 10 re-thresholds: {ms_sweep:.2f} ms "
      f"({ms_full / ms_sweep:.2f}x); results identical: {same}")
