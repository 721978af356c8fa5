"""Randomised GPU-vs-oracle fuzzing (not part of the test suite: minutes of GPU time).  Each case keeps
the previous case's re-threshold result (and so its handle) alive, which varies the allocation layout:
that is how an unguarded read past the event buffer showed up (case 141 of seed 2).
python tools/fuzz.py N_CASES SEED   (FUZZ_CHAIN=1/2: force the runners / the chain split)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2212_07597_b200 as scl, tracegen
from parity import compare

n_cases, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
_keep = []
chain = int(os.environ.get("FUZZ_CHAIN", "0"))
t0 = time.time()
for case in range(n_cases):
    n_traces = int(rng.integers(1, 40))
    n_sites = int(rng.choice([1, 7, 300, 1024, 1025, 2048, 2049, 5000, 1 << 21]))
    max_size = int(rng.choice([8, 300, 5000, 1 << 20, 1 << 27, (1 << 40) - 1]))
    traces = []
    for _ in range(n_traces):
        n = int(rng.choice([0, 1, 7, 8, 9, 255, 256, 257, 2047, 2048, 8191, 8192, 8193, 16385,
                            int(rng.integers(1, 60000))]))
        traces.append(tracegen.random_small_trace(rng, n, n_sites=min(n_sites, 1 << 21), max_size=max_size,
                                                  max_ptrs=int(rng.integers(1, 200))))
    ev = tracegen.from_tuples([e for t in traces for e in t])
    off = np.zeros(n_traces + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in traces])
    tot = int(off[-1])
    T = int(rng.choice([1, 2, 17, 257, 4099, 65537, 1048583, (1 << 40) + 15, int(rng.integers(1, 1 << 24))]))
    hwm = int(rng.integers(0, 2)); formula = int(rng.integers(0, 2))
    desc = (f"case {case}: traces {n_traces}, sites {n_sites}, max_size {max_size}, T {T}, hwm {hwm}, "
            f"formula {formula}, events {tot}")
    if case < int(os.environ.get("FUZZ_START", "0")):          # replay the RNG only
        rng.choice([3, 1031, 1048583])
        continue
    if os.environ.get("FUZZ_SAVE"):
        np.save(f"gpurun_out/fuzz_cur_ev.npy", ev); np.save(f"gpurun_out/fuzz_cur_off.npy", off)
        open("gpurun_out/fuzz_cur.txt", "w").write(desc + "\n")
    try:
        tr = scl.scl_trace_load(ev, off, n_sites)
        r = scl.scl_replay_run(T, tr, tick_ns=1000, hwm_mode=hwm, formula=formula, chain_mode=chain)
        compare(ev, off, n_sites, T, r, hwm_mode=hwm, formula=formula)
        T2 = int(rng.choice([3, 1031, 1048583]))
        if not os.environ.get("FUZZ_NO_RT"):
            r2 = scl.scl_replay_rethreshold(T2, tr, r, tick_ns=1000, hwm_mode=hwm, formula=formula, chain_mode=chain)
            compare(ev, off, n_sites, T2, r2, hwm_mode=hwm, formula=formula)
            _keep.append(r2) if len(_keep) < 1 else (_keep.pop(), _keep.append(r2))
    except (AssertionError, scl.SclError) as e:
        print(f"{desc} FAILED: {e}", flush=True)
        np.save(f"gpurun_out/fuzz_fail_{seed}_{case}_ev.npy", ev); np.save(f"gpurun_out/fuzz_fail_{seed}_{case}_off.npy", off)
        raise
    del tr, r
print(f"{n_cases} cases passed in {time.time() - t0:.0f} s (seed {seed})")
