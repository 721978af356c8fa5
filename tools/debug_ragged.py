import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, oracle, tracegen, paper_2212_07597_b200 as scl
rng = np.random.default_rng(1)
traces = []
for i in range(400):
    n = int(rng.choice([0, 1, 3, 7, 8, 9, 31, 255, 256, 257, 2047, 2048, 2049, 5000, 8191, 8192, 8193,
                        16385, 40000, int(rng.integers(1, 9000))]))
    traces.append(tracegen.random_small_trace(rng, n, n_sites=37, max_size=int(rng.integers(1, 200)),
                                              max_ptrs=int(rng.integers(2, 40))))
ev = tracegen.from_tuples([e for tr in traces for e in tr])
off = np.zeros(len(traces) + 1, dtype=np.uint64); off[1:] = np.cumsum([len(t) for t in traces])
tr = scl.scl_trace_load(ev, off, 37)
r = None
for T in (1, 2, 7, 64, 401, 5000, 10**9):
    for rep in range(2):
        r = scl.scl_replay_run(T, tr, out=r)
        ref = oracle.full(ev, off, 37, T, n_threads=8)
        rows = scl.scl_site_report(r)
        g = np.zeros((37, 10), dtype=np.int64); g[rows["site"]] = rows["col"].astype(np.int64)
        o = ref["result"].site_table.astype(np.int64)
        d = g - o
        bad = np.nonzero(np.any(d != 0, axis=1))[0]
        summ = scl.scl_trace_summaries(r)
        sd = int(np.sum(summ["n_samples"] != ref["result"].summaries["n_samples"]))
        print(f"T={T} rep={rep}: sites differing {len(bad)} (cols {sorted(set(np.nonzero(d)[1].tolist()))}), "
              f"col diffs sum {d.sum(axis=0).tolist()}, summary n_samples mismatches {sd}", flush=True)
