"""Parity of a whole BASELINE configuration on ONE B200 in resident waves (configs 4 and 5 hold
524 / 410 GB of events: more than one GPU's HBM), against the oracle, wave by wave:

  per wave of whole traces: generate (seeded, multi-threaded) -> scl_trace_reload (pinned host ->
  device) -> scl_replay_run(defer_finalize) [config 5: scl_replay_sweep over its 11 thresholds]
  -> compare every trace's summary and samples with the oracle's replay of the same wave ->
  add the wave's summable table on the device (GPU) and in numpy (oracle);
  at the end: scl_finalize of the summed table vs the oracle's a6 on its summed table (report rows,
  flags, probabilities, rates, gate) and planted-leak recall (north star: every planted leak is
  flagged).  Traces are independent, so waves need no carry.

    python tools/fullcfg.py CFG [WAVE_TRACES] [MAX_WAVES]   -> one JSON summary line
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import oracle
import paper_2212_07597_b200 as scl
import tracegen

cid = int(sys.argv[1])
cfg = tracegen.CONFIGS[cid]
wave_tr = int(sys.argv[2]) if len(sys.argv) > 2 else (1024 if cid == 4 else 8)
max_waves = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 30
Ts = list(cfg.t_sweep) if cfg.t_sweep else [cfg.T]
cores = os.cpu_count() or 8
torch.cuda.set_device(0)
n_ev_wave = wave_tr * cfg.events_per_trace
pinned = torch.empty(n_ev_wave * 2, dtype=torch.int64, pin_memory=True)
host = pinned.numpy().view(tracegen.EVENT_DTYPE)
gacc = [None] * len(Ts)                      # summed device tables per threshold
oacc = [np.zeros((cfg.n_sites, oracle.NCOL), dtype=np.uint64) for _ in Ts]
osumm = [[] for _ in Ts]
tr, rs = None, [None] * len(Ts)
t_gen = t_gpu = t_orc = t_cmp = 0.0
n_waves, n_samples = 0, [0] * len(Ts)
for t0 in range(0, cfg.n_traces, wave_tr):
    if n_waves >= max_waves:
        break
    t1 = min(cfg.n_traces, t0 + wave_tr)
    a = time.time()
    ev, off = tracegen.generate(cfg, t0, t1, out=host)
    t_gen += time.time() - a
    a = time.time()
    tr = scl.scl_trace_load(ev, off, cfg.n_sites) if tr is None else scl.scl_trace_reload(tr, ev, off, cfg.n_sites)
    rs[0] = scl.scl_replay_run(Ts[0], tr, defer_finalize=True, out=rs[0])
    for k in range(1, len(Ts)):
        rs[k] = scl.scl_replay_rethreshold(Ts[k], tr, rs[0], defer_finalize=True, out=rs[k])
    for k in range(len(Ts)):
        tab = scl.device_table_tensor(rs[k])
        gacc[k] = tab.clone() if gacc[k] is None else gacc[k].add_(tab)
    torch.cuda.synchronize()
    t_gpu += time.time() - a
    for k, T in enumerate(Ts):
        a = time.time()
        ref = oracle.replay(ev, off, cfg.n_sites, T, n_threads=cores)
        t_orc += time.time() - a
        a = time.time()
        summ = scl.scl_trace_summaries(rs[k])
        for f in ("f_final", "hwm", "n_samples", "n_episodes", "f_first_sample", "f_last_sample"):
            assert np.array_equal(summ[f], ref.summaries[f]), (cid, T, t0, f)
        for t in range(t1 - t0):
            g, o = scl.scl_samples(rs[k], t), ref.trace_samples(t)
            for f in ("idx", "net", "footprint", "site", "kind", "new_max"):
                assert np.array_equal(g[f], o[f]), (cid, T, t0 + t, f)
        oacc[k] += ref.site_table
        osumm[k].append(ref.summaries)
        n_samples[k] += int(ref.summaries["n_samples"].sum())
        t_cmp += time.time() - a
    n_waves += 1
    print(f"wave {n_waves}: traces {t0}..{t1} ok (gen {t_gen:.0f}s gpu {t_gpu:.0f}s oracle {t_orc:.0f}s)", flush=True)

# a6 on the summed tables, both sides
res = []
for k, T in enumerate(Ts):
    scl.device_table_tensor(rs[k]).copy_(gacc[k])
    el = cfg.events_per_trace * 1000
    scl.scl_finalize(rs[k], el)
    rows = scl.scl_site_report(rs[k])
    summ = np.concatenate(osumm[k])
    num, den, op = oracle.gate(summ)
    prob, rate, flag = oracle.finalize(oacc[k], op, el)
    order = oracle.report_order(rate, flag)
    assert np.array_equal(rows["site"], order), (cid, T, "order")
    assert np.array_equal(rows["col"], oacc[k][order]), (cid, T, "site table")
    assert np.array_equal(rows["leak_flag"], flag[order].astype(np.uint32)), (cid, T, "flags")
    for name, x in (("leak_prob", prob), ("leak_rate_mbps", rate)):
        y = x[order]
        assert np.all((rows[name] == y) | (np.abs(rows[name] - y) <= 1e-12 * np.abs(y))), (cid, T, name)
    assert scl.scl_gate(rs[k]) == (num, den, op), (cid, T, "gate")
    pl = tracegen.planted_sites(cfg)
    complete = n_waves * wave_tr >= cfg.n_traces
    recall = int(flag[pl].sum())
    res.append({"T": T, "samples": n_samples[k], "flagged": int(flag.sum()), "planted_flagged": recall,
                "planted": len(pl), "gate_open": bool(op)})
    if complete and T == cfg.T:                    # recall at the config's own threshold (reported for the rest)
        assert recall == len(pl), (cid, T, "planted leak not flagged", oacc[k][pl, 8:])
print(json.dumps({"config": cfg.name, "traces": min(cfg.n_traces, n_waves * wave_tr), "of": cfg.n_traces,
                  "events_per_trace": cfg.events_per_trace, "n_sites": cfg.n_sites, "waves": n_waves,
                  "wave_traces": wave_tr, "parity": "bit-exact (samples, summaries, table, flags, gate; fp64 "
                  "<= 1e-12 rel) vs the oracle, per wave and after the summed a6",
                  "thresholds": res, "seconds": {"generate": t_gen, "gpu_incl_h2d": t_gpu, "oracle": t_orc,
                                                  "compare": t_cmp}, "host_cores": cores}))
