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
    r = scl.scl_replay_run(T, tr, out=r, timing=True)
ms = scl.scl_result_timing(r)[0]
nunits_all = int(sum((cfg.events_per_trace + 8191) // 8192 for _ in range(nt)))
bigbuf = np.zeros(48 + 4 * nunits_all, dtype=np.uint64)
lib.scl_debug_prof(r.handle, bigbuf.ctypes.data)
buf = bigbuf[:32]
nsm = 148
cyc = ms * 1e-3 * 1.965e9
print(f"cfg{cid} traces={nt} T={T}: kernel {ms*1e3:.1f} us = {cyc:.0f} cycles @1.965GHz")
names = {0: ("compute", 16, ["wait_full", "wait_sempty", "summary", "agg+loop", "process"]),
         8: ("producer", 1, ["wait_empty", "fetch+issue"]),
         16: ("lookback", 3, ["idle", "publish", "run"])}
for base, (nm, nw, cats) in names.items():
    tot = buf[base:base + 8].astype(float) / (nw * nsm)
    print(f"  {nm:9s} " + "  ".join(f"{c}={tot[i]/cyc*100:5.1f}%" for i, c in enumerate(cats)))
    if False:
        units = float(buf[base + 6])
        print("  walker per unit (cycles): " + "  ".join(f"{c}={float(buf[base+i])/max(units,1):.0f}" for i, c in enumerate(cats) if c not in ("units", "x")), f" units={units:.0f}")

rc = bigbuf[24:40].astype(float)
pt = bigbuf[40:48].astype(np.int64)
if pt[0] > 0 and pt[1] > 0:
    print(f"  post pass (us from its start): units+traces done {(pt[1]-pt[0])/1e3:.1f}  barrier {(pt[2]-pt[0])/1e3:.1f}  "
          f"re-checks ({int(bigbuf[39])} tasks) done {(pt[3]-pt[0])/1e3:.1f}  report {(pt[4]-pt[0])/1e3:.1f} [gate+sync {(pt[6]-pt[0])/1e3:.1f} pass1+prefix {(pt[7]-pt[0])/1e3:.1f}] -> {(pt[5]-pt[0])/1e3:.1f}")
print(f"  runner: invocations {rc[0]:.0f} batches {rc[1]:.0f} units {rc[2]:.0f} resolves {rc[3]:.0f} "
      f"resolve cyc/each {rc[4]/max(rc[3],1):.0f} ptr-exact {rc[5]:.0f} run cyc/invocation {rc[6]/max(rc[0],1):.0f} lock-fails {rc[7]:.0f}")
nres = max(rc[3], 1)
print(f"  resolve parts per resolve (cycles): record {rc[8]/nres:.0f} rows(+Fc,Mc) {rc[9]/nres:.0f} prefix+scan {rc[10]/nres:.0f} "
      f"walk {rc[12]/nres:.0f} rest {rc[13]/nres:.0f}  cand-chunks {rc[11]/nres:.2f}; batch cycles outside resolves "
      f"{(rc[14])/max(rc[1],1):.0f}/batch")
# per-unit timeline (aggregate published, inclusive published), first unit of each trace = unit 0
if len(sys.argv) > 4:
    nunits = nunits_all
    tl4 = bigbuf[48:].reshape(-1, 4).astype(np.int64); tl = tl4[:, :2]
    t0 = tl[tl > 0].min()
    per = (cfg.events_per_trace + 8191) // 8192
    agg = (tl[:, 0] - t0) / 1e3; inc = (tl[:, 1] - t0) / 1e3
    lag = inc - agg
    print(f"  units={nunits} agg publish: max {agg.max():.0f} us; inclusive publish: max {inc.max():.0f} us; lag mean {lag.mean():.1f} us p50 {np.median(lag):.1f} p90 {np.percentile(lag,90):.1f} max {lag.max():.1f}")
    for t in (0, 1, nt // 2):
        a = agg[t * per:(t + 1) * per]; b = inc[t * per:(t + 1) * per]
        print(f"  trace {t}: " + " ".join(f"{int(x)}/{int(y)}" for x, y in list(zip(a, b))[::8]))

    fin = []
    for t in range(nt):
        us = slice(t * per, (t + 1) * per)
        agg_t = (tl4[us, 0] - t0) / 1e3; be = (tl4[us, 1] - t0) / 1e3; bs = (tl4[us, 2] - t0) / 1e3
        rk = tl4[us, 3] / 1e3
        fin.append((be.max(), agg_t.max(), int((rk > 0).sum()), rk.sum(), t, bs[-1], agg_t[-4:].max()))
    fin.sort(reverse=True)
    rk_all = tl4[:, 3].astype(np.float64); bs_all = (tl4[:, 2] - t0) / 1e3
    end_stream = agg.max()
    sel_b = (rk_all > 0) & (bs_all < end_stream - 5); sel_a = (rk_all > 0) & (bs_all > end_stream + 2)
    print(f"  resolve cycles: during stream mean {rk_all[sel_b].mean():.0f} (n={sel_b.sum()}), after stream end mean "
          f"{rk_all[sel_a].mean() if sel_a.any() else 0:.0f} (n={sel_a.sum()})")
    print("  slowest traces: finish / last publish / resolves / resolve kcyc / last batch start")
    for f_, a_, nr_, rk_, t_, bs_, a4 in fin[:12]:
        print(f"    trace {t_:3d}: finish {f_:6.1f}  last agg {a_:6.1f}  resolves {nr_:3d}  kcyc {rk_:7.1f}  last batch start {bs_:6.1f}")
