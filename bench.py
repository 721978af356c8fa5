#!/usr/bin/env python
"""Benchmark: batched malloc/free trace replay (Scalene, arXiv 2212.07597) on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W [--impl reference]``
prints ONE JSON line on rank 0.  A step is one pass of the whole hot path
a1..a6 over the resident workload: scl_replay_run (streaming
replay kernel [+ the Tier-E reduce of its cold-record stream] + reclaim /
per-sample pass) -> [N>1: NCCL all-reduce of the int64 site table] ->
scl_finalize (probabilities, flags, report order, rows).

Workload: BASELINE configs[2] = config 3, the largest configuration that fits
one B200: 1024 traces x 10^6 events (16.4 GB), 50,000 sites (Zipf 1.0), 16
planted leaks with mixed rates, T = next_prime(10 MiB).  N>1 (launched by
torchrun, or spawned here when --gpus N > 1 and WORLD_SIZE is unset): strong
scaling -- the same 1024 traces split into contiguous shards of 1024/N traces,
and the per-site tables summed with one all-reduce (the method's only exchange
step); --scaling weak gives every rank a full config-sized batch instead.

--impl reference: the CPU oracle (oracle/oracle.c) as it stands, on the host
cores, on the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "malloc/free events/sec replayed (1/2/4/8 B200) and % of HBM peak"
BYTES_PER_EVENT = 16
SAMPLE_BYTES = 32
ROW_BYTES_TABLE = 80


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--traces", type=int, default=0,
                    help="override the total traces (strong) / traces per rank (weak)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the K5 threshold-sweep field")
    return ap.parse_args()


def workload(cfg, n_traces_rank, world, n_traces_total=None, scaling="strong"):
    tot = n_traces_total if n_traces_total is not None else n_traces_rank * world
    return {"workload": f"{cfg.name}: {tot} traces x {cfg.events_per_trace} events ({n_traces_rank} traces/GPU), "
                        f"{cfg.n_sites} sites (Zipf {cfg.zipf_s}), {cfg.n_planted} planted leaks, T={cfg.T}",
            "traces_total": tot, "traces_per_gpu": n_traces_rank, "events_per_trace": cfg.events_per_trace,
            "scaling": scaling,
            "n_sites": cfg.n_sites, "threshold": cfg.T, "event_bytes": BYTES_PER_EVENT,
            "l2": f"inputs larger than L2 ({n_traces_rank * cfg.events_per_trace * 16 / 1e9:.2f} GB > 0.126 GB); no flush needed",
            "parallelism": f"dp{world} (trace shards, int64 all-reduce of the site table)"}


class ClockSampler:
    """NVML polling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.stop, self.first = [], set(), threading.Event(), threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.max = None

    def _run(self):
        nv = self.nv
        names = {getattr(nv, k, None): k for k in (
            "nvmlClocksEventReasonGpuIdle", "nvmlClocksEventReasonApplicationsClocksSetting",
            "nvmlClocksEventReasonSwPowerCap", "nvmlClocksEventReasonHwSlowdown",
            "nvmlClocksEventReasonSwThermalSlowdown", "nvmlClocksEventReasonHwThermalSlowdown",
            "nvmlClocksEventReasonHwPowerBrakeSlowdown", "nvmlClocksEventReasonSyncBoost")}
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if bit and (r & bit):
                        self.reasons.add(name.replace("nvmlClocksEventReason", "").lower())
            except Exception:
                pass
            self.first.set()
            time.sleep(0.0005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            self.first.wait(1.0)                      # polling before the timed work is enqueued
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop.set()
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max, "reasons": sorted(self.reasons - {"gpuidle"}),
                "n_samples": len(self.samples), "source": "nvml, 0.5 ms polling during the timed regions"}


def measured_peak():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy_ read+write, measured)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(config_id):
    """dram bytes per replay_kernel launch from the committed ncu --set full capture, if any."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        e = d.get(f"cfg{config_id}")
        return e["dram_bytes_per_launch"] if e else None
    except Exception:
        return None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_pass(lib, oracle, ev, off, cfg, threads):
    nt = len(off) - 1
    cap = oracle.sample_bound(ev, off, cfg.T)
    soff = np.zeros(nt + 1, dtype=np.uint64)
    soff[1:] = np.cumsum(cap)
    samples = np.zeros(max(int(soff[-1]), 1), dtype=oracle.SAMPLE_DTYPE)
    summ = np.zeros(nt, dtype=oracle.SUMMARY_DTYPE)
    table = np.zeros((cfg.n_sites, oracle.NCOL), dtype=np.uint64)
    t0 = time.perf_counter()
    lib.orc_replay_all(oracle._ptr(ev), oracle._ptr(off), nt, cfg.n_sites, cfg.T, 0, threads,
                       oracle._ptr(samples), oracle._ptr(soff), oracle._ptr(summ), oracle._ptr(table), None)
    num, den, op = oracle.gate(summ)
    prob, rate, flag = oracle.finalize(table, op, oracle.elapsed_ns(off))
    oracle.report_order(rate, flag)
    return time.perf_counter() - t0


def cpu_oracle_baseline(ev, off, cfg, reps=3, one_core_traces=64):
    """The oracle as it stands, on all host cores (the full rank-0 workload) and on 1 core (a
    bounded sample: its first ``one_core_traces`` traces), a1..a6 -- a few core-seconds."""
    import oracle
    lib = oracle._load()
    nt = len(off) - 1
    cores = os.cpu_count() or 1
    best = min(_oracle_pass(lib, oracle, ev, off, cfg, cores) for _ in range(reps))
    n1 = min(nt, one_core_traces)
    ev1, off1 = ev[:int(off[n1])], off[:n1 + 1]
    t1 = _oracle_pass(lib, oracle, ev1, off1, cfg, 1)
    return {"value": len(ev) / best, "unit": "events/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(), "value_1core": len(ev1) / t1,
            "sample": f"all cores: the full rank-0 workload ({len(ev)} events, {nt} traces), a1..a6, best of {reps}; "
                      f"1 core: its first {n1} traces ({len(ev1)} events)"}


def run_reference(args):
    """--impl reference: the oracle on the host cores (rank 0 only; the other ranks exit)."""
    import tracegen
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = tracegen.CONFIGS[args.config]
    ntr = args.traces or cfg.n_traces
    ev, off = tracegen.generate(cfg.with_traces(ntr))
    import oracle
    lib = oracle._load()
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        _oracle_pass(lib, oracle, ev, off, cfg, cores)
    dt = sum(_oracle_pass(lib, oracle, ev, off, cfg, cores) for _ in range(args.steps))
    v = len(ev) * args.steps / dt
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": "events/s",
                      "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
                      "vs_baseline": None, "dtype": "int64", "data": "synthetic",
                      "config": workload(cfg, ntr, 1, ntr, args.scaling),
                      "cpu_baseline": {"value": v, "unit": "events/s", "cores": cores, "kind": "oracle",
                                       "cpu_model": cpu_model(),
                                       "sample": f"full workload ({len(ev)} events) per step"},
                      "e2e": {"value": v, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def plan_launch(gpus: int, world_env, n_devices: int, impl: str = "native"):
    """How this process runs (pure; tested on CPU): ("run", None) -- this process is the
    rank (torchrun set WORLD_SIZE, or N = 1); ("spawn", None) -- start N NCCL ranks here with
    torch.distributed.run; ("error", msg) -- the request cannot be honoured."""
    if gpus < 1:
        return "error", f"--gpus {gpus}: must be >= 1"
    if world_env is not None:
        if int(world_env) != gpus:
            return "error", f"--gpus {gpus} but WORLD_SIZE={world_env}: launch one rank per GPU"
        return "run", None
    if gpus == 1 or impl == "reference":
        return "run", None
    if n_devices < gpus:
        return "error", f"--gpus {gpus} needs {gpus} CUDA devices on this node, {n_devices} visible"
    return "spawn", None


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def rank_traces(n_total: int, rank: int, world: int):
    """Strong scaling: contiguous trace shard [t0, t1) of ``rank`` (sizes differ by at most 1)."""
    q, r = divmod(n_total, world)
    t0 = rank * q + min(rank, r)
    return t0, t0 + q + (1 if rank < r else 0)


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    n_dev = 0
    if world_env is None and args.gpus > 1 and args.impl != "reference":
        import torch
        n_dev = torch.cuda.device_count()
    how, msg = plan_launch(args.gpus, world_env, n_dev, args.impl)
    if how == "error":
        print(f"bench.py: {msg}", file=sys.stderr)
        sys.exit(2)
    if how == "spawn":                               # one NCCL rank per GPU, started here
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                  "--master-port", str(_free_port()), os.path.abspath(__file__), *sys.argv[1:]])
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2212_07597_b200 as scl
    import tracegen

    world = int(world_env or "1")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = tracegen.CONFIGS[args.config]
    if args.scaling == "strong":                    # the config's traces, split across the ranks
        n_total = args.traces or cfg.n_traces
        t0, t1 = rank_traces(n_total, rank, world)
    else:                                           # every rank a config-sized batch of its own
        per = args.traces or cfg.n_traces
        n_total = per * world
        t0, t1 = rank * per, (rank + 1) * per
    ntr = t1 - t0
    gcfg = cfg.with_traces(n_total)
    # pinned host copy of this rank's traces (inputs of the e2e leg)
    n_ev = ntr * cfg.events_per_trace
    pinned = torch.empty(max(n_ev, 1) * 2, dtype=torch.int64, pin_memory=True)
    host_ev = pinned.numpy().view(tracegen.EVENT_DTYPE)
    _, off_local = tracegen.generate(gcfg, t0, t1, out=host_ev)
    host_ev = host_ev[:n_ev]
    stream = torch.cuda.current_stream()
    elapsed_ns = cfg.events_per_trace * 1000          # global max n_t * tick (all traces equal)
    total_events_step = n_total * cfg.events_per_trace

    tr = scl.scl_trace_load(host_ev, off_local, cfg.n_sites, device=local)
    r = None

    def step(r, timing=False, t=tr):
        r = scl.scl_replay_run(cfg.T, t, stream=stream, out=r, defer_finalize=world > 1, elapsed_ns=elapsed_ns,
                               timing=timing)
        if world > 1:
            dist.all_reduce(scl.device_table_tensor(r))
            scl.scl_finalize(r, elapsed_ns)
        return r

    for _ in range(max(args.warmup, 3)):
        r = step(r)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):                    # enqueued back to back: no host sync per step
            r = step(r)
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the stream pass's own duration (roofline): the same K steps again with the library's CUDA
    # events around its kernels (kept out of the timed loop above: ~2.5 us per event record)
    scl.scl_result_kernel_times(r)
    scl.scl_result_pass_times(r)
    with ClockSampler(local) as clk2:
        for _ in range(args.steps):
            r = step(r, timing=True)
        torch.cuda.synchronize()
    kern_ms = scl.scl_result_kernel_times(r)
    pass_ms = scl.scl_result_pass_times(r)
    clk.samples += clk2.samples; clk.reasons |= clk2.reasons
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = total_events_step * args.steps / (ms_max / 1e3)

    summ = scl.scl_trace_summaries(r)
    n_samples = int(summ["n_samples"].sum())

    # NEXT-1: the paper's comparison (Table tab:sampling-comparison) on the same resident traces:
    # the rate-based sampler at R = T (mean one sample per T bytes allocated or freed)
    rr = scl.scl_rate_run(cfg.T, tr, seed=2022, stream=stream)
    rate_ms = []
    for _ in range(3):
        rr = scl.scl_rate_run(cfg.T, tr, seed=2022, stream=stream, out=rr)
        rate_ms.append(scl.scl_rate_timing(rr))
    n_rate = int(scl.scl_rate_counts(rr).sum())
    next1 = {"rate_samples": n_rate, "threshold_samples": n_samples,
             "ratio": (n_rate / n_samples) if n_samples else None,
             "sample_log_bytes": {"rate": n_rate * 24, "threshold": n_samples * 32},
             "rate_kernels_ms": statistics.median(rate_ms),
             "note": "rate-based byte sampler, R = T, seed 2022, same traces (per rank)"}
    del rr
    # K5: a threshold sweep (11 primes above 2^20 .. 2^30) as 11 full replays vs one stream pass
    # + 10 re-thresholds over it (per rank, results reused; device time on the bench stream)
    sweep = None
    if not args.no_sweep:
        Ts = [scl.scl_next_prime(1 << k) for k in range(20, 31)]
        full = [scl.scl_replay_run(T_, tr, stream=stream) for T_ in Ts]
        sw = scl.scl_replay_sweep(Ts, tr, stream=stream)

        def _dev_ms(fn):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a_.record(stream); fn(); b_.record(stream); torch.cuda.synchronize()
            return a_.elapsed_time(b_)
        ms_full = min(_dev_ms(lambda: [scl.scl_replay_run(T_, tr, stream=stream, out=r_) for T_, r_ in zip(Ts, full)])
                      for _ in range(2))
        ms_sweep = min(_dev_ms(lambda: (scl.scl_replay_run(Ts[0], tr, stream=stream, out=sw[0]),
                                        [scl.scl_replay_rethreshold(T_, tr, sw[0], stream=stream, out=r_)
                                         for T_, r_ in zip(Ts[1:], sw[1:])])) for _ in range(2))
        sweep = {"thresholds": len(Ts), "full_replays_ms": ms_full, "one_pass_plus_rethreshold_ms": ms_sweep,
                 "note": "K5: scl_replay_sweep (one stream pass, the other thresholds re-chained over it)"}
        for x in full + sw:
            x.free()
        del full, sw
    kern_avg = statistics.mean(kern_ms)
    pass_avg = statistics.mean(pass_ms)
    alg_bytes = n_ev * BYTES_PER_EVENT + n_samples * SAMPLE_BYTES + cfg.n_sites * ROW_BYTES_TABLE
    achieved = alg_bytes / (kern_avg / 1e3) / 1e9
    peak, peak_src = measured_peak()
    traffic = ncu_traffic(args.config)
    launches = scl.scl_result_launches(r)           # kernels of one step (the library's count)
    cold = launches > 2 + (0 if world == 1 else (1 if cfg.n_sites <= 16384 else 2))

    # a freshly loaded batch on the device: scl_trace_reload from a device copy of the
    # events (one fused copy + load-statistics pass) and one step, CUDA events around both
    fresh = None
    if not args.no_e2e:
        dsrc = torch.from_numpy(host_ev.view(np.int64).reshape(-1)).to(f"cuda:{local}")
        trf = scl.scl_trace_load(dsrc, off_local, cfg.n_sites, device=local)
        rf = scl.scl_replay_run(cfg.T, trf, stream=stream, defer_finalize=world > 1, elapsed_ns=elapsed_ns)
        torch.cuda.synchronize()
        a_, b_, c_ = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a_.record(stream)
        scl.scl_trace_reload(trf, dsrc, off_local, cfg.n_sites, stream=stream)
        b_.record(stream)
        rf = scl.scl_replay_run(cfg.T, trf, stream=stream, out=rf, defer_finalize=world > 1, elapsed_ns=elapsed_ns)
        c_.record(stream)
        torch.cuda.synchronize()
        fresh = {"load_ms": a_.elapsed_time(b_), "step_ms": b_.elapsed_time(c_),
                 "events_per_s": n_ev / ((a_.elapsed_time(c_)) / 1e3),
                 "note": "per rank: scl_trace_reload from a device copy of the batch (the fused copy + load "
                         "statistics pass: sample bounds, event check, size histogram) then one step; host "
                         "sources add the PCIe copy (the e2e line)"}
        rf.free(); trf.free()
        del dsrc
        torch.cuda.synchronize()

    # e2e through the public API: H2D of this step's events from pinned memory, replay, report D2H
    e2e = None
    if not args.no_e2e:
        # the user's batch loop: refill a handle with the next batch of traces from pinned host
        # memory (H2D inside the timed region), replay it, [all-reduce], read the report back (D2H)
        tr.free()
        r.free()
        torch.cuda.synchronize()
        reps = max(3, min(5, args.steps))
        trx = scl.scl_trace_load(host_ev, off_local, cfg.n_sites, device=local)
        rx = None

        def e2e_step(rx):
            scl.scl_trace_reload(trx, host_ev, off_local, cfg.n_sites, stream=stream)
            rx = scl.scl_replay_run(cfg.T, trx, stream=stream, out=rx, defer_finalize=world > 1,
                                    elapsed_ns=elapsed_ns)
            if world > 1:
                dist.all_reduce(scl.device_table_tensor(rx))
                scl.scl_finalize(rx, elapsed_ns)
            return rx, scl.scl_site_report(rx)

        for _ in range(2):                             # warm: buffers sized, result allocated
            rx, rows = e2e_step(rx)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0_ = time.perf_counter()
        for _ in range(reps):
            rx, rows = e2e_step(rx)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0_], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": total_events_step * reps / float(dt.item()), "unit": "events/s",
               "h2d_bytes_per_step": int(n_ev * 16 + off_local.nbytes),
               "d2h_bytes_per_step": int(rows.nbytes + 24),
               "note": "per step and rank: scl_trace_reload(pinned host events -> the handle's device buffers) + "
                       "scl_replay_run [+ all-reduce + scl_finalize] + scl_site_report (wall clock, max over ranks); "
                       "bytes are rank 0's"}
        rx.free()
        trx.free()

    if rank == 0:
        cpu = None
        if not args.no_cpu:
            cpu = cpu_oracle_baseline(host_ev, off_local, cfg)
        out = {
            "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int64", "data": "synthetic (tracegen, seeded)",
            "config": workload(cfg, ntr, world, n_total, args.scaling),
            "hbm_gbs_step": total_events_step * BYTES_PER_EVENT / (ms_max / 1e3) / 1e9 / world,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "scl::replay_kernel",
                         "kernel_ms": kern_avg, "peak_source": peak_src,
                         "stream_pass_ms": pass_avg,
                         "stream_pass": "replay_kernel" + (" + cold_hist_kernel + cold_sum_kernel (Tier E of its "
                                                           "cold-record stream)" if cold else "") + ": a1-a5 before the post pass",
                         "stream_pass_frac": alg_bytes / (pass_avg / 1e3) / 1e9 / peak,
                         "alg_bytes_per_launch": alg_bytes,
                         "alg_bytes_rule": "16 B/event read + 32 B/sample written + 80 B/site table flush",
                         "frac_of_8tbs_spec": achieved / 8000.0,
                         "step_frac": total_events_step * BYTES_PER_EVENT / world / (ms_max / args.steps / 1e3) / 1e9 / peak},
            "clocks": clk.summary(),
            "e2e": e2e,
            "fresh_batch": fresh,
            "gpu_launches": launches * args.steps,
            "gpu_launches_note": "per step: replay_kernel (its CTA 0 prepares the run)" +
                                 (", cold_hist_kernel, cold_sum_kernel" if cold else "") +
                                 ", post_kernel (reclaim + per-sample reduce + a6 grid-wide)" if world == 1 else
                                 ", post_kernel (reclaim + per-sample reduce), then after the all-reduce the a6 "
                                 "kernel(s): report_kernel, or report_flags + report_rows above 16,384 sites",
            "kernel_timing": "stream-pass kernel durations from the library's CUDA events in a second pass of K steps",
            "n_samples_per_step": n_samples,
            "next1_rate_vs_threshold": next1,
            "k5_threshold_sweep": sweep,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
