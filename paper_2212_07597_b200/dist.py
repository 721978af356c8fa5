"""Multi-GPU plumbing: one process per GPU, traces sharded
across ranks, one int64 all-reduce of the summable table (per-site columns +
gate sums) before a6.  Integer addition is associative, so the reduced table
is bit-exact whatever algorithm NCCL picks (NVLS, ring, tree).

torch.distributed is plumbing only; the replay itself runs in libscl.so.
"""
from __future__ import annotations

import numpy as np


def shard_range(offsets, rank: int, world: int):
    """Contiguous trace range [t0, t1) of ``rank``, balanced by event count
    (the cut for rank r is the first trace boundary at or after r/world of the
    events)."""
    off = np.asarray(offsets, dtype=np.uint64)
    n_traces = len(off) - 1
    total = int(off[-1])

    def cut(r):
        if r <= 0:
            return 0
        if r >= world:
            return n_traces
        target = (total * r + world - 1) // world
        return int(np.searchsorted(off[:-1], np.uint64(target), side="left"))

    return cut(rank), cut(rank + 1)


def shard(events, offsets, rank: int, world: int):
    """(events, offsets) of this rank's shard, offsets rebased to 0."""
    t0, t1 = shard_range(offsets, rank, world)
    off = np.asarray(offsets, dtype=np.uint64)
    a, b = int(off[t0]), int(off[t1])
    return events[a:b], (off[t0:t1 + 1] - off[t0]).astype(np.uint64), (t0, t1)


def reduce_table(table, group=None):
    """In-place SUM all-reduce of an int64 tensor (the device table of
    scl_result_device_table, or any same-layout tensor)."""
    import torch.distributed as dist
    dist.all_reduce(table, op=dist.ReduceOp.SUM, group=group)
    return table


def global_elapsed_ns(local_max_len: int, tick_ns: int = 1000, group=None, device="cpu") -> int:
    """Synthetic elapsed time (reading Q11) over ALL ranks: max_t n_t * tick."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(local_max_len)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item()) * tick_ns


def replay_distributed(events, offsets, n_sites: int, T: int, rank: int, world: int, device: int,
                       tick_ns: int = 1000, formula: int = 0, group=None):
    """Shard -> scl_trace_load -> scl_replay_run(defer) -> all-reduce -> scl_finalize.
    Every rank ends with the global report; samples stay rank-local."""
    import torch
    from . import device_table_tensor, scl_finalize, scl_replay_run, scl_trace_load
    torch.cuda.set_device(device)
    ev, off, rng = shard(events, offsets, rank, world)
    tr = scl_trace_load(ev, off, n_sites, device=device)
    r = scl_replay_run(T, tr, tick_ns=tick_ns, formula=formula, defer_finalize=True)
    lens = off[1:] - off[:-1]
    el = global_elapsed_ns(int(lens.max()) if len(lens) else 0, tick_ns, group, device=f"cuda:{device}")
    reduce_table(device_table_tensor(r), group)
    scl_finalize(r, el)
    return tr, r, rng


# ---------------------------------------------------------------- resident waves
# A rank whose shard does not fit in HBM (configs 4/5 at 1/2/4 GPUs) replays it in waves of whole
# traces: traces are independent (every trace starts from F = 0 with its own sampler and tracker),
# so a wave needs no carry; the summable tables of the waves add up (integer sums), and a6 runs
# once on the total.  Per-trace outputs (summaries, samples) are collected per wave.

def plan_waves(offsets, wave_events: int):
    """Consecutive trace ranges [t0, t1) with at most ``wave_events`` events each (a single trace
    longer than that is a wave of its own)."""
    off = np.asarray(offsets, dtype=np.uint64)
    n = len(off) - 1
    waves, t0 = [], 0
    while t0 < n:
        limit = np.uint64(int(off[t0]) + max(int(wave_events), 1))
        t1 = int(np.searchsorted(off, limit, side="right")) - 1      # last boundary <= limit
        t1 = min(max(t1, t0 + 1), n)
        waves.append((t0, t1))
        t0 = t1
    return waves


def replay_waves(events, offsets, n_sites: int, T: int, wave_events: int, device: int = 0,
                 tick_ns: int = 1000, formula: int = 0, rank: int = 0, world: int = 1, group=None,
                 keep_samples: bool = True):
    """Replay this rank's shard in resident waves of at most ``wave_events`` events (one device
    trace buffer, refilled per wave), sum the waves' tables on the device, all-reduce across ranks
    when world > 1, and run a6 once.  Returns (result of the last wave holding the global table and
    report, per-trace summaries of the shard, per-trace sample arrays or None, shard trace range)."""
    import torch
    from . import (device_table_tensor, scl_finalize, scl_replay_run, scl_samples, scl_trace_load,
                   scl_trace_reload, scl_trace_summaries)
    torch.cuda.set_device(device)
    if world > 1:
        ev, off, rng = shard(events, offsets, rank, world)
    else:
        ev, off, rng = events, np.asarray(offsets, dtype=np.uint64), (0, len(offsets) - 1)
    tr, r, acc = None, None, None
    summaries, samples = [], [] if keep_samples else None
    for t0, t1 in plan_waves(off, wave_events):
        a, b = int(off[t0]), int(off[t1])
        wev, woff = ev[a:b], (off[t0:t1 + 1] - off[t0]).astype(np.uint64)
        tr = scl_trace_load(wev, woff, n_sites, device=device) if tr is None else \
            scl_trace_reload(tr, wev, woff, n_sites)
        r = scl_replay_run(T, tr, tick_ns=tick_ns, formula=formula, defer_finalize=True, out=r)
        tab = device_table_tensor(r)
        acc = tab.clone() if acc is None else acc.add_(tab)
        summaries.append(scl_trace_summaries(r).copy())
        if keep_samples:
            samples.extend(scl_samples(r, t) for t in range(t1 - t0))
    if r is None:
        raise ValueError("no traces to replay")
    device_table_tensor(r).copy_(acc)
    lens = off[1:] - off[:-1]
    el = global_elapsed_ns(int(lens.max()) if len(lens) else 0, tick_ns, group, device=f"cuda:{device}") \
        if world > 1 else (int(lens.max()) if len(lens) else 0) * tick_ns
    if world > 1:
        reduce_table(device_table_tensor(r), group)
    scl_finalize(r, el)
    return r, np.concatenate(summaries), samples, rng
