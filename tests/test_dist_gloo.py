"""N>1 host logic on CPU (world_size 2, gloo): trace sharding, the int64 SUM
all-reduce of the summable table and the global elapsed MAX, checked against
the single-process oracle.  The per-rank tables come from the oracle on each
shard (stand-in for the device tables, which need a GPU), laid out exactly
like scl_result_device_table (site table then 3 gate sums)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import tracegen
from paper_2212_07597_b200 import dist as sdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _summable(res, n_sites):
    num, den, _ = oracle.gate(res.summaries)
    cnt = int(np.sum(res.summaries["n_samples"] >= 2))
    return np.concatenate([res.site_table.reshape(-1).astype(np.int64), np.array([num, den, cnt], dtype=np.int64)])


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = tracegen.CONFIGS[2].with_traces(5)
    ev, off = tracegen.generate(cfg, n_threads=2)
    sev, soff, (t0, t1) = sdist.shard(ev, off, rank, world)
    res = oracle.replay(sev, soff, cfg.n_sites, cfg.T)
    tab = torch.from_numpy(_summable(res, cfg.n_sites))
    sdist.reduce_table(tab)
    lens = soff[1:] - soff[:-1]
    el = sdist.global_elapsed_ns(int(lens.max()) if len(lens) else 0, 1000)
    q.put((rank, (t0, t1), tab.numpy().copy(), el))
    dist.destroy_process_group()


def test_shard_range_balanced_and_complete():
    off = np.array([0, 10, 10, 50, 51, 100, 300, 300], dtype=np.uint64)
    for world in (1, 2, 3, 4, 7, 9):
        rngs = [sdist.shard_range(off, r, world) for r in range(world)]
        assert rngs[0][0] == 0 and rngs[-1][1] == len(off) - 1
        for a, b in zip(rngs, rngs[1:]):
            assert a[1] == b[0]
    assert sdist.shard_range(np.array([0, 4, 8, 12, 16], dtype=np.uint64), 1, 2) == (2, 4)


def test_gloo_world2_table_reduce_matches_single_process():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    cfg = tracegen.CONFIGS[2].with_traces(5)
    ev, off = tracegen.generate(cfg)
    full = oracle.replay(ev, off, cfg.n_sites, cfg.T)
    ref = _summable(full, cfg.n_sites)
    assert out[0][1][0] == 0 and out[0][1][1] == out[1][1][0] and out[1][1][1] == 5
    for rank, _, tab, el in out:
        assert np.array_equal(tab, ref)            # bit-exact integer reduction
        assert el == oracle.elapsed_ns(off)
    # a6 on the reduced table equals the single-process report
    num, den, cnt = (int(x) for x in ref[-3:])
    op = cnt > 0 and 100 * num >= den
    assert (num, den, op) == oracle.gate(full.summaries)


def test_plan_waves_cover_in_order_within_limit():
    """Resident waves: consecutive whole-trace ranges covering every trace once, each within the
    event budget unless it is a single longer trace."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        lens = rng.integers(0, 50, size=int(rng.integers(1, 40)))
        off = np.zeros(len(lens) + 1, dtype=np.uint64)
        off[1:] = np.cumsum(lens)
        budget = int(rng.integers(1, 120))
        waves = sdist.plan_waves(off, budget)
        assert waves[0][0] == 0 and waves[-1][1] == len(lens)
        for (a0, a1), (b0, b1) in zip(waves, waves[1:]):
            assert a1 == b0
        for t0, t1 in waves:
            assert t1 > t0
            n = int(off[t1] - off[t0])
            assert n <= budget or t1 == t0 + 1
            if t1 < len(lens):                               # greedy: the next trace would not fit
                assert int(off[t1 + 1] - off[t0]) > budget
