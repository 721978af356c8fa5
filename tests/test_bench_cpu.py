"""bench.py's CPU legs (the reference arm = the oracle on the host cores, and the cpu_baseline
helper) run here without a GPU, so that a signature change in the oracle breaks a CPU test."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "events/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_cpu_baseline_helper():
    sys.path.insert(0, ROOT)
    import bench
    import tracegen
    cfg = tracegen.CONFIGS[1]
    ev, off = tracegen.generate(cfg)
    r = bench.cpu_oracle_baseline(ev, off, cfg, reps=1)
    assert r["value"] > 0 and r["value_1core"] > 0 and r["kind"] == "oracle"


def test_plan_launch():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.plan_launch(1, None, 0) == ("run", None)                 # N = 1: this process
    assert bench.plan_launch(8, "8", 8) == ("run", None)                  # torchrun rank
    assert bench.plan_launch(4, None, 8) == ("spawn", None)               # spawn 4 NCCL ranks here
    assert bench.plan_launch(2, None, 2, impl="reference") == ("run", None)   # oracle: rank 0 only
    how, msg = bench.plan_launch(2, None, 1)
    assert how == "error" and "needs 2 CUDA devices" in msg
    how, msg = bench.plan_launch(2, "4", 4)
    assert how == "error" and "WORLD_SIZE=4" in msg
    assert bench.plan_launch(0, None, 8)[0] == "error"


def test_gpus_without_devices_fails_loudly():
    """--gpus 2 with fewer visible GPUs: a clear error and a nonzero exit, never a silent 1-rank run."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 2, (out.returncode, out.stderr[-2000:])
    assert "needs 2 CUDA devices" in out.stderr and out.stdout.strip() == ""


def test_rank_traces_strong_split():
    sys.path.insert(0, ROOT)
    import bench
    for n, w in ((1024, 8), (1024, 3), (64, 8), (5, 8), (1, 1)):
        shards = [bench.rank_traces(n, r, w) for r in range(w)]
        assert shards[0][0] == 0 and shards[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
        sizes = [b - a for a, b in shards]
        assert max(sizes) - min(sizes) <= 1
