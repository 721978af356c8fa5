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
