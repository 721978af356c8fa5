"""One-line summary of bench JSON lines: python tools/bsum.py FILE..."""
import json, sys
for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        rf = d.get("roofline") or {}
        print(f"{f}: {d['config']['workload'][:60]} value {d['value']:.4g} ms/step {d['ms_per_step']:.4f} "
              f"kernel_ms {rf.get('kernel_ms', 0):.4f} frac {rf.get('frac', 0):.3f} step_frac {rf.get('step_frac', 0) or 0:.3f} "
              f"launches {d.get('gpu_launches')} e2e {(d.get('e2e') or {}).get('value')}")
