"""Per-source-line instruction counts and stall samples of one kernel in an ncu report
(--import-source on, -lineinfo):  python tools/ncu_lines.py REPORT.ncu-rep [TOP] [FILE:LO-HI ...]
Prints the TOP lines by executed warp instructions, and the totals of the given line ranges."""
import csv, io, subprocess, sys

def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, rows = None, []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "":
            continue
        try:
            rows.append((cur, int(r[0]), r[1].strip()[:90], int(r[7]) if r[7] not in ("-", "") else 0,
                         int(r[4]) if r[4] not in ("-", "") else 0))
        except (ValueError, IndexError):
            pass
    return rows

if __name__ == "__main__":
    rows = load(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    tot_i = sum(r[3] for r in rows); tot_s = sum(r[4] for r in rows)
    print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
    for f, ln, src, ins, st in sorted(rows, key=lambda r: -r[3])[:top]:
        print(f"{f}:{ln:5d} {100*ins/tot_i:5.1f}% ins {100*st/max(tot_s,1):5.1f}% smp  {src}")
    for spec in sys.argv[3:]:
        f, rng = spec.split(":"); lo, hi = map(int, rng.split("-"))
        i = sum(r[3] for r in rows if r[0] == f and lo <= r[1] <= hi); s = sum(r[4] for r in rows if r[0] == f and lo <= r[1] <= hi)
        print(f"{spec}: {100*i/tot_i:.1f}% instructions, {100*s/max(tot_s,1):.1f}% stall samples")
