"""Key metrics of one kernel capture (ncu --set full) as a text summary for profiles/:
    python tools/ncu_summary.py REPORT.ncu-rep "header line" [ALG_BYTES] > profiles/rNN_xxx.txt"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "gpc__cycles_elapsed.max", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]

rep, header = sys.argv[1], sys.argv[2]
alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
print("# " + header)
print(f"# kernel: {d.get('Kernel Name', ('', '?'))[1][:100]}")
print()
for k in KEYS:
    if k in d:
        u, v = d[k]
        print(f"{k:90s} {v:>20s} {u}")
print()
print("# top warp stall reasons (warps stalled per issued instruction)")
st = []
for h, (u, v) in d.items():
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v), h))
        except ValueError:
            pass
for v, h in sorted(st, reverse=True)[:10]:
    print(f"{h:90s} {v:20.6f}")


def num(k):
    u, v = d[k]
    x = float(v.replace(",", ""))
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}.get(u, 1)


if alg and "dram__bytes_read.sum" in d:
    traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    t = num("gpu__time_duration.sum")
    tu = d["gpu__time_duration.sum"][0]
    secs = t * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}.get(tu, 1e-9)
    print()
    print(f"# algorithmic bytes per launch {alg:.0f}; dram traffic {traffic:.0f} = {100 * traffic / alg:.1f}% of algorithmic;"
          f" {alg / secs / 1e9:.0f} GB/s algorithmic under ncu (cold, serialised)")
