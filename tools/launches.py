"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, mean, share."""
import csv, collections, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for d in data:
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[d["Kernel Name"].split("(")[0][:70]].append(float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]])
    return agg

if __name__ == "__main__":
    agg = load(sys.argv[1])
    skip = sys.argv[2].split(",") if len(sys.argv) > 2 else ["load_stats"]
    tot = sum(sum(v) for k, v in agg.items() if not any(s in k for s in skip))
    print(f"{'kernel':70s} {'n':>4s} {'mean us':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        sh = "" if any(s in k for s in skip) else f"{100*sum(v)/tot:6.1f}%"
        print(f"{k:70s} {len(v):4d} {sum(v)/len(v):10.2f} {sh:>7s}")
