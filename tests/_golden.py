"""Parser for tests/golden/*.txt hand-worked traces (each file cites its passage)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    T, hwm, events, samples, summary, sites, gate, probs = None, "prefix", [], [], {}, {}, None, {}
    ptrs = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        if tok[0] == "T":
            T = int(tok[1])
        elif tok[0] == "hwm":
            hwm = tok[1]
        elif tok[0] in ("a", "f"):
            p = ptrs.setdefault(tok[1], 0x1000 * (len(ptrs) + 1))
            events.append((tok[0], p, int(tok[2]), int(tok[3])))
        elif tok[0] == "sample":
            i, k, net, F, s, nm = tok[1:]
            samples.append((int(i), k, int(net), int(F), int(s), bool(int(nm))))
        elif tok[0] == "summary":
            summary = {k: int(v) for k, v in (x.split("=") for x in tok[1:])}
        elif tok[0] == "site":
            sites[int(tok[1])] = {k: int(v) for k, v in (x.split("=") for x in tok[2:])}
        elif tok[0] == "gate":
            gate = {k: int(v) for k, v in (x.split("=") for x in tok[1:])}
        elif tok[0] == "prob":
            probs[int(tok[1])] = float(tok[2])
    return dict(T=T, hwm=hwm, events=events, samples=samples, summary=summary, sites=sites,
                gate=gate, probs=probs)


def all_names():
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".txt"))
