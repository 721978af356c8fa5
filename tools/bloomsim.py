"""Debug: emulate the runner's Bloom pointer-match for one trace (CPU), counting positive chunks
per unit for the tracked (unreclaimed) episode pointer."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle, tracegen

t = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10485767
cfg = tracegen.CONFIGS[2].with_traces(t + 1)
ev, off = tracegen.generate(cfg)
e = ev[int(off[t]):int(off[t + 1])]
n = len(e)
r = oracle.replay(e, np.array([0, n], dtype=np.uint64), cfg.n_sites, T)
smp = r.samples
ptr = e["ptr"].astype(np.uint64); meta = e["meta"].astype(np.uint64)
kind = ((meta >> np.uint64(40)) & np.uint64(3)).astype(np.int64)
def bword(p): return ((((p >> np.uint64(4)) & np.uint64(0xffffffff)) * np.uint64(0x9E3779B1)) & np.uint64(0xffffffff)) >> np.uint64(26)
def bmask(p):
    h = (((p >> np.uint64(4)) & np.uint64(0xffffffff)) * np.uint64(0x85EBCA77)) & np.uint64(0xffffffff)
    return (np.uint64(1) << (h >> np.uint64(27))) | (np.uint64(1) << ((h >> np.uint64(22)) & np.uint64(31)))
CH = 256
nch = (n + CH - 1) // CH
bloom = np.zeros((nch, 64), dtype=np.uint64)
fr = np.nonzero(kind == 1)[0]
np.bitwise_or.at(bloom, (fr // CH, bword(ptr[fr]).astype(np.int64)), bmask(ptr[fr]))
# episodes
eps = [(int(s["idx"]), int(ptr[int(s["idx"])])) for s in smp if s["new_max"]]
eps.append((n, 0))
tot_pos = 0; tot_fp = 0
for k in range(len(eps) - 1):
    i0, p = eps[k]; i1 = eps[k + 1][0]
    frees = np.nonzero((kind[i0 + 1:i1] == 1) & (ptr[i0 + 1:i1] == np.uint64(p)))[0]
    end = i0 + 1 + frees[0] if len(frees) else i1
    c0, c1 = i0 // CH, (end - 1) // CH
    w = int(bword(np.uint64(p))); m = bmask(np.uint64(p))
    pos = [(c) for c in range(c0, c1 + 1) if (bloom[c, w] & m) == m]
    tot_pos += len(pos)
    print(f"ep@{i0} unit {i0//8192} ptr {p:#x} reclaimed={len(frees)>0} span units {i0//8192}..{(end-1)//8192} "
          f"chunks {c1-c0+1} positives {len(pos)} word {w} wordpop(avg) {np.mean([bin(int(x)).count('1') for x in bloom[c0:c1+1, w]]):.1f}")
print("samples", len(smp), "episodes", len(eps) - 1, "total positive chunks", tot_pos)
print("mean bits per word", np.mean([bin(int(x)).count('1') for x in bloom.ravel()]))
