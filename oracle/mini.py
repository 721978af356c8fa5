"""Pure-Python mini-oracle for tiny traces -- TEST INFRASTRUCTURE ONLY.

A second, independent transcription of the method (P:429-434 sampler,
P:20-39 leak tracker) written in the A/F-counter vocabulary of the paper
(``|A - F| >= T`` then "resets the counters"), rather than the signed carry
of oracle.c, so that the two transcriptions cross-check each other.  Used
only on small inputs (loops are pure Python).

Events are tuples ``(kind, ptr, size, site)`` with kind 'a' (alloc) or 'f'
(free).  Returns samples as tuples ``(idx, kind, net, F, site, new_max)``
with kind 'G'/'D', the trace summary and per-site dicts.
"""
from __future__ import annotations

from collections import defaultdict


def replay_trace(events, T, hwm_mode="prefix", with_domains=False):
    """with_domains: also return, per sample, (A, managed part of A) -- the allocated bytes since
    the last reset and those of managed-domain events (5th tuple element 1; NEXT-2)."""
    A = 0          # bytes allocated since the last sample
    Am = 0         # of which managed (Python) allocations
    domains = []
    Fr = 0         # bytes freed since the last sample
    footprint = 0
    peak = 0
    peak_at_samples = 0
    tracked = None         # (ptr, site) of the sampled allocation
    reclaimed = False
    samples = []
    cols = defaultdict(lambda: defaultdict(int))
    episodes = 0
    for i, ev in enumerate(events):
        kind, ptr, size, site = ev[:4]
        prev_peak = peak
        if kind == "a":
            A += size
            if len(ev) > 4 and ev[4]:
                Am += size
            footprint += size
            cols[site]["n_malloc"] += 1
            cols[site]["malloc_bytes"] += size
        elif kind == "f":
            Fr += size
            footprint -= size
            cols[site]["n_free"] += 1
            cols[site]["free_bytes"] += size
            if tracked is not None and not reclaimed and tracked[0] == ptr:
                reclaimed = True            # "checks to see whether this object is ever reclaimed"
        else:
            continue
        peak = max(peak, footprint)
        if abs(A - Fr) >= T:                # "|A - F| >= T"
            net = A - Fr
            growth = net > 0
            if hwm_mode == "prefix":
                new_max = growth and footprint > prev_peak
            else:
                new_max = growth and footprint > peak_at_samples
            peak_at_samples = max(peak_at_samples, footprint)
            samples.append((i, "G" if growth else "D", net, footprint, site, new_max))
            domains.append((A, Am))
            if growth:
                cols[site]["n_growth"] += 1
                cols[site]["growth_bytes"] += net
            else:
                cols[site]["n_decline"] += 1
                cols[site]["decline_bytes"] += -net
            if new_max:
                if tracked is not None and reclaimed:
                    cols[tracked[1]]["leak_frees"] += 1
                tracked = (ptr, site)
                reclaimed = False
                cols[site]["leak_mallocs"] += 1
                episodes += 1
            A = Fr = Am = 0                 # "resets the counters"
    if tracked is not None and reclaimed:
        cols[tracked[1]]["leak_frees"] += 1
    summary = dict(f_final=footprint, hwm=peak, n_samples=len(samples), n_episodes=episodes,
                   f_first_sample=samples[0][3] if samples else 0,
                   f_last_sample=samples[-1][3] if samples else 0)
    if with_domains:
        return samples, summary, cols, domains
    return samples, summary, cols
