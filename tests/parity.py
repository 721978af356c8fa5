"""Helpers: run the CUDA path through the C-ABI and compare it element by
element with the oracle on the same seeded inputs (bit-exact for integers and
flags; fp64 probabilities/rates within 1e-12 relative -- BASELINE.json
north_star -- and in practice bit-identical)."""
import numpy as np

import oracle
import paper_2212_07597_b200 as scl

REL_TOL = 1e-12


def gpu_run(events, offsets, n_sites, T, formula=0, tick_ns=1000, traces=None, out=None, validate=False, hwm_mode=0):
    tr = traces if traces is not None else scl.scl_trace_load(events, offsets, n_sites, validate=validate)
    r = scl.scl_replay_run(T, tr, formula=formula, tick_ns=tick_ns, out=out, hwm_mode=hwm_mode)
    return tr, r


def compare(events, offsets, n_sites, T, r, formula=0, tick_ns=1000, traces_to_check=None, ref=None, hwm_mode=0):
    """Assert GPU result r == oracle on (events, offsets). Returns the oracle dict."""
    offsets = np.asarray(offsets, dtype=np.uint64)
    ref = ref or oracle.full(events, offsets, n_sites, T, hwm_mode=hwm_mode, formula=formula, tick_ns=tick_ns, n_threads=8)
    res = ref["result"]
    n_traces = len(offsets) - 1
    # per-trace summaries
    summ = scl.scl_trace_summaries(r)
    for f in ("f_final", "hwm", "n_samples", "n_episodes", "f_first_sample", "f_last_sample"):
        bad = np.nonzero(summ[f] != res.summaries[f])[0]
        assert len(bad) == 0, f"summary {f} differs at traces {bad[:10]}: gpu {summ[f][bad[:5]]} oracle {res.summaries[f][bad[:5]]}"
    # samples, element by element
    check = range(n_traces) if traces_to_check is None else traces_to_check
    for t in check:
        g = scl.scl_samples(r, t)
        o = res.trace_samples(t)
        assert len(g) == len(o), f"trace {t}: {len(g)} samples vs oracle {len(o)}"
        for f in ("idx", "net", "footprint", "site", "kind", "new_max"):
            if not np.array_equal(g[f], o[f]):
                k = int(np.nonzero(g[f] != o[f])[0][0])
                raise AssertionError(f"trace {t} sample {k} field {f}: gpu {g[k]} oracle {o[k]}")
    # site table, report rows, order
    rows = scl.scl_site_report(r)
    order = ref["order"]
    assert np.array_equal(rows["site"], order), "report order differs"
    tab = res.site_table[order]
    for c in range(10):
        if not np.array_equal(rows["col"][:, c], tab[:, c]):
            k = int(np.nonzero(rows["col"][:, c] != tab[:, c])[0][0])
            raise AssertionError(f"site table column {oracle.COLS[c]} differs at site {order[k]}: "
                                 f"gpu {rows['col'][k, c]} oracle {tab[k, c]}")
    assert np.array_equal(rows["leak_flag"], ref["flag"][order].astype(np.uint32)), "leak flags differ"
    for name, key in (("leak_prob", "prob"), ("leak_rate_mbps", "rate")):
        a, b = rows[name], ref[key][order]
        err = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
        assert np.all((a == b) | (err <= REL_TOL)), f"{name} differs beyond 1e-12 rel"
    num, den, op = scl.scl_gate(r)
    assert (num, den, op) == ref["gate"], f"gate {num, den, op} vs oracle {ref['gate']}"
    return ref
