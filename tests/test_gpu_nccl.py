"""scl_run_opts.nccl_comm: the library's own SUM all-reduce of the summable
table and MAX of the elapsed time, on a 1-rank communicator (the only GPU of this box), against
the oracle; and scl_trace_summary_of.  The N-rank arithmetic is covered on CPU (test_dist_gloo)."""
import ctypes

import numpy as np
import pytest

import oracle
import paper_2212_07597_b200 as scl
import tracegen
from parity import compare

pytestmark = pytest.mark.gpu


def _comm_1rank():
    import torch
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")                       # the primary context exists
    nccl = ctypes.CDLL("libnccl.so.2", mode=ctypes.RTLD_GLOBAL)

    class UID(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_char * 128)]
    uid = UID()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, UID, ctypes.c_int]
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    return nccl, comm


def test_nccl_comm_one_rank_matches_oracle_and_summary_of():
    nccl, comm = _comm_1rank()
    try:
        cfg = tracegen.CONFIGS[2].with_traces(3)
        ev, off = tracegen.generate(cfg)
        tr = scl.scl_trace_load(ev, off, cfg.n_sites)
        r = scl.scl_replay_run(cfg.T, tr, tick_ns=1000, nccl_comm=comm.value)
        ref = compare(ev, off, cfg.n_sites, cfg.T, r)
        s = ref["result"].summaries
        for t in range(3):
            assert scl.scl_trace_summary_of(r, t) == (int(s["f_final"][t]), int(s["hwm"][t]),
                                                      int(s["n_samples"][t]), int(s["n_episodes"][t]))
        with pytest.raises(scl.SclError):
            scl.scl_trace_summary_of(r, 3)
        r2 = scl.scl_replay_run(1048583, tr, tick_ns=1000, nccl_comm=comm.value, defer_finalize=True)
        scl.scl_finalize(r2)
        compare(ev, off, cfg.n_sites, 1048583, r2)
    finally:
        nccl.ncclCommDestroy(comm)
