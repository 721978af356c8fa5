"""Parity on subsets of the two configurations that do not fit one GPU (BASELINE configs 4 and
5): config 4's 200,000 Zipf(1.2) sites (most of them on the L2 path) and config 5's heavy-tailed
sizes at its dense threshold T = 65537 and at a sweep threshold (re-threshold), element by
element against the oracle."""
import dataclasses

import numpy as np
import pytest

import paper_2212_07597_b200 as scl
import tracegen
from parity import compare, gpu_run

pytestmark = pytest.mark.gpu


def test_config4_subset():
    cfg = tracegen.CONFIGS[4].with_traces(3)
    ev, off = tracegen.generate(cfg)
    _, r = gpu_run(ev, off, cfg.n_sites, cfg.T)
    compare(ev, off, cfg.n_sites, cfg.T, r)


def test_config5_subset_dense_threshold_and_sweep():
    cfg = dataclasses.replace(tracegen.CONFIGS[5].with_traces(2), events_per_trace=12_000_000)
    ev, off = tracegen.generate(cfg)
    tr, r = gpu_run(ev, off, cfg.n_sites, cfg.T)
    compare(ev, off, cfg.n_sites, cfg.T, r)
    T2 = scl.scl_next_prime(1 << 20)
    r2 = scl.scl_replay_rethreshold(T2, tr, r, tick_ns=1000)
    compare(ev, off, cfg.n_sites, T2, r2)
