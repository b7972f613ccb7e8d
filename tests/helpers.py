"""Shared test fixtures: seeded problems in standard form, comparisons."""
from __future__ import annotations

import numpy as np

from paper_2407_16144_b200 import gen, hplp


def std_from_general(g):
    """Standard form through the PRODUCT's to_standard_form (checked bitwise
    against the reference's own in tests/test_host.py)."""
    s = hplp.to_standard_form(g)
    return s


def problem(name: str):
    """Named parity problems (sizes the CPU oracle finishes in seconds)."""
    P = gen.scaled
    table = {
        "cfg0": lambda: gen.generate(0),
        "cfg1_small": lambda: gen.generate(P(1, m=3000, n=6000)),
        "cfg2_small": lambda: gen.generate(P(2, m=2000, n=4000, infeasible_rows=20, row_scale_log10=0.0)),
        "transport_small": lambda: gen.generate(P(3, sources=40, sinks=50)),
        "zipf_small": lambda: gen.generate(P(4, m=4000, n=8000, zipf_cap=3000, zipf_target_nnz=60000,
                                             zipf_force_cap=3)),
    }
    return table[name]()


def csr_args(s):
    return (s.m, s.n, s.row_ptr, s.col_idx, s.val, s.b, s.c)


def rel_inf(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)) if a.size else 0.0


def random_std_lp(seed, m, n, density=0.2, feasible=True):
    """Small random standard-form LP with a known feasible point."""
    rng = np.random.default_rng(seed)
    mask = rng.random((m, n)) < density
    for i in range(m):
        if not mask[i].any():
            mask[i, rng.integers(n)] = True
    A = np.where(mask, rng.normal(size=(m, n)), 0.0)
    x0 = rng.random(n)
    b = A @ x0
    c = rng.random(n) + 0.1
    rp = np.zeros(m + 1, np.int64)
    cols, vals = [], []
    for i in range(m):
        nz = np.nonzero(A[i])[0]
        cols.extend(nz.tolist())
        vals.extend(A[i, nz].tolist())
        rp[i + 1] = rp[i] + len(nz)
    return m, n, rp, np.array(cols, np.int32), np.array(vals), b, c
