"""Input validation of hplp_solver_create / hplp_solve_csr on the GPU.

A valid CSR with ascending rows goes straight to the device, which checks
ranges, finiteness, order and duplicates itself (hx_upload_csr); anything it
rejects takes the host SparseMatrix path (src/sparse_matrix.cpp semantics:
unsorted rows are sorted, bad input is reported with the reference's
messages).  Both routes must give the reference's behaviour.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2407_16144_b200 import hplp
from tests.helpers import csr_args
from tests.test_gpu_parity import std

pytestmark = pytest.mark.gpu


def _small():
    g, s = std("cfg0")
    m, n, rp, ci, v, b, c = csr_args(s)
    return m, n, rp.copy(), ci.copy(), v.copy(), b.copy(), c.copy()


def test_unsorted_rows_are_sorted(gpu_required):
    m, n, rp, ci, v, b, c = _small()
    ref = hplp.solve(m, n, rp, ci, v, b, c, iteration_limit=200, tolerance=1e-12)
    rng = np.random.default_rng(3)
    ci2, v2 = ci.copy(), v.copy()
    for i in range(m):
        p = rng.permutation(rp[i + 1] - rp[i]) + rp[i]
        ci2[rp[i]:rp[i + 1]], v2[rp[i]:rp[i + 1]] = ci[p], v[p]
    assert not all(np.all(np.diff(ci2[rp[i]:rp[i + 1]]) > 0) for i in range(m))
    got = hplp.solve(m, n, rp, ci2, v2, b, c, iteration_limit=200, tolerance=1e-12)
    assert np.array_equal(got["x"], ref["x"]) and np.array_equal(got["y"], ref["y"])


@pytest.mark.parametrize("case,match", [
    ("duplicate", "duplicate"),
    ("col_range", "out of range"),
    ("nan_value", "non-finite value"),
    ("inf_b", "non-finite b or c"),
    ("nan_c", "non-finite b or c"),
    ("row_ptr", "monotone"),
])
def test_bad_input_rejected(gpu_required, case, match):
    m, n, rp, ci, v, b, c = _small()
    i = int(np.argmax(np.diff(rp) >= 2))  # a row with two entries
    if case == "duplicate":
        ci[rp[i] + 1] = ci[rp[i]]
    elif case == "col_range":
        ci[rp[i]] = n
    elif case == "nan_value":
        v[rp[i]] = np.nan
    elif case == "inf_b":
        b[0] = np.inf
    elif case == "nan_c":
        c[-1] = np.nan
    elif case == "row_ptr":
        rp[i + 1] = rp[i + 2] + 1
    with pytest.raises(ValueError, match=match):
        hplp.Solver(m, n, rp, ci, v, b, c)
    with pytest.raises(ValueError, match=match):
        hplp.solve(m, n, rp, ci, v, b, c, iteration_limit=10)


def test_power_start_reused_across_solves(gpu_required):
    """The start vector drawn for one seed is reused by the next solve with
    that seed and redrawn for another: sigma and iterates follow the seed."""
    m, n, rp, ci, v, b, c = _small()
    s = hplp.Solver(m, n, rp, ci, v, b, c)
    try:
        a1 = s.solve(iteration_limit=50, tolerance=1e-12, seed=7)
        a2 = s.solve(iteration_limit=50, tolerance=1e-12, seed=7)
        b1 = s.solve(iteration_limit=50, tolerance=1e-12, seed=8)
        a3 = s.solve(iteration_limit=50, tolerance=1e-12, seed=7)
    finally:
        s.close()
    one = hplp.solve(m, n, rp, ci, v, b, c, iteration_limit=50, tolerance=1e-12, seed=8)
    assert a1["sigma_estimate"] == a2["sigma_estimate"] == a3["sigma_estimate"]
    assert np.array_equal(a1["x"], a3["x"])
    assert b1["sigma_estimate"] == one["sigma_estimate"] and np.array_equal(b1["x"], one["x"])
