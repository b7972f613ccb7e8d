"""Box form (no reference counterpart), host side and
its CPU restatement.

The box form drops the trailing bound rows x_j + s_j = u_j of the standard
form and enforces x_j <= u_j by the primal projection.  It is a different
iteration from the reference's, so its oracle (the port with
CpuLp.set_box) is pinned by the LP itself: the box form's optimum must match
the standard form's optimum of the same instance.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import CpuLp
from paper_2407_16144_b200 import hplp
from tests.helpers import csr_args, problem, random_std_lp


def box_lp(s):
    mb, nb, up = hplp.box_form(*csr_args(s))
    e = s.row_ptr[mb]
    return (mb, nb, s.row_ptr[: mb + 1], s.col_idx[:e], s.val[:e], s.b[:mb], s.c[:nb]), up


def test_detect_cfg0():
    g = problem("cfg0")
    s = hplp.to_standard_form(g)
    mb, nb, up = hplp.box_form(*csr_args(s))
    # 1000 original rows (300 >= rows get a slack column), every column bounded
    assert (s.m, s.n) == (3000, 4300)
    assert (mb, nb) == (1000, 2300)
    assert np.array_equal(up[:2000], g.col_upper - g.col_lower)
    assert np.all(np.isinf(up[2000:]))


def test_detect_nothing_to_remove():
    m, n, rp, ci, v, b, c = random_std_lp(3, 12, 20)
    mb, nb, up = hplp.box_form(m, n, rp, ci, v, b, c)
    assert (mb, nb) == (m, n) and np.all(np.isinf(up))


def test_detect_stops_at_a_non_bound_row():
    # a trailing row that looks like a bound row but whose slack also appears
    # elsewhere is not removed
    g = problem("cfg0")
    s = hplp.to_standard_form(g)
    ci = s.col_idx.copy()
    ci[s.row_ptr[0]] = s.n - 1 if s.n - 1 not in ci[: s.row_ptr[1]] else ci[s.row_ptr[0]]
    order = np.argsort(ci[: s.row_ptr[1]], kind="stable")
    ci[: s.row_ptr[1]] = ci[: s.row_ptr[1]][order]
    v = s.val.copy()
    v[: s.row_ptr[1]] = v[: s.row_ptr[1]][order]
    mb, nb, up = hplp.box_form(s.m, s.n, s.row_ptr, ci, v, s.b, s.c)
    assert (mb, nb) == (s.m, s.n)  # the last bound row's slack is now shared: nothing removed


def test_oracle_box_step_projects():
    s = hplp.to_standard_form(problem("cfg0"))
    args, up = box_lp(s)
    lp = CpuLp("port", *args).set_box(up)
    rng = np.random.default_rng(0)
    x = rng.random(args[1]) * 20
    y = rng.normal(size=args[0])
    xn, yn, axn, aty = lp.pdhg_step(0.01, x, y, lp.spmv(x))
    assert np.all(xn >= 0) and np.all(xn <= up)
    free = np.clip(x - 0.01 * (aty + args[6]), 0, None)
    assert np.array_equal(xn, np.minimum(free, up))


def test_oracle_box_optimum_matches_standard_form():
    s = hplp.to_standard_form(problem("cfg0"))
    args, up = box_lp(s)
    box = CpuLp("port", *args).set_box(up).solve(tolerance=1e-5, iteration_limit=400000,
                                                 infeasibility_check_period=0)
    std = CpuLp("port", *csr_args(s)).solve(tolerance=1e-5, iteration_limit=400000)
    assert box["status"] == std["status"] == "optimal"
    ob, os_ = float(args[6] @ box["x"]), float(s.c @ std["x"])
    assert abs(ob - os_) <= 1e-4 * max(1.0, abs(os_)), (ob, os_)


def test_oracle_box_rejects_scan():
    s = hplp.to_standard_form(problem("cfg0"))
    args, up = box_lp(s)
    with pytest.raises(ValueError, match="infeasibility"):
        CpuLp("port", *args).set_box(up).solve(iteration_limit=10)
