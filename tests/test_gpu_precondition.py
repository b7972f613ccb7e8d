"""Preconditioning (extension; no reference counterpart) on
the B200: the device transform against a numpy restatement, the loop on the
scaled instance against the oracle given the same instance, and solves whose
results are mapped back to -- and validated on -- the original problem."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import CpuLp
from paper_2407_16144_b200 import hplp
from tests.helpers import csr_args, problem, rel_inf

pytestmark = pytest.mark.gpu


def numpy_ruiz_pc(m, n, rp, ci, v, b, c, ruiz, alpha):
    """Restatement of hx_precondition: same formulas, same rounding order
    ((a * r_i) * c_j); row sums for the PC step compared with a tolerance."""
    rows = np.repeat(np.arange(m), np.diff(rp))
    v = v.copy()
    R, Cs = np.ones(m), np.ones(n)
    b, c = b.copy(), c.copy()

    def apply(dr, dc):
        nonlocal v, b, c
        dr = np.where(dr > 0, 1.0 / np.sqrt(np.where(dr > 0, dr, 1.0)), 1.0)
        dc = np.where(dc > 0, 1.0 / np.sqrt(np.where(dc > 0, dc, 1.0)), 1.0)
        R[:] = R * dr
        Cs[:] = Cs * dc
        v = (v * dr[rows]) * dc[ci]
        b = b * dr
        c = c * dc

    for _ in range(ruiz):
        dr = np.zeros(m)
        np.maximum.at(dr, rows, np.abs(v))
        dc = np.zeros(n)
        np.maximum.at(dc, ci, np.abs(v))
        apply(dr, dc)
    if alpha >= 0:
        dr = np.zeros(m)
        np.add.at(dr, rows, np.abs(v) ** (2 - alpha))
        dc = np.zeros(n)
        np.add.at(dc, ci, np.abs(v) ** alpha)
        apply(dr, dc)
    return v, b, c, R, Cs


@pytest.fixture(scope="module")
def scaled(gpu_required):
    g = problem("cfg1_small")
    s = hplp.to_standard_form(g)
    hx = hplp.HX(device=0)
    hx.upload(*csr_args(s))
    R, Cs = hx.precondition(10, 1.0)
    return g, s, hx, R, Cs, hx.download_problem()


def test_transform_matches_restatement(scaled):
    g, s, hx, R, Cs, (rp, ci, v, b, c) = scaled
    ev, eb, ec, eR, eC = numpy_ruiz_pc(s.m, s.n, s.row_ptr, s.col_idx, s.val, s.b, s.c, 10, 1.0)
    assert np.array_equal(rp, s.row_ptr) and np.array_equal(ci, s.col_idx)
    for got, want in ((v, ev), (b, eb), (c, ec), (R, eR), (Cs, eC)):
        assert rel_inf(got, want) <= 1e-13
    # the scaled rows/columns are close to unit norm (equilibrated)
    rows = np.repeat(np.arange(s.m), np.diff(rp))
    rmax = np.zeros(s.m)
    np.maximum.at(rmax, rows, np.abs(v))
    assert 0.05 < np.median(rmax) < 2.0


def test_loop_parity_on_scaled_instance(scaled):
    g, s, hx, R, Cs, (rp, ci, v, b, c) = scaled
    args = (s.m, s.n, rp, ci, v, b, c)
    cpu = CpuLp("port", *args).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    gpu = hplp.solve(*args, iteration_limit=100, tolerance=1e-12, trace=True)
    for tg, tc in zip(gpu["trace"], cpu["trace"]):
        assert (tg["epoch"], tg["inner"]) == (tc["epoch"], tc["inner"])
        assert rel_inf(np.concatenate([tg["x"], tg["y"]]), np.concatenate([tc["x"], tc["y"]])) <= 1e-10


def test_preconditioned_solve_maps_back(gpu_required):
    g = problem("cfg0")
    s = hplp.to_standard_form(g)
    plain = hplp.solve(*csr_args(s), tolerance=1e-4, iteration_limit=100000)
    pre = hplp.solve(*csr_args(s), tolerance=1e-4, iteration_limit=100000, precondition_ruiz_iters=10,
                     precondition_pc_alpha=1.0)
    assert plain["status"] == pre["status"] == "optimal"
    assert pre["iterations"] < plain["iterations"]  # 4.5k vs 11.3k on configs[0]
    _, obj = s.recover(pre["x"])
    assert abs(obj - g.planted_objective) <= 1e-3 * max(1.0, abs(g.planted_objective))
    # the mapped-back iterate is (approximately) feasible for the ORIGINAL problem
    k = CpuLp("port", *csr_args(s)).kkt_error(pre["x"], pre["y"])
    assert k[0] <= 1e-3 and (pre["x"] >= 0).all()


def test_preconditioning_improves_feasibility_on_row_scaled_instance(gpu_required):
    g = problem("cfg1_small")  # row scales 1e-2..1e2
    s = hplp.to_standard_form(g)
    plain = hplp.solve(*csr_args(s), tolerance=1e-8, iteration_limit=20000)
    pre = hplp.solve(*csr_args(s), tolerance=1e-8, iteration_limit=20000, precondition_ruiz_iters=10,
                     precondition_pc_alpha=1.0)
    assert pre["kkt"][0] < 0.1 * plain["kkt"][0] and pre["kkt"][1] < 0.1 * plain["kkt"][1]
    _, o_pre = s.recover(pre["x"])
    _, o_plain = s.recover(plain["x"])
    assert abs(o_pre - g.planted_objective) < abs(o_plain - g.planted_objective)


def test_preconditioned_infeasibility_certificate_is_valid_on_original(gpu_required):
    # scaled-row infeasible instance (row scales 1e-1..1e1): the loop detects it after scaling
    from paper_2407_16144_b200 import gen

    g = gen.generate(gen.scaled(2, m=1000, n=2000, infeasible_rows=10, row_scale_log10=1.0))
    s = hplp.to_standard_form(g)
    r = hplp.solve(*csr_args(s), tolerance=1e-4, iteration_limit=100000, precondition_ruiz_iters=10,
                   precondition_pc_alpha=1.0)
    assert r["status"] == "primal_infeasible"
    vec, meta = r["primal_cert"]
    assert abs(np.linalg.norm(vec) - 1.0) <= 1e-12
    lp = CpuLp("port", *csr_args(s))
    sigma, _, _, _ = lp.power_iteration()
    rep = lp.validate_primal(vec, 1e-6, sigma * (1 + 1e-4))
    assert rep["valid"], rep


# configs[2] at full size: tests/test_gpu_full_parity.py (validated by the reference itself)
