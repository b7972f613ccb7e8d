"""Box form on the GPU (a flagged mode with no
reference counterpart): hplp_solver_create_box against the port's box form
(CpuLp.set_box) -- per-iteration iterates to 1e-10 over the first 100
iterations, statuses and objectives at tolerance 1e-4 -- plus the mapping
back to the standard form and the standard form's own optimum."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import CpuLp
from paper_2407_16144_b200 import hplp
from tests.helpers import csr_args
from tests.test_box import box_lp
from tests.test_gpu_parity import _trace_cmp, std

pytestmark = pytest.mark.gpu


def box_solve(s, **kw):
    sol = hplp.Solver.box(*csr_args(s))
    try:
        return sol.solve(**kw)
    finally:
        sol.close()


@pytest.mark.parametrize("name", ["cfg0", "cfg1_small", "zipf_small", "transport_small"])
def test_box_iterate_parity_first_100(gpu_required, name):
    g, s = std(name)
    args, up = box_lp(s)
    cpu = CpuLp("port", *args).set_box(up).solve(iteration_limit=100, tolerance=1e-12, trace=True,
                                                 infeasibility_check_period=0)
    gpu = box_solve(s, iteration_limit=100, tolerance=1e-12, trace=True)
    assert len(cpu["trace"]) == 100
    assert len(gpu["trace"][0]["x"]) == args[1] and len(gpu["trace"][0]["y"]) == args[0]
    _trace_cmp(gpu["trace"], cpu["trace"])
    assert [e[:2] for e in gpu["epochs"]] == [e[:2] for e in cpu["epochs"]]
    for k in range(4):
        assert abs(gpu["kkt"][k] - cpu["kkt"][k]) <= 1e-9 * max(abs(cpu["kkt"][k]), 1e-300) + 1e-300


@pytest.mark.parametrize("name", ["cfg0"])
def test_box_solve_tol_1e4(gpu_required, name):
    g, s = std(name)
    args, up = box_lp(s)
    cpu = CpuLp("port", *args).set_box(up).solve(tolerance=1e-4, iteration_limit=300000,
                                                 infeasibility_check_period=0)
    gpu = box_solve(s, tolerance=1e-4, iteration_limit=300000)
    assert gpu["status"] == cpu["status"] == "optimal"
    assert gpu["kkt"][3] <= 1e-4
    ob_g = float(s.c @ gpu["x"])  # standard-form objective of the mapped solution
    ob_c = float(args[6] @ cpu["x"])
    assert abs(ob_g - ob_c) <= 1e-4 * max(1.0, abs(ob_c))
    # the same LP solved in the standard form (the reference's algorithm)
    ref = hplp.solve(*csr_args(s), tolerance=1e-4, iteration_limit=300000)
    assert abs(ob_g - float(s.c @ ref["x"])) <= 1e-3 * max(1.0, abs(ob_c))


@pytest.mark.parametrize("name", ["cfg1_small", "zipf_small"])
def test_box_matches_standard_form_optimum(gpu_required, name):
    """Both forms to 1e-4 (Pock-Chambolle alpha 0.5): the box form's KKT is
    the standard form's at the mapped iterate, so both solutions are 1e-4
    solutions of the same LP and their objectives agree to the gap."""
    g, s = std(name)
    kw = dict(tolerance=1e-4, iteration_limit=2_000_000, precondition_pc_alpha=0.5)
    box = box_solve(s, **kw)
    ref = hplp.solve(*csr_args(s), **kw)
    assert box["status"] == ref["status"] == "optimal"
    ob, orf = float(s.c @ box["x"]), float(s.c @ ref["x"])
    assert abs(ob - orf) <= 5e-4 * (1.0 + abs(orf)), (ob, orf)


def test_box_result_in_standard_form(gpu_required):
    g, s = std("cfg0")
    args, up = box_lp(s)
    mb, nb = args[0], args[1]
    r = box_solve(s, tolerance=1e-6, iteration_limit=300000)
    x, y = r["x"], r["y"]
    assert x.shape == (s.n,) and y.shape == (s.m,)
    # bound rows x_j + s_j = u_j hold exactly up to one rounding; slacks >= 0
    lp = CpuLp("port", *csr_args(s))
    ax = lp.spmv(x)
    assert np.max(np.abs(ax[mb:] - s.b[mb:])) <= 1e-12 * max(1.0, float(np.max(np.abs(s.b[mb:]))))
    assert np.all(x >= 0)
    assert np.all(y[mb:] >= 0)
    # the mapped pair is a near-optimal standard-form pair: its KKT error (the
    # reference's measure) is of the order of the box form's
    k = lp.kkt_error(x, y)
    assert k[3] <= 50 * max(r["kkt"][3], 1e-8), (k, r["kkt"])


def test_box_preconditioned(gpu_required):
    """Ruiz + Pock-Chambolle on the box form: u is rescaled with the columns
    (x = C x'), the mapped solution respects the bounds and matches the
    standard form's optimum."""
    g, s = std("zipf_small")
    args, up = box_lp(s)
    kw = dict(tolerance=1e-4, iteration_limit=400000, precondition_ruiz_iters=10, precondition_pc_alpha=1.0)
    gpu = box_solve(s, **kw)
    ref = hplp.solve(*csr_args(s), **kw)
    assert gpu["status"] == ref["status"] == "optimal"
    ob, orf = float(s.c @ gpu["x"]), float(s.c @ ref["x"])
    assert abs(ob - orf) <= 5e-4 * (1.0 + abs(orf)), (ob, orf)
    assert np.all(gpu["x"] >= 0) and np.all(gpu["x"][: args[1]] <= up * (1 + 1e-12) + 1e-12)


def test_box_rejects_baselines(gpu_required):
    g, s = std("cfg0")
    with pytest.raises(ValueError, match="box form"):
        box_solve(s, iteration_limit=10, scheme=1)
