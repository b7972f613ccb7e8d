"""cmd_solve path on the B200 (SPEC.md [MODULE] cli / mps_io): MPS text ->
to_standard_form -> device solve -> solution JSON + trace CSV, checked
against the CPU oracle on the same instance."""
from __future__ import annotations

import json

import numpy as np
import pytest

from oracle import CpuLp
from paper_2407_16144_b200 import gen, hplp

pytestmark = pytest.mark.gpu

E1 = "NAME E1\nROWS\n N obj\n E r\nCOLUMNS\n    x obj 0 r 1\nRHS\n    RHS r 1\nENDATA\n"
INFEAS = ("NAME INF\nROWS\n N obj\n E r1\n E r2\nCOLUMNS\n    x obj 0 r1 1\n    x r2 1\n"
          "RHS\n    RHS r1 1 r2 2\nENDATA\n")


def test_e1_optimal_report(gpu_required):
    # SPEC.md cli example: E1 with defaults -> "optimal"
    text, csv, status = hplp.solve_mps(E1, tolerance=1e-8)
    d = json.loads(text)
    assert status == d["status"] == "optimal"
    assert abs(d["primal_objective"]) <= 1e-6 and abs(d["primal_solution"][0] - 1.0) <= 1e-6
    assert d["primal_certificate"] is None and d["dual_certificate"] is None
    assert d["kkt"]["max"] <= 1e-8 and "timing" in d
    assert csv.count("\n") == 1  # header only: no trace requested
    # the same numbers as the oracle's solve of the same standard form
    s = hplp.to_standard_form(hplp.parse_mps(E1).general())
    c = CpuLp("port", *s.csr()).solve(tolerance=1e-8)
    assert d["iterations"] == c["iterations"]


def test_infeasible_report_carries_certificate(gpu_required):
    # SPEC.md: infeasible fixture -> certificate in the JSON, no solution
    text, _, status = hplp.solve_mps(INFEAS)
    d = json.loads(text)
    assert status == d["status"] == "primal_infeasible"
    assert d["primal_solution"] is None and d["primal_certificate"] is not None
    v = np.array(d["primal_certificate"]["vector"])
    assert abs(np.linalg.norm(v) - 1.0) <= 1e-12 and v[1] > 0 > v[0]


def test_generated_lp_through_mps_matches_direct_solve(gpu_required):
    g = gen.generate(0)
    text, csv, status = hplp.solve_mps(hplp.mps_from_general(g), tolerance=1e-4, trace_period=500)
    d = json.loads(text)
    direct, x_orig, obj = hplp.solve_general(g, tolerance=1e-4)
    assert status == direct["status"] == "optimal"
    assert d["iterations"] == direct["iterations"]
    assert d["primal_objective"] == obj  # same solve, same recovery
    assert np.array_equal(np.array(d["primal_solution"]), x_orig)
    rows = csv.strip().split("\n")
    assert rows[0].startswith("iteration,epoch,inner,fixed_point_residual")
    assert len(rows) - 1 == d["iterations"] // 500 + 1
    # determinism (SPEC.md cli): identical reports except the timing block
    text2, _, _ = hplp.solve_mps(hplp.mps_from_general(g), tolerance=1e-4, trace_period=500)
    a, b = json.loads(text), json.loads(text2)
    a.pop("timing"), b.pop("timing")
    assert a == b
    # elision of long vectors
    d3 = json.loads(hplp.solve_mps(hplp.mps_from_general(g), tolerance=1e-4, elide_above=10)[0])
    assert d3["primal_solution"] == {"elided": True, "length": g.n}
