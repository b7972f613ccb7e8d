"""Baseline schemes on the B200 (solve_baseline, src/solver.cpp:344-509;
SURVEY.md §8f rank 1): vanilla PDHG, its running average (KKT and
termination on the average), and the average restarted.  Same bars as the
rHPDHG path: per-record iterates (the candidate) to 1e-10 against the CPU
oracle, identical restart sequence, SpMV count and status."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import CpuLp
from paper_2407_16144_b200 import abi, hplp
from tests.helpers import csr_args, rel_inf
from tests.test_gpu_parity import std

pytestmark = pytest.mark.gpu

SCHEMES = [(abi.SCHEME_VANILLA, 0), (abi.SCHEME_AVERAGED, 1), (abi.SCHEME_RESTARTED_AVERAGE, 2)]


def _cmp_traces(tg_list, tc_list):
    assert len(tg_list) == len(tc_list)
    for tg, tc in zip(tg_list, tc_list):
        assert (tg["iteration"], tg["epoch"], tg["inner"]) == (tc["iteration"], tc["epoch"], tc["inner"])
        e = rel_inf(np.concatenate([tg["x"], tg["y"]]), np.concatenate([tc["x"], tc["y"]]))
        assert e <= 1e-10, (tc["iteration"], e)
        for key in ("res", "cand_norm_difference"):
            a, b = tg[key], tc[key]
            assert (math.isnan(a) and math.isnan(b)) or abs(a - b) <= 1e-8 * max(abs(b), 1e-300), (key, a, b)
        assert np.allclose(tg["kkt"], tc["kkt"], rtol=1e-9, atol=1e-300)
        assert sum(len(p) for p in tg["partition"]) == len(tg["x"])


@pytest.mark.parametrize("scheme,mode", SCHEMES)
@pytest.mark.parametrize("name", ["cfg0", "cfg1_small"])
def test_baseline_trace_parity(gpu_required, scheme, mode, name):
    g, s = std(name)
    kw = dict(iteration_limit=300, tolerance=1e-12, trace_period=7)
    cpu = CpuLp("port", *csr_args(s)).solve_baseline(mode, trace=True, **kw)
    gpu = hplp.solve(*csr_args(s), scheme=scheme, trace=True, **kw)
    _cmp_traces(gpu["trace"], cpu["trace"])
    assert gpu["status"] == cpu["status"] == "iteration_limit"
    assert gpu["iterations"] == cpu["iterations"]
    assert gpu["spmv_count"] == cpu["spmv_count"]
    assert [e[:2] for e in gpu["epochs"]] == [e[:2] for e in cpu["epochs"]]
    assert rel_inf(np.concatenate([gpu["x"], gpu["y"]]), np.concatenate([cpu["x"], cpu["y"]])) <= 1e-10


@pytest.mark.parametrize("scheme,mode", SCHEMES)
def test_baseline_solve_parity(gpu_required, scheme, mode):
    """To tolerance (or the limit): same status, iteration count and answer."""
    g, s = std("cfg0")
    kw = dict(iteration_limit=30000, tolerance=1e-4)
    cpu = CpuLp("port", *csr_args(s)).solve_baseline(mode, **kw)
    gpu = hplp.solve(*csr_args(s), scheme=scheme, **kw)
    assert gpu["status"] == cpu["status"]
    assert gpu["iterations"] == cpu["iterations"]
    assert gpu["spmv_count"] == cpu["spmv_count"]
    assert rel_inf(np.concatenate([gpu["x"], gpu["y"]]), np.concatenate([cpu["x"], cpu["y"]])) <= 1e-8


@pytest.mark.parametrize("scheme,mode", SCHEMES)
def test_baseline_infeasibility(gpu_required, scheme, mode):
    # A = [[1],[1]], b = (1, 2): primal infeasible; baselines scan
    # the iterate-difference candidate only
    m, n = 2, 1
    rp, ci, v = np.array([0, 1, 2], np.int64), np.array([0, 0], np.int32), np.array([1.0, 1.0])
    b, c = np.array([1.0, 2.0]), np.array([0.0])
    cpu = CpuLp("port", m, n, rp, ci, v, b, c).solve_baseline(mode, iteration_limit=20000)
    gpu = hplp.solve(m, n, rp, ci, v, b, c, scheme=scheme, iteration_limit=20000)
    assert gpu["status"] == cpu["status"]
    assert gpu["iterations"] == cpu["iterations"]
    if cpu["primal_cert"] is not None:
        assert np.allclose(gpu["primal_cert"][0], cpu["primal_cert"][0], atol=1e-12)
        assert gpu["primal_cert"][1]["source"] == abi.SOURCE_ITERATE_DIFFERENCE


def test_baseline_fixed_restart_frequency(gpu_required):
    g, s = std("cfg0")
    kw = dict(iteration_limit=500, tolerance=1e-12, restart_kind=abi.RESTART_FIXED, k_star=40)
    cpu = CpuLp("port", *csr_args(s)).solve_baseline(2, **kw)
    gpu = hplp.solve(*csr_args(s), scheme=abi.SCHEME_RESTARTED_AVERAGE, **kw)
    assert [e[:2] for e in gpu["epochs"]] == [e[:2] for e in cpu["epochs"]]
    assert rel_inf(np.concatenate([gpu["x"], gpu["y"]]), np.concatenate([cpu["x"], cpu["y"]])) <= 1e-10
