"""B200 parity tests: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  (a) per-iteration iterates, first 100 iterations: ||z_gpu - z_cpu||_inf /
      ||z_cpu||_inf <= 1e-10, identical (epoch, inner) restart sequence;
  (b) solve at tol 1e-4: identical status, objective within 1e-4 relative.
Kernel-level SpMVs: normwise relative error <= 1e-13 (different, fixed
summation order than the reference's sequential sums).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import CpuLp
from paper_2407_16144_b200 import abi, hplp
from tests.helpers import csr_args, problem, random_std_lp, rel_inf

pytestmark = pytest.mark.gpu

PROBLEMS = ["cfg0", "cfg1_small", "cfg2_small", "transport_small", "zipf_small"]
_cache = {}


def std(name):
    if name not in _cache:
        g = problem(name)
        _cache[name] = (g, hplp.to_standard_form(g))
    return _cache[name]


@pytest.fixture(scope="module")
def hx(gpu_required):
    return hplp.HX(device=0)


@pytest.mark.parametrize("name", PROBLEMS)
def test_spmv_parity(hx, name):
    g, s = std(name)
    hx.upload(*csr_args(s))
    cpu = CpuLp("port", *csr_args(s))
    rng = np.random.default_rng(7)
    for _ in range(3):
        x = rng.normal(size=s.n)
        y = rng.normal(size=s.m)
        assert rel_inf(hx.spmv(x), cpu.spmv(x)) <= 1e-13
        assert rel_inf(hx.spmv_transpose(y), cpu.spmv_transpose(y)) <= 1e-13


def test_spmv_adjointness(hx):
    # y'(Ax) == (A'y)'x to 1e-12 relative
    g, s = std("zipf_small")
    hx.upload(*csr_args(s))
    rng = np.random.default_rng(3)
    x, y = rng.normal(size=s.n), rng.normal(size=s.m)
    lhs, rhs = y @ hx.spmv(x), hx.spmv_transpose(y) @ x
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


@pytest.mark.parametrize("name", ["cfg0", "cfg1_small", "transport_small"])
def test_power_iteration_parity(gpu_required, name):
    g, s = std(name)
    cpu = CpuLp("port", *csr_args(s))
    sigma_c, it_c, conv_c, _ = cpu.power_iteration()
    r = hplp.solve(*csr_args(s), iteration_limit=0)
    assert abs(r["sigma_estimate"] / (1 + 1e-4) - sigma_c) <= 1e-10 * sigma_c
    assert r["spmv_count"] == 2 * it_c + 1 + 2


def _trace_cmp(gpu_trace, cpu_trace, tol=1e-10):
    assert len(gpu_trace) == len(cpu_trace)
    worst = 0.0
    for tg, tc in zip(gpu_trace, cpu_trace):
        assert (tg["iteration"], tg["epoch"], tg["inner"]) == (tc["iteration"], tc["epoch"], tc["inner"])
        zc = np.concatenate([tc["x"], tc["y"]])
        zg = np.concatenate([tg["x"], tg["y"]])
        e = rel_inf(zg, zc)
        worst = max(worst, e)
        assert e <= tol, (tg["iteration"], e)
        assert abs(tg["res"] - tc["res"]) <= 1e-8 * max(tc["res"], 1e-300) + 1e-300
    return worst


@pytest.mark.parametrize("kind", ["port", "reference"])
@pytest.mark.parametrize("name", ["cfg0", "cfg1_small", "cfg2_small", "zipf_small"])
def test_iterate_parity_first_100(gpu_required, name, kind):
    """kind "reference": the unmodified reference (oracle/_ref) itself."""
    g, s = std(name)
    cpu = CpuLp(kind, *csr_args(s)).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    gpu = hplp.solve(*csr_args(s), iteration_limit=100, tolerance=1e-12, trace=True)
    assert len(cpu["trace"]) == 100
    _trace_cmp(gpu["trace"], cpu["trace"])
    assert gpu["status"] == cpu["status"] == "iteration_limit"
    assert gpu["iterations"] == cpu["iterations"] == 100
    assert gpu["spmv_count"] == cpu["spmv_count"]
    assert [e[:2] for e in gpu["epochs"]] == [e[:2] for e in cpu["epochs"]]


def _objective(s, x):
    return float(s.c @ x)


@pytest.mark.parametrize("kind", ["port", "reference"])
@pytest.mark.parametrize("name", ["cfg0", "transport_small"])
def test_solve_parity_tol_1e4(gpu_required, name, kind):
    g, s = std(name)
    cpu = CpuLp(kind, *csr_args(s)).solve(tolerance=1e-4, iteration_limit=200000)
    gpu = hplp.solve(*csr_args(s), tolerance=1e-4, iteration_limit=200000)
    assert gpu["status"] == cpu["status"] == "optimal"
    oc, og = _objective(s, cpu["x"]), _objective(s, gpu["x"])
    assert abs(og - oc) <= 1e-4 * max(1.0, abs(oc))
    assert gpu["kkt"][3] <= 1e-4
    if not math.isnan(g.planted_objective):
        _, obj = s.recover(gpu["x"])
        assert abs(obj - g.planted_objective) <= 1e-3 * max(1.0, abs(g.planted_objective))


@pytest.mark.parametrize("kind", ["port", "reference"])
def test_infeasible_certificate(gpu_required, kind):
    g, s = std("cfg2_small")
    gpu = hplp.solve(*csr_args(s), tolerance=1e-4, iteration_limit=100000)
    cpu = CpuLp(kind, *csr_args(s)).solve(tolerance=1e-4, iteration_limit=100000)
    assert gpu["status"] == cpu["status"] == "primal_infeasible"
    assert gpu["iterations"] == cpu["iterations"]
    vec, meta = gpu["primal_cert"]
    rep = CpuLp(kind, *csr_args(s)).validate_primal(vec, 1e-6, gpu["sigma_estimate"])
    assert rep["valid"] and rep["orientation"] == abi.ORIENT_AS_IS
    assert abs(np.linalg.norm(vec) - 1.0) <= 1e-12
    assert meta["at_iteration"] == gpu["iterations"]


# ---- SPEC.md known-answer instances through the GPU path -------------------
def _csr(rows, m, n):
    rp = [0]
    ci, v = [], []
    for r in rows:
        for c, val in r:
            ci.append(c)
            v.append(val)
        rp.append(len(ci))
    return m, n, np.array(rp, np.int64), np.array(ci, np.int32), np.array(v)


def test_kat_e1_optimal(gpu_required):
    # E1: c=(0), A=[1], b=(1) -> x ~ 1, y ~ 0
    m, n, rp, ci, v = _csr([[(0, 1.0)]], 1, 1)
    r = hplp.solve(m, n, rp, ci, v, np.array([1.0]), np.array([0.0]), tolerance=1e-8)
    assert r["status"] == "optimal"
    assert abs(r["x"][0] - 1.0) <= 1e-6 and abs(r["y"][0]) <= 1e-6
    c = CpuLp("port", m, n, rp, ci, v, [1.0], [0.0]).solve(tolerance=1e-8)
    assert r["iterations"] == c["iterations"]


def test_kat_primal_infeasible(gpu_required):
    # A=[[1],[1]], b=(1,2), c=0 -> PrimalInfeasible (AC6)
    m, n, rp, ci, v = _csr([[(0, 1.0)], [(0, 1.0)]], 2, 1)
    r = hplp.solve(m, n, rp, ci, v, np.array([1.0, 2.0]), np.array([0.0]))
    assert r["status"] == "primal_infeasible" and r["iterations"] <= 10000
    c = CpuLp("port", m, n, rp, ci, v, [1.0, 2.0], [0.0]).solve()
    assert r["iterations"] == c["iterations"]
    assert np.allclose(r["primal_cert"][0], c["primal_cert"][0], rtol=0, atol=1e-12)


def test_kat_dual_infeasible(gpu_required):
    # c=(-1,0), A=[1,-1], b=0 -> DualInfeasible with ray ~ (1,1)/sqrt2
    m, n, rp, ci, v = _csr([[(0, 1.0), (1, -1.0)]], 1, 2)
    r = hplp.solve(m, n, rp, ci, v, np.array([0.0]), np.array([-1.0, 0.0]))
    assert r["status"] == "dual_infeasible"
    c = CpuLp("port", m, n, rp, ci, v, [0.0], [-1.0, 0.0]).solve()
    assert r["iterations"] == c["iterations"]
    assert np.allclose(r["dual_cert"][0], c["dual_cert"][0], atol=1e-9)


@pytest.mark.parametrize("seed", range(4))
def test_random_small_lps(gpu_required, seed):
    args = random_std_lp(seed, 6, 10)
    cpu = CpuLp("port", *args).solve(tolerance=1e-8, iteration_limit=20000)
    gpu = hplp.solve(*args, tolerance=1e-8, iteration_limit=20000)
    assert gpu["status"] == cpu["status"]
    assert gpu["iterations"] == cpu["iterations"]
    assert rel_inf(np.concatenate([gpu["x"], gpu["y"]]), np.concatenate([cpu["x"], cpu["y"]])) <= 1e-8


def test_determinism(gpu_required):
    g, s = std("cfg1_small")
    a = hplp.solve(*csr_args(s), iteration_limit=500, tolerance=1e-12)
    b = hplp.solve(*csr_args(s), iteration_limit=500, tolerance=1e-12)
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])
    assert a["kkt"] == b["kkt"] and a["epochs"] == b["epochs"]


def test_zero_iteration_limit(gpu_required):
    g, s = std("cfg0")
    cpu = CpuLp("port", *csr_args(s)).solve(iteration_limit=0)
    gpu = hplp.solve(*csr_args(s), iteration_limit=0)
    assert gpu["status"] == cpu["status"] == "iteration_limit"
    assert np.all(gpu["x"] == 0) and np.all(gpu["y"] == 0)
    assert np.allclose(gpu["kkt"], cpu["kkt"], rtol=1e-12)
    assert gpu["spmv_count"] == cpu["spmv_count"]


def test_empty_matrix(gpu_required):
    # nnz = 0: sigma = 0, eta = 1 (src/pdhg_core.cpp:32-33)
    m, n = 2, 3
    rp = np.zeros(m + 1, np.int64)
    b, c = np.array([0.0, 0.0]), np.array([1.0, 2.0, 0.5])
    cpu = CpuLp("port", m, n, rp, np.zeros(0, np.int32), np.zeros(0), b, c).solve()
    gpu = hplp.solve(m, n, rp, np.zeros(0, np.int32), np.zeros(0), b, c)
    assert gpu["status"] == cpu["status"]
    assert gpu["iterations"] == cpu["iterations"]
    assert gpu["eta"] == cpu["eta"] == 1.0


def test_fixed_and_none_restarts(gpu_required):
    g, s = std("cfg0")
    for kw in (dict(restart_kind=abi.RESTART_FIXED, k_star=50), dict(restart_kind=abi.RESTART_NONE)):
        cpu = CpuLp("port", *csr_args(s)).solve(iteration_limit=300, tolerance=1e-12, **kw)
        gpu = hplp.solve(*csr_args(s), iteration_limit=300, tolerance=1e-12, **kw)
        assert [e[:2] for e in gpu["epochs"]] == [e[:2] for e in cpu["epochs"]]
        assert rel_inf(np.concatenate([gpu["x"], gpu["y"]]), np.concatenate([cpu["x"], cpu["y"]])) <= 1e-9


def test_invalid_inputs_raise(gpu_required):
    m, n, rp, ci, v = _csr([[(0, 1.0), (0, 2.0)]], 1, 1)
    with pytest.raises(ValueError):
        hplp.solve(m, n, rp, ci, v, np.array([1.0]), np.array([0.0]))
    m, n, rp, ci, v = _csr([[(0, 1.0)]], 1, 1)
    with pytest.raises(ValueError):
        hplp.solve(m, n, rp, ci, v, np.array([1.0]), np.array([0.0]), tolerance=0.0)


def test_trace_diagnostics_parity(gpu_required):
    """TraceRecord's partition estimate and normalized-candidate norm
    (src/solver.cpp:279-287) from the device path equal the oracle's: sets
    identical (a reduced cost within rounding of the tol*sigma threshold may
    flip one index), norms to 1e-9 relative."""
    g, s = std("cfg1_small")
    kw = dict(iteration_limit=100, tolerance=1e-12, trace=True)
    cpu = CpuLp("port", *csr_args(s)).solve(**kw)
    gpu = hplp.solve(*csr_args(s), **kw)
    flips = 0
    for tg, tc in zip(gpu["trace"], cpu["trace"]):
        for u, v in zip(tg["partition"], tc["partition"]):
            flips += len(np.setxor1d(u, v))
        a, b = tg["cand_norm_normalized"], tc["cand_norm_normalized"]
        if tc["inner"] == 0:
            assert np.isnan(a) and np.isnan(b)
        else:
            assert abs(a - b) <= 1e-9 * max(abs(b), 1e-300), (tc["iteration"], a, b)
        assert sum(len(p) for p in tg["partition"]) == s.n
    assert flips <= 2


def _ragged_lp(seed=11, m=600, n=90000):
    """Empty rows and columns, 1-entry rows, a 70k-entry row and a dense-ish
    column: every task kind (stream rows, single pieces, multi-piece long rows
    folded by their owner CTA) in one matrix."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(m):
        if i % 97 == 0:
            rows.append([])  # empty row
        elif i == 5:
            rows.append(sorted(rng.choice(n, 70000, replace=False).tolist()))  # very long row
        elif i % 7 == 0:
            rows.append([int(rng.integers(n))])  # single entry
        else:
            cols = set(rng.choice(n, int(rng.integers(2, 60)), replace=False).tolist())
            cols.add(17)  # a column present in most rows
            rows.append(sorted(cols))
    rp = [0]
    ci, v = [], []
    for r in rows:
        ci += r
        v += rng.normal(size=len(r)).tolist()
        rp.append(len(ci))
    x0 = rng.random(n)
    A_x0 = np.array([sum(v[p] * x0[ci[p]] for p in range(rp[i], rp[i + 1])) for i in range(m)])
    c = rng.random(n) + 0.1
    return m, n, np.array(rp, np.int64), np.array(ci, np.int32), np.array(v), A_x0, c


def test_ragged_structure_parity(gpu_required):
    args = _ragged_lp()
    cpu = CpuLp("port", *args).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    gpu = hplp.solve(*args, iteration_limit=100, tolerance=1e-12, trace=True)
    _trace_cmp(gpu["trace"], cpu["trace"])
    assert gpu["spmv_count"] == cpu["spmv_count"]
    cpu_s = CpuLp("port", *args)
    rng = np.random.default_rng(5)
    x, y = rng.normal(size=args[1]), rng.normal(size=args[0])
    h = hplp.HX(device=0)
    h.upload(*args)
    assert rel_inf(h.spmv(x), cpu_s.spmv(x)) <= 1e-13
    assert rel_inf(h.spmv_transpose(y), cpu_s.spmv_transpose(y)) <= 1e-13
    h.close()


def test_ragged_structure_team_parity(gpu_required):
    args = _ragged_lp()
    cpu = CpuLp("port", *args).solve(iteration_limit=60, tolerance=1e-12, trace=True)
    t = hplp.Solver.team(*args, nranks=3)
    gpu = t.solve(iteration_limit=60, tolerance=1e-12, trace=True)
    t.close()
    _trace_cmp(gpu["trace"], cpu["trace"])


@pytest.mark.parametrize("name,blocks", [("cfg1_small", 2), ("zipf_small", 2), ("ragged", 2), ("cfg1_small", 3),
                                         ("zipf_small", 4), ("ragged", 8)])
def test_column_blocked_phase_b_parity(gpu_required, name, blocks, monkeypatch):
    """loop_kernel_stream_cb (phase B swept in K column blocks, the path
    configs[4] takes; forced here with HX_COLBLOCK=K on the stream kernel):
    first 100 iterates within 1e-10 of the oracle, same restarts and SpMV
    counts, then a solve to 1e-4 with the same status and objective."""
    monkeypatch.setenv("HX_COLBLOCK", str(blocks))
    monkeypatch.setenv("HPLP_L2_STREAM", "1")
    monkeypatch.setenv("HPLP_TRACE_RING", "0")  # traced iterations from the blocked kernel itself
    args = _ragged_lp() if name == "ragged" else csr_args(std(name)[1])
    cpu = CpuLp("port", *args).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    sol = hplp.Solver(*args)
    assert sol.hx.loop_kernel() == "hx::loop_kernel_stream_cb"
    gpu = sol.solve(iteration_limit=100, tolerance=1e-12, trace=True)
    _trace_cmp(gpu["trace"], cpu["trace"])
    assert gpu["spmv_count"] == cpu["spmv_count"]
    assert [e[:2] for e in gpu["epochs"]] == [e[:2] for e in cpu["epochs"]]
    if name != "ragged":  # to 1e-4 against the unblocked kernel
        g4 = sol.solve(iteration_limit=300000, tolerance=1e-4)
        monkeypatch.setenv("HX_COLBLOCK", "0")
        ref = hplp.Solver(*args)
        assert ref.hx.loop_kernel() == "hx::loop_kernel_stream"
        r4 = ref.solve(iteration_limit=300000, tolerance=1e-4)
        ref.close()
        assert g4["status"] == r4["status"]
        c = args[6]
        assert abs(float(c @ g4["x"]) - float(c @ r4["x"])) <= 1e-4 * max(1.0, abs(float(c @ r4["x"])))
    sol.close()


def test_column_blocked_preconditioned_parity(gpu_required, monkeypatch):
    """hx_precondition rescales every copy of A the loop reads -- the column
    blocks of loop_kernel_stream_cb included (they kept the
    unscaled values, so A x+ used the original matrix while A^T y used the
    scaled one).  The device loop on the preconditioned instance must match
    the oracle run on the instance downloaded from the device."""
    monkeypatch.setenv("HX_COLBLOCK", "4")
    monkeypatch.setenv("HPLP_L2_STREAM", "1")
    monkeypatch.setenv("HPLP_TRACE_RING", "0")  # traced iterations from the blocked kernel itself
    s = std("cfg1_small")[1]
    sol = hplp.Solver(*csr_args(s))
    assert sol.hx.loop_kernel() == "hx::loop_kernel_stream_cb"
    sol.hx.precondition(3, 0.5)
    rp, ci, v, b, c = sol.hx.download_problem()
    assert rel_inf(v, s.val) > 1e-3  # the instance really changed
    cpu = CpuLp("port", s.m, s.n, rp, ci, v, b, c).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    gpu = sol.solve(iteration_limit=100, tolerance=1e-12, trace=True)
    _trace_cmp(gpu["trace"], cpu["trace"])
    assert gpu["spmv_count"] == cpu["spmv_count"]
    sol.close()


@pytest.mark.parametrize("name", ["zipf_small", "cfg1_small", "transport_small"])
def test_reference_sum_order_spmv_bit_exact(gpu_required, name):
    """hx_set_sum_order(HX_SUM_REFERENCE): every row of A and A^T is one
    sequential chain in ascending index order, so both SpMVs are BIT-identical
    to the reference's loops (src/sparse_matrix.cpp:108-115, :127-134) --
    long Zipf rows (pieces carried by one warp) included."""
    g, s = std(name)
    hx = hplp.HX(device=0)
    hx.set_sum_order(hplp.SUM_REFERENCE)
    hx.upload(*csr_args(s))
    assert hx.sum_order() == hplp.SUM_REFERENCE
    ref = CpuLp("reference", *csr_args(s))
    rng = np.random.default_rng(11)
    for _ in range(3):
        x, y = rng.normal(size=s.n), rng.normal(size=s.m)
        assert np.array_equal(hx.spmv(x), ref.spmv(x))
        assert np.array_equal(hx.spmv_transpose(y), ref.spmv_transpose(y))
    with pytest.raises(hplp.HplpError):
        hx.set_sum_order(hplp.SUM_FAST)  # fixed once uploaded
    hx.close()


def test_reference_sum_order_iterates(gpu_required, monkeypatch):
    """The loop in the reference order (loop_kernel_exact) on a Zipf instance
    with rows of several thousand nonzeros: 100 iterates against the
    reference itself, identical restarts and SpMV counts."""
    monkeypatch.setenv("HPLP_TRACE_RING", "0")  # traced iterations from loop_kernel_exact itself
    g, s = std("zipf_small")
    with hplp.sum_order("reference"):
        sol = hplp.Solver(*csr_args(s))
    assert sol.hx.loop_kernel() == "hx::loop_kernel_exact"
    gpu = sol.solve(iteration_limit=100, tolerance=1e-12, trace=True)
    sol.close()
    cpu = CpuLp("reference", *csr_args(s)).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    worst = _trace_cmp(gpu["trace"], cpu["trace"], tol=1e-12)
    assert gpu["spmv_count"] == cpu["spmv_count"]
    print(f"zipf_small reference order: worst {worst:.2e}")


def test_trace_ring_runs_at_full_batch_rate(gpu_required):
    """Device trace ring: with trace_period = 1 the loop
    records every iteration on the device (iterate, partition classes,
    normalized-candidate norm) and does NOT end its launch per record -- the
    traced solve launches the loop kernel as often as the untraced one, and
    its records equal the oracle's (iterates to 1e-10, partition sets, norms
    to 1e-9)."""
    g, s = std("cfg1_small")
    kw = dict(iteration_limit=300, tolerance=1e-12)
    sol = hplp.Solver(*csr_args(s))
    l0 = sol.hx.launches()
    plain = sol.solve(**kw)
    l1 = sol.hx.launches()
    traced = sol.solve(trace=True, **kw)
    l2 = sol.hx.launches()
    sol.close()
    assert len(traced["trace"]) == 300
    assert l2 - l1 == l1 - l0, (l1 - l0, l2 - l1)  # no launch per traced iteration
    assert np.array_equal(plain["x"], traced["x"]) and np.array_equal(plain["y"], traced["y"])
    cpu = CpuLp("port", *csr_args(s)).solve(trace=True, **kw)
    _trace_cmp(traced["trace"], cpu["trace"])
    flips = 0
    for tg, tc in zip(traced["trace"], cpu["trace"]):
        for u, v in zip(tg["partition"], tc["partition"]):
            flips += len(np.setxor1d(u, v))
        a, b = tg["cand_norm_normalized"], tc["cand_norm_normalized"]
        if tc["inner"] == 0:
            assert np.isnan(a) and np.isnan(b)
        else:
            assert abs(a - b) <= 1e-9 * max(abs(b), 1e-300), (tc["iteration"], a, b)
    assert flips <= 3


def test_trace_ring_minimum_capacity_and_disabled(gpu_required, monkeypatch):
    """The ring at its minimum of 2 slots (a launch ends after every record)
    and switched off (HPLP_TRACE_RING=0: the pause-per-record path with the
    host's partition estimate) give the same records as the default ring."""
    g, s = std("cfg0")
    kw = dict(iteration_limit=120, tolerance=1e-12, trace=True, trace_period=3)
    base = hplp.solve(*csr_args(s), **kw)
    monkeypatch.setenv("HPLP_TRACE_RING_MB", "0.0001")
    small = hplp.solve(*csr_args(s), **kw)
    monkeypatch.delenv("HPLP_TRACE_RING_MB")
    monkeypatch.setenv("HPLP_TRACE_RING", "0")
    off = hplp.solve(*csr_args(s), **kw)
    assert len(base["trace"]) == len(small["trace"]) == len(off["trace"]) == 40
    for a, b, c in zip(base["trace"], small["trace"], off["trace"]):
        assert (a["iteration"], a["epoch"], a["inner"]) == (b["iteration"], b["epoch"], b["inner"])
        assert (a["iteration"], a["epoch"], a["inner"]) == (c["iteration"], c["epoch"], c["inner"])
        assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])
        assert np.array_equal(a["x"], c["x"]) and np.array_equal(a["y"], c["y"])
        assert all(np.array_equal(u, v) for u, v in zip(a["partition"], b["partition"]))
        assert sum(len(np.setxor1d(u, v)) for u, v in zip(a["partition"], c["partition"])) <= 1
        assert a["kkt"] == b["kkt"] == c["kkt"]
    assert np.array_equal(base["x"], small["x"]) and np.array_equal(base["x"], off["x"])


@pytest.mark.parametrize("name", ["cfg1_small", "zipf_small", "transport_small", "ragged"])
def test_bank_staggered_layout_bit_identical(gpu_required, name, monkeypatch):
    """Bank-staggered stream tasks (build_schedule stagger, HX_STAGGER): the
    pad slots only append +0.0 to a row's sum and no row sum is -0.0, so on a
    matrix of stream rows only (<= 64 nonzeros) both SpMVs are bit-identical
    to the unpadded layout -- with the most padding allowed (15 slots before
    every row) and with the default.  Rows beyond 64 nonzeros are cut into
    pieces of 256 slots from their aligned start in the staggered copy
    (equal pieces in the plain one), which moves the fast order's partial sums:
    those SpMVs agree to 1e-13.  The solve's norms and KKT sums follow the
    schedule's row -> lane map, which the pads move, so iterates agree to
    rounding, with identical statuses, iteration counts and restarts -- on a
    preconditioned instance too (the padded copies are rescaled with the
    CSR)."""
    args = _ragged_lp() if name == "ragged" else csr_args(std(name)[1])
    long_rows = max(np.diff(np.asarray(args[2])).max(), np.bincount(np.asarray(args[3]), minlength=args[1]).max()) > 64
    rng = np.random.default_rng(5)
    x, y = rng.normal(size=args[1]), rng.normal(size=args[0])
    runs = {}
    for layout in ("0,0,4", "15,1,4", "15,15,1"):
        monkeypatch.setenv("HX_STAGGER", layout)
        hx = hplp.HX(device=0)
        hx.upload(*args)
        prods = (hx.spmv(x), hx.spmv_transpose(y))
        hx.close()
        out = []
        for pc in (False, True):
            sol = hplp.Solver(*args)
            if pc:
                sol.hx.precondition(2, 0.5)
            r = sol.solve(iteration_limit=400, tolerance=1e-12)
            out.append((r["x"], r["y"], r["status"], r["iterations"], [e[:2] for e in r["epochs"]]))
            sol.close()
        runs[layout] = (prods, out)
    base_p, base = runs["0,0,4"]
    for layout in ("15,1,4", "15,15,1"):
        p, o = runs[layout]
        if long_rows:
            assert rel_inf(p[0], base_p[0]) <= 1e-13 and rel_inf(p[1], base_p[1]) <= 1e-13, layout
        else:
            assert np.array_equal(p[0], base_p[0]) and np.array_equal(p[1], base_p[1]), layout
        for a, b in zip(o, base):
            tol = 1e-11 if long_rows else 1e-12
            assert rel_inf(a[0], b[0]) <= tol and rel_inf(a[1], b[1]) <= tol, layout
            assert a[2:] == b[2:], layout
