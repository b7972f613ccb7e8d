"""CPU tests of the product's host side (no GPU): the generator, the
standard-form conversion against the reference's own to_standard_form, the
C ABI surface (every symbol include/*.h declares is exported; struct sizes
agree with the ctypes mirrors) and that the CUDA path fails loudly -- never
falls back -- when no B200 is visible."""
from __future__ import annotations

import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
from oracle import CpuStd
from paper_2407_16144_b200 import abi, gen, hplp
from paper_2407_16144_b200.build import GEN_LIB, GPU_LIB
from tests.conftest import has_gpu

ROOT = Path(__file__).resolve().parent.parent
CHECKERS = ["port"] + (["reference"] if oracle.available("reference") else [])


def test_generator_deterministic_and_sized():
    a, b = gen.generate(0), gen.generate(0)
    for f in ("row_ptr", "col_idx", "val", "row_rhs", "objective", "col_upper"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    assert (a.m, a.n, a.nnz) == (1000, 2000, 10000)
    assert (a.row_relation[:700] == abi.ROW_EQ).all() and (a.row_relation[700:] == abi.ROW_GE).all()
    # planted optimum is primal feasible: A x* = b on '=' rows, >= b on '>=' rows, bounds hold
    rows = np.repeat(np.arange(a.m), np.diff(a.row_ptr))
    ax = np.bincount(rows, weights=a.val * a.x_star[a.col_idx], minlength=a.m)
    eq = a.row_relation == abi.ROW_EQ
    assert np.allclose(ax[eq], a.row_rhs[eq], atol=1e-9)
    assert (ax[~eq] >= a.row_rhs[~eq] - 1e-9).all()
    assert (a.x_star >= 0).all() and (a.x_star <= a.col_upper).all()
    assert math.isclose(a.planted_objective, float(a.objective @ a.x_star), rel_tol=1e-12)


def test_generator_presets_shapes():
    p = gen.preset(1)
    assert (p.m, p.n, p.nnz_per_row, p.row_scale_log10) == (100000, 200000, 20, 2.0)
    t = gen.generate(gen.scaled(3, sources=30, sinks=20))
    assert (t.m, t.n, t.nnz) == (50, 600, 1200)
    supply, demand = t.row_rhs[:30], t.row_rhs[30:]
    assert math.isclose(supply.sum(), 1.1 * demand.sum(), rel_tol=1e-12)
    z = gen.generate(gen.scaled(4, m=2000, n=4000, zipf_cap=500, zipf_target_nnz=20000, zipf_force_cap=2))
    lens = np.diff(z.row_ptr)
    assert lens.max() == 500 and lens.min() >= 1
    i2 = gen.generate(gen.scaled(2, m=300, n=600, infeasible_rows=7))
    assert i2.m == 307 and math.isnan(i2.planted_objective)


def _random_general(seed):
    """General-form LP exercising every conversion branch: <=, =, >= rows with
    and without RANGES, free / lower-only / upper-only / boxed / fixed
    columns, maximize, an objective constant, unsorted row entries."""
    rng = np.random.default_rng(seed)
    m, n = 9, 12
    rp, ci, v = [0], [], []
    for i in range(m):
        cols = rng.choice(n, size=rng.integers(1, 5), replace=False)
        ci.extend(cols.tolist())
        v.extend(np.round(rng.normal(size=len(cols)), 3).tolist())
        rp.append(len(ci))
    rel = rng.integers(0, 3, size=m).astype(np.int32)
    rng_ = np.where(rng.random(m) < 0.4, np.round(rng.normal(size=m), 2), np.nan)
    base = np.round(rng.normal(size=n), 2)
    lo = np.where(rng.random(n) < 0.2, -np.inf, base)
    hi = np.where(rng.random(n) < 0.5, np.inf, base + np.abs(np.round(rng.normal(size=n), 2)))
    hi[0], lo[0] = np.inf, -np.inf  # free
    lo[1] = -np.inf  # upper only
    g = gen.GeneralLP(m, n, np.array(rp, np.int64), np.array(ci, np.int32), np.array(v), rel,
                      np.round(rng.normal(size=m), 2), lo, hi, np.round(rng.normal(size=n), 2))
    g.row_range = rng_
    g.maximize = bool(seed % 2)
    g.objective_constant = 1.25
    return g


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("kind", CHECKERS)
def test_to_standard_form_matches_checker(seed, kind):
    g = _random_general(seed)
    mine = hplp.to_standard_form(g)
    ref = CpuStd(kind, g.as_abi())
    assert (mine.m, mine.n, mine.nnz) == (ref.m, ref.n, ref.nnz)
    for f in ("row_ptr", "col_idx", "val", "b", "c"):
        assert np.array_equal(getattr(mine, f), getattr(ref, f)), f
    x = np.random.default_rng(seed).random(mine.n)
    xo, obj = mine.recover(x, 3.5)
    xo2, obj2 = ref.recover(x, 3.5, g.n)
    assert np.array_equal(xo, xo2) and obj == obj2


def test_to_standard_form_planted_config0():
    g = gen.generate(0)
    mine = hplp.to_standard_form(g)
    ref = CpuStd(CHECKERS[-1], g.as_abi())
    assert (mine.m, mine.n, mine.nnz) == (3000, 4300, 14300)
    for f in ("row_ptr", "col_idx", "val", "b", "c"):
        assert np.array_equal(getattr(mine, f), getattr(ref, f))


@pytest.mark.parametrize("kind", CHECKERS)
def test_to_standard_form_nonfinite_b_rejected_like_reference(kind):
    # a column with lower = upper = -inf mirrors to an infinite shift of b:
    # the reference's StandardFormLP ctor throws (src/lp_model.cpp:40-42), so must we
    g = _random_general(2)
    g.col_lower = g.col_lower.copy()
    g.col_upper = g.col_upper.copy()
    j = int(g.col_idx[0])
    g.col_lower[j], g.col_upper[j] = -np.inf, -np.inf
    with pytest.raises(ValueError, match="non-finite b or c"):
        hplp.to_standard_form(g)
    with pytest.raises(ValueError, match="non-finite b or c"):
        CpuStd(kind, g.as_abi())


def test_to_standard_form_errors():
    g = _random_general(0)
    g.col_lower = g.col_lower.copy()
    g.col_upper = g.col_upper.copy()
    g.col_lower[3], g.col_upper[3] = 2.0, 1.0
    with pytest.raises(ValueError, match="inconsistent bounds"):
        hplp.to_standard_form(g)
    g = _random_general(1)
    g.col_idx = g.col_idx.copy()
    g.col_idx[1] = g.col_idx[0] if g.row_ptr[1] >= 2 else g.col_idx[1]
    if g.row_ptr[1] >= 2:
        with pytest.raises(ValueError, match="duplicate"):
            hplp.to_standard_form(g)


def _declared(header):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(h[xp]\w*)\s*\(", text, flags=re.M)) - {"hplp_config_default"})


@pytest.mark.parametrize("header,lib", [("hx.h", GPU_LIB), ("hplp_gpu.h", GPU_LIB), ("hplp_gen.h", GEN_LIB)])
def test_c_abi_exports(header, lib):
    hplp.lib()  # builds if needed
    names = _declared(header)
    assert len(names) >= 5
    L = C.CDLL(str(lib))
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_struct_sizes_match_header():
    L = hplp.lib()
    for i, t in enumerate((abi.Config, abi.Result, abi.IO, abi.Epoch, abi.Trace, abi.General, hplp.HxProgress)):
        assert L.hx_sizeof(i) == C.sizeof(t), t.__name__


def test_config_validation_matches_reference():
    L = hplp.lib()
    ok = abi.Config.default()
    assert L.hplp_validate_config(C.byref(ok)) == 0
    for bad in (dict(tolerance=0.0), dict(iteration_limit=-1), dict(restart_kind=abi.RESTART_FIXED, k_star=0),
                dict(beta=1.0), dict(tau0=0), dict(infeasibility_check_period=-1)):
        c = abi.Config.default(**bad)
        assert L.hplp_validate_config(C.byref(c)) == abi.HPLP_EINVAL, bad


def test_status_strings():
    assert [hplp.to_string(i) for i in range(6)] == list(abi.STATUS_NAMES)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_cuda_path_fails_loudly_without_gpu():
    rp = np.array([0, 1], np.int64)
    with pytest.raises(hplp.HplpError):
        hplp.solve(1, 1, rp, np.array([0], np.int32), np.array([1.0]), np.array([1.0]), np.array([0.0]))
    with pytest.raises(hplp.HplpError):
        hplp.HX(device=0)


@pytest.mark.parametrize("seed", [12345, 1, 2**63 + 5])
def test_power_start_bit_identical_to_sequential_draw(seed):
    """hplp_power_start (parallel uniform conversion and log/sqrt) equals the
    reference's sequential std::normal_distribution loop bit for bit
    (src/sparse_matrix.cpp:145-151), checked against the oracle's restatement;
    odd and even lengths, including configs[1]'s 430,000."""
    import oracle
    from oracle.loader import load

    lo = load("port")
    for n in (1, 2, 3, 7, 1000, 1001, 40_001, 430_000):
        want = np.empty(n)
        assert lo.orc_power_start(n, C.c_uint64(seed), want.ctypes.data_as(C.POINTER(C.c_double))) == 0
        got = hplp.power_start(n, seed)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (n, seed)


def _sched_matrix(seed, rows, lo, hi, long_every=0, long_len=0):
    rng = np.random.default_rng(seed)
    lens = rng.integers(lo, hi + 1, size=rows)
    if long_every:
        lens[::long_every] = long_len
    return np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)


@pytest.mark.parametrize("rows,lo,hi,long_every,long_len", [(20000, 1, 40, 0, 0), (5000, 0, 64, 997, 5000),
                                                            (30000, 1, 2, 0, 0), (0, 1, 1, 0, 0)])
def test_schedule_covers_every_nonzero_once(rows, lo, hi, long_every, long_len):
    """hx_schedule_info (host only): the warp schedule the loop kernels walk
    covers every row and nonzero exactly once -- stream tasks of <= 64 rows /
    <= 256 nonzeros, longer rows cut into pieces of <= 256 -- and the same
    input always gives the same table (what makes the device reductions
    reproducible)."""
    rp = _sched_matrix(1, rows, lo, hi, long_every, long_len)
    tasks, st = hplp.schedule_info(rp, ctas=148)
    tasks2, _ = hplp.schedule_info(rp, ctas=148)
    assert np.array_equal(tasks, tasks2)
    live = tasks[~((tasks[:, 0] == 0) & (tasks[:, 1] == 0) & (tasks[:, 3] == 0))]
    kind = (live[:, 1].astype(np.int64) & 0xFFFFFFFF) >> 30
    r1 = live[:, 1] & ((1 << 30) - 1)
    nz = np.zeros(int(rp[-1]) + 1, np.int64)
    for (r0, _, p0, p1), e, k in zip(live, r1, kind):
        assert 0 < p1 - p0 <= 256 or (p1 == p0 and k == 0)
        if k == 0:  # stream task: whole rows, their nonzeros exactly
            assert e - r0 <= 64 and rp[r0] == p0 and rp[e] == p1
        else:  # a piece of one long row
            assert e == r0 + 1 and rp[r0] <= p0 < p1 <= rp[r0 + 1]
        nz[p0:p1] += 1
    assert np.all(nz[: int(rp[-1])] == 1)
    covered = np.zeros(max(rows, 1), np.int64)
    for (r0, _, p0, p1), e, k in zip(live, r1, kind):
        if k == 0:
            covered[r0:e] += 1
        elif p0 == rp[r0]:
            covered[r0] += 1
    if rows:
        assert np.all(covered[:rows] == 1)


def test_schedule_balances_ctas_and_leads_warp0():
    """Units are dealt to the least-loaded CTA first (its warps share one L1
    pipe), so CTA sums end within ~1% of each other even where warp sums
    differ by 20%; warp 0's lead (it runs the controller while the others
    start phase A) moves work to the CTA's other warps."""
    rp = _sched_matrix(7, 230000, 1, 20)
    tasks, st = hplp.schedule_info(rp, ctas=148)
    assert st["max_cta"] <= 1.02 * st["mean_cta"], st
    W = st["W"]
    live = ~((tasks[:, 0] == 0) & (tasks[:, 1] == 0) & (tasks[:, 3] == 0))
    warp = np.arange(len(tasks)) % W
    w0 = np.count_nonzero(live & (warp % 16 == 0))
    tasks_l, st_l = hplp.schedule_info(rp, ctas=148, lead=3000.0)
    live_l = ~((tasks_l[:, 0] == 0) & (tasks_l[:, 1] == 0) & (tasks_l[:, 3] == 0))
    warp_l = np.arange(len(tasks_l)) % W
    assert np.count_nonzero(live_l & (warp_l % 16 == 0)) < w0
    assert st_l["max_cta"] <= 1.02 * st_l["mean_cta"], st_l


def test_schedule_info_rejects_bad_input():
    with pytest.raises(ValueError, match="monotone"):
        hplp.schedule_info(np.array([0, 5, 3], np.int32))
    with pytest.raises(ValueError, match="bad arguments"):
        hplp.schedule_info(np.array([0, 1], np.int32), ctas=0)
