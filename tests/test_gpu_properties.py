"""The paper's properties on the device path (SPEC.md ACCEPTANCE CRITERIA),
checked on what the B200 loop computes:
  AC3  adaptive per-epoch contraction (epoch log residuals);
  AC9  nonexpansiveness of T in the canonical norm (single device steps);
  AC8  partition identification from device traces, rHPDHG vs vanilla PDHG.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2407_16144_b200 import abi, hplp
from tests.helpers import random_std_lp

pytestmark = pytest.mark.gpu


def test_ac3_adaptive_epoch_contraction(gpu_required):
    """residual at z^{n+1,0} <= (1/e) residual at z^{n,0} + 1e-10 for every
    epoch ended by the decay rule (the stall cap ends epochs regardless)."""
    checked = 0
    for seed in range(10):
        args = random_std_lp(seed, 5, 8)
        r = hplp.solve(*args, tolerance=1e-8, iteration_limit=20000)
        eps = r["epochs"]
        for n in range(1, len(eps) - 1):
            if eps[n][1] >= 2000:  # stall-capped epoch
                continue
            assert eps[n + 1][2] <= math.exp(-1) * eps[n][2] + 1e-10, (seed, n, eps[n], eps[n + 1])
            checked += 1
    assert checked >= 10


def _canon(A, eta, dx, dy):
    # ||(dx, dy)||_P^2 = ||dx||^2/eta - 2 dy'A dx + ||dy||^2/eta (src/pdhg_core.cpp:37-51)
    return math.sqrt(max(dx @ dx / eta - 2.0 * dy @ (A @ dx) + dy @ dy / eta, 0.0))


def test_ac9_nonexpansive_device_step(gpu_required):
    """||T(z) - T(z')||_P <= ||z - z'||_P + 1e-10 for random pairs, T taken
    from one device iteration (hx_setup(z) + hx_run(1) -> ITERATE_NEXT)."""
    rng = np.random.default_rng(9)
    for seed in range(6):
        m, n, rp, ci, v, b, c = random_std_lp(seed, 6, 10)
        A = sp.csr_matrix((v, ci, rp), shape=(m, n))
        sol = hplp.Solver(m, n, rp, ci, v, b, c)
        r0 = sol.solve(iteration_limit=0)
        eta = r0["eta"]
        cfg = abi.Config.default(iteration_limit=1, tolerance=1e-300, infeasibility_check_period=0)

        def T(x, y):
            sol.hx.setup(cfg, r0["sigma_estimate"], eta, x, y)
            sol.hx.run(1)
            return sol.hx.get_iterate(hplp.ITERATE_NEXT)

        for _ in range(10):
            x1, y1 = rng.normal(size=n) * 3, rng.normal(size=m) * 3
            x2, y2 = rng.normal(size=n) * 3, rng.normal(size=m) * 3
            tx1, ty1 = T(x1, y1)
            tx2, ty2 = T(x2, y2)
            assert _canon(A, eta, tx1 - tx2, ty1 - ty2) <= _canon(A, eta, x1 - x2, y1 - y2) + 1e-10
        sol.close()


def _identification(trace, oracle_n, oracle_b1):
    """Smallest logged iteration after which (N, B1) equals the oracle on
    every later record (inc/diagnostics.hpp:86-89); None if never."""
    ident = None
    for rec in trace:
        ok = np.array_equal(rec["partition"][0], oracle_n) and np.array_equal(rec["partition"][1], oracle_b1)
        if ok and ident is None:
            ident = rec["iteration"]
        elif not ok:
            ident = None
    return ident


def test_ac8_partition_identification(gpu_required):
    """The (N, B1) estimate of the device traces stabilises to the partition of
    a high-accuracy solve before termination, and rHPDHG identifies no later
    than vanilla PDHG on at least half of the instances (SPEC.md AC8 floor)."""
    wins = total = 0
    for seed in range(20):
        args = random_std_lp(100 + seed, 6, 12)
        ref = hplp.solve(*args, tolerance=1e-12, iteration_limit=200000, trace=True, trace_period=100000)
        if ref["status"] != "optimal":
            continue
        last = hplp.solve(*args, tolerance=1e-12, iteration_limit=ref["iterations"] + 1, trace=True,
                          trace_period=max(ref["iterations"], 1))["trace"][-1]["partition"]
        on, ob1 = last[0], last[1]
        # every 10th iteration logged (the identification iteration to within 10)
        rh = hplp.solve(*args, tolerance=1e-8, iteration_limit=200000, trace=True, trace_period=10)
        va = hplp.solve(*args, tolerance=1e-8, iteration_limit=200000, trace=True, trace_period=10,
                        scheme=abi.SCHEME_VANILLA)
        i_rh, i_va = _identification(rh["trace"], on, ob1), _identification(va["trace"], on, ob1)
        if i_rh is None or i_va is None:
            continue
        total += 1
        wins += i_rh <= i_va
    assert total >= 10, total
    assert wins >= total / 2, (wins, total)
