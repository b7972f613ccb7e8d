"""Multi-GPU row partition on ONE B200.

The team's ranks run as CTA groups of ONE cooperative launch
(loop_kernel_team): each group owns a row block of A and a column block
(rows of A^T), pushes the slices its peers gather (x+, y+, the Halpern y
combo, certificate vectors) and its partial-sum records into the other
groups' buffers, and crosses the two-level team barrier -- the same kernel,
push protocol and barrier a multi-GPU node runs with CUDA-IPC peer pointers
(B200_PROFILING.md: ranks whose kernels wait on one another must not be
separate launches on one GPU, so emulation is one launch).

Bars: the oracle's per-iteration iterates to 1e-10 with the identical
(epoch, inner) sequence; identical status; bit-identical controllers on
every rank (every rank reduces all records in one fixed order).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import CpuLp
from paper_2407_16144_b200 import abi, hplp
from tests.helpers import csr_args, problem, rel_inf
from tests.test_gpu_parity import _trace_cmp, std

pytestmark = pytest.mark.gpu


def team_solve(s, nranks, **kw):
    t = hplp.Solver.team(*csr_args(s), nranks=nranks)
    try:
        r = t.solve(**kw)
        prog = [t.rank_hx(q).progress() for q in range(nranks)]
    finally:
        t.close()
    return r, prog


def _same_controllers(prog):
    """Every rank's replicated controller ends in the same state."""
    keys = ("it", "n", "k", "spmv_count", "status", "error", "res_epoch_start", "best_kkt", "trace_it", "trace_n",
            "trace_k", "trace_res", "n_epochs")
    for p in prog[1:]:
        for k in keys:
            assert getattr(p, k) == getattr(prog[0], k), k
        assert p.best_err.as_tuple() == prog[0].best_err.as_tuple()
        assert p.trace_kkt.as_tuple() == prog[0].trace_kkt.as_tuple()


@pytest.mark.parametrize("name,nranks", [("cfg0", 2), ("cfg1_small", 3), ("cfg2_small", 4), ("zipf_small", 2),
                                         ("zipf_small", 8), ("transport_small", 5)])
def test_team_iterate_parity_first_100(gpu_required, name, nranks):
    g, s = std(name)
    cpu = CpuLp("port", *csr_args(s)).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    gpu, prog = team_solve(s, nranks, iteration_limit=100, tolerance=1e-12, trace=True)
    assert len(cpu["trace"]) == 100
    _trace_cmp(gpu["trace"], cpu["trace"])
    assert gpu["status"] == cpu["status"] == "iteration_limit"
    assert gpu["spmv_count"] == cpu["spmv_count"]
    assert [e[:2] for e in gpu["epochs"]] == [e[:2] for e in cpu["epochs"]]
    _same_controllers(prog)


@pytest.mark.parametrize("nranks", [2, 4])
def test_team_solve_tol_1e4(gpu_required, nranks):
    g, s = std("cfg0")
    cpu = CpuLp("port", *csr_args(s)).solve(tolerance=1e-4, iteration_limit=200000)
    gpu, prog = team_solve(s, nranks, tolerance=1e-4, iteration_limit=200000)
    assert gpu["status"] == cpu["status"] == "optimal"
    oc, og = float(s.c @ cpu["x"]), float(s.c @ gpu["x"])
    assert abs(og - oc) <= 1e-4 * max(1.0, abs(oc))
    assert gpu["kkt"][3] <= 1e-4
    # the restart sequence only diverges through last-bit reduction-order effects
    assert abs(gpu["iterations"] - cpu["iterations"]) <= 0.02 * cpu["iterations"]
    _same_controllers(prog)


@pytest.mark.parametrize("name,nranks", [("cfg1_small", 3), ("zipf_small", 8), ("cfg0", 2)])
def test_team_rank_records_path(gpu_required, monkeypatch, name, nranks):
    """The rank-record reduction (each rank's leader pre-reduces its CTAs'
    phase records at the end-of-iteration barrier; the default once
    nranks * grid > 320 records, i.e. real multi-GPU teams) forced on for
    the one-device team: same iterate bar, identical controllers."""
    monkeypatch.setenv("HPLP_TEAM_PREREDUCE", "1")
    g, s = std(name)
    cpu = CpuLp("port", *csr_args(s)).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    gpu, prog = team_solve(s, nranks, iteration_limit=100, tolerance=1e-12, trace=True)
    _trace_cmp(gpu["trace"], cpu["trace"])
    assert [e[:2] for e in gpu["epochs"]] == [e[:2] for e in cpu["epochs"]]
    _same_controllers(prog)
    long, prog = team_solve(s, nranks, tolerance=1e-4, iteration_limit=200000)
    # the long run against the single-device solve (itself pinned to the
    # oracle by test_gpu_parity; the oracle's own 1e-4 run takes minutes here)
    ref = hplp.solve(*csr_args(s), tolerance=1e-4, iteration_limit=200000)
    assert long["status"] == ref["status"]
    assert abs(long["iterations"] - ref["iterations"]) <= max(10, ref["iterations"] // 100)
    _same_controllers(prog)


def test_team_matches_single_gpu_long_run(gpu_required):
    """2000 iterations (restarts, certificate scans every 100) on the team
    stay within rounding of the single-context solve."""
    g, s = std("cfg1_small")
    one = hplp.solve(*csr_args(s), iteration_limit=2000, tolerance=1e-12)
    team, prog = team_solve(s, 3, iteration_limit=2000, tolerance=1e-12)
    assert [e[:2] for e in team["epochs"]] == [e[:2] for e in one["epochs"]]
    assert rel_inf(np.concatenate([team["x"], team["y"]]), np.concatenate([one["x"], one["y"]])) <= 1e-9
    _same_controllers(prog)


def test_team_infeasible_certificate(gpu_required):
    g, s = std("cfg2_small")
    gpu, prog = team_solve(s, 3, tolerance=1e-4, iteration_limit=100000)
    cpu = CpuLp("port", *csr_args(s)).solve(tolerance=1e-4, iteration_limit=100000)
    assert gpu["status"] == cpu["status"] == "primal_infeasible"
    vec, meta = gpu["primal_cert"]
    rep = CpuLp("port", *csr_args(s)).validate_primal(vec, 1e-6, gpu["sigma_estimate"])
    assert rep["valid"]
    assert abs(np.linalg.norm(vec) - 1.0) <= 1e-12
    _same_controllers(prog)


def test_team_dual_infeasible_kat(gpu_required):
    # c=(-1,0), A=[1,-1], b=0 -> DualInfeasible; 2 ranks on 1 row
    rp, ci, v = np.array([0, 2], np.int64), np.array([0, 1], np.int32), np.array([1.0, -1.0])
    t = hplp.Solver.team(1, 2, rp, ci, v, np.array([0.0]), np.array([-1.0, 0.0]), nranks=2)
    r = t.solve()
    t.close()
    c = CpuLp("port", 1, 2, rp, ci, v, [0.0], [-1.0, 0.0]).solve()
    assert r["status"] == c["status"] == "dual_infeasible"
    assert r["iterations"] == c["iterations"]
    assert np.allclose(r["dual_cert"][0], c["dual_cert"][0], atol=1e-9)


def test_team_preconditioned(gpu_required):
    g, s = std("cfg1_small")
    kw = dict(iteration_limit=300, tolerance=1e-12, precondition_ruiz_iters=10, precondition_pc_alpha=1.0)
    one = hplp.solve(*csr_args(s), **kw)
    team, _ = team_solve(s, 2, **kw)
    assert [e[:2] for e in team["epochs"]] == [e[:2] for e in one["epochs"]]
    assert rel_inf(np.concatenate([team["x"], team["y"]]), np.concatenate([one["x"], one["y"]])) <= 1e-10


def test_team_low_level_api(gpu_required):
    """hx_set_partition / hx_upload_csr / hx_team_bind / hx_team_run by hand,
    plus the error paths."""
    g, s = std("cfg0")
    rb, cb = hplp.plan_partition(s.m, s.n, s.row_ptr, s.col_idx, 2)
    hxs = [hplp.HX(device=0) for _ in range(2)]
    grid = hxs[0].info()["grid"]
    for r, h in enumerate(hxs):
        h.set_partition(2, r, rb, cb, grid // 2)
        h.upload(*csr_args(s))
    assert len(hxs[0].team_export()) > 0
    with pytest.raises(hplp.HplpError):  # not bound yet: the peers are unknown
        cfg = abi.Config.default(iteration_limit=10)
        hxs[0].setup(cfg, 1.0, 0.1)
        hxs[0].run(10)
    hplp.team_bind(hxs)
    sigma, _, _, _ = hxs[0].power_iteration(np.ones(s.n) / np.sqrt(s.n))
    sig_used = sigma * (1 + 1e-4)
    cfg = abi.Config.default(iteration_limit=50, tolerance=1e-12)
    for h in hxs:
        h.setup(cfg, sig_used, 1.0 / (2 * sig_used))
    prog = hplp.team_run(hxs, 50)
    assert [p.it for p in prog] == [50, 50]
    assert prog[0].status == prog[1].status == abi.STATUS_ITERATION_LIMIT
    with pytest.raises(hplp.HplpError):  # bound ranks run together
        hxs[0].run(10)
    x0, y0 = hxs[0].get_iterate(hplp.ITERATE_BEST)
    x1, y1 = hxs[1].get_iterate(hplp.ITERATE_BEST)
    assert np.array_equal(x0, x1) and np.array_equal(y0, y1)
    with pytest.raises(ValueError):
        hplp.HX(device=0).set_partition(9, 0, [0, 1], [0, 1])
    with pytest.raises(ValueError):  # bounds must ascend from 0
        hplp.HX(device=0).set_partition(2, 0, [0, 5, 3], [0, 1, 2])
    for h in hxs:
        h.close()


# ---- one process per GPU (CUDA IPC) ----------------------------------------
def test_rank_solver_parity(gpu_required):
    """hplp_solver_create_rank + export/import + solve, as one rank of one: the
    launch path a torchrun rank takes (team of one, IPC blob of itself)."""
    g, s = std("cfg1_small")
    r = hplp.Solver.rank(*csr_args(s), nranks=1, rank=0, device=0)
    r.team_import(r.team_export())
    got = r.solve(iteration_limit=100, tolerance=1e-12, trace=True)
    r.close()
    cpu = CpuLp("port", *csr_args(s)).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    _trace_cmp(got["trace"], cpu["trace"])
    assert got["spmv_count"] == cpu["spmv_count"]


def _ipc_worker(rank, port, q):
    import os

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2407_16144_b200 import gen, hplp as H, team

        s = H.to_standard_form(gen.generate(0))
        sol = H.Solver.rank(*s.csr(), nranks=2, rank=rank, device=0)
        blobs = team.exchange(sol.team_export())
        for b in blobs:  # opens the peer's CUDA IPC mappings (same device, other process)
            sol.team_import(b)
        dist.barrier()  # both mapped before either unmaps
        sol.close()
        q.put((rank, "ok", len(blobs), blobs[0] != blobs[1]))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), 0, False))
    finally:
        dist.destroy_process_group()


def test_rank_ipc_mapping_two_processes(gpu_required):
    """Two processes exchange IPC blobs over torch.distributed and map each
    other's buffers.  No loop runs: two ranks whose kernels wait on one another
    must not share one GPU (B200_PROFILING.md); the loop itself is covered by
    the one-launch emulation above."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [o[1] for o in out] == ["ok", "ok"], out
    assert all(o[2] == 2 and o[3] for o in out)


# ---- memory partition: a rank stores only its blocks -----------------------
@pytest.mark.parametrize("name,nranks", [("cfg1_small", 2), ("zipf_small", 4), ("transport_small", 8)])
def test_rank_stores_only_its_blocks(gpu_required, name, nranks):
    """Every rank keeps its row block of A and its column block (rows of A^T)
    only: together the ranks store each nonzero exactly twice (once per
    copy), and each rank about 2 nnz / nranks -- the full matrix is on no
    rank's device (hx_stored_nonzeros), which is what lets an LP larger than
    one GPU run on the team."""
    g, s = std(name)
    rb, cb = hplp.plan_partition(s.m, s.n, s.row_ptr, s.col_idx, nranks)
    t = hplp.Solver.team(*csr_args(s), nranks=nranks)
    try:
        stored = [t.rank_hx(q).stored_nonzeros() for q in range(nranks)]
        for q, (na, nt) in enumerate(stored):
            assert na == s.row_ptr[rb[q + 1]] - s.row_ptr[rb[q]]
            assert nt == int(np.count_nonzero((s.col_idx >= cb[q]) & (s.col_idx < cb[q + 1])))
            assert na + nt <= 2 * s.nnz / nranks * 1.6 + 4 * 256, (q, na + nt, 2 * s.nnz / nranks)
        assert sum(a for a, _ in stored) == sum(b for _, b in stored) == s.nnz
        one = hplp.Solver(*csr_args(s))
        assert one.hx.stored_nonzeros() == (s.nnz, s.nnz)
        one.close()
        # the partitioned team still solves the LP: 100 iterates against the oracle
        got = t.solve(iteration_limit=100, tolerance=1e-12, trace=True)
    finally:
        t.close()
    cpu = CpuLp("port", *csr_args(s)).solve(iteration_limit=100, tolerance=1e-12, trace=True)
    _trace_cmp(got["trace"], cpu["trace"])
    assert got["spmv_count"] == cpu["spmv_count"]


def test_team_power_iteration_and_zero_iteration_kkt(gpu_required):
    """Power iteration on the team (each rank its rows of A x and columns of
    A^T w, the slices pushed to the peers, sigma from every rank's records)
    and the zero-iteration solve's KKT with fresh products (kModeKkt), against
    the oracle."""
    g, s = std("cfg1_small")
    cpu = CpuLp("port", *csr_args(s)).solve(iteration_limit=0, tolerance=1e-4)
    for nranks in (2, 5):
        t = hplp.Solver.team(*csr_args(s), nranks=nranks)
        try:
            got = t.solve(iteration_limit=0, tolerance=1e-4)
        finally:
            t.close()
        assert abs(got["sigma_estimate"] - cpu["sigma_estimate"]) <= 1e-12 * cpu["sigma_estimate"]
        assert got["spmv_count"] == cpu["spmv_count"]
        for a, b in zip(got["kkt"], cpu["kkt"]):
            assert abs(a - b) <= 1e-12 * max(abs(b), 1e-300)


def test_team_preconditioning_matches_single_device(gpu_required):
    """Ruiz + Pock-Chambolle on the team (kModeScale: each rank scales its
    blocks with the row / column scales its peers pushed): the scaled
    instance is the one the single device builds, so the solves agree."""
    g, s = std("zipf_small")
    kw = dict(iteration_limit=200, tolerance=1e-12, precondition_ruiz_iters=5, precondition_pc_alpha=0.5,
              trace=True, trace_period=20)
    one = hplp.solve(*csr_args(s), **kw)
    team, prog = team_solve(s, 4, **kw)
    _same_controllers(prog)
    assert [e[:2] for e in team["epochs"]] == [e[:2] for e in one["epochs"]]
    for a, b in zip(team["trace"], one["trace"]):
        assert rel_inf(np.concatenate([a["x"], a["y"]]), np.concatenate([b["x"], b["y"]])) <= 1e-10
        # the partition estimate from the team's trace slots (hx_trace_reduced_costs);
        # long-row sums may differ in the last bit between the two schedules
        moved = sum(len(np.setxor1d(pa, pb)) for pa, pb in zip(a["partition"], b["partition"]))
        assert moved <= 2, moved
