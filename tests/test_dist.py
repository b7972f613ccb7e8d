"""Multi-GPU path, host side (CPU, gloo, world_size 2): the partition planner
and the row-partitioned iteration's exchange pattern, checked against the
single-process oracle."""
from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import CpuLp
from paper_2407_16144_b200 import hplp
from paper_2407_16144_b200.abi import i32ptr, i64ptr
from tests.helpers import csr_args, problem, rel_inf


def plan(s, parts):
    L = hplp.lib()
    L.hplp_plan_partition.argtypes = [C.c_int64, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.c_int32,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    rb, cb = np.empty(parts + 1, np.int64), np.empty(parts + 1, np.int64)
    assert L.hplp_plan_partition(s.m, s.n, i64ptr(s.row_ptr), i32ptr(s.col_idx), parts, i64ptr(rb), i64ptr(cb)) == 0
    return rb, cb


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_partition_plan_balanced(parts):
    s = hplp.to_standard_form(problem("zipf_small"))
    rb, cb = plan(s, parts)
    assert rb[0] == 0 and rb[-1] == s.m and cb[0] == 0 and cb[-1] == s.n
    assert (np.diff(rb) >= 0).all() and (np.diff(cb) >= 0).all()
    cost = np.array([s.row_ptr[rb[p + 1]] - s.row_ptr[rb[p]] + 3 * (rb[p + 1] - rb[p]) for p in range(parts)])
    longest = int(np.diff(s.row_ptr).max()) + 3
    assert cost.max() - cost.min() <= 2 * longest  # contiguous cut: within two rows of even
    col_nnz = np.bincount(s.col_idx, minlength=s.n)
    ccost = np.array([col_nnz[cb[p]:cb[p + 1]].sum() + 3 * (cb[p + 1] - cb[p]) for p in range(parts)])
    assert ccost.max() - ccost.min() <= 2 * (int(col_nnz.max()) + 3)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, args, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests.dist_emulation import run_rank

    run_rank(rank, world, *args, q)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,restart", [("cfg0", "adaptive"), ("cfg1_small", "adaptive"), ("zipf_small", "fixed")])
def test_row_partitioned_iteration_matches_oracle(name, restart):
    s = hplp.to_standard_form(problem(name))
    world = 2
    rb, cb = plan(s, world)
    lp = CpuLp("port", *csr_args(s))
    sigma, _, _, _ = lp.power_iteration()
    sigma_used = sigma * (1.0 + 1e-4)
    iters = 80
    kw = dict(restart_kind=0, k_star=25) if restart == "fixed" else {}
    cpu = lp.solve(iteration_limit=iters, tolerance=1e-12, infeasibility_check_period=0, trace=True, **kw)
    cfg = dict(tolerance=1e-12, restart=restart, k_star=25, tau0=32, beta=0.36787944117144233, stall_cap=2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    args = (s.m, s.n, s.row_ptr, s.col_idx, s.val, s.b, s.c, rb, cb, iters, sigma_used, cfg)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue

    trace = None
    for _ in range(600):
        try:
            trace = q.get(timeout=0.5)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    assert trace is not None, [p.exitcode for p in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(trace) == len(cpu["trace"]) == iters
    for (it, n_ep, k, x, y, _), tc in zip(trace, cpu["trace"]):
        assert (it, n_ep, k) == (tc["iteration"], tc["epoch"], tc["inner"])
        assert rel_inf(np.concatenate([x, y]), np.concatenate([tc["x"], tc["y"]])) <= 1e-10


def _exchange_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_16144_b200 import team

    q.put((rank, team.exchange(bytes([rank]) * (rank + 3))))
    dist.destroy_process_group()


def test_team_blob_exchange_gloo():
    """The multi-process join plumbing (paper_2407_16144_b200/team.py): every
    rank receives every rank's IPC blob in rank order."""
    world = 2
    q = mp.get_context("spawn").SimpleQueue()
    port = _free_port()
    ps = [mp.get_context("spawn").Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get() for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert got[r] == [bytes([k]) * (k + 3) for k in range(world)]


def _agree_worker(rank, world, port, fail_rank, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_16144_b200 import team

    out = []
    for phase in ("create", "join", "power"):
        try:
            team.agree(not (rank == fail_rank and phase == "join"), phase)
            out.append(phase)
        except RuntimeError as e:
            out.append(f"raised:{phase}:{'join' in str(e)}")
            break
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [None, 0, 1])
def test_team_setup_failure_fails_every_rank(fail_rank):
    """team.agree (the bench's team setup, paper_2407_16144_b200/team.py): a
    rank that fails a setup phase makes EVERY rank raise at that phase -- no
    rank goes on into a collective its peers skipped, and there is no
    fallback to independent replicas."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    ps = [ctx.Process(target=_agree_worker, args=(r, world, port, fail_rank, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get() for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        if fail_rank is None:
            assert got[r] == ["create", "join", "power"]
        else:
            assert got[r] == ["create", "raised:join:True"], got
