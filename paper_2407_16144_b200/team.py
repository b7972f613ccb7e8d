"""Multi-process team plumbing (one process per GPU, e.g. under torchrun).

Each rank's solver exports a blob of CUDA IPC handles for the buffers its
peers write into (iterate pools, certificate vectors, partial-sum records,
barrier word); the blobs travel over torch.distributed (NCCL or gloo
process group -- plumbing only, the data path is the fused P2P kernel) and
every rank imports all of them.  See include/hplp_gpu.h
(hplp_solver_create_rank) and DESIGN.md §6.
"""
from __future__ import annotations


def exchange(blob: bytes, group=None) -> list:
    """All ranks' blobs in rank order (torch.distributed all_gather_object)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


def join(solver, group=None) -> None:
    """Bind this rank's solver to every peer of the process group."""
    for b in exchange(solver.team_export(), group):
        solver.team_import(b)


def agree(ok: bool, what: str, group=None) -> None:
    """Every rank learns whether every rank succeeded at `what` (all_reduce
    MIN of a flag); if any failed, every rank raises -- so no rank ever enters
    a collective its peers skipped."""
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag.item()) == 0:
        raise RuntimeError(f"team setup failed on some rank during {what}")


def rank_solver(std, device: int, group=None):
    """Solver for this process's block of `std` (a StdForm), joined to the
    team.  Setup runs in phases (create, join, first power iteration) with an
    agreement after each, so a failure on one rank fails every rank instead
    of leaving peers stuck in a collective."""
    import torch.distributed as dist

    from .hplp import Solver

    s, err = None, None
    try:
        s = Solver.rank(*std.csr(), nranks=dist.get_world_size(group), rank=dist.get_rank(group), device=device)
    except Exception as e:  # noqa: BLE001 -- re-raised after the agreement
        err = e
    agree(err is None, "hplp_solver_create_rank", group)
    blobs = exchange(s.team_export(), group)
    try:
        for b in blobs:
            s.team_import(b)
    except Exception as e:  # noqa: BLE001
        err = e
    agree(err is None, "team_import", group)
    return s
