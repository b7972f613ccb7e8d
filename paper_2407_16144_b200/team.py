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


def rank_solver(std, device: int, group=None):
    """Solver for this process's block of `std` (a StdForm), joined to the team."""
    import torch.distributed as dist

    from .hplp import Solver

    s = Solver.rank(*std.csr(), nranks=dist.get_world_size(group), rank=dist.get_rank(group), device=device)
    join(s, group)
    return s
