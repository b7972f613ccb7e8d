"""TEST INFRASTRUCTURE: a host (numpy) emulation of the row-partitioned
multi-GPU rHPDHG iteration, one process per
rank over torch.distributed (gloo).  It exercises exactly the exchange
pattern the multi-GPU device path uses:

  all-gather y slices   -> local A^T y on the owned columns (phase A)
  all-gather x+ slices  -> local A x+ on the owned rows      (phase B)
  all-gather the 7 per-rank partial sums, reduced in rank order
  -> bit-identical totals on every rank -> replicated controller

and the ownership from the product's partition planner
(hplp_plan_partition).  The controller follows src/solver.cpp:241-341
(termination, adaptive/fixed restarts with the stall cap, Halpern combine
with the carried A x, best tracking); certificate scans are disabled
(infeasibility_check_period = 0) on both sides of the comparison.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp


def run_rank(rank, world, m, n, row_ptr, col_idx, val, b, c, row_bounds, col_bounds, iters, sigma_used, cfg,
             out_queue):
    import torch
    import torch.distributed as dist

    A = sp.csr_matrix((val, col_idx, row_ptr), shape=(m, n))
    r0, r1 = int(row_bounds[rank]), int(row_bounds[rank + 1])
    c0, c1 = int(col_bounds[rank]), int(col_bounds[rank + 1])
    A_loc = A[r0:r1, :]                    # owned rows of A
    AT_loc = A.T.tocsr()[c0:c1, :]          # owned rows of A^T (owned columns of A)
    b_loc, c_loc = b[r0:r1], c[c0:c1]
    eta = 1.0 / (2.0 * sigma_used)

    def gather(v_loc, total):
        """all-gather of the owned slices (gloo needs equal sizes: pad to the
        largest slice, then trim)."""
        bounds = row_bounds if total == m else col_bounds
        sizes = [int(bounds[r + 1] - bounds[r]) for r in range(world)]
        big = max(sizes)
        buf = torch.zeros(big, dtype=torch.float64)
        buf[: len(v_loc)] = torch.from_numpy(np.ascontiguousarray(v_loc))
        parts = [torch.zeros(big, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, buf)
        return np.concatenate([p.numpy()[: sizes[r]] for r, p in enumerate(parts)])

    def reduce_ordered(vals):
        t = torch.tensor(vals, dtype=torch.float64)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        tot = parts[0].clone()
        for p in parts[1:]:
            tot = tot + p  # rank order: identical on every rank
        return tot.numpy()

    b_norm = math.sqrt(reduce_ordered([float(b_loc @ b_loc)])[0])
    c_norm = math.sqrt(reduce_ordered([float(c_loc @ c_loc)])[0])
    x = np.zeros(c1 - c0)
    y = np.zeros(r1 - r0)
    a_x = np.zeros(r1 - r0)
    ax_anchor, x_anchor, y_anchor = a_x.copy(), x.copy(), y.copy()
    n_ep, k, res_start = 0, 0, 0.0
    trace = []
    for it in range(iters):
        y_full = gather(y, m)
        aty = AT_loc @ y_full
        xp = np.maximum(x - eta * (aty + c_loc), 0.0)
        xp_full = gather(xp, n)
        axp = A_loc @ xp_full
        yp = y + eta * ((2.0 * axp - a_x) - b_loc)
        dres = np.maximum(-(c_loc + aty), 0.0)
        tot = reduce_ordered([float(dres @ dres), float(c_loc @ x), float((x - xp) @ (x - xp)),
                              float((a_x - b_loc) @ (a_x - b_loc)), float(b_loc @ y), float((y - yp) @ (y - yp)),
                              float((y - yp) @ (a_x - axp))])
        kkt_p = math.sqrt(tot[3]) / (1.0 + b_norm)
        kkt_d = math.sqrt(tot[0]) / (1.0 + c_norm)
        kkt_g = abs(tot[1] + tot[4]) / (1.0 + abs(tot[1]) + abs(tot[4]))
        kmax = max(kkt_p, kkt_d, kkt_g)
        q = tot[2] / eta - 2.0 * tot[6] + tot[5] / eta
        res = math.sqrt(q) if q > 0 else 0.0
        if k == 0:
            res_start = res
        trace.append((it, n_ep, k, gather(x, n), gather(y, m), kmax))
        if kmax <= cfg["tolerance"]:
            break
        if cfg["restart"] == "fixed":
            restart = k >= cfg["k_star"]
        else:
            restart = (k > cfg["tau0"]) if n_ep == 0 else (res <= cfg["beta"] * res_start)
            restart = restart or (cfg["stall_cap"] > 0 and k >= cfg["stall_cap"])
        if restart:
            x, y, a_x = xp, yp, axp
            x_anchor, y_anchor, ax_anchor = x.copy(), y.copy(), a_x.copy()
            n_ep += 1
            k = 0
        else:
            w = 1.0 / (k + 2)
            x = (1.0 - w) * xp + w * x_anchor
            y = (1.0 - w) * yp + w * y_anchor
            a_x = (1.0 - w) * axp + w * ax_anchor
            k += 1
    if rank == 0:
        out_queue.put(trace)
    dist.barrier()
