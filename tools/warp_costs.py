"""Fit the schedule's cost model from measured per-warp SpMV times.

Needs the per-warp timer build:
  make -C paper_2407_16144_b200/csrc LIB=../lib_wprof EXTRA=-DHX_WPROF
  HPLP_GPU_LIB=$PWD/paper_2407_16144_b200/lib_wprof/libhplp_gpu.so python tools/warp_costs.py 1
Per warp: time ~ a * nnz + b * rows + c * stream_tasks + d * piece_tasks
(least squares, per phase); prints the fit and the cost-model constants it
implies (row and task cost in nnz units, kRowCost / kTaskCost).
"""
import os
import sys
from pathlib import Path

os.environ["HX_PROFILE"] = "1"
# task positions must index the CSR arrays below (no bank-staggered copy)
os.environ.setdefault("HX_STAGGER", "0,0,4")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 1
s = hplp.to_standard_form(gen.generate(cfg_id))
solver = hplp.Solver.from_std(s)
r0 = solver.solve(iteration_limit=0)
hx = solver.hx
hx.setup(abi.Config.default(tolerance=1e-6, iteration_limit=10**9, infeasibility_check_period=0),
         r0["sigma_estimate"], r0["eta"])
g = hx.info()["grid"]
W = g * hx.WARPS
hx.run(200)
hx.warp_profile(reset=True)
iters = 1000
hx.run(iters)
wt, cta = hx.warp_profile(reset=True)
wt = wt / iters / 1965.0  # us per iteration (SM clock ~1965 MHz)


import scipy.sparse as sp  # noqa: E402

A = sp.csr_matrix((s.val, s.col_idx, s.row_ptr), shape=(s.m, s.n))
AT = A.T.tocsr()
AT.sort_indices()
IDX = {0: A.indices, 1: AT.indices}


def features(tasks, idx):
    f = np.zeros((W, 5))
    kind = tasks[:, 1] >> 30
    rows = (tasks[:, 1] & ((1 << 30) - 1)) - tasks[:, 0]
    nnz = tasks[:, 3] - tasks[:, 2]
    empty = (tasks == 0).all(axis=1)
    for t in range(len(tasks)):
        if empty[t]:
            continue
        w = t % W
        f[w, 0] += nnz[t]
        f[w, 4] += len(np.unique(idx[tasks[t, 2]:tasks[t, 3]] >> 2))  # distinct 32-byte sectors gathered
        if kind[t] == 0:
            f[w, 1] += rows[t]
            f[w, 2] += 1
        else:
            f[w, 3] += 1
    return f


for phase, which, name in ((0, 1, "A (rows of A^T)"), (1, 0, "B (rows of A)")):
    f = features(hx.sched_tasks(which), IDX[which])
    y = wt[phase]
    m = f[:, 0] > 0
    coef, *_ = np.linalg.lstsq(f[m], y[m], rcond=None)
    pred = f[m] @ coef
    r2 = 1 - ((y[m] - pred) ** 2).sum() / ((y[m] - y[m].mean()) ** 2).sum()
    a, b, c, d, e = coef
    print(f"phase {name}: warps {m.sum()}, time us/warp mean {y[m].mean():.2f} min {y[m].min():.2f} max {y[m].max():.2f}")
    print(f"   fit us = {a*1e3:.3f}e-3*nnz + {b*1e3:.3f}e-3*rows + {c:.4f}*stream_tasks + {d:.4f}*pieces "
          f"+ {e*1e3:.3f}e-3*sectors (R^2 {r2:.3f})")
    c4, *_ = np.linalg.lstsq(f[m][:, :4], y[m], rcond=None)
    p4 = f[m][:, :4] @ c4
    print(f"   without the sector feature: R^2 {1 - ((y[m] - p4) ** 2).sum() / ((y[m] - y[m].mean()) ** 2).sum():.3f}; "
          f"sectors in nnz units {e / a:.2f}")
    cta_t = y.reshape(g, hx.WARPS).max(axis=1)
    print(f"   CTA max-warp time: mean {cta_t.mean():.2f} max {cta_t.max():.2f}; warp time sd {y[m].std():.3f}")
    yw = y.reshape(g, hx.WARPS)
    cta_mean = yw.mean(axis=1)
    cta_mean_nolead = yw[:, 1:].mean(axis=1)
    print(f"   CTA mean-warp time (all warps): mean {cta_mean.mean():.2f} max {cta_mean.max():.2f} min {cta_mean.min():.2f}; "
          f"warps 1..15 only: max {cta_mean_nolead.max():.2f}; warp0 mean {yw[:, 0].mean():.2f}")
    print(f"   in nnz units: row {b/a:.2f}, stream task {c/a:.1f}, piece task {d/a:.1f}")
    print(f"   per-warp features mean: nnz {f[m,0].mean():.0f} rows {f[m,1].mean():.0f} "
          f"stream {f[m,2].mean():.1f} pieces {f[m,3].mean():.1f}")
    resid = y[m] - pred
    print(f"   residual sd {resid.std():.3f} us; slowest warps (t, pred):",
          [(round(float(y[m][i]), 2), round(float(pred[i]), 2)) for i in np.argsort(y[m])[-5:]])
solver.close()
