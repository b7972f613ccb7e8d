"""Run the large BASELINE configs on one B200: iterations/s of the device
loop, memory footprint, and (configs[3], or any config with --parity N) the
first N iterates against the CPU oracle.

  python tools/big_configs.py 3 --parity 20
  python tools/big_configs.py 4
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("--iters", type=int, default=300)
ap.add_argument("--parity", type=int, default=0)
a = ap.parse_args()
t = time.perf_counter()
g = gen.generate(a.cfg)
t_gen = time.perf_counter() - t
t = time.perf_counter()
s = hplp.to_standard_form(g)
t_std = time.perf_counter() - t
print(f"cfg{a.cfg}: general {g.m}x{g.n} nnz {g.nnz} (gen {t_gen:.1f}s); standard {s.m}x{s.n} nnz {s.nnz} "
      f"(to_standard_form {t_std:.1f}s); max row {int(np.diff(s.row_ptr).max())}", flush=True)
t = time.perf_counter()
solver = hplp.Solver.from_std(s)
t_up = time.perf_counter() - t
r0 = solver.solve(iteration_limit=0)
print(f"upload {t_up:.2f}s; sigma {r0['sigma_estimate']:.6g} eta {r0['eta']:.6g} power spmvs {r0['spmv_count'] - 3}",
      flush=True)
hx = solver.hx
hx.setup(abi.Config.default(tolerance=1e-4, iteration_limit=10**9), r0["sigma_estimate"], r0["eta"])
hx.run(20)
p = hx.run(a.iters)
b_iter = 24 * s.nnz + 68 * s.m + 44 * s.n + 8
ips = a.iters / p.device_ms * 1e3
print(f"loop: {a.iters} its in {p.device_ms:.2f} ms -> {ips:.1f} it/s, {b_iter * ips / 1e9:.1f} GB/s algorithmic "
      f"({b_iter * ips / 6537.6e9:.3f} of measured HBM); kkt {p.trace_kkt.max_relative:.3e}", flush=True)
if a.parity:
    import oracle

    gpu = hplp.solve(*s.csr(), iteration_limit=a.parity, tolerance=1e-12, trace=True)
    cpu = oracle.CpuLp("port", *s.csr()).solve(iteration_limit=a.parity, tolerance=1e-12, trace=True)
    worst = 0.0
    for tg, tc in zip(gpu["trace"], cpu["trace"]):
        assert (tg["epoch"], tg["inner"]) == (tc["epoch"], tc["inner"])
        zc = np.concatenate([tc["x"], tc["y"]])
        zg = np.concatenate([tg["x"], tg["y"]])
        worst = max(worst, float(np.max(np.abs(zg - zc)) / max(np.max(np.abs(zc)), 1e-300)))
    print(f"parity over {a.parity} iterations: max rel inf-norm diff {worst:.3e}; spmv {gpu['spmv_count']} vs "
          f"{cpu['spmv_count']}", flush=True)
solver.close()
