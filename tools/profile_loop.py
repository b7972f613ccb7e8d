"""Short driver for ncu captures of the loop kernel (configs[1] by default).

  python tools/profile_loop.py [--cfg 1] [--iters 200] [--launches 3]
Runs setup (power iteration) then `launches` hx_run batches of `iters`
iterations; under ncu use -k regex:loop_kernel -s <skip> -c 1.
"""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=1)
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--launches", type=int, default=3)
ap.add_argument("--box", action="store_true", help="the box form (loop_kernel_box)")
a = ap.parse_args()
g = gen.generate(a.cfg)
s = hplp.to_standard_form(g)
solver = hplp.Solver.box(*s.csr()) if a.box else hplp.Solver.from_std(s)
r0 = solver.solve(iteration_limit=0)
cfg = abi.Config.default(tolerance=1e-4, iteration_limit=10**9, infeasibility_check_period=0 if a.box else 100)
solver.hx.setup(cfg, r0["sigma_estimate"], r0["eta"])
for i in range(a.launches):
    t = time.perf_counter()
    p = solver.hx.run(a.iters)
    print(f"launch {i}: {a.iters} its in {p.device_ms:.3f} ms -> {a.iters / p.device_ms * 1e3:.0f} it/s; "
          f"it={p.it} n={p.n} k={p.k} kkt={p.trace_kkt.max_relative:.3e}", flush=True)
if os.environ.get("HX_PROFILE") == "1":
    import json
    print(json.dumps(solver.hx.phase_profile(), indent=1))
solver.close()
