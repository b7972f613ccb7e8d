"""Iterations/s of each scheme on configs[1] (best of 5 batches of 1000,
device-resident, L2 not flushed): rHPDHG and the three baselines."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

s = hplp.to_standard_form(gen.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 1))
sol = hplp.Solver.from_std(s)
r0 = sol.solve(iteration_limit=0)
b_iter = 24 * s.nnz + 68 * s.m + 44 * s.n + 8
for name, scheme in (("rHPDHG", 0), ("vanilla", 1), ("averaged", 2), ("restarted_average", 3)):
    cfg = abi.Config.default(tolerance=1e-4, iteration_limit=10**9, scheme=scheme)
    sol.hx.setup(cfg, r0["sigma_estimate"], r0["eta"])
    best = min(sol.hx.run(1000).device_ms for _ in range(5))
    print(f"{name:18s} {1e6 / best:9.0f} it/s  ({b_iter * 1e6 / best / 6453.1e9:.3f} of the HBM roofline on B_iter)",
          flush=True)
