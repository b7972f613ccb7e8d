"""Box-form loop throughput on configs[1] (best of 6 batches of 1000)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

s = hplp.to_standard_form(gen.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 1))
sol = hplp.Solver.box(*s.csr())
cfg = abi.Config.default(tolerance=1e-4, iteration_limit=10**9, infeasibility_check_period=0)
r0 = sol.solve(iteration_limit=0)
sol.hx.setup(cfg, r0["sigma_estimate"], r0["eta"])
best = min(sol.hx.run(1000).device_ms for _ in range(6))
print(os.environ.get("HPLP_L2_STREAM", "auto"), f"box loop {1e6 / best:8.0f} it/s", flush=True)
sol.close()
