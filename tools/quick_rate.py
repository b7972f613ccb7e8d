"""Loop throughput on configs[1] for the library HPLP_GPU_LIB points at:
the single-GPU kernel (loop_kernel) and the one-rank team kernel
(loop_kernel_team), best of 5 batches of 1000 iterations (L2 not flushed).
  HPLP_GPU_LIB=build_variants/X/libhplp_gpu.so python tools/quick_rate.py"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
s = hplp.to_standard_form(gen.generate(cid))
cfg = abi.Config.default(tolerance=1e-4, iteration_limit=10**9)
out = []
for kind in ("loop", "team1"):
    if kind == "loop":
        sol = hplp.Solver.from_std(s)
    else:
        sol = hplp.Solver.rank(*s.csr(), nranks=1, rank=0)
        sol.team_import(sol.team_export())
    r0 = sol.solve(iteration_limit=0)
    sol.hx.setup(cfg, r0["sigma_estimate"], r0["eta"])
    best = min(sol.hx.run(1000).device_ms for _ in range(6))
    out.append(f"{kind} {1e6 / best:8.0f} it/s")
    sol.close()
print(os.environ.get("HPLP_GPU_LIB", "default"), " | ".join(out), flush=True)
