"""Per-iteration phase breakdown of the loop kernel on configs[1] (HX_PROFILE=1
per-CTA timers): phase A, barrier 1, phase B, barrier 2, controller, scans /
redone phases.  python tools/phase_breakdown.py [config] [--box]"""
import os
import sys
from pathlib import Path

os.environ["HX_PROFILE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1
box = "--box" in sys.argv
s = hplp.to_standard_form(gen.generate(cid))
sol = hplp.Solver.box(*s.csr()) if box else hplp.Solver.from_std(s)
cfg = abi.Config.default(tolerance=1e-6, iteration_limit=10**9, infeasibility_check_period=0 if box else 100)
r0 = sol.solve(iteration_limit=0)
hx = sol.hx
hx.setup(cfg, r0["sigma_estimate"], r0["eta"])
hx.run(500)
hx.phase_profile(reset=True)
p = hx.run(2000)
prof = hx.phase_profile(reset=True)
print(f"configs[{cid}]{' box' if box else ''}: {2000 / (p.device_ms / 1e3):.0f} it/s "
      f"({p.device_ms / 2:.2f} us per iteration)")
tot = 0.0
for k, v in prof.items():
    print(f"  {k:13s} mean {v['mean_us']:6.2f}  max {v['max_us']:6.2f}  min {v['min_us']:6.2f} us/iter")
sol.close()
