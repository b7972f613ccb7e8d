"""Preconditioning settings for the box form vs the standard form on one
config: seconds / iterations to 1e-4 and the objective's distance to the
planted optimum.  python tools/box_precond_sweep.py [config]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import gen, hplp  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = gen.generate(cid)
s = hplp.to_standard_form(g)
args = s.csr()
for ruiz in (0, 3, 10):
    for alpha in (0.0, 0.3, 0.5, 0.7, 1.0):
        row = []
        for form in ("standard", "box"):
            t0 = time.perf_counter()
            sol = hplp.Solver.box(*args) if form == "box" else hplp.Solver(*args)
            r = sol.solve(tolerance=1e-4, iteration_limit=3_000_000, time_limit_seconds=20.0,
                          precondition_ruiz_iters=ruiz, precondition_pc_alpha=alpha)
            sol.close()
            dt = time.perf_counter() - t0
            _, obj = s.recover(r["x"])
            rel = abs(obj - g.planted_objective) / abs(g.planted_objective)
            row.append(f"{form} {r['status'][:8]:8s} {r['iterations']:8d} its {dt:6.2f}s objerr {rel:.1e}")
        print(f"ruiz {ruiz:2d} alpha {alpha:.1f}: " + " | ".join(row), flush=True)
