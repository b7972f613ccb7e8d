"""Quality of preconditioned solves on the ORIGINAL LP: the loop's tolerance
is checked on the scaled instance, so evaluate the returned (unscaled)
iterate's relative KKT error on the unscaled problem (hx_kkt_current) and its
objective against the planted optimum."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

g = gen.generate(1)
s = hplp.to_standard_form(g)
plain = hplp.Solver.from_std(s)
r0 = plain.solve(iteration_limit=0)
for ruiz, alpha in ((0, -1.0), (10, 1.0), (0, 1.0), (0, 0.5), (10, 0.5)):
    r = hplp.solve(*s.csr(), tolerance=1e-4, time_limit_seconds=60, precondition_ruiz_iters=ruiz,
                   precondition_pc_alpha=alpha)
    plain.hx.setup(abi.Config.default(), r0["sigma_estimate"], r0["eta"], r["x"], r["y"])
    k = plain.hx.kkt_current()
    _, obj = s.recover(r["x"])
    rel = abs(obj - g.planted_objective) / abs(g.planted_objective)
    print(f"ruiz={ruiz:2d} pc={alpha:4.1f}: {r['status']} it={r['iterations']:7d} {r['wall_seconds']:.2f}s | scaled KKT "
          f"{r['kkt'][3]:.2e} | original KKT max {k[3]:.2e} (p {k[0]:.1e} d {k[1]:.1e} g {k[2]:.1e}) | objective rel err "
          f"{rel:.1e}", flush=True)
