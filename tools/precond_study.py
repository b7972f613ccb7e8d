"""KKT after N iterations with / without preconditioning (convergence study)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import gen, hplp  # noqa: E402
from tests.helpers import problem  # noqa: E402

for name in sys.argv[1:]:
    g = gen.generate(int(name[3:])) if name.startswith("cfg") and name[3:].isdigit() else problem(name)
    s = hplp.to_standard_form(g)
    for ruiz, alpha in ((0, -1.0), (10, -1.0), (10, 1.0), (0, 1.0)):
        for its in (20000, 100000):
            r = hplp.solve(*s.csr(), tolerance=1e-4, iteration_limit=its, precondition_ruiz_iters=ruiz,
                           precondition_pc_alpha=alpha)
            _, obj = s.recover(r["x"])
            print(f"{name:14s} ruiz={ruiz:2d} pc={alpha:4.1f} its={its:6d}: {r['status']:17s} it={r['iterations']:6d} "
                  f"kkt={r['kkt'][3]:.2e} (p {r['kkt'][0]:.1e} d {r['kkt'][1]:.1e} g {r['kkt'][2]:.1e}) "
                  f"obj={obj:.6g} planted={g.planted_objective:.6g} {r['wall_seconds']:.1f}s", flush=True)
