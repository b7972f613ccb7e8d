"""Box form vs standard form on the GPU: iterations and seconds to relative
KKT 1e-4 (each form's own KKT), objective of the standard-form solution, with
and without preconditioning.  python tools/box_study.py [names...]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import gen, hplp  # noqa: E402
from tests.helpers import problem  # noqa: E402

names = sys.argv[1:] or ["cfg0", "cfg1_small", "zipf_small", "configs1"]
for name in names:
    g = gen.generate(1) if name == "configs1" else problem(name)
    s = hplp.to_standard_form(g)
    args = (s.m, s.n, s.row_ptr, s.col_idx, s.val, s.b, s.c)
    for pre in ({}, {"precondition_ruiz_iters": 0, "precondition_pc_alpha": 0.5},
                {"precondition_ruiz_iters": 10, "precondition_pc_alpha": 1.0}):
        for form in ("standard", "box"):
            sol = hplp.Solver.box(*args) if form == "box" else hplp.Solver(*args)
            t0 = time.perf_counter()
            r = sol.solve(tolerance=1e-4, iteration_limit=2_000_000, time_limit_seconds=60.0, **pre)
            dt = time.perf_counter() - t0
            sol.close()
            print(f"{name:12s} {form:8s} pre={pre or '-'}: {r['status']:15s} its {r['iterations']:8d} "
                  f"{dt:7.2f}s  obj {float(s.c @ r['x']):.8e} (planted {g.planted_objective:.8e}) "
                  f"kkt {r['kkt'][3]:.2e}", flush=True)
