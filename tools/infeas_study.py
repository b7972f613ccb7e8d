"""configs[2] (primal infeasible): iterations to a valid Farkas certificate
under different stall caps / preconditioning (time-boxed)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import gen, hplp  # noqa: E402

cid = 2
g = gen.generate(cid)
s = hplp.to_standard_form(g)
print(f"configs[2]: std {s.m} x {s.n}, nnz {s.nnz}", flush=True)
runs = [dict(), dict(adaptive_stall_cap=0), dict(adaptive_stall_cap=20000),
        dict(precondition_ruiz_iters=10, precondition_pc_alpha=1.0, adaptive_stall_cap=0),
        dict(precondition_ruiz_iters=10, precondition_pc_alpha=1.0)]
for kw in runs:
    t0 = time.time()
    r = hplp.solve(*s.csr(), tolerance=1e-4, iteration_limit=3_000_000, time_limit_seconds=100, **kw)
    pc = r["primal_cert"][1] if r["primal_cert"] else None
    print(f"{kw}: {r['status']} it={r['iterations']} epochs={r['n_epochs']} t={time.time() - t0:.1f}s cert={pc}", flush=True)
