"""Time to 1e-4 / to a certificate for preconditioning variants (configs[1], configs[2])."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import gen, hplp  # noqa: E402

for cid in (1, 2):
    s = hplp.to_standard_form(gen.generate(cid))
    for ruiz, alpha in ((0, 1.0), (10, 1.0), (4, 1.0), (0, 0.5)):
        kw = dict(adaptive_stall_cap=0, iteration_limit=2_000_000) if cid == 2 else {}
        t0 = time.time()
        r = hplp.solve(*s.csr(), tolerance=1e-4, time_limit_seconds=60, precondition_ruiz_iters=ruiz,
                       precondition_pc_alpha=alpha, **kw)
        cert = r["primal_cert"][1]["residual"] if r["primal_cert"] else None
        print(f"cfg{cid} ruiz={ruiz} pc={alpha}: {r['status']} it={r['iterations']} t={time.time() - t0:.1f}s "
              f"cert_res={cert}", flush=True)
