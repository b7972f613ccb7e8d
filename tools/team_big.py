"""Team path at configs[4] scale on ONE device (2 emulated ranks): upload
(partition, masks), 50 iterations, agreement with the single-context solve."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2407_16144_b200 import gen, hplp  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = hplp.to_standard_form(gen.generate(cid))
print(f"configs[{cid}]: {s.m} x {s.n}, nnz {s.nnz}", flush=True)
t0 = time.time()
t = hplp.Solver.team(*s.csr(), nranks=2)
print(f"team create {time.time() - t0:.1f}s", flush=True)
t0 = time.time()
rt = t.solve(iteration_limit=40, tolerance=1e-12, trace=True, trace_period=10)
print(f"team solve {time.time() - t0:.1f}s ({rt['iterations']} its)", flush=True)
t.close()
r1 = hplp.solve(*s.csr(), iteration_limit=40, tolerance=1e-12, trace=True, trace_period=10)
for a, b in zip(rt["trace"], r1["trace"]):
    za, zb = np.concatenate([a["x"], a["y"]]), np.concatenate([b["x"], b["y"]])
    print(f"it {a['iteration']} (n,k)=({a['epoch']},{a['inner']}) vs ({b['epoch']},{b['inner']}): max|z| {np.max(np.abs(zb)):.3e} "
          f"rel diff {np.max(np.abs(za - zb)) / max(np.max(np.abs(zb)), 1e-300):.2e} kkt {a['kkt'][3]:.6e} {b['kkt'][3]:.6e}",
          flush=True)
print("epochs", [e[:2] for e in rt["epochs"]], [e[:2] for e in r1["epochs"]])
