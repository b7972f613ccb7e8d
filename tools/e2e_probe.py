"""Where the end-to-end solve time goes (create / solve / free), repeated."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import gen, hplp  # noqa: E402

s = hplp.to_standard_form(gen.generate(1))
args = s.csr()
for rep in range(8):
    t0 = time.perf_counter()
    sol = hplp.Solver(*args)
    t1 = time.perf_counter()
    r = sol.solve(iteration_limit=5000, tolerance=1e-4)
    t2 = time.perf_counter()
    sol.close()
    t3 = time.perf_counter()
    r2 = hplp.solve(*args, iteration_limit=5000, tolerance=1e-4)
    t4 = time.perf_counter()
    print(f"create {t1-t0:.3f}s solve {t2-t1:.3f}s close {t3-t2:.3f}s | one-shot hplp.solve {t4-t3:.3f}s", flush=True)
