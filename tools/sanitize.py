"""Small solves touching every device code path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):
  compute-sanitizer --tool memcheck python tools/sanitize.py
Standard loop with certificate scans and restarts, traces, the box form, the
three baseline schemes, a two-rank team emulated on one device,
preconditioning, an infeasible LP (certificate readback)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

g = gen.generate(gen.scaled(0, m=200, n=400, nnz_per_row=8))
s = hplp.to_standard_form(g)
args = s.csr()
r = hplp.solve(*args, iteration_limit=250, tolerance=1e-12)
print("loop", r["status"], r["iterations"], flush=True)
r = hplp.solve(*args, iteration_limit=30, tolerance=1e-12, trace=True, trace_period=10)
print("trace", len(r["trace"]), flush=True)
r = hplp.solve(*args, iteration_limit=120, tolerance=1e-12, precondition_ruiz_iters=2, precondition_pc_alpha=1.0)
print("precondition", r["status"], flush=True)
b = hplp.Solver.box(*args)
r = b.solve(iteration_limit=120, tolerance=1e-12)
b.close()
print("box", r["status"], flush=True)
for scheme in (abi.SCHEME_VANILLA, abi.SCHEME_AVERAGED, abi.SCHEME_RESTARTED_AVERAGE):
    r = hplp.solve(*args, iteration_limit=120, tolerance=1e-12, scheme=scheme)
    print("scheme", scheme, r["status"], flush=True)
t = hplp.Solver.team(*args, nranks=2)
r = t.solve(iteration_limit=150, tolerance=1e-12)
t.close()
print("team", r["status"], flush=True)
inf = hplp.solve(2, 1, [0, 1, 2], [0, 0], [1.0, 1.0], [1.0, 2.0], [0.0])
print("infeasible", inf["status"], flush=True)
print("sanitize done", flush=True)
