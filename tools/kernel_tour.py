"""Run every hx kernel at least once on configs[1] (for the per-kernel ncu
table in profiles/): upload (validation, A^T build), preconditioning, power
iteration, setup SpMV, the rHPDHG loop with certificate scans, result
readback (combine, certificate, fresh KKT), trace diagnostics, the three
baseline schemes, and a two-rank team emulated on one device."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

s = hplp.to_standard_form(gen.generate(1))
sol = hplp.Solver.from_std(s)
sol.solve(iteration_limit=300, tolerance=1e-12, precondition_ruiz_iters=2, precondition_pc_alpha=1.0)
sol.solve(iteration_limit=40, tolerance=1e-12, precondition_ruiz_iters=2, precondition_pc_alpha=1.0, trace=True,
          trace_period=20)
hx = sol.hx
hx.kkt_current()
hx.get_iterate(hplp.ITERATE_CURRENT)
for scheme in (abi.SCHEME_VANILLA, abi.SCHEME_AVERAGED, abi.SCHEME_RESTARTED_AVERAGE):
    sol.solve(iteration_limit=100, tolerance=1e-12, precondition_ruiz_iters=2, precondition_pc_alpha=1.0,
              scheme=scheme)
sol.close()
inf = hplp.solve(2, 1, [0, 1, 2], [0, 0], [1.0, 1.0], [1.0, 2.0], [0.0])  # certificate readback (cert_kernel)
assert inf["status"] == "primal_infeasible"
t = hplp.Solver.team(*s.csr(), nranks=2)
t.solve(iteration_limit=200, tolerance=1e-12)
t.close()
print("tour done", flush=True)
