"""Emulated team rates on ONE device (ranks = CTA groups of one launch):
the protocol's overhead (pushes to every rank's buffers, two-level team
barrier) against the single-context loop.  Not a multi-GPU number."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

s = hplp.to_standard_form(gen.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 1))
cfg = abi.Config.default(tolerance=1e-4, iteration_limit=10**9)
ranks = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4]
iters = 1000 if s.nnz < 50_000_000 else 50
for nr in ranks:
    t = hplp.Solver.team(*s.csr(), nranks=nr) if nr > 1 else hplp.Solver.from_std(s)
    r0 = t.solve(iteration_limit=0)
    hxs = [t.rank_hx(q) for q in range(nr)]
    for h in hxs:
        h.setup(cfg, r0["sigma_estimate"], r0["eta"])
    best = 1e30
    for _ in range(3):
        p = hplp.team_run(hxs, iters) if nr > 1 else [hxs[0].run(iters)]
        best = min(best, p[0].device_ms)
    stored = [h.stored_nonzeros() for h in hxs]
    print(f"ranks {nr}: {iters * 1e3 / best:8.1f} it/s (one device: {148 // nr} CTAs per rank; "
          f"nonzeros stored per rank (A, A^T): {stored[0]} .. {stored[-1]})", flush=True)
    t.close()
