"""Emulated team rates on ONE device (ranks = CTA groups of one launch):
the protocol's overhead (pushes to every rank's buffers, two-level team
barrier) against the single-context loop.  Not a multi-GPU number."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

s = hplp.to_standard_form(gen.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 1))
cfg = abi.Config.default(tolerance=1e-4, iteration_limit=10**9)
for nr in (1, 2, 4):
    t = hplp.Solver.team(*s.csr(), nranks=nr) if nr > 1 else hplp.Solver.from_std(s)
    r0 = t.solve(iteration_limit=0)
    hxs = [t.rank_hx(q) for q in range(nr)]
    for h in hxs:
        h.setup(cfg, r0["sigma_estimate"], r0["eta"])
    best = 1e30
    for _ in range(5):
        p = hplp.team_run(hxs, 1000) if nr > 1 else [hxs[0].run(1000)]
        best = min(best, p[0].device_ms)
    print(f"ranks {nr}: {1e6 / best:8.0f} it/s (one device: {148 // nr} CTAs per rank)", flush=True)
    t.close()
