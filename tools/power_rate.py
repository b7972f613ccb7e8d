"""Device time per power iteration (hx_power_iteration, kModePower inside the
loop kernel) against one loop iteration, configs[1].  python tools/power_rate.py [cfg]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
s = hplp.to_standard_form(gen.generate(cid))
sol = hplp.Solver.from_std(s)
hx = sol.hx
stream = torch.cuda.ExternalStream(hx.stream())
x0 = hplp.power_start(s.n)
for its in (10, 86, 200):
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sig, it, conv, _ = hx.power_iteration(x0, tol=0.0, max_iters=its)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"power iteration x{it}: {best:.3f} ms, {1e3 * best / it:.1f} us per iteration", flush=True)
r0 = sol.solve(iteration_limit=0)
hx.setup(abi.Config.default(tolerance=0.0, iteration_limit=10**9), r0["sigma_estimate"], r0["eta"])
hx.run(500)
print(f"loop: {1e3 * hx.run(2000).device_ms / 2000:.1f} us per iteration")
sol.close()
