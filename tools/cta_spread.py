"""Per-CTA phase times (HX_PROFILE=1): is the spread systematic per CTA (the
schedule) or per SM (hardware), or noise?  Compares two repetitions."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["HX_PROFILE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2407_16144_b200 import abi, gen, hplp  # noqa: E402

s = hplp.to_standard_form(gen.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 1))
solver = hplp.Solver.from_std(s)
r0 = solver.solve(iteration_limit=0)
hx = solver.hx
hx.setup(abi.Config.default(tolerance=1e-4, iteration_limit=10**9), r0["sigma_estimate"], r0["eta"])
g = hx.info()["grid"]
reps = []
for rep in range(3):
    buf = (C.c_uint64 * (g * 48))()
    hplp.lib().hx_profile(hx.h, buf, 1)
    hx.run(1000)
    buf = (C.c_uint64 * (g * 48))()
    hplp.lib().hx_profile(hx.h, buf, 1)
    a = np.array(buf[: g * 16], dtype=np.float64).reshape(g, 16)
    its = a[0, 5]
    k = 1.0 / its / 1965.0
    reps.append(dict(A=a[:, 0] * k + a[:, 4] * k, B=a[:, 2] * k, B1=a[:, 1] * k, B2=a[:, 3] * k, sm=a[:, 6].astype(int)))
for key in ("A", "B"):
    v = [r[key] for r in reps]
    print(f"{key}: per-CTA mean {v[0].mean():.2f} min {v[0].min():.2f} max {v[0].max():.2f} us; "
          f"corr by CTA rep0/rep1 {np.corrcoef(v[0], v[1])[0, 1]:.3f}, rep0/rep2 {np.corrcoef(v[0], v[2])[0, 1]:.3f}")
    o = np.argsort(v[0])
    print("   slowest (cta, sm, t0, t1):", [(int(i), int(reps[0]['sm'][i]), round(v[0][i], 2), round(v[1][i], 2)) for i in o[-8:]])
    print("   fastest (cta, sm, t0, t1):", [(int(i), int(reps[0]['sm'][i]), round(v[0][i], 2), round(v[1][i], 2)) for i in o[:8]])
print("smid same across reps:", all((r["sm"] == reps[0]["sm"]).all() for r in reps))
for key in ("B1", "B2"):
    print(key, "mean", round(reps[0][key].mean(), 2), "min", round(reps[0][key].min(), 2))
