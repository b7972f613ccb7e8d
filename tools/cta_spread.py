"""Per-CTA phase time vs SM id (HX_PROFILE=1): is the CTA spread hardware?"""
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
for rep in range(2):
    buf = (C.c_uint64 * (g * 16))()
    hplp.lib().hx_profile(hx.h, buf, 1)
    hx.run(500)
    buf = (C.c_uint64 * (g * 16))()
    hplp.lib().hx_profile(hx.h, buf, 1)
    a = np.array(buf[:], dtype=np.float64).reshape(g, 16)
    its = a[0, 5]
    pa, pb = a[:, 0] / its / 1e3, a[:, 2] / its / 1e3
    sm = a[:, 6].astype(int)
    order = np.argsort(pa + pb)
    print(f"rep {rep}: phaseA+B per CTA: min {np.min(pa+pb):.1f} med {np.median(pa+pb):.1f} max {np.max(pa+pb):.1f} us")
    print("  slowest 12 (cta, sm, A, B):", [(int(i), int(sm[i]), round(pa[i], 1), round(pb[i], 1)) for i in order[-12:]])
    print("  fastest 6 (cta, sm, A, B):", [(int(i), int(sm[i]), round(pa[i], 1), round(pb[i], 1)) for i in order[:6]])
    # same-SM pairs: correlation of the two CTAs on one SM
    bysm = {}
    for i in range(g):
        bysm.setdefault(sm[i], []).append(pa[i] + pb[i])
    pairs = np.array([v for v in bysm.values() if len(v) == 2])
    if len(pairs):
        print(f"  corr between the 2 CTAs sharing an SM: {np.corrcoef(pairs[:, 0], pairs[:, 1])[0, 1]:.3f}")
    cta_idx = np.arange(g)
    print(f"  corr(time, cta index): {np.corrcoef(cta_idx, pa + pb)[0, 1]:.3f}; corr(time, smid): {np.corrcoef(sm, pa + pb)[0, 1]:.3f}")
