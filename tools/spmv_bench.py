"""Calibration: hx SpMV engine vs cuSPARSE (torch CSR) on a config's A, A^T."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_16144_b200 import gen, hplp  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = gen.generate(cfg)
s = hplp.to_standard_form(g)
L = hplp.lib()
L.hx_bench_spmv.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
hx = hplp.HX()
hx.upload(*s.csr())
print("grid", hx.info())
for tr in (0, 1):
    ms = C.c_double()
    assert L.hx_bench_spmv(hx.h, tr, 50, C.byref(ms)) == 0
    rows = s.n if tr else s.m
    by = 12 * s.nnz + 4 * rows + 8 * rows + 8 * (s.m if tr else s.n)
    print(f"hx  {'A^T y' if tr else 'A x  '}: {ms.value*1e3:8.2f} us  ({by/ms.value/1e6:7.1f} GB/s min-traffic)")
A = torch.sparse_csr_tensor(torch.tensor(s.row_ptr), torch.tensor(s.col_idx.astype(np.int64)), torch.tensor(s.val),
                            size=(s.m, s.n), device="cuda")
AT = A.t().to_sparse_csr()
x = torch.randn(s.n, 1, dtype=torch.float64, device="cuda")
y = torch.randn(s.m, 1, dtype=torch.float64, device="cuda")
for name, M, v in (("A x  ", A, x), ("A^T y", AT, y)):
    for _ in range(3):
        M @ v
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        M @ v
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / 50
    print(f"cuSPARSE {name}: {t*1e3:8.2f} us")
