"""Dump a config's A and A^T as CSR binaries and run tools/spmv_micro."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2407_16144_b200 import gen, hplp  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = gen.generate(cfg)
s = hplp.to_standard_form(g)
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
import scipy.sparse as sp  # noqa: E402

A = sp.csr_matrix((s.val, s.col_idx, s.row_ptr), shape=(s.m, s.n))
for name, M in (("A", A), ("AT", A.T.tocsr())):
    M.sort_indices()
    p = out / f"cfg{cfg}_{name}.bin"
    with open(p, "wb") as f:
        np.array([M.shape[0], M.shape[1], M.nnz], np.int64).tofile(f)
        M.indptr.astype(np.int32).tofile(f)
        M.indices.astype(np.int32).tofile(f)
        M.data.astype(np.float64).tofile(f)
    print(f"== cfg{cfg} {name}: {M.shape} nnz={M.nnz}", flush=True)
    subprocess.run(["tools/spmv_micro", str(p)], check=True)
