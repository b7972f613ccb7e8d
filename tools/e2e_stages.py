"""Stage times of the bench's end-to-end call (hplp_solve_csr from pinned host
buffers, configs[1], 5000 iterations) with HPLP_TIMING=1 (printed on stderr by
the C++ driver and hx_upload_csr).  python tools/e2e_stages.py [config] [iterations]"""
import os
import sys
import time
from pathlib import Path

os.environ["HPLP_TIMING"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_16144_b200 import gen, hplp  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
its = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
s = hplp.to_standard_form(gen.generate(cid))
rp, ci, v, b, c = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
                   for a in (s.row_ptr, s.col_idx, s.val, s.b, s.c))
for rep in range(int(os.environ.get("E2E_REPS", "2"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = hplp.solve(s.m, s.n, rp, ci, v, b, c, iteration_limit=its, tolerance=1e-4)
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {dt * 1e3:.1f} ms, {its / dt:.0f} it/s end to end", file=sys.stderr, flush=True)
