"""Elements pushed between ranks per rHPDHG iteration for a row partition
(hplp_plan_partition): every owned x+ / y-combo element to every peer (dense)
vs only to the peers that gather it (the xneed / yneed masks)."""
import sys
from pathlib import Path

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_16144_b200 import gen, hplp  # noqa: E402

s = hplp.to_standard_form(gen.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 1))
A = sp.csr_matrix((s.val, s.col_idx, s.row_ptr), shape=(s.m, s.n))
rows_of = A.tocoo()
for P in (2, 4, 8):
    rb, cb = hplp.plan_partition(s.m, s.n, s.row_ptr, s.col_idx, P)
    ro = np.searchsorted(rb, rows_of.row, side="right") - 1  # owner of each entry's row
    co = np.searchsorted(cb, rows_of.col, side="right") - 1  # owner of its column
    # x+_j goes to the owners of the rows in column j (other than its own);
    # y_i to the owners of the columns in row i
    x_pairs = np.unique(rows_of.col.astype(np.int64) * 8 + ro)
    x_need = np.count_nonzero((x_pairs % 8) != (np.searchsorted(cb, x_pairs // 8, side="right") - 1))
    y_pairs = np.unique(rows_of.row.astype(np.int64) * 8 + co)
    y_need = np.count_nonzero((y_pairs % 8) != (np.searchsorted(rb, y_pairs // 8, side="right") - 1))
    dense = (s.n + s.m) * (P - 1)
    print(f"P={P}: dense {dense / 1e6:.2f} M elements/iteration, selective {(x_need + y_need) / 1e6:.2f} M "
          f"({(x_need + y_need) / dense:.1%}); per GPU received {8 * (x_need + y_need) / P / 1e6:.1f} MB")
