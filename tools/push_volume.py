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

# Structure-aware ownership: original rows and columns in
# nnz-balanced contiguous blocks; each bound row x_j + s_j = u_j and its
# slack s_j with column j; each row slack with its row.  Pushes left: only
# what crosses between the original blocks.
col_nnz = np.diff(A.tocsc().indptr)
row_nnz = np.diff(A.indptr)
single = col_nnz == 1  # slack columns: one entry
Acoo = rows_of
slack_row = np.full(s.n, -1)
slack_row[Acoo.col[single[Acoo.col]]] = Acoo.row[single[Acoo.col]]
is_bound = np.zeros(s.m, bool)
bound_col = np.full(s.m, -1)
for i in np.nonzero(row_nnz == 2)[0]:
    cols = A.indices[A.indptr[i]:A.indptr[i + 1]]
    sl = cols[single[cols]]
    if len(sl) == 1:
        is_bound[i] = True
        bound_col[i] = cols[~single[cols]][0]


def blocks(weights, P):
    cum = np.cumsum(weights)
    return np.minimum((cum * P - 1) // max(cum[-1], 1), P - 1).astype(np.int64)


orig_rows = np.nonzero(~is_bound)[0]
orig_cols = np.nonzero(~single)[0]
for P in (2, 4, 8):
    rown = np.zeros(s.m, np.int64)
    coln = np.zeros(s.n, np.int64)
    rown[orig_rows] = blocks(row_nnz[orig_rows], P)
    coln[orig_cols] = blocks(col_nnz[orig_cols], P)
    rown[is_bound] = coln[bound_col[is_bound]]
    sl = np.nonzero(single)[0]
    coln[sl] = rown[slack_row[sl]]
    ro, co = rown[Acoo.row], coln[Acoo.col]
    x_pairs = np.unique(Acoo.col.astype(np.int64) * 8 + ro)
    x_need = np.count_nonzero((x_pairs % 8) != coln[x_pairs // 8])
    y_pairs = np.unique(Acoo.row.astype(np.int64) * 8 + co)
    y_need = np.count_nonzero((y_pairs % 8) != rown[y_pairs // 8])
    dense = (s.n + s.m) * (P - 1)
    lo, hi = np.bincount(ro, minlength=P), np.bincount(co, minlength=P)
    print(f"P={P} structure-aware: selective {(x_need + y_need) / 1e6:.2f} M ({(x_need + y_need) / dense:.1%} of dense);"
          f" per GPU received {8 * (x_need + y_need) / P / 1e6:.1f} MB; nnz per rank (rows of A) "
          f"{lo.min() / 1e6:.2f}-{lo.max() / 1e6:.2f} M")
