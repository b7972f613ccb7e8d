// Row partition of the rHPDHG problem across P GPUs.
//
// Rank p owns a contiguous block of rows of A (dual variables y, A x, b) and a
// contiguous block of rows of A^T (primal variables x, c), each balanced by
// cost = nnz + kRowCost * rows so skewed (Zipf) matrices split evenly.  Per
// iteration the ranks all-gather the y slices before A^T y and the x+ slices
// before A x+, and all-gather their ~7 partial sums, which every rank reduces
// in rank order -- bit-identical totals, so the replicated controller takes
// identical decisions on every rank (the same scheme the device uses across
// CTAs).  Host C++; exported through include/hplp_gpu.h.
#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "hplp_gpu.h"

namespace {

constexpr double kRowCost = 3.0;

// Contiguous cut of rows [0, rows) into parts of about equal cost; bounds has
// parts + 1 entries.
void cut(const int64_t* ptr, int64_t rows, int32_t parts, int64_t* bounds) {
  const double total = static_cast<double>(ptr[rows]) + kRowCost * static_cast<double>(rows);
  bounds[0] = 0;
  int64_t r = 0;
  for (int32_t p = 1; p < parts; ++p) {
    const double target = total * p / parts;
    while (r < rows && static_cast<double>(ptr[r + 1]) + kRowCost * static_cast<double>(r + 1) <= target) ++r;
    // take the row that straddles the target if that lands closer
    if (r < rows) {
      const double before = static_cast<double>(ptr[r]) + kRowCost * r;
      const double after = static_cast<double>(ptr[r + 1]) + kRowCost * (r + 1);
      if (after - target < target - before) ++r;
    }
    bounds[p] = std::max(bounds[p - 1], r);
  }
  bounds[parts] = rows;
}

}  // namespace

extern "C" int hplp_plan_partition(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                                   int32_t parts, int64_t* row_bounds, int64_t* col_bounds) {
  if (parts < 1 || m < 0 || n < 0) return HPLP_EINVAL;
  try {
    cut(row_ptr, m, parts, row_bounds);
    std::vector<int64_t> col_ptr(static_cast<std::size_t>(n) + 1, 0);
    for (int64_t p = 0; p < row_ptr[m]; ++p) {
      if (col_idx[p] < 0 || col_idx[p] >= n) return HPLP_EINVAL;
      ++col_ptr[static_cast<std::size_t>(col_idx[p]) + 1];
    }
    for (int64_t j = 0; j < n; ++j) col_ptr[j + 1] += col_ptr[j];
    cut(col_ptr.data(), n, parts, col_bounds);
  } catch (const std::exception&) {
    return HPLP_ENOMEM;
  }
  return HPLP_OK;
}
