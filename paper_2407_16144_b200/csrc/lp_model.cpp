// Host-side problem model of the B200 solver: SparseMatrix (CSR), the
// StandardFormLP checks, and to_standard_form.  A new implementation that
// builds the standard-form CSR directly (no global triplet sort) while
// reproducing the reference's output exactly: the same row order
// [original rows, bound rows], column order [original columns (split ones
// take two), row slacks, bound slacks] and the same b-shift summation order
// (src/lp_model.cpp:155-325), so iterates stay comparable bit for bit.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>

#include "hplp_gpu.hpp"

namespace hplp_gpu {

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();

// Sort each row's (col, value) pairs by column if needed; throw on duplicates.
void sort_rows(Index m, const std::vector<int64_t>& rp, std::vector<int32_t>& ci, std::vector<double>& v,
               const char* who) {
  std::vector<std::pair<int32_t, double>> row;
  for (Index i = 0; i < m; ++i) {
    const int64_t p0 = rp[i], p1 = rp[i + 1];
    bool sorted = true;
    for (int64_t p = p0 + 1; p < p1; ++p) {
      if (ci[p] < ci[p - 1]) sorted = false;
      if (ci[p] == ci[p - 1])
        throw std::invalid_argument(std::string(who) + ": duplicate entry at (" + std::to_string(i) + ", " +
                                    std::to_string(ci[p]) + ")");
    }
    if (sorted) continue;
    row.clear();
    for (int64_t p = p0; p < p1; ++p) row.push_back({ci[p], v[p]});
    std::stable_sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (std::size_t q = 0; q < row.size(); ++q) {
      if (q && row[q].first == row[q - 1].first)
        throw std::invalid_argument(std::string(who) + ": duplicate entry at (" + std::to_string(i) + ", " +
                                    std::to_string(row[q].first) + ")");
      ci[p0 + static_cast<int64_t>(q)] = row[q].first;
      v[p0 + static_cast<int64_t>(q)] = row[q].second;
    }
  }
}
}  // namespace

// src/sparse_matrix.cpp:24-66
SparseMatrix::SparseMatrix(Index n_rows, Index n_cols, const std::vector<Triplet>& entries)
    : rows_(n_rows), cols_(n_cols) {
  if (n_rows < 0 || n_cols < 0) throw std::invalid_argument("SparseMatrix: negative dimension");
  if (n_cols > std::numeric_limits<int32_t>::max())
    throw std::invalid_argument("SparseMatrix: column count exceeds the int32 index range");
  for (const Triplet& t : entries) {
    if (t.row < 0 || t.row >= n_rows || t.col < 0 || t.col >= n_cols)
      throw std::invalid_argument("SparseMatrix: entry (" + std::to_string(t.row) + ", " + std::to_string(t.col) +
                                  ") out of range for " + std::to_string(n_rows) + "x" + std::to_string(n_cols));
    if (!std::isfinite(t.value))
      throw std::invalid_argument("SparseMatrix: non-finite value at (" + std::to_string(t.row) + ", " +
                                  std::to_string(t.col) + ")");
  }
  row_ptr_.assign(static_cast<std::size_t>(n_rows) + 1, 0);
  for (const Triplet& t : entries) ++row_ptr_[static_cast<std::size_t>(t.row) + 1];
  for (Index i = 0; i < n_rows; ++i) row_ptr_[i + 1] += row_ptr_[i];
  col_idx_.resize(entries.size());
  val_.resize(entries.size());
  std::vector<int64_t> fill(row_ptr_.begin(), row_ptr_.end() - 1);
  for (const Triplet& t : entries) {
    const int64_t p = fill[t.row]++;
    col_idx_[p] = static_cast<int32_t>(t.col);
    val_[p] = t.value;
  }
  sort_rows(n_rows, row_ptr_, col_idx_, val_, "SparseMatrix");
}

SparseMatrix SparseMatrix::from_csr(Index n_rows, Index n_cols, const int64_t* row_ptr, const int32_t* col_idx,
                                    const double* val) {
  if (n_rows < 0 || n_cols < 0) throw std::invalid_argument("SparseMatrix: negative dimension");
  SparseMatrix a;
  a.rows_ = n_rows;
  a.cols_ = n_cols;
  if (row_ptr[0] != 0) throw std::invalid_argument("SparseMatrix: row_ptr[0] must be 0");
  for (Index i = 0; i < n_rows; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) throw std::invalid_argument("SparseMatrix: row_ptr not monotone");
  const int64_t nnz = row_ptr[n_rows];
  a.row_ptr_.assign(row_ptr, row_ptr + n_rows + 1);
  a.col_idx_.assign(col_idx, col_idx + nnz);
  a.val_.assign(val, val + nnz);
  for (Index i = 0; i < n_rows; ++i)
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      if (col_idx[p] < 0 || col_idx[p] >= n_cols)
        throw std::invalid_argument("SparseMatrix: entry (" + std::to_string(i) + ", " + std::to_string(col_idx[p]) +
                                    ") out of range for " + std::to_string(n_rows) + "x" + std::to_string(n_cols));
      if (!std::isfinite(val[p]))
        throw std::invalid_argument("SparseMatrix: non-finite value at (" + std::to_string(i) + ", " +
                                    std::to_string(col_idx[p]) + ")");
    }
  sort_rows(n_rows, a.row_ptr_, a.col_idx_, a.val_, "SparseMatrix");
  return a;
}

std::vector<Triplet> SparseMatrix::triplets_row_order() const {
  std::vector<Triplet> out;
  out.reserve(val_.size());
  for (Index i = 0; i < rows_; ++i)
    for (int64_t p = row_ptr_[i]; p < row_ptr_[i + 1]; ++p) out.push_back({i, col_idx_[p], val_[p]});
  return out;
}

// src/lp_model.cpp:35-43
StandardFormLP::StandardFormLP(SparseMatrix a_in, Vector b_in, Vector c_in)
    : a(std::move(a_in)), b(std::move(b_in)), c(std::move(c_in)) {
  if (static_cast<Index>(b.size()) != a.rows() || static_cast<Index>(c.size()) != a.cols())
    throw std::invalid_argument("StandardFormLP: inconsistent dimensions");
  for (double v : b)
    if (!std::isfinite(v)) throw std::invalid_argument("StandardFormLP: non-finite b or c");
  for (double v : c)
    if (!std::isfinite(v)) throw std::invalid_argument("StandardFormLP: non-finite b or c");
}

// src/lp_model.cpp:65-85
Vector VariableMap::recover_primal(const Vector& x_std) const {
  if (static_cast<Index>(x_std.size()) != standard_cols)
    throw std::invalid_argument("recover_primal: wrong standard-form length");
  Vector x(recoveries.size());
  for (std::size_t j = 0; j < recoveries.size(); ++j) {
    const VariableRecovery& r = recoveries[j];
    switch (r.kind) {
      case VariableRecovery::Kind::kShifted:
        x[j] = r.offset + x_std[r.col];
        break;
      case VariableRecovery::Kind::kMirrored:
        x[j] = r.offset - x_std[r.col];
        break;
      case VariableRecovery::Kind::kSplit:
        x[j] = x_std[r.col] - x_std[r.neg_col];
        break;
    }
  }
  return x;
}

namespace {

// Rows of the general form as CSR in entry order (a view for both inputs).
struct RowsView {
  Index m = 0, n = 0;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
};

struct ColumnInfo {
  double lower, upper, obj;
};

struct RowInfo {
  int relation;  // HPLP_ROW_*
  double rhs;
  bool has_range;
  double range;
  std::string name;
};

std::pair<StandardFormLP, VariableMap> convert(const RowsView& A, const std::vector<RowInfo>& rows,
                                               const std::vector<ColumnInfo>& cols,
                                               const std::vector<std::string>* col_names, bool maximize,
                                               double objective_constant) {
  const Index m = A.m, n = A.n;
  auto col_name = [&](Index j) { return col_names ? (*col_names)[j] : "c" + std::to_string(j); };
  // validate_general_form, src/lp_model.cpp:96-134
  for (Index j = 0; j < n; ++j) {
    const ColumnInfo& c = cols[j];
    if (std::isnan(c.lower) || std::isnan(c.upper) || !std::isfinite(c.obj))
      throw std::invalid_argument("GeneralFormLP: non-finite data for column '" + col_name(j) + "'");
    if (c.lower > c.upper)
      throw std::invalid_argument("GeneralFormLP: inconsistent bounds for '" + col_name(j) + "' (lower > upper)");
  }
  for (const RowInfo& r : rows)
    if (!std::isfinite(r.rhs) || (r.has_range && !std::isfinite(r.range)))
      throw std::invalid_argument("GeneralFormLP: non-finite rhs/range for row '" + r.name + "'");
  for (int64_t p = 0; p < A.rp[m]; ++p) {
    if (A.ci[p] < 0 || A.ci[p] >= n) throw std::invalid_argument("GeneralFormLP: entry index out of range");
    if (!std::isfinite(A.v[p])) throw std::invalid_argument("GeneralFormLP: non-finite matrix entry");
  }
  {
    std::vector<int32_t> tmp;
    for (Index i = 0; i < m; ++i) {
      tmp.assign(A.ci.begin() + A.rp[i], A.ci.begin() + A.rp[i + 1]);
      std::sort(tmp.begin(), tmp.end());
      if (std::adjacent_find(tmp.begin(), tmp.end()) != tmp.end())
        throw std::invalid_argument("GeneralFormLP: duplicate matrix entry");
    }
  }
  const double sense = maximize ? -1.0 : 1.0;
  VariableMap map;
  map.objective_sign = sense;
  map.recoveries.resize(static_cast<std::size_t>(n));
  map.row_conversions.resize(static_cast<std::size_t>(m));

  // Stage 1 (src/lp_model.cpp:175-199): row intervals (row_interval :139-151),
  // slack items appended after the original columns in row order.
  struct Work {
    double lower, upper, obj;
  };
  std::vector<Work> work(static_cast<std::size_t>(n));
  for (Index j = 0; j < n; ++j) work[j] = {cols[j].lower, cols[j].upper, sense * cols[j].obj};
  Vector row_b(static_cast<std::size_t>(m), 0.0);
  std::vector<Index> slack_item(static_cast<std::size_t>(m), -1);
  for (Index i = 0; i < m; ++i) {
    const RowInfo& r = rows[i];
    double lo, hi;
    switch (r.relation) {
      case HPLP_ROW_LE:
        lo = r.has_range ? r.rhs - std::abs(r.range) : -kInf;
        hi = r.rhs;
        break;
      case HPLP_ROW_GE:
        lo = r.rhs;
        hi = r.has_range ? r.rhs + std::abs(r.range) : kInf;
        break;
      default:
        if (!r.has_range) lo = hi = r.rhs;
        else if (r.range >= 0) lo = r.rhs, hi = r.rhs + r.range;
        else lo = r.rhs + r.range, hi = r.rhs;
    }
    RowConversion& conv = map.row_conversions[i];
    conv.lower = lo;
    conv.upper = hi;
    if (lo == hi) {
      row_b[i] = lo;
    } else if (hi < kInf) {
      row_b[i] = hi;
      conv.slack_sign = 1.0;
      slack_item[i] = static_cast<Index>(work.size());
      work.push_back({0.0, lo > -kInf ? hi - lo : kInf, 0.0});
    } else {
      row_b[i] = lo;
      conv.slack_sign = -1.0;
      slack_item[i] = static_cast<Index>(work.size());
      work.push_back({0.0, kInf, 0.0});
    }
  }
  // Stage 2 (:201-253): shift / mirror / split, columns numbered in work order.
  enum : uint8_t { kShift, kMirror, kSplit };
  std::vector<uint8_t> kind(work.size());
  std::vector<int64_t> tcol(work.size()), tneg(work.size(), 0);
  std::vector<double> toff(work.size(), 0.0);
  Vector c_std;
  c_std.reserve(work.size() * 2);
  double shift_const = 0.0;
  std::vector<std::pair<int64_t, double>> pending;  // (column, rhs) of bound rows
  int64_t next_col = 0;
  for (std::size_t w = 0; w < work.size(); ++w) {
    const Work& wc = work[w];
    if (wc.lower == -kInf && wc.upper == kInf) {
      kind[w] = kSplit;
      tcol[w] = next_col++;
      tneg[w] = next_col++;
      c_std.push_back(wc.obj);
      c_std.push_back(-wc.obj);
    } else if (wc.lower > -kInf) {
      kind[w] = kShift;
      tcol[w] = next_col++;
      toff[w] = wc.lower;
      c_std.push_back(wc.obj);
      shift_const += wc.obj * wc.lower;
      if (wc.upper < kInf) pending.push_back({tcol[w], wc.upper - wc.lower});
    } else {
      kind[w] = kMirror;
      tcol[w] = next_col++;
      toff[w] = wc.upper;
      c_std.push_back(-wc.obj);
      shift_const += wc.obj * wc.upper;
    }
  }
  const Index m_std = m + static_cast<Index>(pending.size());
  map.bound_rows.reserve(pending.size());
  for (std::size_t t = 0; t < pending.size(); ++t) {
    map.bound_rows.push_back({m + static_cast<Index>(t), pending[t].first, next_col, pending[t].second});
    ++next_col;
    c_std.push_back(0.0);
  }
  const Index n_std = next_col;
  if (n_std > std::numeric_limits<int32_t>::max())
    throw std::invalid_argument("to_standard_form: standard form exceeds the int32 column range");
  for (Index j = 0; j < n; ++j) {
    VariableRecovery& rec = map.recoveries[j];
    rec.col = tcol[j];
    rec.neg_col = kind[j] == kSplit ? tneg[j] : 0;
    rec.offset = toff[j];
    rec.kind = kind[j] == kShift    ? VariableRecovery::Kind::kShifted
               : kind[j] == kMirror ? VariableRecovery::Kind::kMirrored
                                    : VariableRecovery::Kind::kSplit;
  }
  for (Index i = 0; i < m; ++i)
    if (slack_item[i] >= 0) map.row_conversions[i].slack_col = tcol[slack_item[i]];

  // Emission (:279-313), straight into CSR: row i = its transformed entries
  // in entry order, then its slack; bound rows = (column, slack).  b shifts
  // accumulate in entry order, as the reference's single pass over entries.
  std::vector<int64_t> rp(static_cast<std::size_t>(m_std) + 1, 0);
  for (Index i = 0; i < m; ++i) {
    int64_t len = slack_item[i] >= 0 ? 1 : 0;
    for (int64_t p = A.rp[i]; p < A.rp[i + 1]; ++p) len += kind[A.ci[p]] == kSplit ? 2 : 1;
    rp[i + 1] = rp[i] + len;
  }
  for (Index t = 0; t < static_cast<Index>(pending.size()); ++t) rp[m + t + 1] = rp[m + t] + 2;
  std::vector<int32_t> ci(static_cast<std::size_t>(rp[m_std]));
  std::vector<double> cv(ci.size());
  Vector b_std(static_cast<std::size_t>(m_std), 0.0);
  for (Index i = 0; i < m; ++i) {
    int64_t q = rp[i];
    b_std[i] = row_b[i];
    for (int64_t p = A.rp[i]; p < A.rp[i + 1]; ++p) {
      const int32_t j = A.ci[p];
      const double val = A.v[p];
      switch (kind[j]) {
        case kShift:
          ci[q] = static_cast<int32_t>(tcol[j]), cv[q++] = val;
          b_std[i] -= val * toff[j];
          break;
        case kMirror:
          ci[q] = static_cast<int32_t>(tcol[j]), cv[q++] = -val;
          b_std[i] -= val * toff[j];
          break;
        default:
          ci[q] = static_cast<int32_t>(tcol[j]), cv[q++] = val;
          ci[q] = static_cast<int32_t>(tneg[j]), cv[q++] = -val;
      }
    }
    if (slack_item[i] >= 0) ci[q] = static_cast<int32_t>(tcol[slack_item[i]]), cv[q++] = map.row_conversions[i].slack_sign;
  }
  for (std::size_t t = 0; t < pending.size(); ++t) {
    const BoundRow& br = map.bound_rows[t];
    const int64_t q = rp[br.row];
    ci[q] = static_cast<int32_t>(br.col), cv[q] = 1.0;
    ci[q + 1] = static_cast<int32_t>(br.slack_col), cv[q + 1] = 1.0;
    b_std[br.row] = br.rhs;
  }
  map.objective_constant = sense * shift_const + objective_constant;
  map.standard_rows = m_std;
  map.standard_cols = n_std;
  SparseMatrix a = SparseMatrix::from_csr(m_std, n_std, rp.data(), ci.data(), cv.data());
  return {StandardFormLP(std::move(a), std::move(b_std), std::move(c_std)), std::move(map)};
}

}  // namespace

std::pair<StandardFormLP, VariableMap> to_standard_form(const GeneralFormLP& g) {
  const Index m = g.num_rows(), n = g.num_cols();
  if (static_cast<Index>(g.objective.size()) != n)
    throw std::invalid_argument("GeneralFormLP: objective length mismatch");
  for (const Triplet& t : g.entries)
    if (t.row < 0 || t.row >= m || t.col < 0 || t.col >= n)
      throw std::invalid_argument("GeneralFormLP: entry index out of range");
  RowsView A;
  A.m = m;
  A.n = n;
  A.rp.assign(static_cast<std::size_t>(m) + 1, 0);
  for (const Triplet& t : g.entries) ++A.rp[t.row + 1];
  for (Index i = 0; i < m; ++i) A.rp[i + 1] += A.rp[i];
  A.ci.resize(g.entries.size());
  A.v.resize(g.entries.size());
  std::vector<int64_t> fill(A.rp.begin(), A.rp.end() - 1);
  for (const Triplet& t : g.entries) {  // stable: entry order kept within rows
    const int64_t p = fill[t.row]++;
    A.ci[p] = static_cast<int32_t>(t.col);
    A.v[p] = t.value;
  }
  std::vector<RowInfo> rows(static_cast<std::size_t>(m));
  for (Index i = 0; i < m; ++i) {
    const GeneralFormRow& r = g.rows[i];
    rows[i] = {r.relation == RowRelation::kLessEqual ? HPLP_ROW_LE
               : r.relation == RowRelation::kGreaterEqual ? HPLP_ROW_GE
                                                          : HPLP_ROW_EQ,
               r.rhs, r.range.has_value(), r.range.value_or(0.0), r.name};
  }
  std::vector<ColumnInfo> cols(static_cast<std::size_t>(n));
  std::vector<std::string> names(static_cast<std::size_t>(n));
  for (Index j = 0; j < n; ++j) {
    cols[j] = {g.columns[j].lower, g.columns[j].upper, g.objective[j]};
    names[j] = g.columns[j].name;
  }
  return convert(A, rows, cols, &names, g.maximize, g.objective_constant);
}

std::pair<StandardFormLP, VariableMap> to_standard_form(const hplp_general_t& g) {
  if (g.m < 0 || g.n < 0) throw std::invalid_argument("GeneralFormLP: negative dimension");
  if (g.row_ptr[0] != 0) throw std::invalid_argument("GeneralFormLP: row_ptr[0] must be 0");
  for (int64_t i = 0; i < g.m; ++i)
    if (g.row_ptr[i + 1] < g.row_ptr[i]) throw std::invalid_argument("GeneralFormLP: row_ptr not monotone");
  RowsView A;
  A.m = g.m;
  A.n = g.n;
  A.rp.assign(g.row_ptr, g.row_ptr + g.m + 1);
  A.ci.assign(g.col_idx, g.col_idx + g.row_ptr[g.m]);
  A.v.assign(g.val, g.val + g.row_ptr[g.m]);
  std::vector<RowInfo> rows(static_cast<std::size_t>(g.m));
  for (int64_t i = 0; i < g.m; ++i) {
    const bool hr = g.row_range && !std::isnan(g.row_range[i]);
    rows[i] = {g.row_relation[i], g.row_rhs[i], hr, hr ? g.row_range[i] : 0.0, "r" + std::to_string(i)};
  }
  std::vector<ColumnInfo> cols(static_cast<std::size_t>(g.n));
  for (int64_t j = 0; j < g.n; ++j) cols[j] = {g.col_lower[j], g.col_upper[j], g.objective[j]};
  return convert(A, rows, cols, nullptr, g.maximize != 0, g.objective_constant);
}

}  // namespace hplp_gpu
