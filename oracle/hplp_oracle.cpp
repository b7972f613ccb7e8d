// TEST INFRASTRUCTURE ONLY -- the CPU checker for the B200 rHPDHG path.
//
// A plain C++ (std::vector, no Eigen) restatement of the reference solver's
// hot path, following /root/reference/proj line by line; every function cites
// the reference file:line it restates.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline leg may load this library; the product never
// links or calls it (and fails loudly without its CUDA library instead).
//
// Parity pin: tests/test_oracle.py checks this restatement bit for bit
// against the unmodified reference compiled by oracle/Makefile
// (oracle/_ref/libhplp_ref.so) and against the SPEC.md known-answer tests
// committed under tests/golden/.
//
// Arithmetic: one IEEE rounding per scalar op (built with -ffp-contract=off),
// reductions sequential in ascending index order (the order of the Eigen
// subset the reference is compiled against here, oracle/eigen_shim).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "hplp_types.h"

namespace orc {

using Vec = std::vector<double>;
constexpr double kInf = std::numeric_limits<double>::infinity();

// ---- BLAS-1 (Eigen semantics: eager element-wise, sequential reductions) --
double sqnorm(const Vec& v) {
  double s = 0.0;
  for (double a : v) s += a * a;
  return s;
}
double norm(const Vec& v) { return std::sqrt(sqnorm(v)); }
double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double inf_norm(const Vec& v) {  // src/infeasibility.cpp:22-24
  if (v.empty()) return 0.0;
  double m = std::abs(v[0]);
  for (std::size_t i = 1; i < v.size(); ++i) m = std::abs(v[i]) > m ? std::abs(v[i]) : m;
  return m;
}
bool all_finite(const Vec& v) {
  for (double a : v)
    if (!std::isfinite(a)) return false;
  return true;
}
Vec sub(const Vec& a, const Vec& b) {
  Vec r(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) r[i] = a[i] - b[i];
  return r;
}
Vec scale(double s, const Vec& a) {
  Vec r(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) r[i] = s * a[i];
  return r;
}
// (1-w)*a + w*b evaluated as Eigen does: two products, then one sum.
Vec combine(double w, const Vec& a, const Vec& b) {
  Vec r(a.size());
  const double omw = 1.0 - w;
  for (std::size_t i = 0; i < a.size(); ++i) r[i] = omw * a[i] + w * b[i];
  return r;
}

// ---- SparseMatrix: src/sparse_matrix.cpp:24-66 ------------------------------
struct Csr {
  int64_t rows = 0, cols = 0;
  std::vector<int64_t> rp, cp;     // row / column pointers
  std::vector<int32_t> ci, ri;     // column index (by row), row index (by col)
  std::vector<double> rv, cv;      // values by row / by column
  int64_t nnz() const { return static_cast<int64_t>(rv.size()); }
};

// Validation and storage: range check, finiteness, duplicates are a hard
// error (src/sparse_matrix.cpp:27-53); both traversals keep ascending inner
// indices (inc/sparse_matrix.hpp:34-38).
Csr make_csr(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
             const double* val) {
  if (m < 0 || n < 0) throw std::invalid_argument("SparseMatrix: negative dimension");
  Csr a;
  a.rows = m;
  a.cols = n;
  const int64_t nnz = row_ptr[m];
  a.rp.assign(row_ptr, row_ptr + m + 1);
  a.ci.resize(static_cast<std::size_t>(nnz));
  a.rv.resize(static_cast<std::size_t>(nnz));
  std::vector<std::pair<int32_t, double>> row;
  for (int64_t i = 0; i < m; ++i) {
    row.clear();
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      if (col_idx[p] < 0 || col_idx[p] >= n)
        throw std::invalid_argument("SparseMatrix: entry (" + std::to_string(i) + ", " +
                                    std::to_string(col_idx[p]) + ") out of range for " +
                                    std::to_string(m) + "x" + std::to_string(n));
      if (!std::isfinite(val[p]))
        throw std::invalid_argument("SparseMatrix: non-finite value at (" + std::to_string(i) +
                                    ", " + std::to_string(col_idx[p]) + ")");
      row.push_back({col_idx[p], val[p]});
    }
    std::stable_sort(row.begin(), row.end(),
                     [](const auto& x, const auto& y) { return x.first < y.first; });
    for (std::size_t q = 0; q < row.size(); ++q) {
      if (q && row[q].first == row[q - 1].first)
        throw std::invalid_argument("SparseMatrix: duplicate entry at (" + std::to_string(i) +
                                    ", " + std::to_string(row[q].first) + ")");
      a.ci[static_cast<std::size_t>(row_ptr[i]) + q] = row[q].first;
      a.rv[static_cast<std::size_t>(row_ptr[i]) + q] = row[q].second;
    }
  }
  // Column-compressed copy: counting sort, stable in row order.
  a.cp.assign(static_cast<std::size_t>(n) + 1, 0);
  for (int64_t p = 0; p < nnz; ++p) ++a.cp[static_cast<std::size_t>(a.ci[p]) + 1];
  for (int64_t j = 0; j < n; ++j) a.cp[j + 1] += a.cp[j];
  a.ri.resize(static_cast<std::size_t>(nnz));
  a.cv.resize(static_cast<std::size_t>(nnz));
  std::vector<int64_t> fill(a.cp.begin(), a.cp.end() - 1);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t p = a.rp[i]; p < a.rp[i + 1]; ++p) {
      const int64_t q = fill[a.ci[p]]++;
      a.ri[q] = static_cast<int32_t>(i);
      a.cv[q] = a.rv[p];
    }
  return a;
}

// spmv: src/sparse_matrix.cpp:101-117 (ascending-column sequential sum).
Vec spmv(const Csr& a, const Vec& x) {
  if (static_cast<int64_t>(x.size()) != a.cols)
    throw std::invalid_argument("spmv: x has length " + std::to_string(x.size()) +
                                ", expected " + std::to_string(a.cols));
  Vec out(static_cast<std::size_t>(a.rows), 0.0);
  for (int64_t i = 0; i < a.rows; ++i) {
    double acc = 0.0;
    for (int64_t p = a.rp[i]; p < a.rp[i + 1]; ++p) acc += a.rv[p] * x[a.ci[p]];
    out[i] = acc;
  }
  return out;
}

// spmv_transpose: src/sparse_matrix.cpp:119-136 (ascending-row sum per column).
Vec spmv_t(const Csr& a, const Vec& y) {
  if (static_cast<int64_t>(y.size()) != a.rows)
    throw std::invalid_argument("spmv_transpose: y has length " + std::to_string(y.size()) +
                                ", expected " + std::to_string(a.rows));
  Vec out(static_cast<std::size_t>(a.cols), 0.0);
  for (int64_t j = 0; j < a.cols; ++j) {
    double acc = 0.0;
    for (int64_t p = a.cp[j]; p < a.cp[j + 1]; ++p) acc += a.cv[p] * y[a.ri[p]];
    out[j] = acc;
  }
  return out;
}

struct Power {
  double sigma = 0.0;
  int64_t iterations = 0;
  bool converged = false;
};

// power_iteration: src/sparse_matrix.cpp:138-179.
Power power_iteration(const Csr& a, double tol, int64_t max_iters, uint64_t seed) {
  Power res;
  if (a.rows == 0 || a.cols == 0 || a.nnz() == 0) {
    res.converged = true;
    return res;
  }
  std::mt19937_64 gen(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  Vec x(static_cast<std::size_t>(a.cols));
  for (auto& v : x) v = dist(gen);
  double xn = norm(x);
  if (xn == 0.0) std::fill(x.begin(), x.end(), 1.0), xn = norm(x);
  for (auto& v : x) v /= xn;
  double sigma_prev = 0.0;
  for (int64_t k = 0; k < max_iters; ++k) {
    Vec w = spmv(a, x);
    const double sigma = norm(w);
    res.iterations = k + 1;
    if (sigma == 0.0) {  // :158-163 re-draw from the same stream
      for (auto& v : x) v = dist(gen);
      const double nn = norm(x);
      for (auto& v : x) v /= nn;
      continue;
    }
    Vec z = spmv_t(a, w);
    res.sigma = sigma;
    if (k > 0 && std::abs(sigma - sigma_prev) <= tol * sigma) {
      res.converged = true;
      return res;
    }
    sigma_prev = sigma;
    const double zn = norm(z);
    if (zn == 0.0) {
      res.converged = true;
      return res;
    }
    for (std::size_t i = 0; i < x.size(); ++i) x[i] = z[i] / zn;
  }
  return res;
}

struct Lp {
  Csr a;
  Vec b, c;
  // Box form (no reference counterpart): column upper
  // bounds enforced by the projection; empty = the reference's standard form.
  Vec u;
};

struct Kkt {
  double p = 0, d = 0, g = 0, max = 0;
};

// kkt_error_with_products: src/pdhg_core.cpp:57-68.
Kkt kkt(const Vec& x, const Vec& y, const Lp& lp, const Vec& a_x, const Vec& at_y) {
  Kkt e;
  double b_norm = norm(lp.b);
  if (!lp.u.empty()) {  // box form: ||b|| of the standard form (b, then the bound rows' u)
    double sq = sqnorm(lp.b);
    for (double u : lp.u)
      if (u < kInf) sq += u * u;
    b_norm = std::sqrt(sq);
  }
  e.p = norm(sub(a_x, lp.b)) / (1.0 + b_norm);
  Vec r(lp.c.size());
  double ul = 0.0;  // box form: sum over bounded columns of u_j [-(c + A^T y)_j]^+
  for (std::size_t j = 0; j < r.size(); ++j) {
    const double v = -(lp.c[j] + at_y[j]);
    r[j] = v < 0.0 ? 0.0 : v;
    if (!lp.u.empty() && lp.u[j] < kInf) {
      ul += lp.u[j] * r[j];
      r[j] = 0.0;
    }
  }
  e.d = norm(r) / (1.0 + norm(lp.c));
  const double cx = dot(lp.c, x);
  const double by = dot(lp.b, y) + ul;
  e.g = std::abs(cx + by) / (1.0 + std::abs(cx) + std::abs(by));
  e.max = std::max({e.p, e.d, e.g});
  return e;
}

// canonical_norm_with_product: src/pdhg_core.cpp:37-51.
double canonical(const Vec& dx, const Vec& dy, const Vec& a_dx, double eta) {
  const double q = sqnorm(dx) / eta - 2.0 * dot(dy, a_dx) + sqnorm(dy) / eta;
  if (q < 0.0) {
    const double sc = (sqnorm(dx) + sqnorm(dy)) / eta;
    if (q < -1e-9 * sc)
      throw std::domain_error(
          "canonical norm: quadratic form is negative (eta too large for this matrix)");
    return 0.0;
  }
  return std::sqrt(q);
}

struct Step {
  Vec x, y, a_x_next, at_y;
};

// pdhg_step_with_products: src/pdhg_core.cpp:75-87.
Step pdhg_step(const Vec& x, const Vec& y, const Lp& lp, double eta, const Vec& a_x) {
  Step r;
  r.at_y = spmv_t(lp.a, y);
  r.x.resize(x.size());
  for (std::size_t j = 0; j < x.size(); ++j) {
    const double v = x[j] - eta * (r.at_y[j] + lp.c[j]);
    r.x[j] = v < 0.0 ? 0.0 : v;
    if (!lp.u.empty() && r.x[j] > lp.u[j]) r.x[j] = lp.u[j];  // box form
  }
  r.a_x_next = spmv(lp.a, r.x);
  r.y.resize(y.size());
  for (std::size_t i = 0; i < y.size(); ++i)
    r.y[i] = y[i] + eta * ((2.0 * r.a_x_next[i] - a_x[i]) - lp.b[i]);
  return r;
}

struct Farkas {
  double residual = kInf, margin = 0.0;
  int orientation = HPLP_ORIENT_AS_IS;
  bool valid = false;
};

// validate_primal_infeasibility: src/infeasibility.cpp:41-67.
Farkas validate_primal(const Vec& v, const Lp& lp, double tol, double sigma) {
  Farkas rep;
  const double n2 = norm(v);
  if (n2 == 0.0 || !all_finite(v)) return rep;
  Vec u(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) u[i] = v[i] / n2;
  const double threshold = tol * std::max(1.0, inf_norm(u) * sigma);
  const Vec at_u = spmv_t(lp.a, u);
  const double b_norm = norm(lp.b);
  for (double s : {1.0, -1.0}) {
    Vec t(at_u.size());
    for (std::size_t j = 0; j < t.size(); ++j) {
      const double q = s * at_u[j];
      t[j] = q < 0.0 ? 0.0 : q;
    }
    const double residual = inf_norm(t);
    const double margin = s * dot(lp.b, u);
    const bool ok = residual <= threshold && margin > 0.0 && margin >= tol * b_norm;
    if (ok || (!rep.valid && residual < rep.residual)) {
      rep.residual = residual;
      rep.margin = margin;
      rep.orientation = s > 0 ? HPLP_ORIENT_AS_IS : HPLP_ORIENT_NEGATED;
    }
    if (ok) {
      rep.valid = true;
      break;
    }
  }
  return rep;
}

// validate_dual_infeasibility: src/infeasibility.cpp:76-106.
Farkas validate_dual(const Vec& v, const Lp& lp, double tol, double sigma) {
  Farkas rep;
  const double n2 = norm(v);
  if (n2 == 0.0 || !all_finite(v)) return rep;
  Vec u(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) u[i] = v[i] / n2;
  const double threshold = tol * std::max(1.0, inf_norm(u) * sigma);
  const double nonneg_threshold = tol * std::max(1.0, inf_norm(u));
  const Vec a_u = spmv(lp.a, u);
  const double margin_threshold = -tol * std::max(1.0, norm(lp.c));
  for (double s : {1.0, -1.0}) {
    const double ray = inf_norm(scale(s, a_u));
    Vec t(u.size());
    for (std::size_t j = 0; j < t.size(); ++j) {
      const double q = -s * u[j];
      t[j] = q < 0.0 ? 0.0 : q;
    }
    const double sign = inf_norm(t);
    const double residual = std::max(ray, sign);
    const double margin = s * dot(lp.c, u);
    const bool ok = ray <= threshold && sign <= nonneg_threshold && margin <= margin_threshold;
    if (ok || (!rep.valid && residual < rep.residual)) {
      rep.residual = residual;
      rep.margin = margin;
      rep.orientation = s > 0 ? HPLP_ORIENT_AS_IS : HPLP_ORIENT_NEGATED;
    }
    if (ok) {
      rep.valid = true;
      break;
    }
  }
  return rep;
}

// should_restart: src/solver.cpp:162-174.
bool should_restart(const hplp_config_t& c, int64_t n, int64_t k, double now, double start) {
  switch (c.restart_kind) {
    case HPLP_RESTART_FIXED:
      return k >= c.k_star;
    case HPLP_RESTART_ADAPTIVE:
      if (n == 0) return k > c.tau0;
      return now <= c.beta * start;
    default:
      return false;
  }
}

// validate_config: src/solver.cpp:40-65.
void validate_config(const hplp_config_t& c) {
  if (!(c.tolerance > 0.0)) throw std::invalid_argument("SolverConfig: tolerance must be > 0");
  if (c.iteration_limit < 0)
    throw std::invalid_argument("SolverConfig: iteration_limit must be >= 0");
  if (!(c.certificate_tolerance > 0.0))
    throw std::invalid_argument("SolverConfig: certificate_tolerance must be > 0");
  if (c.infeasibility_check_period < 0 || c.trace_period < 0 || c.adaptive_stall_cap < 0)
    throw std::invalid_argument("SolverConfig: periods must be >= 0");
  if (c.restart_kind == HPLP_RESTART_FIXED && c.k_star < 1)
    throw std::invalid_argument("RestartScheme: k_star must be >= 1");
  if (c.restart_kind == HPLP_RESTART_ADAPTIVE &&
      (!(c.beta > 0.0) || !(c.beta < 1.0) || c.tau0 < 1))
    throw std::invalid_argument("RestartScheme: adaptive needs beta in (0,1) and tau0 >= 1");
}

// StepSize ctor / largest_stable: src/pdhg_core.cpp:21-35.
double step_size(double eta, double sigma) {
  if (!(eta > 0.0) || !std::isfinite(eta))
    throw std::invalid_argument("StepSize: eta must be positive and finite");
  if (sigma > 0.0 && eta > 1.0 / (2.0 * sigma) * (1 + 1e-12))
    throw std::invalid_argument("StepSize: eta exceeds 1/(2 ||A||_2-estimate) = " +
                                std::to_string(1.0 / (2.0 * sigma)));
  return eta;
}

struct Cert {
  bool present = false;
  Vec vec;
  int source = HPLP_SOURCE_ITERATE_DIFFERENCE;
  int64_t at = 0;
  int orientation = HPLP_ORIENT_AS_IS;
  double residual = 0, margin = 0;
};

// make_certificate: src/solver.cpp:89-101.
Cert make_cert(const Vec& raw, int source, int64_t at, const Farkas& f) {
  Cert c;
  c.present = true;
  const double s = f.orientation == HPLP_ORIENT_NEGATED ? -1.0 : 1.0;
  c.vec = scale(s / norm(raw), raw);
  c.source = source;
  c.at = at;
  c.orientation = f.orientation;
  c.residual = f.residual;
  c.margin = f.margin;
  return c;
}

struct Epoch {
  int64_t epoch = 0, len = 0;
  double res = 0;
  Kkt kkt;
};

using Clock = std::chrono::steady_clock;

// solve: src/solver.cpp:206-342 (make_setup :67-78, initial_point :80-87).
void solve(const Lp& lp, const hplp_config_t& cfg, hplp_io_t* io, hplp_result_t* out) {
  const auto t0 = Clock::now();
  auto since = [&] { return std::chrono::duration<double>(Clock::now() - t0).count(); };
  validate_config(cfg);
  if (!lp.u.empty() && cfg.infeasibility_check_period > 0)
    throw std::invalid_argument("box form: no infeasibility scan (set infeasibility_check_period 0)");
  const Power pi = power_iteration(lp.a, 1e-4, 5000, cfg.seed);
  const double sigma_used = pi.sigma * (1.0 + 1e-4);
  int64_t n_spmv = 2 * pi.iterations;
  double eta;
  if (cfg.has_eta_override) {
    eta = step_size(cfg.eta_override, sigma_used);
  } else {
    eta = sigma_used <= 0.0 ? step_size(1.0, 0.0) : step_size(1.0 / (2.0 * sigma_used), sigma_used);
  }
  const int64_t m = lp.a.rows, n = lp.a.cols;
  Vec x(static_cast<std::size_t>(n), 0.0), y(static_cast<std::size_t>(m), 0.0);
  if (io && io->init_x && io->init_y) {
    x.assign(io->init_x, io->init_x + n);
    y.assign(io->init_y, io->init_y + m);
  }
  Vec a_x = spmv(lp.a, x);
  ++n_spmv;
  Vec anc_x = x, anc_y = y, a_x_anchor = a_x;
  int64_t ep = 0, k = 0, it = 0;
  double res_epoch_start = 0.0;
  std::vector<Epoch> epochs;
  double best_kkt = kInf;
  Vec best_x = x, best_y = y;
  Kkt best_err;
  Cert primal, dual;

  auto finish = [&](int status, const Vec& fx, const Vec& fy, const Kkt& e) {
    std::memset(out, 0, sizeof(*out));
    out->status = status;
    if (!epochs.empty() && epochs.back().len == 0) epochs.back().len = k;
    out->iterations = it;
    out->spmv_count = n_spmv;
    out->wall_seconds = since();
    out->eta = eta;
    out->sigma_estimate = sigma_used;
    out->final_kkt = {e.p, e.d, e.g, e.max};
    out->n_epochs = static_cast<int64_t>(epochs.size());
    auto put_cert = [&](const Cert& c, hplp_cert_meta_t* meta, double* dst) {
      if (!c.present) return;
      meta->present = 1;
      meta->source = c.source;
      meta->orientation = c.orientation;
      meta->at_iteration = c.at;
      meta->residual = c.residual;
      meta->margin = c.margin;
      if (dst) std::copy(c.vec.begin(), c.vec.end(), dst);
    };
    put_cert(primal, &out->primal_cert, io ? io->primal_cert : nullptr);
    put_cert(dual, &out->dual_cert, io ? io->dual_cert : nullptr);
    if (io) {
      if (io->x) std::copy(fx.begin(), fx.end(), io->x);
      if (io->y) std::copy(fy.begin(), fy.end(), io->y);
      if (io->epochs)
        for (std::size_t e2 = 0; e2 < epochs.size() && static_cast<int64_t>(e2) < io->epochs_capacity; ++e2)
          io->epochs[e2] = {epochs[e2].epoch, epochs[e2].len, epochs[e2].res,
                            {epochs[e2].kkt.p, epochs[e2].kkt.d, epochs[e2].kkt.g, epochs[e2].kkt.max}};
    }
  };
  auto limit = [&](int status) {  // :242-254
    if (std::isfinite(best_kkt)) {
      finish(status, best_x, best_y, best_err);
    } else {
      const Kkt e = kkt(x, y, lp, spmv(lp.a, x), spmv_t(lp.a, y));
      finish(status, x, y, e);
      out->spmv_count += 2;
    }
  };

  while (true) {
    if (it >= cfg.iteration_limit) return limit(HPLP_STATUS_ITERATION_LIMIT);
    if (since() > cfg.time_limit_seconds) return limit(HPLP_STATUS_TIME_LIMIT);

    Step sr = pdhg_step(x, y, lp, eta, a_x);  // :256
    n_spmv += 2;
    const Kkt e = kkt(x, y, lp, a_x, sr.at_y);  // :258
    const double res = canonical(sub(x, sr.x), sub(y, sr.y), sub(a_x, sr.a_x_next), eta);
    if (k == 0) {  // :261-264
      res_epoch_start = res;
      epochs.push_back({ep, 0, res, e});
    }
    if (e.max < best_kkt) {  // :265-269
      best_kkt = e.max;
      best_x = x;
      best_y = y;
      best_err = e;
    }
    if (cfg.trace_period > 0 && it % cfg.trace_period == 0 && io && io->trace_fn) {
      hplp_trace_t t;  // :271-290
      t.epoch = ep;
      t.inner = k;
      t.iteration = it;
      t.fixed_point_residual = res;
      t.kkt = {e.p, e.d, e.g, e.max};
      t.candidate_norm_difference =
          canonical(sub(sr.x, x), sub(sr.y, y), sub(sr.a_x_next, a_x), eta);
      t.candidate_norm_normalized = std::numeric_limits<double>::quiet_NaN();
      if (k >= 1) {
        const double s = 2.0 / static_cast<double>(k);
        t.candidate_norm_normalized = canonical(scale(s, sub(x, anc_x)), scale(s, sub(y, anc_y)),
                                                scale(s, sub(a_x, a_x_anchor)), eta);
      }
      t.wall_seconds = since();
      // partition_estimate_from_reduced_costs(z, c + A^T y, tol_active, sigma),
      // src/diagnostics.cpp:26-43 via src/solver.cpp:279-280
      std::vector<int64_t> pn, pb1, pb2;
      const double r_tol = cfg.tol_active * sigma_used;
      for (int64_t j = 0; j < n; ++j) {
        const double r = lp.c[j] + sr.at_y[j];
        if (r > r_tol) pn.push_back(j);
        else if (std::abs(r) <= r_tol && x[j] > cfg.tol_active) pb1.push_back(j);
        else pb2.push_back(j);
      }
      t.partition_n = static_cast<int64_t>(pn.size());
      t.partition_b1 = static_cast<int64_t>(pb1.size());
      t.partition_b2 = static_cast<int64_t>(pb2.size());
      pn.insert(pn.end(), pb1.begin(), pb1.end());
      pn.insert(pn.end(), pb2.begin(), pb2.end());
      t.partition_sets = pn.data();
      io->trace_fn(&t, x.data(), n, y.data(), m, io->trace_user);
    }
    if (e.max <= cfg.tolerance) {  // :292-295
      finish(HPLP_STATUS_OPTIMAL, x, y, e);
      return;
    }
    if (cfg.infeasibility_check_period > 0 && it > 0 &&
        (it % cfg.infeasibility_check_period == 0 || k == 0)) {  // :297-317
      auto check = [&](const Vec& v_x, const Vec& v_y, int source) {  // CertificateScan::check :108-129
        if (!primal.present && norm(v_y) > 0.0) {
          Farkas f = validate_primal(v_y, lp, cfg.certificate_tolerance, sigma_used);
          ++n_spmv;
          if (f.valid) primal = make_cert(v_y, source, it, f);
        }
        if (!dual.present && norm(v_x) > 0.0) {
          Farkas f = validate_dual(v_x, lp, cfg.certificate_tolerance, sigma_used);
          ++n_spmv;
          if (f.valid) dual = make_cert(v_x, source, it, f);
        }
      };
      check(sub(sr.x, x), sub(sr.y, y), HPLP_SOURCE_ITERATE_DIFFERENCE);
      if (k >= 1) {
        const double s = 2.0 / static_cast<double>(k);
        check(scale(s, sub(x, anc_x)), scale(s, sub(y, anc_y)), HPLP_SOURCE_NORMALIZED_ITERATE);
      }
      if (primal.present || dual.present) {
        const int status = primal.present && dual.present ? HPLP_STATUS_PRIMAL_DUAL_INFEASIBLE
                           : primal.present               ? HPLP_STATUS_PRIMAL_INFEASIBLE
                                                          : HPLP_STATUS_DUAL_INFEASIBLE;
        finish(status, x, y, e);
        return;
      }
    }
    bool restart = should_restart(cfg, ep, k, res, res_epoch_start);  // :319-324
    if (!restart && cfg.restart_kind == HPLP_RESTART_ADAPTIVE && cfg.adaptive_stall_cap > 0 &&
        k >= cfg.adaptive_stall_cap)
      restart = true;
    if (restart) {  // :325-332
      epochs.back().len = k;
      x = std::move(sr.x);
      y = std::move(sr.y);
      a_x = std::move(sr.a_x_next);
      anc_x = x;
      anc_y = y;
      a_x_anchor = a_x;
      ++ep;
      k = 0;
    } else {  // :333-339
      const double w = 1.0 / static_cast<double>(k + 2);
      x = combine(w, sr.x, anc_x);
      y = combine(w, sr.y, anc_y);
      a_x = combine(w, sr.a_x_next, a_x_anchor);
      ++k;
    }
    ++it;
  }
}

// solve_baseline: src/solver.cpp:344-509 (mode 0 vanilla, 1 averaged, 2
// restarted average) and update_average (src/baselines.cpp:20-31).
void solve_baseline(const Lp& lp, const hplp_config_t& cfg, int mode, hplp_io_t* io, hplp_result_t* out) {
  const auto t0 = Clock::now();
  auto since = [&] { return std::chrono::duration<double>(Clock::now() - t0).count(); };
  validate_config(cfg);
  if (!lp.u.empty()) throw std::invalid_argument("box form: rHPDHG only");
  const Power pi = power_iteration(lp.a, 1e-4, 5000, cfg.seed);
  const double sigma_used = pi.sigma * (1.0 + 1e-4);
  int64_t n_spmv = 2 * pi.iterations;
  double eta;
  if (cfg.has_eta_override) eta = step_size(cfg.eta_override, sigma_used);
  else eta = sigma_used <= 0.0 ? step_size(1.0, 0.0) : step_size(1.0 / (2.0 * sigma_used), sigma_used);
  const bool averaged = mode != 0, restarted = mode == 2;
  const int64_t m = lp.a.rows, n = lp.a.cols;
  Vec x(static_cast<std::size_t>(n), 0.0), y(static_cast<std::size_t>(m), 0.0);
  if (io && io->init_x && io->init_y) {
    x.assign(io->init_x, io->init_x + n);
    y.assign(io->init_y, io->init_y + m);
  }
  Vec a_x = spmv(lp.a, x);
  ++n_spmv;
  Vec mx, my, a_x_avg, at_y_avg;  // running mean (z-bar) and its products
  int64_t count = 0;
  bool ready = false;
  int64_t ep = 0, k = 0, it = 0;
  double res_epoch_start = 0.0;
  std::vector<Epoch> epochs;
  double best_kkt = kInf;
  Vec best_x = x, best_y = y;
  Kkt best_err;
  Cert primal, dual;
  auto finish = [&](int status, const Vec& fx, const Vec& fy, const Kkt& e) {
    std::memset(out, 0, sizeof(*out));
    out->status = status;
    if (!epochs.empty() && epochs.back().len == 0) epochs.back().len = k;
    out->iterations = it;
    out->spmv_count = n_spmv;
    out->wall_seconds = since();
    out->eta = eta;
    out->sigma_estimate = sigma_used;
    out->final_kkt = {e.p, e.d, e.g, e.max};
    out->n_epochs = static_cast<int64_t>(epochs.size());
    auto put_cert = [&](const Cert& c, hplp_cert_meta_t* meta, double* dst) {
      if (!c.present) return;
      meta->present = 1;
      meta->source = c.source;
      meta->orientation = c.orientation;
      meta->at_iteration = c.at;
      meta->residual = c.residual;
      meta->margin = c.margin;
      if (dst) std::copy(c.vec.begin(), c.vec.end(), dst);
    };
    put_cert(primal, &out->primal_cert, io ? io->primal_cert : nullptr);
    put_cert(dual, &out->dual_cert, io ? io->dual_cert : nullptr);
    if (io) {
      if (io->x) std::copy(fx.begin(), fx.end(), io->x);
      if (io->y) std::copy(fy.begin(), fy.end(), io->y);
      if (io->epochs)
        for (std::size_t e2 = 0; e2 < epochs.size() && static_cast<int64_t>(e2) < io->epochs_capacity; ++e2)
          io->epochs[e2] = {epochs[e2].epoch, epochs[e2].len, epochs[e2].res,
                            {epochs[e2].kkt.p, epochs[e2].kkt.d, epochs[e2].kkt.g, epochs[e2].kkt.max}};
    }
  };
  while (true) {
    if (it >= cfg.iteration_limit || since() > cfg.time_limit_seconds) {  // :387-399
      const int status = it >= cfg.iteration_limit ? HPLP_STATUS_ITERATION_LIMIT : HPLP_STATUS_TIME_LIMIT;
      if (std::isfinite(best_kkt)) {
        finish(status, best_x, best_y, best_err);
      } else {
        finish(status, x, y, kkt(x, y, lp, spmv(lp.a, x), spmv_t(lp.a, y)));
        out->spmv_count += 2;
      }
      return;
    }
    Step sr = pdhg_step(x, y, lp, eta, a_x);  // :401-402
    n_spmv += 2;
    if (averaged) {  // :404-416
      if (!ready) {
        mx = x, my = y, count = 1;
        a_x_avg = a_x;
        at_y_avg = sr.at_y;
        ready = true;
      } else {
        const double w = 1.0 / static_cast<double>(count + 1);
        for (int64_t j = 0; j < n; ++j) mx[j] += w * (x[j] - mx[j]);
        for (int64_t i = 0; i < m; ++i) my[i] += w * (y[i] - my[i]);
        count += 1;
        const double w2 = 1.0 / static_cast<double>(count);
        for (int64_t i = 0; i < m; ++i) a_x_avg[i] += w2 * (a_x[i] - a_x_avg[i]);
        for (int64_t j = 0; j < n; ++j) at_y_avg[j] += w2 * (sr.at_y[j] - at_y_avg[j]);
      }
    }
    const Vec& cx = averaged ? mx : x;
    const Vec& cy = averaged ? my : y;
    const Kkt e = averaged ? kkt(mx, my, lp, a_x_avg, at_y_avg) : kkt(x, y, lp, a_x, sr.at_y);  // :418-421
    const bool tracing = cfg.trace_period > 0 && it % cfg.trace_period == 0 && io && io->trace_fn;
    double res;
    if (averaged && (restarted || tracing || k == 0)) {  // :424-433
      Step as = pdhg_step(mx, my, lp, eta, a_x_avg);
      n_spmv += 2;
      res = canonical(sub(mx, as.x), sub(my, as.y), sub(a_x_avg, as.a_x_next), eta);
    } else if (!averaged) {
      res = canonical(sub(x, sr.x), sub(y, sr.y), sub(a_x, sr.a_x_next), eta);
    } else {
      res = std::numeric_limits<double>::quiet_NaN();
    }
    if (k == 0) {  // :434-437
      res_epoch_start = res;
      epochs.push_back({ep, 0, res, e});
    }
    if (e.max < best_kkt) {  // :438-442
      best_kkt = e.max;
      best_x = cx;
      best_y = cy;
      best_err = e;
    }
    if (tracing) {  // :444-460
      hplp_trace_t t;
      t.epoch = ep;
      t.inner = k;
      t.iteration = it;
      t.fixed_point_residual = res;
      t.kkt = {e.p, e.d, e.g, e.max};
      t.candidate_norm_difference = canonical(sub(sr.x, x), sub(sr.y, y), sub(sr.a_x_next, a_x), eta);
      t.candidate_norm_normalized = std::numeric_limits<double>::quiet_NaN();
      t.wall_seconds = since();
      std::vector<int64_t> pn, pb1, pb2;
      const double r_tol = cfg.tol_active * sigma_used;
      const Vec& aty = averaged ? at_y_avg : sr.at_y;
      for (int64_t j = 0; j < n; ++j) {
        const double r = lp.c[j] + aty[j];
        if (r > r_tol) pn.push_back(j);
        else if (std::abs(r) <= r_tol && cx[j] > cfg.tol_active) pb1.push_back(j);
        else pb2.push_back(j);
      }
      t.partition_n = static_cast<int64_t>(pn.size());
      t.partition_b1 = static_cast<int64_t>(pb1.size());
      t.partition_b2 = static_cast<int64_t>(pb2.size());
      pn.insert(pn.end(), pb1.begin(), pb1.end());
      pn.insert(pn.end(), pb2.begin(), pb2.end());
      t.partition_sets = pn.data();
      io->trace_fn(&t, cx.data(), n, cy.data(), m, io->trace_user);
    }
    if (e.max <= cfg.tolerance) {  // :462-465
      finish(HPLP_STATUS_OPTIMAL, cx, cy, e);
      return;
    }
    if (cfg.infeasibility_check_period > 0 && it > 0 && it % cfg.infeasibility_check_period == 0) {  // :467-481
      const Vec vx = sub(sr.x, x), vy = sub(sr.y, y);
      if (norm(vy) > 0.0) {
        Farkas f = validate_primal(vy, lp, cfg.certificate_tolerance, sigma_used);
        ++n_spmv;
        if (f.valid) primal = make_cert(vy, HPLP_SOURCE_ITERATE_DIFFERENCE, it, f);
      }
      if (norm(vx) > 0.0) {
        Farkas f = validate_dual(vx, lp, cfg.certificate_tolerance, sigma_used);
        ++n_spmv;
        if (f.valid) dual = make_cert(vx, HPLP_SOURCE_ITERATE_DIFFERENCE, it, f);
      }
      if (primal.present || dual.present) {
        const int status = primal.present && dual.present ? HPLP_STATUS_PRIMAL_DUAL_INFEASIBLE
                           : primal.present               ? HPLP_STATUS_PRIMAL_INFEASIBLE
                                                          : HPLP_STATUS_DUAL_INFEASIBLE;
        finish(status, cx, cy, e);
        return;
      }
    }
    bool restart = restarted && should_restart(cfg, ep, k, res, res_epoch_start);  // :483-489
    if (restarted && !restart && cfg.restart_kind == HPLP_RESTART_ADAPTIVE && cfg.adaptive_stall_cap > 0 &&
        k >= cfg.adaptive_stall_cap)
      restart = true;
    if (restart) {  // :490-500
      epochs.back().len = k;
      x = mx, y = my;
      a_x = a_x_avg;
      count = 0;
      ready = false;
      ++ep;
      k = 0;
    } else {
      x = std::move(sr.x);
      y = std::move(sr.y);
      a_x = std::move(sr.a_x_next);
      ++k;
    }
    ++it;
  }
}

// ---- to_standard_form: src/lp_model.cpp:155-325 ----------------------------
struct StdForm {
  Lp lp;
  // VariableMap (inc/lp_model.hpp:102-119), flattened.
  std::vector<int> kind;  // 0 shifted, 1 mirrored, 2 split
  std::vector<int64_t> col, neg_col;
  std::vector<double> offset;
  double objective_sign = 1.0, objective_constant = 0.0;
};

StdForm to_standard_form(const hplp_general_t* g) {
  const int64_t m = g->m, n = g->n;
  // validate_general_form: src/lp_model.cpp:96-134.
  for (int64_t j = 0; j < n; ++j) {
    if (std::isnan(g->col_lower[j]) || std::isnan(g->col_upper[j]) || !std::isfinite(g->objective[j]))
      throw std::invalid_argument("GeneralFormLP: non-finite data for column 'c" + std::to_string(j) + "'");
    if (g->col_lower[j] > g->col_upper[j])
      throw std::invalid_argument("GeneralFormLP: inconsistent bounds for 'c" + std::to_string(j) +
                                  "' (lower > upper)");
  }
  auto has_range = [&](int64_t i) { return g->row_range && !std::isnan(g->row_range[i]); };
  for (int64_t i = 0; i < m; ++i)
    if (!std::isfinite(g->row_rhs[i]) || (has_range(i) && !std::isfinite(g->row_range[i])))
      throw std::invalid_argument("GeneralFormLP: non-finite rhs/range for row 'r" + std::to_string(i) + "'");
  for (int64_t p = 0; p < g->row_ptr[m]; ++p) {
    if (g->col_idx[p] < 0 || g->col_idx[p] >= n)
      throw std::invalid_argument("GeneralFormLP: entry index out of range");
    if (!std::isfinite(g->val[p])) throw std::invalid_argument("GeneralFormLP: non-finite matrix entry");
  }
  for (int64_t i = 0; i < m; ++i) {
    std::vector<int32_t> cols(g->col_idx + g->row_ptr[i], g->col_idx + g->row_ptr[i + 1]);
    std::sort(cols.begin(), cols.end());
    if (std::adjacent_find(cols.begin(), cols.end()) != cols.end())
      throw std::invalid_argument("GeneralFormLP: duplicate matrix entry");
  }
  const double sense = g->maximize ? -1.0 : 1.0;
  struct Work { double lo, hi, obj; };
  std::vector<Work> work(static_cast<std::size_t>(n));
  for (int64_t j = 0; j < n; ++j) work[j] = {g->col_lower[j], g->col_upper[j], sense * g->objective[j]};
  // Stage 1 (:175-199): rows become equalities, row_interval (:139-151).
  Vec row_b(static_cast<std::size_t>(m), 0.0);
  std::vector<int64_t> slack_item(static_cast<std::size_t>(m), -1);
  std::vector<double> slack_sign(static_cast<std::size_t>(m), 0.0);
  for (int64_t i = 0; i < m; ++i) {
    double lo, hi;
    const double rhs = g->row_rhs[i];
    switch (g->row_relation[i]) {
      case HPLP_ROW_LE:
        lo = has_range(i) ? rhs - std::abs(g->row_range[i]) : -kInf;
        hi = rhs;
        break;
      case HPLP_ROW_GE:
        lo = rhs;
        hi = has_range(i) ? rhs + std::abs(g->row_range[i]) : kInf;
        break;
      default:
        if (!has_range(i)) {
          lo = hi = rhs;
        } else if (g->row_range[i] >= 0) {
          lo = rhs;
          hi = rhs + g->row_range[i];
        } else {
          lo = rhs + g->row_range[i];
          hi = rhs;
        }
    }
    if (lo == hi) {
      row_b[i] = lo;
    } else if (hi < kInf) {
      row_b[i] = hi;
      slack_sign[i] = 1.0;
      slack_item[i] = static_cast<int64_t>(work.size());
      work.push_back({0.0, lo > -kInf ? hi - lo : kInf, 0.0});
    } else {
      row_b[i] = lo;
      slack_sign[i] = -1.0;
      slack_item[i] = static_cast<int64_t>(work.size());
      work.push_back({0.0, kInf, 0.0});
    }
  }
  // Stage 2 (:201-253): variable transforms and pending bound rows.
  std::vector<int> kind(work.size());
  std::vector<int64_t> tcol(work.size()), tneg(work.size(), 0);
  std::vector<double> toff(work.size(), 0.0);
  Vec c_std;
  double shift_const = 0.0;
  std::vector<std::pair<int64_t, double>> pending;
  int64_t next_col = 0;
  for (std::size_t w = 0; w < work.size(); ++w) {
    const Work& wc = work[w];
    if (wc.lo == -kInf && wc.hi == kInf) {
      kind[w] = 2;
      tcol[w] = next_col++;
      tneg[w] = next_col++;
      c_std.push_back(wc.obj);
      c_std.push_back(-wc.obj);
    } else if (wc.lo > -kInf) {
      kind[w] = 0;
      tcol[w] = next_col++;
      toff[w] = wc.lo;
      c_std.push_back(wc.obj);
      shift_const += wc.obj * wc.lo;
      if (wc.hi < kInf) pending.push_back({tcol[w], wc.hi - wc.lo});
    } else {
      kind[w] = 1;
      tcol[w] = next_col++;
      toff[w] = wc.hi;
      c_std.push_back(-wc.obj);
      shift_const += wc.obj * wc.hi;
    }
  }
  const int64_t m_std = m + static_cast<int64_t>(pending.size());
  std::vector<int64_t> bound_slack(pending.size());
  for (std::size_t t = 0; t < pending.size(); ++t) {
    bound_slack[t] = next_col++;
    c_std.push_back(0.0);
  }
  const int64_t n_std = next_col;
  // Emission (:279-313): entries in input order, then row slacks, then the
  // bound rows; b shifted by lower/upper offsets in entry order.
  struct T { int64_t r, c; double v; };
  std::vector<T> trip;
  Vec b_std(static_cast<std::size_t>(m_std), 0.0);
  for (int64_t i = 0; i < m; ++i) b_std[i] = row_b[i];
  for (int64_t i = 0; i < m; ++i)
    for (int64_t p = g->row_ptr[i]; p < g->row_ptr[i + 1]; ++p) {
      const int64_t j = g->col_idx[p];
      const double v = g->val[p];
      switch (kind[j]) {
        case 0:
          trip.push_back({i, tcol[j], v});
          b_std[i] -= v * toff[j];
          break;
        case 1:
          trip.push_back({i, tcol[j], -v});
          b_std[i] -= v * toff[j];
          break;
        default:
          trip.push_back({i, tcol[j], v});
          trip.push_back({i, tneg[j], -v});
      }
    }
  for (int64_t i = 0; i < m; ++i)
    if (slack_item[i] >= 0) trip.push_back({i, tcol[slack_item[i]], slack_sign[i]});
  for (std::size_t t = 0; t < pending.size(); ++t) {
    const int64_t r = m + static_cast<int64_t>(t);
    trip.push_back({r, pending[t].first, 1.0});
    trip.push_back({r, bound_slack[t], 1.0});
    b_std[r] = pending[t].second;
  }
  std::vector<int64_t> rp(static_cast<std::size_t>(m_std) + 1, 0);
  for (const T& t : trip) ++rp[t.r + 1];
  for (int64_t i = 0; i < m_std; ++i) rp[i + 1] += rp[i];
  std::vector<int32_t> ci(trip.size());
  std::vector<double> cv(trip.size());
  std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
  for (const T& t : trip) {
    ci[fill[t.r]] = static_cast<int32_t>(t.c);
    cv[fill[t.r]++] = t.v;
  }
  StdForm s;
  s.lp.a = make_csr(m_std, n_std, rp.data(), ci.data(), cv.data());
  if (!all_finite(b_std) || !all_finite(c_std))  // StandardFormLP ctor, src/lp_model.cpp:40-42
    throw std::invalid_argument("StandardFormLP: non-finite b or c");
  s.lp.b = std::move(b_std);
  s.lp.c = std::move(c_std);
  for (int64_t j = 0; j < n; ++j) {
    s.kind.push_back(kind[j]);
    s.col.push_back(tcol[j]);
    s.neg_col.push_back(tneg[j]);
    s.offset.push_back(toff[j]);
  }
  s.objective_sign = sense;
  s.objective_constant = sense * shift_const + g->objective_constant;
  return s;
}

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HPLP_OK;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return HPLP_EDOMAIN;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return HPLP_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HPLP_ESTATE;
  }
}

Vec vec(const double* p, int64_t n) { return Vec(p, p + n); }
void put(const Vec& v, double* o) {
  if (o) std::copy(v.begin(), v.end(), o);
}

}  // namespace orc

using orc::guarded;

extern "C" {

const char* orc_last_error(void) { return orc::g_err.c_str(); }

int orc_lp_create(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                  const double* val, const double* b, const double* c, void** out) {
  return guarded([&] {
    auto* lp = new orc::Lp{orc::make_csr(m, n, row_ptr, col_idx, val), orc::vec(b, m), orc::vec(c, n), {}};
    if (!orc::all_finite(lp->b) || !orc::all_finite(lp->c)) {
      delete lp;
      throw std::invalid_argument("StandardFormLP: non-finite b or c");
    }
    *out = lp;
  });
}

void orc_lp_free(void* h) { delete static_cast<orc::Lp*>(h); }

// The start vector of power_iteration above (src/sparse_matrix.cpp:145-151),
// drawn sequentially: the checker for hplp_power_start.
int orc_power_start(int64_t n, uint64_t seed, double* x) {
  return guarded([&] {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> dist(0.0, 1.0);
    orc::Vec v(static_cast<std::size_t>(n));
    for (auto& e : v) e = dist(gen);
    double xn = orc::norm(v);
    if (xn == 0.0) std::fill(v.begin(), v.end(), 1.0), xn = orc::norm(v);
    for (std::size_t i = 0; i < v.size(); ++i) x[i] = v[i] / xn;
  });
}

// Box form: upper bounds u (n values, >= 0, +inf = none); NULL clears.
int orc_lp_set_box(void* h, const double* u) {
  return guarded([&] {
    auto& lp = *static_cast<orc::Lp*>(h);
    if (!u) {
      lp.u.clear();
      return;
    }
    lp.u = orc::vec(u, lp.a.cols);
    for (double v : lp.u)
      if (std::isnan(v) || v < 0.0) throw std::invalid_argument("box form: upper bounds must be >= 0 (or +inf)");
  });
}

int orc_spmv(void* h, const double* x, double* out) {
  return guarded([&] {
    auto& lp = *static_cast<orc::Lp*>(h);
    orc::put(orc::spmv(lp.a, orc::vec(x, lp.a.cols)), out);
  });
}

int orc_spmv_transpose(void* h, const double* y, double* out) {
  return guarded([&] {
    auto& lp = *static_cast<orc::Lp*>(h);
    orc::put(orc::spmv_t(lp.a, orc::vec(y, lp.a.rows)), out);
  });
}

int orc_power_iteration(void* h, double tol, int64_t max_iters, uint64_t seed, double* sigma,
                        int64_t* iters, int32_t* converged, double* seconds) {
  return guarded([&] {
    auto t0 = orc::Clock::now();
    orc::Power p = orc::power_iteration(static_cast<orc::Lp*>(h)->a, tol, max_iters, seed);
    if (seconds) *seconds = std::chrono::duration<double>(orc::Clock::now() - t0).count();
    *sigma = p.sigma;
    *iters = p.iterations;
    *converged = p.converged ? 1 : 0;
  });
}

int orc_pdhg_step(void* h, double eta, const double* x, const double* y, const double* a_x,
                  double* x_next, double* y_next, double* a_x_next, double* at_y) {
  return guarded([&] {
    auto& lp = *static_cast<orc::Lp*>(h);
    orc::Step s = orc::pdhg_step(orc::vec(x, lp.a.cols), orc::vec(y, lp.a.rows), lp, eta,
                                 orc::vec(a_x, lp.a.rows));
    orc::put(s.x, x_next);
    orc::put(s.y, y_next);
    orc::put(s.a_x_next, a_x_next);
    orc::put(s.at_y, at_y);
  });
}

int orc_kkt_error(void* h, const double* x, const double* y, hplp_kkt_t* out) {
  return guarded([&] {
    auto& lp = *static_cast<orc::Lp*>(h);
    orc::Vec xv = orc::vec(x, lp.a.cols), yv = orc::vec(y, lp.a.rows);
    orc::Kkt e = orc::kkt(xv, yv, lp, orc::spmv(lp.a, xv), orc::spmv_t(lp.a, yv));
    *out = {e.p, e.d, e.g, e.max};
  });
}

int orc_canonical_norm_with_product(int64_t n, int64_t m, const double* dx, const double* dy,
                                    const double* a_dx, double eta, double* out) {
  return guarded([&] { *out = orc::canonical(orc::vec(dx, n), orc::vec(dy, m), orc::vec(a_dx, m), eta); });
}

int orc_validate_primal(void* h, const double* v_y, double tol, double sigma, double* rep4) {
  return guarded([&] {
    auto& lp = *static_cast<orc::Lp*>(h);
    orc::Farkas f = orc::validate_primal(orc::vec(v_y, lp.a.rows), lp, tol, sigma);
    rep4[0] = f.residual;
    rep4[1] = f.margin;
    rep4[2] = f.orientation;
    rep4[3] = f.valid ? 1.0 : 0.0;
  });
}

int orc_validate_dual(void* h, const double* v_x, double tol, double sigma, double* rep4) {
  return guarded([&] {
    auto& lp = *static_cast<orc::Lp*>(h);
    orc::Farkas f = orc::validate_dual(orc::vec(v_x, lp.a.cols), lp, tol, sigma);
    rep4[0] = f.residual;
    rep4[1] = f.margin;
    rep4[2] = f.orientation;
    rep4[3] = f.valid ? 1.0 : 0.0;
  });
}

int orc_should_restart(int32_t kind, int64_t k_star, double beta, int64_t tau0, int64_t n,
                       int64_t k, double res_now, double res_start) {
  hplp_config_t c = hplp_config_default();
  c.restart_kind = kind;
  c.k_star = k_star;
  c.beta = beta;
  c.tau0 = tau0;
  return orc::should_restart(c, n, k, res_now, res_start) ? 1 : 0;
}

int orc_lp_solve(void* h, const hplp_config_t* cfg, hplp_io_t* io, hplp_result_t* res) {
  return guarded([&] { orc::solve(*static_cast<orc::Lp*>(h), *cfg, io, res); });
}

int orc_lp_solve_baseline(void* h, int32_t mode, const hplp_config_t* cfg, hplp_io_t* io, hplp_result_t* res) {
  return guarded([&] {
    if (mode < 0 || mode > 2) throw std::invalid_argument("solve_baseline: mode in 0..2");
    orc::solve_baseline(*static_cast<orc::Lp*>(h), *cfg, mode, io, res);
  });
}

int orc_to_standard_form(const hplp_general_t* g, void** out, int64_t* m_s, int64_t* n_s,
                         int64_t* nnz_s) {
  return guarded([&] {
    auto* s = new orc::StdForm(orc::to_standard_form(g));
    *m_s = s->lp.a.rows;
    *n_s = s->lp.a.cols;
    *nnz_s = s->lp.a.nnz();
    *out = s;
  });
}

int orc_std_export(void* h, int64_t* row_ptr, int32_t* col_idx, double* val, double* b, double* c) {
  return guarded([&] {
    auto& s = *static_cast<orc::StdForm*>(h);
    std::copy(s.lp.a.rp.begin(), s.lp.a.rp.end(), row_ptr);
    std::copy(s.lp.a.ci.begin(), s.lp.a.ci.end(), col_idx);
    std::copy(s.lp.a.rv.begin(), s.lp.a.rv.end(), val);
    orc::put(s.lp.b, b);
    orc::put(s.lp.c, c);
  });
}

// VariableMap::recover_primal (src/lp_model.cpp:65-85) / recover_objective
// (inc/lp_model.hpp:116-118).
int orc_std_recover(void* h, const double* x_std, double* x_orig, double std_objective,
                    double* objective) {
  return guarded([&] {
    auto& s = *static_cast<orc::StdForm*>(h);
    if (x_std && x_orig)
      for (std::size_t j = 0; j < s.kind.size(); ++j) {
        switch (s.kind[j]) {
          case 0: x_orig[j] = s.offset[j] + x_std[s.col[j]]; break;
          case 1: x_orig[j] = s.offset[j] - x_std[s.col[j]]; break;
          default: x_orig[j] = x_std[s.col[j]] - x_std[s.neg_col[j]];
        }
      }
    if (objective) *objective = s.objective_sign * std_objective + s.objective_constant;
  });
}

int orc_std_lp(void* h, void** out) {
  return guarded([&] { *out = new orc::Lp(static_cast<orc::StdForm*>(h)->lp); });
}

void orc_std_free(void* h) { delete static_cast<orc::StdForm*>(h); }

}  // extern "C"
