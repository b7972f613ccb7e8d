// Seeded synthetic LP generator (include/hplp_gen.h).  Host C++ only.
//
// Planted instances follow BASELINE.json configs[0,1,2,4] as resolved in
// x* has 40% of entries at a bound (0 or u, 50/50) and the rest
// U(0,u); y* is N(0,1) on '=' rows and, on '>=' rows, |N(0,1)| on the active
// half and 0 on the rest; b = A x* except on inactive '>=' rows, where
// b = A x* - U[0,1] (BASELINE says "plus slack", which would make x* violate
// A x >= b); c = A^T y* + s with s >= 0 at the lower bound, <= 0 at the
// upper bound and 0 in the interior, so (x*, y*) is a KKT pair and c^T x* is
// the optimum.  Transport follows configs[3].
#include "hplp_gen.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "hplp_types.h"

namespace {

thread_local std::string g_err;

struct Gen {
  int64_t m = 0, n = 0;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
  std::vector<int32_t> rel;
  std::vector<double> rhs, lo, hi, obj, x_star;
  double planted = std::numeric_limits<double>::quiet_NaN();
};

struct Rng {
  std::mt19937_64 g;
  std::normal_distribution<double> nd{0.0, 1.0};
  explicit Rng(uint64_t s) : g(s) {}
  double u01() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  double uni(double a, double b) { return a + (b - a) * u01(); }
  double normal() { return nd(g); }
  int64_t below(int64_t k) { return static_cast<int64_t>(g() % static_cast<uint64_t>(k)); }
};

// k distinct uniform columns of [0, n), ascending.
void distinct_cols(Rng& r, int64_t n, int64_t k, std::vector<int32_t>& out) {
  out.clear();
  if (k >= n) {
    out.resize(static_cast<std::size_t>(n));
    std::iota(out.begin(), out.end(), 0);
    return;
  }
  while (static_cast<int64_t>(out.size()) < k) {
    const int64_t need = k - static_cast<int64_t>(out.size());
    for (int64_t t = 0; t < need; ++t) out.push_back(static_cast<int32_t>(r.below(n)));
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
  }
}

std::vector<int64_t> zipf_lengths(Rng& r, const hplp_gen_params_t& p) {
  const int64_t cap = p.zipf_cap;
  std::vector<double> cdf(static_cast<std::size_t>(cap));
  double acc = 0.0;
  for (int64_t k = 1; k <= cap; ++k) cdf[k - 1] = (acc += std::pow(static_cast<double>(k), -p.zipf_s));
  std::vector<int64_t> z(static_cast<std::size_t>(p.m));
  double total = 0.0;
  for (auto& zi : z) {
    const double t = r.u01() * acc;
    zi = static_cast<int64_t>(std::upper_bound(cdf.begin(), cdf.end(), t) - cdf.begin()) + 1;
    zi = std::min(zi, cap);
    total += static_cast<double>(zi);
  }
  const double scale = static_cast<double>(p.zipf_target_nnz) / total;
  std::vector<int64_t> len(z.size());
  for (std::size_t i = 0; i < z.size(); ++i)
    len[i] = std::clamp<int64_t>(std::llround(static_cast<double>(z[i]) * scale), 1, cap);
  if (p.zipf_force_cap > 0) {
    std::vector<int64_t> order(z.size());
    std::iota(order.begin(), order.end(), 0);
    const int64_t f = std::min<int64_t>(p.zipf_force_cap, p.m);
    std::partial_sort(order.begin(), order.begin() + f, order.end(),
                      [&](int64_t a, int64_t b) { return z[a] != z[b] ? z[a] > z[b] : a < b; });
    for (int64_t t = 0; t < f; ++t) len[order[t]] = cap;
  }
  return len;
}

void planted(const hplp_gen_params_t& p, Gen& g) {
  if (p.m < 1 || p.n < 1) throw std::invalid_argument("generator: m, n must be >= 1");
  Rng r(p.seed);
  const int64_t m = p.m, n = p.n;
  const int64_t m_eq = static_cast<int64_t>(std::llround(p.eq_frac * static_cast<double>(m)));
  std::vector<int64_t> len;
  if (p.zipf) {
    len = zipf_lengths(r, p);
  } else {
    len.assign(static_cast<std::size_t>(m), std::min(p.nnz_per_row, n));
  }
  g.m = m + p.infeasible_rows;
  g.n = n;
  g.rp.assign(1, 0);
  std::vector<int32_t> cols;
  for (int64_t i = 0; i < m; ++i) {
    distinct_cols(r, n, len[i], cols);
    const double scale = p.row_scale_log10 > 0
                             ? std::pow(10.0, r.uni(-p.row_scale_log10, p.row_scale_log10))
                             : 1.0;
    for (int32_t c : cols) {
      g.ci.push_back(c);
      g.v.push_back(r.normal() * scale);
    }
    g.rp.push_back(static_cast<int64_t>(g.ci.size()));
  }
  // Bounds and planted primal.
  g.lo.assign(static_cast<std::size_t>(n), 0.0);
  g.hi.resize(static_cast<std::size_t>(n));
  g.x_star.resize(static_cast<std::size_t>(n));
  std::vector<int8_t> at(static_cast<std::size_t>(n), 0);  // -1 lower, +1 upper, 0 interior
  for (int64_t j = 0; j < n; ++j) {
    g.hi[j] = r.uni(p.ub_lo, p.ub_hi);
    if (r.u01() < 0.4) {
      at[j] = r.u01() < 0.5 ? -1 : 1;
      g.x_star[j] = at[j] < 0 ? 0.0 : g.hi[j];
    } else {
      g.x_star[j] = r.u01() * g.hi[j];
      if (g.x_star[j] == 0.0) at[j] = -1;
    }
  }
  // Planted dual.
  std::vector<double> y(static_cast<std::size_t>(m), 0.0);
  std::vector<int8_t> active(static_cast<std::size_t>(m), 1);
  for (int64_t i = 0; i < m; ++i) {
    if (i < m_eq) {
      y[i] = r.normal();
    } else if (r.u01() < 0.5) {
      y[i] = std::abs(r.normal());
    } else {
      active[i] = 0;
    }
  }
  g.rel.resize(static_cast<std::size_t>(g.m));
  g.rhs.resize(static_cast<std::size_t>(g.m));
  for (int64_t i = 0; i < m; ++i) {
    double ax = 0.0;
    for (int64_t q = g.rp[i]; q < g.rp[i + 1]; ++q) ax += g.v[q] * g.x_star[g.ci[q]];
    g.rel[i] = i < m_eq ? HPLP_ROW_EQ : HPLP_ROW_GE;
    g.rhs[i] = active[i] ? ax : ax - r.u01();
  }
  std::vector<double> aty(static_cast<std::size_t>(n), 0.0);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t q = g.rp[i]; q < g.rp[i + 1]; ++q) aty[g.ci[q]] += g.v[q] * y[i];
  g.obj.resize(static_cast<std::size_t>(n));
  double cx = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    const double s = at[j] < 0 ? std::abs(r.normal()) : at[j] > 0 ? -std::abs(r.normal()) : 0.0;
    g.obj[j] = aty[j] + s;
    cx += g.obj[j] * g.x_star[j];
  }
  g.planted = cx;
  // Contradictory copies of '=' rows (configs[2]).
  if (p.infeasible_rows > 0) {
    if (m_eq < 1) throw std::invalid_argument("generator: infeasible rows need '=' rows");
    for (int64_t t = 0; t < p.infeasible_rows; ++t) {
      const int64_t src = r.below(m_eq);
      for (int64_t q = g.rp[src]; q < g.rp[src + 1]; ++q) {
        g.ci.push_back(g.ci[q]);
        g.v.push_back(g.v[q]);
      }
      g.rp.push_back(static_cast<int64_t>(g.ci.size()));
      g.rel[m + t] = HPLP_ROW_EQ;
      g.rhs[m + t] = g.rhs[src] + r.uni(5.0, 10.0);
    }
    g.planted = std::numeric_limits<double>::quiet_NaN();
    std::fill(g.x_star.begin(), g.x_star.end(), std::numeric_limits<double>::quiet_NaN());
  }
}

void transport(const hplp_gen_params_t& p, Gen& g) {
  const int64_t S = p.sources, D = p.sinks;
  if (S < 1 || D < 1) throw std::invalid_argument("generator: sources, sinks must be >= 1");
  if (S * D > std::numeric_limits<int32_t>::max())
    throw std::invalid_argument("generator: transport too large for int32 columns");
  Rng r(p.seed);
  g.m = S + D;
  g.n = S * D;
  g.obj.resize(static_cast<std::size_t>(g.n));
  for (auto& c : g.obj) c = r.uni(1.0, 100.0);
  std::vector<double> s(static_cast<std::size_t>(S)), d(static_cast<std::size_t>(D));
  double ss = 0.0, sd = 0.0;
  for (auto& v : s) ss += (v = r.uni(50.0, 150.0));
  for (auto& v : d) sd += (v = r.uni(50.0, 150.0));
  const double f = 1.1 * sd / ss;
  for (auto& v : s) v *= f;
  g.rp.assign(1, 0);
  g.ci.reserve(static_cast<std::size_t>(2 * g.n));
  for (int64_t i = 0; i < S; ++i) {  // supply rows: sum_j x_ij <= s_i
    for (int64_t j = 0; j < D; ++j) g.ci.push_back(static_cast<int32_t>(i * D + j));
    g.rp.push_back(static_cast<int64_t>(g.ci.size()));
  }
  for (int64_t j = 0; j < D; ++j) {  // demand rows: sum_i x_ij >= d_j
    for (int64_t i = 0; i < S; ++i) g.ci.push_back(static_cast<int32_t>(i * D + j));
    g.rp.push_back(static_cast<int64_t>(g.ci.size()));
  }
  g.v.assign(g.ci.size(), 1.0);
  g.rel.resize(static_cast<std::size_t>(g.m));
  g.rhs.resize(static_cast<std::size_t>(g.m));
  for (int64_t i = 0; i < S; ++i) g.rel[i] = HPLP_ROW_LE, g.rhs[i] = s[i];
  for (int64_t j = 0; j < D; ++j) g.rel[S + j] = HPLP_ROW_GE, g.rhs[S + j] = d[j];
  g.lo.assign(static_cast<std::size_t>(g.n), 0.0);
  g.hi.assign(static_cast<std::size_t>(g.n), std::numeric_limits<double>::infinity());
  g.x_star.assign(static_cast<std::size_t>(g.n), std::numeric_limits<double>::quiet_NaN());
}

}  // namespace

extern "C" {

const char* hplp_gen_last_error(void) { return g_err.c_str(); }

int hplp_gen_preset(int32_t cfg, hplp_gen_params_t* p) {
  *p = hplp_gen_params_t{};
  p->kind = HPLP_GEN_PLANTED;
  p->eq_frac = 0.7;
  p->ub_lo = 1.0;
  p->ub_hi = 10.0;
  p->zipf_s = 1.5;
  switch (cfg) {
    case 0:  // small feasible, 0.5% per row
      p->m = 1000, p->n = 2000, p->nnz_per_row = 10, p->seed = 20240722ull;
      return HPLP_OK;
    case 1:  // medium planted, ~2M nnz, row scales 1e-2..1e2
      p->m = 100000, p->n = 200000, p->nnz_per_row = 20, p->row_scale_log10 = 2.0;
      p->seed = 20240723ull;
      return HPLP_OK;
    case 2:  // infeasible: medium generator at half size + 200 contradictory rows
      p->m = 50000, p->n = 100000, p->nnz_per_row = 20, p->row_scale_log10 = 2.0;
      p->infeasible_rows = 200, p->seed = 20240724ull;
      return HPLP_OK;
    case 3:  // transportation 2000 x 2000
      p->kind = HPLP_GEN_TRANSPORT, p->sources = 2000, p->sinks = 2000, p->seed = 20240725ull;
      return HPLP_OK;
    case 4:  // large skewed: Zipf(1.5) rows capped at 50k, ~100M nnz
      p->m = 5000000, p->n = 10000000, p->eq_frac = 0.6, p->zipf = 1, p->zipf_cap = 50000;
      p->zipf_target_nnz = 100000000, p->zipf_force_cap = 8, p->seed = 20240726ull;
      return HPLP_OK;
    default:
      g_err = "generator: unknown preset";
      return HPLP_EINVAL;
  }
}

int hplp_gen_create(const hplp_gen_params_t* p, void** handle) {
  try {
    auto* g = new Gen();
    try {
      if (p->kind == HPLP_GEN_TRANSPORT) transport(*p, *g);
      else planted(*p, *g);
    } catch (...) {
      delete g;
      throw;
    }
    *handle = g;
    return HPLP_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return HPLP_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HPLP_ENOMEM;
  }
}

void hplp_gen_dims(void* h, int64_t* m, int64_t* n, int64_t* nnz) {
  const Gen& g = *static_cast<Gen*>(h);
  *m = g.m;
  *n = g.n;
  *nnz = static_cast<int64_t>(g.ci.size());
}

int hplp_gen_export(void* h, int64_t* row_ptr, int32_t* col_idx, double* val, int32_t* row_relation,
                    double* row_rhs, double* col_lower, double* col_upper, double* objective,
                    double* planted_objective) {
  const Gen& g = *static_cast<Gen*>(h);
  std::copy(g.rp.begin(), g.rp.end(), row_ptr);
  std::copy(g.ci.begin(), g.ci.end(), col_idx);
  std::copy(g.v.begin(), g.v.end(), val);
  std::copy(g.rel.begin(), g.rel.end(), row_relation);
  std::copy(g.rhs.begin(), g.rhs.end(), row_rhs);
  std::copy(g.lo.begin(), g.lo.end(), col_lower);
  std::copy(g.hi.begin(), g.hi.end(), col_upper);
  std::copy(g.obj.begin(), g.obj.end(), objective);
  if (planted_objective) *planted_objective = g.planted;
  return HPLP_OK;
}

int hplp_gen_planted_x(void* h, double* x_star) {
  const Gen& g = *static_cast<Gen*>(h);
  std::copy(g.x_star.begin(), g.x_star.end(), x_star);
  return HPLP_OK;
}

void hplp_gen_free(void* h) { delete static_cast<Gen*>(h); }

}  // extern "C"
