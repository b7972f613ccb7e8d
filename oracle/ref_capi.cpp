// TEST INFRASTRUCTURE ONLY.  Never linked into the product.
//
// C-ABI harness around the UNMODIFIED reference library (/root/reference/proj,
// compiled by oracle/build_ref.sh against oracle/eigen_shim).  It lets the
// Python tests and bench.py's reference arm call the reference's own public
// API -- SparseMatrix, to_standard_form, power_iteration, pdhg_step,
// kkt_error, validate_*_infeasibility, should_restart, solve() -- with plain
// pointers.  Output lands in oracle/_ref/libhplp_ref.so (git-ignored).
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hplp/baselines.hpp"
#include "hplp/infeasibility.hpp"
#include "hplp/lp_model.hpp"
#include "hplp/pdhg_core.hpp"
#include "hplp/solver.hpp"
#include "hplp/sparse_matrix.hpp"
#include "hplp_types.h"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HPLP_OK;
  } catch (const std::domain_error& e) {
    return fail(e, HPLP_EDOMAIN);
  } catch (const std::invalid_argument& e) {
    return fail(e, HPLP_EINVAL);
  } catch (const std::exception& e) {
    return fail(e, HPLP_ESTATE);
  }
}

std::vector<hplp::Triplet> csr_triplets(int64_t m, const int64_t* row_ptr,
                                        const int32_t* col_idx, const double* val) {
  std::vector<hplp::Triplet> t;
  t.reserve(static_cast<std::size_t>(row_ptr[m]));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
      t.push_back({i, col_idx[p], val[p]});
  return t;
}

hplp::Vector vec(const double* p, int64_t n) {
  hplp::Vector v(n);
  if (n) std::memcpy(v.data(), p, sizeof(double) * static_cast<std::size_t>(n));
  return v;
}

void put(const hplp::Vector& v, double* out) {
  if (out && v.size()) std::memcpy(out, v.data(), sizeof(double) * static_cast<std::size_t>(v.size()));
}

hplp::SolverConfig to_config(const hplp_config_t* c) {
  hplp::SolverConfig s;
  switch (c->restart_kind) {
    case HPLP_RESTART_FIXED:
      s.restart = hplp::RestartScheme::fixed(c->k_star);
      break;
    case HPLP_RESTART_NONE:
      s.restart = hplp::RestartScheme::none();
      break;
    default:
      s.restart = hplp::RestartScheme::adaptive(c->beta, c->tau0);
  }
  s.restart.k_star = c->k_star;
  s.tolerance = c->tolerance;
  s.iteration_limit = c->iteration_limit;
  s.time_limit_seconds = c->time_limit_seconds;
  if (c->has_eta_override) s.eta_override = c->eta_override;
  s.infeasibility_check_period = c->infeasibility_check_period;
  s.trace_period = c->trace_period;
  s.certificate_tolerance = c->certificate_tolerance;
  s.tol_active = c->tol_active;
  s.adaptive_stall_cap = c->adaptive_stall_cap;
  s.seed = c->seed;
  return s;
}

void put_kkt(const hplp::KktError& e, hplp_kkt_t* o) {
  o->primal_residual = e.primal_residual;
  o->dual_residual = e.dual_residual;
  o->gap_residual = e.gap_residual;
  o->max_relative = e.max_relative;
}

void put_cert(const std::optional<hplp::Certificate>& c, hplp_cert_meta_t* m, double* vec_out) {
  std::memset(m, 0, sizeof(*m));
  if (!c) return;
  m->present = 1;
  m->source = c->source == hplp::CandidateSource::kNormalizedIterate
                  ? HPLP_SOURCE_NORMALIZED_ITERATE
                  : HPLP_SOURCE_ITERATE_DIFFERENCE;
  m->orientation = c->orientation == hplp::Orientation::kAsIs ? HPLP_ORIENT_AS_IS
                                                              : HPLP_ORIENT_NEGATED;
  m->at_iteration = c->at_iteration;
  m->residual = c->residual;
  m->margin = c->margin;
  put(c->vector, vec_out);
}

struct RefLp {
  hplp::StandardFormLP lp;
};

struct RefStd {
  hplp::StandardFormLP lp;
  hplp::VariableMap map;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_lp_create(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                  const double* val, const double* b, const double* c, void** out) {
  return guarded([&] {
    hplp::SparseMatrix a(m, n, csr_triplets(m, row_ptr, col_idx, val));
    *out = new RefLp{hplp::StandardFormLP(std::move(a), vec(b, m), vec(c, n))};
  });
}

void ref_lp_free(void* h) { delete static_cast<RefLp*>(h); }

int ref_spmv(void* h, const double* x, double* out) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    put(hplp::spmv(lp.a, vec(x, lp.num_cols())), out);
  });
}

int ref_spmv_transpose(void* h, const double* y, double* out) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    put(hplp::spmv_transpose(lp.a, vec(y, lp.num_rows())), out);
  });
}

int ref_power_iteration(void* h, double tol, int64_t max_iters, uint64_t seed,
                        double* sigma, int64_t* iters, int32_t* converged,
                        double* seconds) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    auto t0 = std::chrono::steady_clock::now();
    hplp::PowerIterationResult r = hplp::power_iteration(lp.a, tol, max_iters, seed);
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *sigma = r.sigma;
    *iters = r.iterations;
    *converged = r.converged ? 1 : 0;
  });
}

// One application of T with a caller-supplied A*x (pdhg_step_with_products,
// src/pdhg_core.cpp:75-87).
int ref_pdhg_step(void* h, double eta, const double* x, const double* y, const double* a_x,
                  double* x_next, double* y_next, double* a_x_next, double* at_y) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    hplp::Iterate z{vec(x, lp.num_cols()), vec(y, lp.num_rows())};
    hplp::PdhgStepResult r = hplp::pdhg_step_with_products(
        z, lp, hplp::StepSize(eta, 0.0), vec(a_x, lp.num_rows()));
    put(r.next.x, x_next);
    put(r.next.y, y_next);
    put(r.a_x_next, a_x_next);
    put(r.at_y, at_y);
  });
}

int ref_kkt_error(void* h, const double* x, const double* y, hplp_kkt_t* out) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    hplp::Iterate z{vec(x, lp.num_cols()), vec(y, lp.num_rows())};
    put_kkt(hplp::kkt_error(z, lp), out);
  });
}

int ref_canonical_norm_with_product(int64_t n, int64_t m, const double* dx, const double* dy,
                                    const double* a_dx, double eta, double* out) {
  return guarded([&] {
    hplp::Iterate z{vec(dx, n), vec(dy, m)};
    *out = hplp::canonical_norm_with_product(z, vec(a_dx, m), eta);
  });
}

int ref_fixed_point_residual(void* h, double eta, const double* x, const double* y, double* out) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    hplp::Iterate z{vec(x, lp.num_cols()), vec(y, lp.num_rows())};
    hplp::StepSize step(eta, 0.0);
    *out = hplp::fixed_point_residual(z, lp, step, hplp::CanonicalNorm(lp, step));
  });
}

// FarkasReport flattened: [residual, margin, orientation, valid].
int ref_validate_primal(void* h, const double* v_y, double tol, double sigma, double* rep4) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    hplp::FarkasReport r =
        hplp::validate_primal_infeasibility(vec(v_y, lp.num_rows()), lp, tol, sigma);
    rep4[0] = r.primal_cert_residual;
    rep4[1] = r.primal_margin;
    rep4[2] = r.primal_orientation == hplp::Orientation::kAsIs ? 0.0 : 1.0;
    rep4[3] = r.primal_valid ? 1.0 : 0.0;
  });
}

int ref_validate_dual(void* h, const double* v_x, double tol, double sigma, double* rep4) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    hplp::FarkasReport r =
        hplp::validate_dual_infeasibility(vec(v_x, lp.num_cols()), lp, tol, sigma);
    rep4[0] = r.dual_cert_residual;
    rep4[1] = r.dual_margin;
    rep4[2] = r.dual_orientation == hplp::Orientation::kAsIs ? 0.0 : 1.0;
    rep4[3] = r.dual_valid ? 1.0 : 0.0;
  });
}

int ref_should_restart(int32_t kind, int64_t k_star, double beta, int64_t tau0, int64_t n,
                       int64_t k, double res_now, double res_start) {
  hplp::RestartScheme s = kind == HPLP_RESTART_FIXED    ? hplp::RestartScheme::fixed(k_star)
                          : kind == HPLP_RESTART_NONE   ? hplp::RestartScheme::none()
                                                        : hplp::RestartScheme::adaptive(beta, tau0);
  return hplp::should_restart(s, n, k, res_now, res_start) ? 1 : 0;
}

const char* ref_status_string(int32_t status) {
  return hplp::to_string(static_cast<hplp::SolveStatus>(status));
}

int ref_lp_solve_impl(void* h, int32_t baseline, const hplp_config_t* cfg, hplp_io_t* io, hplp_result_t* res);

int ref_lp_solve(void* h, const hplp_config_t* cfg, hplp_io_t* io, hplp_result_t* res) {
  return ref_lp_solve_impl(h, -1, cfg, io, res);
}

// solve_baseline (src/solver.cpp:344-509): mode 0 vanilla, 1 averaged,
// 2 restarted average.
int ref_lp_solve_baseline(void* h, int32_t mode, const hplp_config_t* cfg, hplp_io_t* io, hplp_result_t* res) {
  if (mode < 0 || mode > 2) return guarded([] { throw std::invalid_argument("solve_baseline: mode in 0..2"); });
  return ref_lp_solve_impl(h, mode, cfg, io, res);
}

int ref_lp_solve_impl(void* h, int32_t baseline, const hplp_config_t* cfg, hplp_io_t* io, hplp_result_t* res) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    hplp::SolverConfig config = to_config(cfg);
    if (io && io->init_x && io->init_y)
      config.initial_iterate =
          hplp::Iterate{vec(io->init_x, lp.num_cols()), vec(io->init_y, lp.num_rows())};
    if (io && io->trace_fn && cfg->trace_period > 0) {
      config.trace_sink = [io](const hplp::TraceRecord& rec, const hplp::Iterate& z) {
        hplp_trace_t t;
        t.epoch = rec.epoch;
        t.inner = rec.inner;
        t.iteration = rec.iteration;
        t.fixed_point_residual = rec.fixed_point_residual;
        put_kkt(rec.kkt, &t.kkt);
        t.candidate_norm_normalized = rec.candidate_norm_normalized;
        t.candidate_norm_difference = rec.candidate_norm_difference;
        t.wall_seconds = rec.wall_seconds;
        std::vector<int64_t> sets;
        for (auto v : {&rec.partition.n_set, &rec.partition.b1_set, &rec.partition.b2_set})
          for (auto i : *v) sets.push_back(static_cast<int64_t>(i));
        t.partition_n = static_cast<int64_t>(rec.partition.n_set.size());
        t.partition_b1 = static_cast<int64_t>(rec.partition.b1_set.size());
        t.partition_b2 = static_cast<int64_t>(rec.partition.b2_set.size());
        t.partition_sets = sets.data();
        io->trace_fn(&t, z.x.data(), z.x.size(), z.y.data(), z.y.size(), io->trace_user);
      };
    }
    hplp::SolveResult r =
        baseline < 0 ? hplp::solve(lp, config)
                     : hplp::solve_baseline(lp, config,
                                            baseline == 0   ? hplp::BaselineMode::kVanilla
                                            : baseline == 1 ? hplp::BaselineMode::kAveraged
                                                            : hplp::BaselineMode::kRestartedAverage);
    std::memset(res, 0, sizeof(*res));
    res->status = static_cast<int32_t>(r.status);
    res->iterations = r.totals.iterations;
    res->spmv_count = r.totals.spmv_count;
    res->wall_seconds = r.totals.wall_seconds;
    res->eta = r.totals.eta;
    res->sigma_estimate = r.totals.sigma_estimate;
    put_kkt(r.final_kkt, &res->final_kkt);
    res->n_epochs = static_cast<int64_t>(r.epochs.size());
    if (io) {
      put(r.final_iterate.x, io->x);
      put(r.final_iterate.y, io->y);
      put_cert(r.primal_certificate, &res->primal_cert, io->primal_cert);
      put_cert(r.dual_certificate, &res->dual_cert, io->dual_cert);
      if (io->epochs) {
        for (std::size_t e = 0; e < r.epochs.size() && static_cast<int64_t>(e) < io->epochs_capacity; ++e) {
          io->epochs[e].epoch = r.epochs[e].epoch;
          io->epochs[e].restart_length = r.epochs[e].restart_length;
          io->epochs[e].residual_at_start = r.epochs[e].residual_at_start;
          put_kkt(r.epochs[e].kkt_at_start, &io->epochs[e].kkt_at_start);
        }
      }
    } else {
      put_cert(r.primal_certificate, &res->primal_cert, nullptr);
      put_cert(r.dual_certificate, &res->dual_cert, nullptr);
    }
  });
}

// General form -> standard form through the reference's to_standard_form.
int ref_to_standard_form(const hplp_general_t* g, void** out, int64_t* m_s, int64_t* n_s,
                         int64_t* nnz_s) {
  return guarded([&] {
    hplp::GeneralFormLP gl;
    gl.maximize = g->maximize != 0;
    gl.objective_constant = g->objective_constant;
    gl.rows.resize(static_cast<std::size_t>(g->m));
    for (int64_t i = 0; i < g->m; ++i) {
      auto& r = gl.rows[static_cast<std::size_t>(i)];
      r.name = "r" + std::to_string(i);
      r.relation = g->row_relation[i] == HPLP_ROW_LE   ? hplp::RowRelation::kLessEqual
                   : g->row_relation[i] == HPLP_ROW_GE ? hplp::RowRelation::kGreaterEqual
                                                       : hplp::RowRelation::kEqual;
      r.rhs = g->row_rhs[i];
      if (g->row_range && !std::isnan(g->row_range[i])) r.range = g->row_range[i];
    }
    gl.columns.resize(static_cast<std::size_t>(g->n));
    gl.objective.resize(static_cast<std::size_t>(g->n));
    for (int64_t j = 0; j < g->n; ++j) {
      auto& c = gl.columns[static_cast<std::size_t>(j)];
      c.name = "c" + std::to_string(j);
      c.lower = g->col_lower[j];
      c.upper = g->col_upper[j];
      gl.objective[static_cast<std::size_t>(j)] = g->objective[j];
    }
    gl.entries = csr_triplets(g->m, g->row_ptr, g->col_idx, g->val);
    auto [lp, map] = hplp::to_standard_form(gl);
    auto* h = new RefStd{std::move(lp), std::move(map)};
    *m_s = h->lp.num_rows();
    *n_s = h->lp.num_cols();
    *nnz_s = h->lp.a.nonzeros();
    *out = h;
  });
}

// Standard-form CSR (row-major traversal order of the reference's storage).
int ref_std_export(void* h, int64_t* row_ptr, int32_t* col_idx, double* val, double* b,
                   double* c) {
  return guarded([&] {
    const auto& s = *static_cast<RefStd*>(h);
    const auto& br = s.lp.a.by_row();
    for (int64_t i = 0; i <= s.lp.num_rows(); ++i) row_ptr[i] = br.outerIndexPtr()[i];
    for (int64_t p = 0; p < s.lp.a.nonzeros(); ++p) {
      col_idx[p] = br.innerIndexPtr()[p];
      val[p] = br.valuePtr()[p];
    }
    put(s.lp.b, b);
    put(s.lp.c, c);
  });
}

int ref_std_recover(void* h, const double* x_std, double* x_orig, double std_objective,
                    double* objective) {
  return guarded([&] {
    const auto& s = *static_cast<RefStd*>(h);
    if (x_std && x_orig) put(s.map.recover_primal(vec(x_std, s.map.standard_cols)), x_orig);
    if (objective) *objective = s.map.recover_objective(std_objective);
  });
}

// Standard-form LP handle (for ref_lp_* calls) built from a converted problem.
int ref_std_lp(void* h, void** out) {
  return guarded([&] { *out = new RefLp{static_cast<RefStd*>(h)->lp}; });
}

void ref_std_free(void* h) { delete static_cast<RefStd*>(h); }

// Proposition-1 harness (src/baselines.cpp:33-55), used by the KAT tests.
int ref_trajectory_deviation(void* h, const double* x0, const double* y0, int64_t k_max,
                             double eta, int32_t unconstrained, double* out) {
  return guarded([&] {
    const auto& lp = static_cast<RefLp*>(h)->lp;
    hplp::Iterate z0{vec(x0, lp.num_cols()), vec(y0, lp.num_rows())};
    *out = hplp::trajectory_deviation(lp, z0, k_max, hplp::StepSize(eta, 0.0), unconstrained != 0);
  });
}

}  // extern "C"
