// C ABI (include/hplp_gpu.h) over the C++ host driver (hplp_gpu.hpp).
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "hplp_gpu.h"
#include "hplp_gpu.hpp"
#include "hx.h"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HPLP_OK;
  } catch (const hplp_gpu::MpsParseError& e) {
    g_err = e.what();
    return HPLP_EPARSE;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return HPLP_EDOMAIN;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return HPLP_EINVAL;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return HPLP_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HPLP_ECUDA;
  }
}

void put_kkt(const hplp_gpu::KktError& e, hplp_kkt_t* o) {
  *o = {e.primal_residual, e.dual_residual, e.gap_residual, e.max_relative};
}

void put_cert(const std::optional<hplp_gpu::Certificate>& c, hplp_cert_meta_t* m, double* vec) {
  std::memset(m, 0, sizeof(*m));
  if (!c) return;
  m->present = 1;
  m->source = c->source == hplp_gpu::CandidateSource::kNormalizedIterate ? HPLP_SOURCE_NORMALIZED_ITERATE
                                                                          : HPLP_SOURCE_ITERATE_DIFFERENCE;
  m->orientation = c->orientation == hplp_gpu::Orientation::kNegated ? HPLP_ORIENT_NEGATED : HPLP_ORIENT_AS_IS;
  m->at_iteration = c->at_iteration;
  m->residual = c->residual;
  m->margin = c->margin;
  if (vec) std::memcpy(vec, c->vector.data(), c->vector.size() * sizeof(double));
}

void fill_result(const hplp_gpu::SolveResult& r, hplp_io_t* io, hplp_result_t* res) {
  std::memset(res, 0, sizeof(*res));
  res->status = static_cast<int32_t>(r.status);
  res->iterations = r.totals.iterations;
  res->spmv_count = r.totals.spmv_count;
  res->wall_seconds = r.totals.wall_seconds;
  res->eta = r.totals.eta;
  res->sigma_estimate = r.totals.sigma_estimate;
  put_kkt(r.final_kkt, &res->final_kkt);
  res->n_epochs = static_cast<int64_t>(r.epochs.size());
  put_cert(r.primal_certificate, &res->primal_cert, io ? io->primal_cert : nullptr);
  put_cert(r.dual_certificate, &res->dual_cert, io ? io->dual_cert : nullptr);
  if (!io) return;
  // (an empty final_iterate was read straight into io->x / io->y: SolverConfig::out_x)
  if (io->x && !r.final_iterate.x.empty())
    std::memcpy(io->x, r.final_iterate.x.data(), r.final_iterate.x.size() * sizeof(double));
  if (io->y && !r.final_iterate.y.empty())
    std::memcpy(io->y, r.final_iterate.y.data(), r.final_iterate.y.size() * sizeof(double));
  if (io->epochs)
    for (std::size_t e = 0; e < r.epochs.size() && static_cast<int64_t>(e) < io->epochs_capacity; ++e) {
      io->epochs[e].epoch = r.epochs[e].epoch;
      io->epochs[e].restart_length = r.epochs[e].restart_length;
      io->epochs[e].residual_at_start = r.epochs[e].residual_at_start;
      put_kkt(r.epochs[e].kkt_at_start, &io->epochs[e].kkt_at_start);
    }
}

hplp_gpu::SolverConfig config_with_io(const hplp_config_t* cfg, hplp_io_t* io, int64_t m, int64_t n) {
  hplp_gpu::SolverConfig c = hplp_gpu::from_pod(*cfg);
  if (io && io->init_x && io->init_y)
    c.initial_iterate = hplp_gpu::Iterate{std::vector<double>(io->init_x, io->init_x + n),
                                          std::vector<double>(io->init_y, io->init_y + m)};
  if (io && io->trace_fn && cfg->trace_period > 0) {
    c.trace_sink = [io](const hplp_gpu::TraceRecord& rec, const hplp_gpu::Iterate& z) {
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
      io->trace_fn(&t, z.x.data(), static_cast<int64_t>(z.x.size()), z.y.data(), static_cast<int64_t>(z.y.size()),
                   io->trace_user);
    };
  }
  return c;
}

struct StdHandle {
  hplp_gpu::StandardFormLP lp;
  hplp_gpu::VariableMap map;
};

}  // namespace

extern "C" {

const char* hplp_last_error(void) { return g_err.c_str(); }

const char* hplp_status_string(int32_t status) {
  if (status < 0 || status > 5) return "unknown";
  return hplp_gpu::to_string(static_cast<hplp_gpu::SolveStatus>(status));
}

int hplp_validate_config(const hplp_config_t* cfg) {
  return guarded([&] {
    const hplp_gpu::SolverConfig c = hplp_gpu::from_pod(*cfg);
    if (!(c.tolerance > 0.0)) throw std::invalid_argument("SolverConfig: tolerance must be > 0");
    if (c.iteration_limit < 0) throw std::invalid_argument("SolverConfig: iteration_limit must be >= 0");
    if (!(c.certificate_tolerance > 0.0))
      throw std::invalid_argument("SolverConfig: certificate_tolerance must be > 0");
    if (c.infeasibility_check_period < 0 || c.trace_period < 0 || c.adaptive_stall_cap < 0)
      throw std::invalid_argument("SolverConfig: periods must be >= 0");
    if (c.restart.kind == hplp_gpu::RestartScheme::Kind::kFixedFrequency && c.restart.k_star < 1)
      throw std::invalid_argument("RestartScheme: k_star must be >= 1");
    if (c.restart.kind == hplp_gpu::RestartScheme::Kind::kAdaptiveResidualDecay &&
        (!(c.restart.beta > 0.0) || !(c.restart.beta < 1.0) || c.restart.tau0 < 1))
      throw std::invalid_argument("RestartScheme: adaptive needs beta in (0,1) and tau0 >= 1");
  });
}

namespace {
// SparseMatrix semantics (src/sparse_matrix.cpp: rows given in any order are
// sorted, duplicates and bad entries rejected with the reference's messages).
// A matrix that is already valid CSR with ascending rows -- the common case --
// goes straight to the device, which validates ranges, finiteness, order and
// duplicates itself (hx_upload_csr); only a matrix it rejects takes the host
// path, which sorts it or reports the reference's error.
hplp_gpu::Solver* create_solver(int32_t device, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                                const double* val, const double* b, const double* c) {
  if (m >= 0 && n >= 0 && row_ptr && row_ptr[0] == 0) {
    try {
      return new hplp_gpu::Solver(device, m, n, row_ptr, col_idx, val, b, c);
    } catch (const std::invalid_argument&) {
      // fall through: the host path sorts or reports
    }
  }
  hplp_gpu::SparseMatrix a = hplp_gpu::SparseMatrix::from_csr(m, n, row_ptr, col_idx, val);
  hplp_gpu::StandardFormLP lp(std::move(a), std::vector<double>(b, b + m), std::vector<double>(c, c + n));
  return new hplp_gpu::Solver(lp, device);
}
}  // namespace

int hplp_solver_create(int32_t device, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                       const double* val, const double* b, const double* c, void** solver) {
  return guarded([&] { *solver = create_solver(device, m, n, row_ptr, col_idx, val, b, c); });
}

int hplp_solver_create_box(int32_t device, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                           const double* val, const double* b, const double* c, void** solver) {
  return guarded([&] {
    // validated with SparseMatrix semantics first (the box form keeps the
    // caller's ascending rows as they are)
    hplp_gpu::SparseMatrix a = hplp_gpu::SparseMatrix::from_csr(m, n, row_ptr, col_idx, val);
    hplp_gpu::StandardFormLP lp(std::move(a), std::vector<double>(b, b + m), std::vector<double>(c, c + n));
    *solver = new hplp_gpu::Solver(hplp_gpu::Solver::BoxFormTag{}, device, m, n, lp.a.row_ptr().data(),
                                   lp.a.col_idx().data(), lp.a.values().data(), lp.b.data(), lp.c.data());
  });
}

int hplp_box_form_dims(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                       const double* b, const double* c, int64_t* m_box, int64_t* n_box, double* upper) {
  return guarded([&] {
    hplp_gpu::SparseMatrix a = hplp_gpu::SparseMatrix::from_csr(m, n, row_ptr, col_idx, val);
    const hplp_gpu::BoxForm f = hplp_gpu::detect_box_form(m, n, a.row_ptr().data(), a.col_idx().data(),
                                                          a.values().data(), b, c);
    *m_box = f.m, *n_box = f.n;
    if (upper) std::copy(f.upper.begin(), f.upper.end(), upper);
  });
}

int hplp_solver_create_team(const int32_t* devices, int32_t ndevices, int32_t nranks, int32_t ctas_per_rank,
                            int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                            const double* b, const double* c, void** solver) {
  return guarded([&] {
    if (!devices || ndevices < 1) throw std::invalid_argument("hplp_solver_create_team: no devices");
    hplp_gpu::SparseMatrix a = hplp_gpu::SparseMatrix::from_csr(m, n, row_ptr, col_idx, val);
    std::vector<int> devs(devices, devices + ndevices);
    *solver = new hplp_gpu::Solver(devs, nranks, m, n, a.row_ptr().data(), a.col_idx().data(), a.values().data(), b, c,
                                   ctas_per_rank);
  });
}

int hplp_solver_create_rank(int32_t device, int32_t nranks, int32_t rank, int64_t m, int64_t n,
                            const int64_t* row_ptr, const int32_t* col_idx, const double* val, const double* b,
                            const double* c, void** solver) {
  return guarded([&] {
    hplp_gpu::SparseMatrix a = hplp_gpu::SparseMatrix::from_csr(m, n, row_ptr, col_idx, val);
    *solver = new hplp_gpu::Solver(device, nranks, rank, m, n, a.row_ptr().data(), a.col_idx().data(),
                                   a.values().data(), b, c);
  });
}

int hplp_solver_team_export(void* solver, void* blob, int64_t capacity, int64_t* size) {
  return guarded([&] {
    const std::vector<unsigned char> v = static_cast<hplp_gpu::Solver*>(solver)->team_export();
    if (size) *size = static_cast<int64_t>(v.size());
    if (blob) {
      if (capacity < static_cast<int64_t>(v.size())) throw std::invalid_argument("hplp_solver_team_export: blob too small");
      std::memcpy(blob, v.data(), v.size());
    }
  });
}

int hplp_solver_team_import(void* solver, const void* blob, int64_t size) {
  return guarded([&] { static_cast<hplp_gpu::Solver*>(solver)->team_import(blob, static_cast<std::size_t>(size)); });
}

int hplp_solver_solve(void* solver, const hplp_config_t* cfg, hplp_io_t* io, hplp_result_t* result) {
  return guarded([&] {
    auto* s = static_cast<hplp_gpu::Solver*>(solver);
    hplp_gpu::SolverConfig c = config_with_io(cfg, io, s->rows(), s->cols());
    if (io && io->x && io->y) c.out_x = io->x, c.out_y = io->y;  // no host staging copy of the result
    fill_result(s->solve(c), io, result);
  });
}

void* hplp_solver_hx(void* solver) { return static_cast<hplp_gpu::Solver*>(solver)->hx(); }

void* hplp_solver_rank_hx(void* solver, int32_t rank) { return static_cast<hplp_gpu::Solver*>(solver)->rank_hx(rank); }

void hplp_solver_free(void* solver) { delete static_cast<hplp_gpu::Solver*>(solver); }

int hplp_solve_csr(int32_t device, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                   const double* val, const double* b, const double* c, const hplp_config_t* cfg, hplp_io_t* io,
                   hplp_result_t* result) {
  void* s = nullptr;
  // the power iteration's start vector is drawn on a host thread while the
  // problem uploads
  hplp_gpu::PowerStartFuture start;
  if (cfg && n > 0) start = hplp_gpu::draw_power_start_async(n, cfg->seed);
  // HPLP_TIMING=1: the three stages' wall times on stderr
  const char* te = std::getenv("HPLP_TIMING");
  const bool timing = te && te[0] == '1';
  const auto t0 = std::chrono::steady_clock::now();
  auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  int rc = hplp_solver_create(device, m, n, row_ptr, col_idx, val, b, c, &s);
  if (rc != HPLP_OK) return rc;
  const auto t1 = std::chrono::steady_clock::now();
  if (start.valid()) static_cast<hplp_gpu::Solver*>(s)->use_power_start(cfg->seed, start);
  rc = hplp_solver_solve(s, cfg, io, result);
  const auto t2 = std::chrono::steady_clock::now();
  hplp_solver_free(s);
  if (timing)
    std::fprintf(stderr, "hplp_solve_csr: create+upload %.3f ms, solve %.3f ms, free %.3f ms\n", ms(t0, t1), ms(t1, t2),
                 ms(t2, std::chrono::steady_clock::now()));
  return rc;
}

int hplp_power_start(int64_t n, uint64_t seed, double* x) {
  return guarded([&] {
    if (n < 0 || (n > 0 && !x)) throw std::invalid_argument("hplp_power_start: n < 0 or x is NULL");
    const std::vector<double> v = hplp_gpu::power_start(n, seed);
    std::copy(v.begin(), v.end(), x);
  });
}

int hplp_to_standard_form(const hplp_general_t* g, void** std_form, int64_t* m, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    auto conv = hplp_gpu::to_standard_form(*g);
    auto* h = new StdHandle{std::move(conv.first), std::move(conv.second)};
    *m = h->lp.num_rows();
    *n = h->lp.num_cols();
    *nnz = h->lp.a.nonzeros();
    *std_form = h;
  });
}

int hplp_std_export(void* std_form, int64_t* row_ptr, int32_t* col_idx, double* val, double* b, double* c) {
  return guarded([&] {
    const auto& h = *static_cast<StdHandle*>(std_form);
    const auto& a = h.lp.a;
    if (row_ptr) std::memcpy(row_ptr, a.row_ptr().data(), a.row_ptr().size() * sizeof(int64_t));
    if (col_idx) std::memcpy(col_idx, a.col_idx().data(), a.col_idx().size() * sizeof(int32_t));
    if (val) std::memcpy(val, a.values().data(), a.values().size() * sizeof(double));
    if (b) std::memcpy(b, h.lp.b.data(), h.lp.b.size() * sizeof(double));
    if (c) std::memcpy(c, h.lp.c.data(), h.lp.c.size() * sizeof(double));
  });
}

int hplp_std_recover(void* std_form, const double* x_std, double* x_orig, double std_objective, double* objective) {
  return guarded([&] {
    const auto& h = *static_cast<StdHandle*>(std_form);
    if (x_std && x_orig) {
      std::vector<double> xs(x_std, x_std + h.map.standard_cols);
      std::vector<double> xo = h.map.recover_primal(xs);
      std::memcpy(x_orig, xo.data(), xo.size() * sizeof(double));
    }
    if (objective) *objective = h.map.recover_objective(std_objective);
  });
}

void hplp_std_free(void* std_form) { delete static_cast<StdHandle*>(std_form); }

int hplp_solve_general(int32_t device, const hplp_general_t* g, const hplp_config_t* cfg, hplp_io_t* io,
                       hplp_result_t* result, double* x_orig, double* objective) {
  return guarded([&] {
    auto conv = hplp_gpu::to_standard_form(*g);
    const hplp_gpu::StandardFormLP& lp = conv.first;
    hplp_gpu::Solver s(lp, device);
    hplp_gpu::SolverConfig c = config_with_io(cfg, io, lp.num_rows(), lp.num_cols());
    hplp_gpu::SolveResult r = s.solve(c);
    fill_result(r, io, result);
    double cx = 0.0;
    for (std::size_t j = 0; j < lp.c.size(); ++j) cx += lp.c[j] * r.final_iterate.x[j];
    if (x_orig) {
      std::vector<double> xo = conv.second.recover_primal(r.final_iterate.x);
      std::memcpy(x_orig, xo.data(), xo.size() * sizeof(double));
    }
    if (objective) *objective = conv.second.recover_objective(cx);
  });
}

// ---- MPS ingestion and reports (inc/hplp/mps_io.hpp; csrc/mps_io.cpp) ----

namespace {
struct MpsHandle {
  hplp_gpu::GeneralFormLP g;
  hplp_gpu::MpsDocument doc;
  // hplp_general_t view (CSR rows from the triplets, row order kept)
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v, rhs, range, lo, up, obj;
  std::vector<int32_t> rel;
  hplp_general_t view{};
  void build() {
    const int64_t m = g.num_rows(), n = g.num_cols();
    rp.assign(static_cast<std::size_t>(m) + 1, 0);
    for (const auto& t : g.entries) ++rp[static_cast<std::size_t>(t.row) + 1];
    for (int64_t i = 0; i < m; ++i) rp[i + 1] += rp[i];
    ci.resize(g.entries.size());
    v.resize(g.entries.size());
    std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
    for (const auto& t : g.entries) {
      const int64_t k = fill[t.row]++;
      ci[k] = static_cast<int32_t>(t.col);
      v[k] = t.value;
    }
    rel.resize(m), rhs.resize(m), range.resize(m);
    for (int64_t i = 0; i < m; ++i) {
      const auto& r = g.rows[i];
      rel[i] = r.relation == hplp_gpu::RowRelation::kLessEqual      ? HPLP_ROW_LE
               : r.relation == hplp_gpu::RowRelation::kGreaterEqual ? HPLP_ROW_GE
                                                                    : HPLP_ROW_EQ;
      rhs[i] = r.rhs;
      range[i] = r.range ? *r.range : std::nan("");
    }
    lo.resize(n), up.resize(n), obj.resize(n);
    for (int64_t j = 0; j < n; ++j) lo[j] = g.columns[j].lower, up[j] = g.columns[j].upper, obj[j] = g.objective[j];
    view = hplp_general_t{m,          n,          static_cast<int64_t>(ci.size()), rp.data(), ci.data(), v.data(),
                          rel.data(), rhs.data(), range.data(),                    lo.data(), up.data(), obj.data(),
                          g.maximize ? 1 : 0,     0,          g.objective_constant};
  }
};

int put_text(const std::string& s, char* out, int64_t cap, int64_t* size) {
  if (size) *size = static_cast<int64_t>(s.size());
  if (out) {
    if (cap < static_cast<int64_t>(s.size()) + 1) throw std::invalid_argument("output buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  }
  return HPLP_OK;
}
}  // namespace

int hplp_mps_parse(const char* text, void** handle, int64_t* m, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    auto h = std::make_unique<MpsHandle>();
    h->g = hplp_gpu::parse_mps(std::string(text), &h->doc);
    h->build();
    if (m) *m = h->view.m;
    if (n) *n = h->view.n;
    if (nnz) *nnz = h->view.nnz;
    *handle = h.release();
  });
}

int hplp_mps_view(void* handle, hplp_general_t* view) {
  return guarded([&] { *view = static_cast<MpsHandle*>(handle)->view; });
}

int hplp_mps_names(void* handle, int32_t what, char* out, int64_t cap, int64_t* size) {
  return guarded([&] {
    const auto& h = *static_cast<MpsHandle*>(handle);
    std::string s;
    if (what == 0) s = h.g.name;
    else if (what == 1) s = h.g.objective_name;
    else if (what == 2)
      for (const auto& w : h.doc.warnings) s += w + "\n";
    else if (what == 3)
      for (const auto& r : h.g.rows) s += r.name + "\n";
    else if (what == 4)
      for (const auto& c : h.g.columns) s += c.name + "\n";
    else throw std::invalid_argument("hplp_mps_names: what in 0..4");
    put_text(s, out, cap, size);
  });
}

int hplp_mps_write(void* handle, char* out, int64_t cap, int64_t* size) {
  return guarded([&] { put_text(hplp_gpu::write_mps(static_cast<MpsHandle*>(handle)->g), out, cap, size); });
}

void hplp_mps_free(void* handle) { delete static_cast<MpsHandle*>(handle); }

int hplp_mps_from_general(const hplp_general_t* g, char* out, int64_t cap, int64_t* size) {
  return guarded([&] {
    hplp_gpu::GeneralFormLP lp;
    lp.name = "GENERAL";
    lp.objective_name = "OBJ";
    lp.maximize = g->maximize != 0;
    lp.objective_constant = g->objective_constant;
    lp.rows.resize(static_cast<std::size_t>(g->m));
    for (int64_t i = 0; i < g->m; ++i) {
      auto& r = lp.rows[i];
      r.name = "R" + std::to_string(i);
      r.relation = g->row_relation[i] == HPLP_ROW_LE   ? hplp_gpu::RowRelation::kLessEqual
                   : g->row_relation[i] == HPLP_ROW_GE ? hplp_gpu::RowRelation::kGreaterEqual
                                                       : hplp_gpu::RowRelation::kEqual;
      r.rhs = g->row_rhs[i];
      if (g->row_range && !std::isnan(g->row_range[i])) r.range = g->row_range[i];
    }
    lp.columns.resize(static_cast<std::size_t>(g->n));
    lp.objective.assign(g->objective, g->objective + g->n);
    for (int64_t j = 0; j < g->n; ++j) {
      lp.columns[j].name = "C" + std::to_string(j);
      lp.columns[j].lower = g->col_lower[j];
      lp.columns[j].upper = g->col_upper[j];
    }
    // column-major entries (the order an MPS COLUMNS section gives)
    std::vector<std::vector<hplp_gpu::Triplet>> by_col(static_cast<std::size_t>(g->n));
    for (int64_t i = 0; i < g->m; ++i)
      for (int64_t p = g->row_ptr[i]; p < g->row_ptr[i + 1]; ++p)
        by_col[g->col_idx[p]].push_back(hplp_gpu::Triplet{i, g->col_idx[p], g->val[p]});
    for (const auto& v : by_col) lp.entries.insert(lp.entries.end(), v.begin(), v.end());
    put_text(hplp_gpu::write_mps(lp), out, cap, size);
  });
}

int hplp_solve_mps(int32_t device, const char* mps_text, const hplp_config_t* cfg, const char* instance,
                   int64_t elide_above, char* json, int64_t json_cap, int64_t* json_size, char* trace_csv,
                   int64_t trace_cap, int64_t* trace_size, int32_t* status) {
  return guarded([&] {
    hplp_gpu::MpsDocument doc;
    const hplp_gpu::GeneralFormLP g = hplp_gpu::parse_mps(std::string(mps_text), &doc);
    auto conv = hplp_gpu::to_standard_form(g);
    const hplp_gpu::StandardFormLP& lp = conv.first;
    hplp_gpu::Solver s(lp, device);
    if (const int rc = hplp_validate_config(cfg); rc != HPLP_OK) throw std::invalid_argument(g_err);
    hplp_gpu::SolverConfig c = hplp_gpu::from_pod(*cfg);
    c.device = device;
    std::vector<hplp_gpu::TraceRecord> trace;
    if (c.trace_period > 0) c.trace_sink = [&](const hplp_gpu::TraceRecord& r, const hplp_gpu::Iterate&) { trace.push_back(r); };
    const hplp_gpu::SolveResult r = s.solve(c);
    hplp_gpu::SolutionReport rep;
    rep.instance = instance ? instance : g.name;
    rep.status = r.status;
    double cx = 0.0, by = 0.0;
    for (std::size_t j = 0; j < lp.c.size(); ++j) cx += lp.c[j] * r.final_iterate.x[j];
    for (std::size_t i = 0; i < lp.b.size(); ++i) by += lp.b[i] * r.final_iterate.y[i];
    rep.primal_objective = conv.second.recover_objective(cx);
    rep.dual_objective = conv.second.recover_objective(-by);  // gap |c'x + b'y| -> dual value -b'y
    rep.kkt = r.final_kkt;
    rep.iterations = r.totals.iterations;
    rep.epochs = static_cast<long>(r.epochs.size());
    rep.spmv_count = r.totals.spmv_count;
    rep.eta = r.totals.eta;
    rep.sigma_estimate = r.totals.sigma_estimate;
    rep.solve_seconds = r.totals.wall_seconds;
    const bool infeasible = r.status == hplp_gpu::SolveStatus::kPrimalInfeasible ||
                            r.status == hplp_gpu::SolveStatus::kDualInfeasible ||
                            r.status == hplp_gpu::SolveStatus::kPrimalDualInfeasible;
    if (!infeasible) {
      rep.primal_solution = conv.second.recover_primal(r.final_iterate.x);
      rep.dual_solution = r.final_iterate.y;
    }
    rep.primal_certificate = r.primal_certificate;
    rep.dual_certificate = r.dual_certificate;
    rep.config_echo = {{"tolerance", std::to_string(c.tolerance)},
                       {"iteration_limit", std::to_string(c.iteration_limit)},
                       {"restart", c.restart.kind == hplp_gpu::RestartScheme::Kind::kFixedFrequency ? "fixed"
                                   : c.restart.kind == hplp_gpu::RestartScheme::Kind::kNone           ? "none"
                                                                                                      : "adaptive"},
                       {"infeasibility_check_period", std::to_string(c.infeasibility_check_period)},
                       {"seed", std::to_string(c.seed)},
                       {"device", std::to_string(device)}};
    hplp_gpu::JsonWriteOptions opt;
    if (elide_above >= 0) opt.vector_elision_threshold = elide_above;
    put_text(hplp_gpu::write_solution_json(rep, opt), json, json_cap, json_size);
    if (trace_csv || trace_size) put_text(hplp_gpu::write_trace_csv(trace), trace_csv, trace_cap, trace_size);
    if (status) *status = static_cast<int32_t>(r.status);
  });
}

int hplp_json_normalize(const char* json, int32_t include_timing, char* out, int64_t cap, int64_t* size) {
  return guarded([&] {
    hplp_gpu::JsonWriteOptions opt;
    opt.include_timing = include_timing != 0;
    put_text(hplp_gpu::write_solution_json(hplp_gpu::parse_solution_json(json), opt), out, cap, size);
  });
}

}  // extern "C"
