// hplp_gpu::solve -- the C++ host driver of the B200 rHPDHG solver.
//
// Mirrors src/solver.cpp:206-342 of the reference: setup (power iteration
// with the reference's seeded std::mt19937_64 start vector, step size),
// initial iterate, then the iteration loop -- which runs ON THE DEVICE in
// batches through hx_run (include/hx.h), the controller making every
// per-iteration decision there.  The host only drains epoch records, feeds
// the synchronous trace sink (trace_period > 0 pauses the device after each
// traced iteration) and assembles the SolveResult.  There is no CPU compute
// path: without a B200 the hx layer fails and solve() throws.
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <future>
#include <cmath>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "hplp_gpu.hpp"
#include "hplp_gpu.h"
#include "hx.h"

namespace hplp_gpu {

namespace {

using Clock = std::chrono::steady_clock;
constexpr double kPowerTol = 1e-4;          // src/solver.cpp:24
constexpr int64_t kPowerMaxIters = 5000;    // src/solver.cpp:25
constexpr int64_t kBatch = 4096;            // iterations per hx_run when not tracing

[[noreturn]] void throw_hx(hx_ctx* ctx, int rc) {
  const std::string msg = hx_last_error(ctx);
  if (rc == HPLP_EINVAL) throw std::invalid_argument(msg);
  if (rc == HPLP_EDOMAIN) throw std::domain_error(msg);
  throw std::runtime_error("hplp_gpu: " + msg);
}

void check(hx_ctx* ctx, int rc) {
  if (rc != HPLP_OK) throw_hx(ctx, rc);
}

// validate_config, src/solver.cpp:40-65
void validate_config(const SolverConfig& config) {
  if (!(config.tolerance > 0.0)) throw std::invalid_argument("SolverConfig: tolerance must be > 0");
  if (config.iteration_limit < 0) throw std::invalid_argument("SolverConfig: iteration_limit must be >= 0");
  if (!(config.certificate_tolerance > 0.0))
    throw std::invalid_argument("SolverConfig: certificate_tolerance must be > 0");
  if (config.infeasibility_check_period < 0 || config.trace_period < 0 || config.adaptive_stall_cap < 0)
    throw std::invalid_argument("SolverConfig: periods must be >= 0");
  if (config.scheme < HPLP_SCHEME_RHPDHG || config.scheme > HPLP_SCHEME_RESTARTED_AVERAGE)
    throw std::invalid_argument("SolverConfig: unknown scheme");
  if (config.restart.kind == RestartScheme::Kind::kFixedFrequency && config.restart.k_star < 1)
    throw std::invalid_argument("RestartScheme: k_star must be >= 1");
  if (config.restart.kind == RestartScheme::Kind::kAdaptiveResidualDecay &&
      (!(config.restart.beta > 0.0) || !(config.restart.beta < 1.0) || config.restart.tau0 < 1))
    throw std::invalid_argument("RestartScheme: adaptive needs beta in (0,1) and tau0 >= 1");
}

// StepSize ctor, src/pdhg_core.cpp:21-35
double step_size(double eta, double sigma_estimate) {
  if (!(eta > 0.0) || !std::isfinite(eta)) throw std::invalid_argument("StepSize: eta must be positive and finite");
  if (sigma_estimate > 0.0 && eta > 1.0 / (2.0 * sigma_estimate) * (1 + 1e-12))
    throw std::invalid_argument("StepSize: eta exceeds 1/(2 ||A||_2-estimate) = " +
                                std::to_string(1.0 / (2.0 * sigma_estimate)));
  return eta;
}

double seq_norm(const Vector& v) {  // Vector::norm with a sequential sum
  double s = 0.0;
  for (double a : v) s += a * a;
  return std::sqrt(s);
}

KktError kkt_of(const hplp_kkt_t& k) {
  return {k.primal_residual, k.dual_residual, k.gap_residual, k.max_relative};
}

struct PowerResult {
  double sigma = 0.0;
  int64_t iterations = 0;
  bool converged = false;
};

}  // namespace

struct PowerStart {
  Vector x;  // normalised
  uint64_t seed = 0;
  // The generator state after drawing x (for a re-draw on sigma == 0, which
  // continues the same stream): replayed from the seed, only when needed.
  void stream_after(std::mt19937_64& gen, std::normal_distribution<double>& dist) const {
    gen.seed(seed);
    dist = std::normal_distribution<double>(0.0, 1.0);
    for (std::size_t i = 0; i < x.size(); ++i) (void)dist(gen);
  }
};

namespace {

// The raw engine outputs replayed through libstdc++'s own generate_canonical
// (same template, same long double arithmetic as _Adaptor in
// std::normal_distribution), so every uniform is bit-identical.
struct ReplayEngine {
  using result_type = std::mt19937_64::result_type;
  const result_type* p;
  static constexpr result_type min() { return std::mt19937_64::min(); }
  static constexpr result_type max() { return std::mt19937_64::max(); }
  result_type operator()() { return *p++; }
};

}  // namespace

// n draws of std::normal_distribution<double>(0, 1) from std::mt19937_64(seed)
// -- bit for bit what the reference's loop `for (auto& v : x) v = dist(gen)`
// gives (src/sparse_matrix.cpp:145-151; libstdc++'s Marsaglia polar method,
// bits/random.tcc) -- with the expensive parts on host threads.  The polar
// method draws uniforms in pairs (u[2p], u[2p+1]) until a pair lands inside
// the unit disc, so pair p's fate depends on its own two engine outputs only:
// the outputs are drawn in order (cheap), then each thread converts a range of
// pairs with libstdc++'s own generate_canonical (the long double division is
// most of the sequential cost) and tests them, a prefix count over the ranges
// places every accepted pair in the output, and the threads compute the
// accepted pairs' log/sqrt.  Accepted pair k yields out[2k] = y * mult and
// out[2k + 1] = x * mult (the value the distribution saves for its next call).
// Scratch buffers are kept between calls (first-touch page faults cost more
// than the arithmetic).
void draw_normals(std::vector<double>& out, uint64_t seed) {
  const std::size_t n = out.size(), need = (n + 1) / 2;
  if (n == 0) return;
  const unsigned threads = std::clamp(std::thread::hardware_concurrency(), 1u, 8u);
  static std::mutex scratch_mu;
  static std::vector<std::mt19937_64::result_type> s_raw;
  static std::vector<double> s_u;
  static std::vector<unsigned char> s_ok;
  std::unique_lock<std::mutex> own(scratch_mu, std::try_to_lock);
  std::vector<std::mt19937_64::result_type> l_raw;
  std::vector<double> l_u;
  std::vector<unsigned char> l_ok;
  auto& raw = own.owns_lock() ? s_raw : l_raw;
  auto& u = own.owns_lock() ? s_u : l_u;
  auto& ok = own.owns_lock() ? s_ok : l_ok;
  std::mt19937_64 gen(seed);
  std::size_t done = 0;  // accepted pairs written so far
  while (done < need) {
    // acceptance pi/4 per pair: ~1.3x the pairs still needed, plus slack
    const std::size_t np = (need - done) * 13 / 10 + 64;
    raw.resize(2 * np);
    u.resize(2 * np);
    ok.resize(np);
    for (auto& r : raw) r = gen();
    const unsigned T = static_cast<unsigned>(std::min<std::size_t>(threads, (np + 8191) / 8192));
    std::vector<std::size_t> cnt(T + 1, 0);
    auto range = [&](unsigned t, std::size_t len) { return std::pair<std::size_t, std::size_t>{len * t / T, len * (t + 1) / T}; };
    auto run = [&](auto&& f) {
      std::vector<std::thread> pool;
      for (unsigned t = 1; t < T; ++t) pool.emplace_back(f, t);
      f(0u);
      for (auto& th : pool) th.join();
    };
    run([&](unsigned t) {
      const auto [a, b] = range(t, np);
      ReplayEngine e{raw.data() + 2 * a};
      std::size_t c = 0;
      for (std::size_t p = a; p < b; ++p) {
        const double u0 = std::generate_canonical<double, std::numeric_limits<double>::digits>(e);
        const double u1 = std::generate_canonical<double, std::numeric_limits<double>::digits>(e);
        u[2 * p] = u0, u[2 * p + 1] = u1;
        const double x = 2.0 * u0 - 1.0;
        const double y = 2.0 * u1 - 1.0;
        const double r2 = x * x + y * y;
        ok[p] = !(r2 > 1.0 || r2 == 0.0);
        c += ok[p];
      }
      cnt[t + 1] = c;
    });
    for (unsigned t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
    run([&](unsigned t) {
      const auto [a, b] = range(t, np);
      std::size_t k = done + cnt[t];
      for (std::size_t p = a; p < b && k < need; ++p) {
        if (!ok[p]) continue;
        const double x = 2.0 * u[2 * p] - 1.0;
        const double y = 2.0 * u[2 * p + 1] - 1.0;
        const double r2 = x * x + y * y;
        const double mult = std::sqrt(-2 * std::log(r2) / r2);
        out[2 * k] = y * mult * 1.0 + 0.0;  // ret * stddev + mean
        if (2 * k + 1 < n) out[2 * k + 1] = x * mult * 1.0 + 0.0;
        ++k;
      }
    });
    done = std::min(need, done + cnt[T]);
    // the engine must continue right after the last pair used: outputs drawn
    // past it are never consumed (a re-draw replays the stream from the seed)
  }
}

std::vector<double> power_start(int64_t n, uint64_t seed) {
  PowerStart s;
  s.seed = seed;
  s.x.resize(static_cast<std::size_t>(std::max<int64_t>(n, 0)));
  draw_normals(s.x, seed);
  double xn = seq_norm(s.x);
  if (xn == 0.0) std::fill(s.x.begin(), s.x.end(), 1.0), xn = seq_norm(s.x);
  for (auto& v : s.x) v /= xn;
  return std::move(s.x);
}

PowerStartFuture draw_power_start_async(int64_t n, uint64_t seed) {
  return std::async(std::launch::async, [n, seed] {
           auto s = std::make_shared<PowerStart>();
           s->seed = seed;
           s->x.resize(static_cast<std::size_t>(std::max<int64_t>(n, 0)));
           draw_normals(s->x, seed);
           double xn = seq_norm(s->x);
           if (xn == 0.0) std::fill(s->x.begin(), s->x.end(), 1.0), xn = seq_norm(s->x);
           for (auto& v : s->x) v /= xn;
           return s;
         })
      .share();
}

namespace {

// power_iteration, src/sparse_matrix.cpp:138-179: the start vector (and any
// re-draw) comes from the same std::mt19937_64 stream as the reference; the
// SpMVs and norms run on the device (hx_power_iteration).
PowerResult power_iteration(hx_ctx* ctx, int64_t m, int64_t n, int64_t nnz, double tol, int64_t max_iters,
                            const PowerStart& start) {
  PowerResult res;
  if (m == 0 || n == 0 || nnz == 0) {
    res.converged = true;
    return res;
  }
  std::mt19937_64 gen;  // a re-draw continues the stream (rebuilt when needed)
  std::normal_distribution<double> dist;
  bool stream_ready = false;
  Vector x = start.x;
  int64_t k0 = 0;
  double sigma_prev = 0.0;
  while (true) {
    double sigma = 0.0;
    int64_t iters = 0;
    int32_t conv = 0, redraw = 0;
    check(ctx, hx_power_iteration(ctx, x.data(), tol, k0, max_iters, sigma_prev, &sigma, &iters, &conv, &redraw));
    res.iterations = iters;
    res.sigma = sigma;
    if (!redraw) {
      res.converged = conv != 0;
      return res;
    }
    // sigma == 0 at iteration iters-1: re-draw and continue (:158-163)
    if (!stream_ready) start.stream_after(gen, dist), stream_ready = true;
    for (auto& v : x) v = dist(gen);
    const double nn = seq_norm(x);
    for (auto& v : x) v /= nn;
    k0 = iters;
    sigma_prev = sigma;
    if (k0 >= max_iters) return res;
  }
}

}  // namespace

RestartScheme RestartScheme::fixed(long k_star) {
  RestartScheme s;
  s.kind = Kind::kFixedFrequency;
  s.k_star = k_star;
  return s;
}

RestartScheme RestartScheme::adaptive(double beta, long tau0) {
  RestartScheme s;
  s.kind = Kind::kAdaptiveResidualDecay;
  s.beta = beta;
  s.tau0 = tau0;
  return s;
}

RestartScheme RestartScheme::none() {
  RestartScheme s;
  s.kind = Kind::kNone;
  return s;
}

// src/solver.cpp:162-174 (the device controller implements the same rule).
bool should_restart(const RestartScheme& scheme, long n, long k, double residual_now, double residual_epoch_start) {
  switch (scheme.kind) {
    case RestartScheme::Kind::kFixedFrequency:
      return k >= scheme.k_star;
    case RestartScheme::Kind::kAdaptiveResidualDecay:
      if (n == 0) return k > scheme.tau0;
      return residual_now <= scheme.beta * residual_epoch_start;
    case RestartScheme::Kind::kNone:
      return false;
  }
  return false;
}

// src/solver.cpp:176-192
const char* to_string(SolveStatus status) {
  switch (status) {
    case SolveStatus::kOptimal:
      return "optimal";
    case SolveStatus::kPrimalInfeasible:
      return "primal_infeasible";
    case SolveStatus::kDualInfeasible:
      return "dual_infeasible";
    case SolveStatus::kPrimalDualInfeasible:
      return "primal_dual_infeasible";
    case SolveStatus::kIterationLimit:
      return "iteration_limit";
    case SolveStatus::kTimeLimit:
      return "time_limit";
  }
  return "unknown";
}

hplp_config_t to_pod(const SolverConfig& c) {
  hplp_config_t p = hplp_config_default();
  p.restart_kind = c.restart.kind == RestartScheme::Kind::kFixedFrequency ? HPLP_RESTART_FIXED
                   : c.restart.kind == RestartScheme::Kind::kNone        ? HPLP_RESTART_NONE
                                                                         : HPLP_RESTART_ADAPTIVE;
  p.k_star = c.restart.k_star;
  p.beta = c.restart.beta;
  p.tau0 = c.restart.tau0;
  p.tolerance = c.tolerance;
  p.iteration_limit = c.iteration_limit;
  p.time_limit_seconds = c.time_limit_seconds;
  p.has_eta_override = c.eta_override.has_value();
  p.eta_override = c.eta_override.value_or(0.0);
  p.infeasibility_check_period = c.infeasibility_check_period;
  p.trace_period = c.trace_period;
  p.certificate_tolerance = c.certificate_tolerance;
  p.tol_active = c.tol_active;
  p.adaptive_stall_cap = c.adaptive_stall_cap;
  p.seed = c.seed;
  p.precondition_ruiz_iters = c.precondition_ruiz_iters;
  p.precondition_pc_alpha = c.precondition_pc_alpha;
  p.scheme = c.scheme;
  return p;
}

SolverConfig from_pod(const hplp_config_t& p) {
  SolverConfig c;
  c.restart = p.restart_kind == HPLP_RESTART_FIXED  ? RestartScheme::fixed(p.k_star)
              : p.restart_kind == HPLP_RESTART_NONE ? RestartScheme::none()
                                                    : RestartScheme::adaptive(p.beta, p.tau0);
  c.restart.k_star = p.k_star;
  c.tolerance = p.tolerance;
  c.iteration_limit = p.iteration_limit;
  c.time_limit_seconds = p.time_limit_seconds;
  if (p.has_eta_override) c.eta_override = p.eta_override;
  c.infeasibility_check_period = p.infeasibility_check_period;
  c.trace_period = p.trace_period;
  c.certificate_tolerance = p.certificate_tolerance;
  c.tol_active = p.tol_active;
  c.adaptive_stall_cap = p.adaptive_stall_cap;
  c.seed = p.seed;
  c.precondition_ruiz_iters = p.precondition_ruiz_iters;
  c.precondition_pc_alpha = p.precondition_pc_alpha;
  c.scheme = p.scheme;
  return c;
}

Solver::Solver(const StandardFormLP& lp, int device)
    : Solver(device, lp.num_rows(), lp.num_cols(), lp.a.row_ptr().data(), lp.a.col_idx().data(),
             lp.a.values().data(), lp.b.data(), lp.c.data()) {}

Solver::Solver(int device, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
               const double* b, const double* c)
    : m_(m), n_(n), nnz_(row_ptr[m]) {
  int rc = hx_create(device, &ctx_);
  if (rc != HPLP_OK) throw_hx(nullptr, rc);
  rc = hx_upload_csr(ctx_, m, n, row_ptr, col_idx, val, b, c);
  if (rc != HPLP_OK) {
    const std::string msg = hx_last_error(ctx_);
    hx_destroy(ctx_);
    ctx_ = nullptr;
    if (rc == HPLP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("hplp_gpu: " + msg);
  }
}

Solver::Solver(const std::vector<int>& devices, int nranks, int64_t m, int64_t n, const int64_t* row_ptr,
               const int32_t* col_idx, const double* val, const double* b, const double* c, int ctas_per_rank)
    : m_(m), n_(n), nnz_(row_ptr[m]) {
  if (devices.empty() || nranks < 1) throw std::invalid_argument("Solver: a team needs devices and nranks >= 1");
  std::vector<int64_t> rb(static_cast<std::size_t>(nranks) + 1), cb(static_cast<std::size_t>(nranks) + 1);
  if (hplp_plan_partition(m, n, row_ptr, col_idx, nranks, rb.data(), cb.data()) != HPLP_OK)
    throw std::invalid_argument("Solver: partition plan failed");
  auto fail = [&](hx_ctx* ctx, int rc) {
    const std::string msg = hx_last_error(ctx);
    for (hx_ctx* x : ranks_) hx_destroy(x);
    ranks_.clear();
    ctx_ = nullptr;
    if (rc == HPLP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("hplp_gpu: " + msg);
  };
  for (int r = 0; r < nranks; ++r) {
    const int dev = devices[static_cast<std::size_t>(r) % devices.size()];
    hx_ctx* ctx = nullptr;
    int rc = hx_create(dev, &ctx);
    if (rc != HPLP_OK) fail(nullptr, rc);
    ranks_.push_back(ctx);
    int ctas = ctas_per_rank;
    if (ctas == 0) {  // ranks sharing this device split its SMs
      int sharing = 0;
      for (int q = 0; q < nranks; ++q) sharing += devices[static_cast<std::size_t>(q) % devices.size()] == dev;
      int32_t grid = 0;
      hx_device_info(ctx, nullptr, &grid, nullptr);
      ctas = sharing > 1 ? std::max(1, grid / sharing) : 0;
    }
    rc = hx_set_partition(ctx, nranks, r, rb.data(), cb.data(), ctas);
    if (rc != HPLP_OK) fail(ctx, rc);
    rc = hx_upload_csr(ctx, m, n, row_ptr, col_idx, val, b, c);
    if (rc != HPLP_OK) fail(ctx, rc);
  }
  const int rc = hx_team_bind(ranks_.data(), nranks);
  if (rc != HPLP_OK) fail(ranks_[0], rc);
  ctx_ = ranks_[0];
}

Solver::Solver(int device, int nranks, int rank, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
               const double* val, const double* b, const double* c)
    : m_(m), n_(n), nnz_(row_ptr[m]) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("Solver: need 0 <= rank < nranks");
  std::vector<int64_t> rb(static_cast<std::size_t>(nranks) + 1), cb(static_cast<std::size_t>(nranks) + 1);
  if (hplp_plan_partition(m, n, row_ptr, col_idx, nranks, rb.data(), cb.data()) != HPLP_OK)
    throw std::invalid_argument("Solver: partition plan failed");
  int rc = hx_create(device, &ctx_);
  if (rc != HPLP_OK) throw_hx(nullptr, rc);
  rc = hx_set_partition(ctx_, nranks, rank, rb.data(), cb.data(), 0);
  if (rc == HPLP_OK) rc = hx_upload_csr(ctx_, m, n, row_ptr, col_idx, val, b, c);
  if (rc != HPLP_OK) {
    const std::string msg = hx_last_error(ctx_);
    hx_destroy(ctx_);
    ctx_ = nullptr;
    if (rc == HPLP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("hplp_gpu: " + msg);
  }
}

std::vector<unsigned char> Solver::team_export() const {
  int64_t size = 0;
  check(ctx_, hx_team_export(ctx_, nullptr, 0, &size));
  std::vector<unsigned char> blob(static_cast<std::size_t>(size));
  check(ctx_, hx_team_export(ctx_, blob.data(), size, &size));
  return blob;
}

void Solver::team_import(const void* blob, std::size_t size) {
  check(ctx_, hx_team_import(ctx_, blob, static_cast<int64_t>(size)));
}

Solver::~Solver() {
  if (ranks_.empty()) hx_destroy(ctx_);
  for (hx_ctx* x : ranks_) hx_destroy(x);
}

BoxForm detect_box_form(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                        const double* b, const double* c) {
  BoxForm f;
  f.m = m, f.n = n;
  if (m <= 0 || n <= 0) {
    f.upper.assign(static_cast<std::size_t>(std::max<int64_t>(n, 0)), std::numeric_limits<double>::infinity());
    return f;
  }
  std::vector<int32_t> count(static_cast<std::size_t>(n), 0);
  for (int64_t p = 0; p < row_ptr[m]; ++p) ++count[col_idx[p]];
  // trailing rows t = 0, 1, ... from the end: row m-1-t pairs a column with slack n-1-t
  std::vector<int64_t> cols;
  std::vector<double> rhs;
  while (static_cast<int64_t>(cols.size()) < std::min(m, n - 1)) {
    const int64_t k = static_cast<int64_t>(cols.size());
    const int64_t i = m - 1 - k, s = n - 1 - k;
    if (row_ptr[i + 1] - row_ptr[i] != 2) break;
    const int64_t p = row_ptr[i];
    if (col_idx[p + 1] != s || col_idx[p] >= s || val[p] != 1.0 || val[p + 1] != 1.0) break;
    if (count[s] != 1 || c[s] != 0.0 || !(b[i] >= 0.0)) break;
    cols.push_back(col_idx[p]);
    rhs.push_back(b[i]);
  }
  // the bounded columns must lie in the remaining block, one bound each
  int64_t T = static_cast<int64_t>(cols.size());
  while (T > 0) {
    std::vector<char> seen(static_cast<std::size_t>(n - T), 0);
    bool ok = true;
    for (int64_t t = 0; t < T && ok; ++t) {
      const int64_t j = cols[static_cast<std::size_t>(t)];
      if (j >= n - T || seen[static_cast<std::size_t>(j)]) ok = false;
      else seen[static_cast<std::size_t>(j)] = 1;
    }
    if (ok) break;
    --T;
  }
  f.m = m - T, f.n = n - T;
  f.upper.assign(static_cast<std::size_t>(f.n), std::numeric_limits<double>::infinity());
  f.bound_col.resize(static_cast<std::size_t>(T));
  for (int64_t t = 0; t < T; ++t) {  // row f.m + t is cols[T - 1 - t] (found from the end)
    const int64_t j = cols[static_cast<std::size_t>(T - 1 - t)];
    f.bound_col[static_cast<std::size_t>(t)] = j;
    f.upper[static_cast<std::size_t>(j)] = rhs[static_cast<std::size_t>(T - 1 - t)];
  }
  return f;
}

Solver::Solver(BoxFormTag, int device, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
               const double* val, const double* b, const double* c) {
  BoxForm f = detect_box_form(m, n, row_ptr, col_idx, val, b, c);
  // the leading block: its rows reference only leading columns (each slack
  // appears in its bound row alone), so the caller's arrays serve as they are
  m_ = f.m, n_ = f.n, nnz_ = row_ptr[f.m];
  int rc = hx_create(device, &ctx_);
  if (rc != HPLP_OK) throw_hx(nullptr, rc);
  auto fail = [&](int code) {
    const std::string msg = hx_last_error(ctx_);
    hx_destroy(ctx_);
    ctx_ = nullptr;
    if (code == HPLP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("hplp_gpu: " + msg);
  };
  rc = hx_upload_csr(ctx_, f.m, f.n, row_ptr, col_idx, val, b, c);
  if (rc != HPLP_OK) fail(rc);
  rc = hx_set_box(ctx_, f.upper.data());
  if (rc != HPLP_OK) fail(rc);
  BoxInfo info;
  info.m_std = m, info.n_std = n;
  info.bound_col = std::move(f.bound_col);
  info.bound_upper.resize(info.bound_col.size());
  for (std::size_t t = 0; t < info.bound_col.size(); ++t)
    info.bound_upper[t] = f.upper[static_cast<std::size_t>(info.bound_col[t])];
  box_ = std::move(info);
}

SolveResult Solver::solve(const SolverConfig& config) {
  if (!box_) return solve_core(config);
  const BoxInfo& B = *box_;
  if (config.scheme != HPLP_SCHEME_RHPDHG) throw std::invalid_argument("box form: rHPDHG only");
  SolverConfig cfg = config;
  cfg.infeasibility_check_period = 0;  // no certificates in the box form
  cfg.out_x = cfg.out_y = nullptr;     // the result is mapped back to the standard form below
  if (cfg.initial_iterate) {  // standard-form dimensions: the leading parts
    Iterate z = *cfg.initial_iterate;
    if (static_cast<int64_t>(z.x.size()) == B.n_std && static_cast<int64_t>(z.y.size()) == B.m_std) {
      z.x.resize(static_cast<std::size_t>(n_));
      z.y.resize(static_cast<std::size_t>(m_));
      cfg.initial_iterate = std::move(z);
    }
  }
  SolveResult r = solve_core(cfg);
  // back to the standard form: slack s_j = u_j - x_j, bound-row dual
  // max(0, -(c + A^T y)_j), evaluated on the device problem (scaled by C, R
  // when preconditioned: c' + A'^T y' = C (c + A^T y), y' = y / R)
  Iterate& z = r.final_iterate;
  Vector ys(z.y);
  if (scaled_)
    for (std::size_t i = 0; i < ys.size(); ++i) ys[i] /= row_scale_[i];
  Vector aty(static_cast<std::size_t>(n_)), cdev(static_cast<std::size_t>(n_));
  check(ctx_, hx_spmv_transpose(ctx_, ys.data(), aty.data()));
  check(ctx_, hx_download_problem(ctx_, nullptr, nullptr, nullptr, nullptr, cdev.data()));
  const std::size_t T = B.bound_col.size();
  z.x.resize(static_cast<std::size_t>(B.n_std));
  z.y.resize(static_cast<std::size_t>(B.m_std));
  for (std::size_t t = 0; t < T; ++t) {
    const std::size_t j = static_cast<std::size_t>(B.bound_col[t]);
    // (a Halpern combination of two points at u_j may exceed it by an ulp)
    const double slack = B.bound_upper[t] - z.x[j];
    z.x[static_cast<std::size_t>(n_) + t] = slack < 0.0 ? 0.0 : slack;
    double lam = cdev[j] + aty[j];
    if (scaled_) lam /= col_scale_[j];
    z.y[static_cast<std::size_t>(m_) + t] = lam < 0.0 ? -lam : 0.0;
  }
  return r;
}

// solve(): src/solver.cpp:206-342.
SolveResult Solver::solve_core(const SolverConfig& config) {
  const auto t0 = Clock::now();
  auto since = [&] { return std::chrono::duration<double>(Clock::now() - t0).count(); };
  // HPLP_TIMING=1: cumulative wall time of the solve stages on stderr
  const bool timing = [] {
    const char* e = std::getenv("HPLP_TIMING");
    return e && e[0] == '1';
  }();
  auto stage = [&](const char* what) {
    if (timing) std::fprintf(stderr, "solve: %-16s at %8.3f ms\n", what, 1e3 * since());
  };
  validate_config(config);
  hx_ctx* ctx = ctx_;
  // optional diagonal preconditioning (extension), applied once per Solver
  const bool want_scale = config.precondition_ruiz_iters > 0 || config.precondition_pc_alpha >= 0.0;
  if (want_scale || scaled_) {
    if (config.precondition_ruiz_iters < 0) throw std::invalid_argument("SolverConfig: precondition_ruiz_iters < 0");
    if (scaled_ && (config.precondition_ruiz_iters != ruiz_ || config.precondition_pc_alpha != pc_alpha_))
      throw std::invalid_argument("Solver: preconditioning is applied once per Solver; settings cannot change");
    if (!scaled_) {
      row_scale_.assign(static_cast<std::size_t>(m_), 1.0);
      col_scale_.assign(static_cast<std::size_t>(n_), 1.0);
      check(ctx, hx_precondition(ctx, config.precondition_ruiz_iters, config.precondition_pc_alpha, row_scale_.data(),
                                 col_scale_.data()));
      // a team: that one call scaled every rank's blocks together (the
      // exchange of the row / column scales runs inside the team kernel)
      scaled_ = true;
      ruiz_ = config.precondition_ruiz_iters;
      pc_alpha_ = config.precondition_pc_alpha;
    }
  }
  auto unscale = [&](Vector& x, Vector& y) {  // x = C x', y = R y'
    if (!scaled_) return;
    for (std::size_t j = 0; j < x.size(); ++j) x[j] *= col_scale_[j];
    for (std::size_t i = 0; i < y.size(); ++i) y[i] *= row_scale_[i];
  };
  // make_setup (:67-78)
  if (!start_.valid() || start_seed_ != config.seed) use_power_start(config.seed, draw_power_start_async(n_, config.seed));
  const PowerStart& pstart = *start_.get();
  stage("power start");
  const PowerResult pi = power_iteration(ctx, m_, n_, nnz_, kPowerTol, kPowerMaxIters, pstart);
  stage("power iteration");
  const double sigma_used = pi.sigma * (1.0 + kPowerTol);
  long n_spmv = 2 * static_cast<long>(pi.iterations);
  const double eta = config.eta_override ? step_size(*config.eta_override, sigma_used)
                     : sigma_used <= 0.0 ? step_size(1.0, 0.0)
                                         : step_size(1.0 / (2.0 * sigma_used), sigma_used);
  // initial_point (:80-87)
  const double* x0 = nullptr;
  const double* y0 = nullptr;
  Vector xs0, ys0;
  if (config.initial_iterate) {
    const Iterate& z = *config.initial_iterate;
    if (static_cast<int64_t>(z.x.size()) != n_ || static_cast<int64_t>(z.y.size()) != m_)
      throw std::invalid_argument("SolverConfig: initial iterate has wrong size");
    x0 = z.x.data();
    y0 = z.y.data();
    if (scaled_) {  // x' = x / C, y' = y / R
      xs0 = z.x;
      ys0 = z.y;
      for (std::size_t j = 0; j < xs0.size(); ++j) xs0[j] /= col_scale_[j];
      for (std::size_t i = 0; i < ys0.size(); ++i) ys0[i] /= row_scale_[i];
      x0 = xs0.data();
      y0 = ys0.data();
    }
  }
  hplp_config_t pod = to_pod(config);
  pod.time_limit_seconds = config.time_limit_seconds - since();  // device clock starts at the loop
  check(ctx, hx_setup(ctx, &pod, sigma_used, eta, x0, y0));
  for (std::size_t r = 1; r < ranks_.size(); ++r) check(ranks_[r], hx_setup(ranks_[r], &pod, sigma_used, eta, x0, y0));
  stage("setup");
  n_spmv += 1;  // a_x = A x (:213-214)
  // one batch of the loop: the context, or every rank of the team together
  auto run_batch = [&](int64_t batch, hx_progress_t* prog) {
    if (ranks_.empty()) return hx_run(ctx, batch, prog);
    std::vector<hx_progress_t> all(ranks_.size());
    const int rc = hx_team_run(ranks_.data(), static_cast<int32_t>(ranks_.size()), batch, all.data());
    *prog = all[0];
    return rc;
  };

  SolveResult out;
  std::vector<hplp_epoch_t> epochs;
  hx_progress_t p{};
  check(ctx, hx_progress(ctx, &p));
  auto drain_epochs = [&] {
    const int64_t have = static_cast<int64_t>(epochs.size());
    const int64_t from = have > 0 ? have - 1 : 0;  // re-read the open epoch (restart_length)
    if (p.n_epochs > from) {
      epochs.resize(static_cast<std::size_t>(p.n_epochs));
      check(ctx, hx_epochs(ctx, from, p.n_epochs - from, epochs.data() + from));
    }
  };
  // a rank of a multi-rank team: the time limit is decided on the device by
  // rank 0 (a per-rank host check could split the team)
  const int32_t team_size = hx_team_size(ctx);
  // the device trace ring (hx_trace_take): records of whole batches, drained
  // between launches; without it (box form, baselines) a traced iteration
  // ends its launch
  const bool ring = config.trace_period > 0 && hx_trace_ring_capacity(ctx) > 0;
  auto drain_ring = [&] {
    while (hx_trace_pending(ctx) > 0) {
      hplp_trace_t t{};
      Iterate z{Vector(static_cast<std::size_t>(n_)), Vector(static_cast<std::size_t>(m_))};
      std::vector<unsigned char> cls(static_cast<std::size_t>(n_));
      check(ctx, hx_trace_take(ctx, &t, z.x.data(), z.y.data(), cls.data()));
      if (!config.trace_sink) continue;
      TraceRecord rec;
      rec.epoch = t.epoch;
      rec.inner = t.inner;
      rec.iteration = t.iteration;
      rec.fixed_point_residual = t.fixed_point_residual;
      rec.kkt = kkt_of(t.kkt);
      rec.candidate_norm_difference = t.candidate_norm_difference;
      if (t.inner >= 1) rec.candidate_norm_normalized = t.candidate_norm_normalized;
      // the sets from the device classes (the reference's index order)
      rec.partition.tol_active = config.tol_active;
      rec.partition.n_set.reserve(static_cast<std::size_t>(t.partition_n));
      rec.partition.b1_set.reserve(static_cast<std::size_t>(t.partition_b1));
      rec.partition.b2_set.reserve(static_cast<std::size_t>(t.partition_b2));
      for (std::size_t j = 0; j < cls.size(); ++j)
        (cls[j] == 0 ? rec.partition.n_set : cls[j] == 1 ? rec.partition.b1_set : rec.partition.b2_set)
            .push_back(static_cast<Index>(j));
      rec.wall_seconds = since();
      unscale(z.x, z.y);
      config.trace_sink(rec, z);
    }
  };
  while (p.status < 0) {
    if (team_size == 1 && since() > config.time_limit_seconds && p.it < config.iteration_limit) {
      // host-side guard for the time limit between batches (:249-254)
      break;
    }
    const int64_t batch = config.trace_period > 0 && !ring ? config.trace_period : kBatch;
    const int rc = run_batch(batch, &p);
    if (rc != HPLP_OK) throw_hx(ctx, rc);
    drain_epochs();
    if (ring) {
      drain_ring();
    } else if (p.paused && config.trace_sink) {
      TraceRecord rec;
      rec.epoch = p.trace_n;
      rec.inner = p.trace_k;
      rec.iteration = p.trace_it;
      rec.fixed_point_residual = p.trace_res;
      rec.kkt = kkt_of(p.trace_kkt);
      rec.candidate_norm_difference = p.trace_res_diff;  // ||T(z) - z|| (== the residual for rHPDHG)
      Iterate z{Vector(static_cast<std::size_t>(n_)), Vector(static_cast<std::size_t>(m_))};
      check(ctx, hx_get_iterate(ctx, HX_ITERATE_LAST, z.x.data(), z.y.data()));
      // partition estimate from the reduced costs c + A^T y and the
      // normalized candidate's norm (src/solver.cpp:279-287), on the LP the
      // loop iterates (the scaled one when preconditioned)
      Vector rcost(static_cast<std::size_t>(n_));
      double cnn = std::numeric_limits<double>::quiet_NaN();
      check(ctx, hx_trace_reduced_costs(ctx, rcost.data()));
      check(ctx, hx_trace_extras(ctx, nullptr, nullptr, &cnn));
      rec.partition = partition_estimate_from_reduced_costs(z, rcost, config.tol_active, sigma_used);
      rec.candidate_norm_normalized = cnn;
      rec.wall_seconds = since();
      unscale(z.x, z.y);
      config.trace_sink(rec, z);
    }
  }
  SolveStatus status = p.status >= 0 ? static_cast<SolveStatus>(p.status) : SolveStatus::kTimeLimit;
  out.status = status;
  stage("loop");
  // the final iterate: straight into the caller's buffers when given
  const bool direct = config.out_x && config.out_y;
  if (!direct) {
    out.final_iterate.x.resize(static_cast<std::size_t>(n_));
    out.final_iterate.y.resize(static_cast<std::size_t>(m_));
  }
  double* fx = direct ? config.out_x : out.final_iterate.x.data();
  double* fy = direct ? config.out_y : out.final_iterate.y.data();
  long extra_spmv = 0;
  if (status == SolveStatus::kIterationLimit || status == SolveStatus::kTimeLimit) {
    // (:242-254) best iterate if any KKT value was finite, else z with fresh products
    if (p.best_valid) {
      check(ctx, hx_get_iterate(ctx, HX_ITERATE_BEST, fx, fy));
      out.final_kkt = kkt_of(p.best_err);
    } else {
      check(ctx, hx_get_iterate(ctx, HX_ITERATE_CURRENT, fx, fy));
      hplp_kkt_t k;
      check(ctx, hx_kkt_current(ctx, &k));
      out.final_kkt = kkt_of(k);
      extra_spmv = 2;
    }
  } else {
    check(ctx, hx_get_iterate(ctx, HX_ITERATE_LAST, fx, fy));
    out.final_kkt = kkt_of(p.final_kkt);
  }
  if (scaled_) {  // x = C x', y = R y'
    for (int64_t j = 0; j < n_; ++j) fx[j] *= col_scale_[static_cast<std::size_t>(j)];
    for (int64_t i = 0; i < m_; ++i) fy[i] *= row_scale_[static_cast<std::size_t>(i)];
  }
  auto take_cert = [&](int kind, const hplp_cert_meta_t& meta, std::optional<Certificate>& dst, int64_t len) {
    if (!meta.present) return;
    Certificate c;
    c.vector.resize(static_cast<std::size_t>(len));
    check(ctx, hx_get_certificate(ctx, kind, c.vector.data()));
    if (scaled_) {  // y = R y' (primal certificate), u = C u' (dual ray), unit norm again
      const Vector& sc = kind == 0 ? row_scale_ : col_scale_;
      double nn = 0.0;
      for (std::size_t i = 0; i < c.vector.size(); ++i) nn += (c.vector[i] *= sc[i]) * c.vector[i];
      nn = std::sqrt(nn);
      if (nn > 0.0)
        for (double& v2 : c.vector) v2 /= nn;
    }
    c.source = meta.source == HPLP_SOURCE_NORMALIZED_ITERATE ? CandidateSource::kNormalizedIterate
                                                             : CandidateSource::kIterateDifference;
    c.at_iteration = static_cast<long>(meta.at_iteration);
    c.orientation = meta.orientation == HPLP_ORIENT_NEGATED ? Orientation::kNegated : Orientation::kAsIs;
    c.residual = meta.residual;
    c.margin = meta.margin;
    dst = std::move(c);
  };
  stage("loop+readback");
  take_cert(0, p.primal_cert, out.primal_certificate, m_);
  take_cert(1, p.dual_cert, out.dual_certificate, n_);
  out.epochs.reserve(epochs.size());
  for (const hplp_epoch_t& e : epochs)
    out.epochs.push_back({static_cast<long>(e.epoch), static_cast<long>(e.restart_length), e.residual_at_start,
                          kkt_of(e.kkt_at_start)});
  if (!out.epochs.empty() && out.epochs.back().restart_length == 0) out.epochs.back().restart_length = p.k;
  out.totals = {static_cast<long>(p.it), n_spmv + static_cast<long>(p.spmv_count) + extra_spmv, since(), eta,
                sigma_used};
  return out;
}

// src/diagnostics.cpp:26-43
PartitionEstimate partition_estimate_from_reduced_costs(const Iterate& z, const Vector& reduced_costs,
                                                        double tol_active, double sigma_estimate) {
  PartitionEstimate p;
  p.tol_active = tol_active;
  const double r_tol = tol_active * sigma_estimate;
  for (std::size_t i = 0; i < reduced_costs.size(); ++i) {
    const double r = reduced_costs[i];
    if (r > r_tol) p.n_set.push_back(static_cast<Index>(i));
    else if (std::abs(r) <= r_tol && z.x[i] > tol_active) p.b1_set.push_back(static_cast<Index>(i));
    else p.b2_set.push_back(static_cast<Index>(i));
  }
  return p;
}

SolveResult solve(const StandardFormLP& lp, const SolverConfig& config) {
  Solver s(lp, config.device);
  return s.solve(config);
}

SolveResult solve_baseline(const StandardFormLP& lp, const SolverConfig& config, BaselineMode mode) {
  SolverConfig c = config;
  c.scheme = mode == BaselineMode::kVanilla    ? HPLP_SCHEME_VANILLA
             : mode == BaselineMode::kAveraged ? HPLP_SCHEME_AVERAGED
                                               : HPLP_SCHEME_RESTARTED_AVERAGE;
  Solver s(lp, config.device);
  return s.solve(c);
}

}  // namespace hplp_gpu
