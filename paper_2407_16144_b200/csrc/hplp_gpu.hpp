// hplp_gpu: C++ mirror of the reference hplp public API
// (/root/reference/proj/include/hplp/{sparse_matrix,lp_model,pdhg_core,solver}.hpp)
// whose solve() runs the rHPDHG loop on a B200 through the hx C-ABI layer
// (include/hx.h).  Same type names, field meanings, defaults and exception
// types; Eigen::VectorXd becomes std::vector<double>.  A C++ caller of the
// reference switches by replacing `hplp::` with `hplp_gpu::`.
#pragma once

#include <cstdint>
#include <functional>
#include <future>
#include <iosfwd>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hplp_types.h"

struct hx_ctx;  // include/hx.h

namespace hplp_gpu {

using Index = std::ptrdiff_t;
using Vector = std::vector<double>;

// inc/sparse_matrix.hpp:28-32
struct Triplet {
  Index row = 0;
  Index col = 0;
  double value = 0.0;
};

// inc/sparse_matrix.hpp:39-70.  Host CSR with ascending columns per row; the
// device builds the column-major copy (A^T) itself.  Throws
// std::invalid_argument on out-of-range indices, non-finite values and
// duplicate (row, col) pairs (src/sparse_matrix.cpp:27-53).
class SparseMatrix {
 public:
  SparseMatrix() = default;
  SparseMatrix(Index n_rows, Index n_cols, const std::vector<Triplet>& entries);
  static SparseMatrix from_csr(Index n_rows, Index n_cols, const int64_t* row_ptr, const int32_t* col_idx,
                               const double* val);

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index nonzeros() const { return static_cast<Index>(val_.size()); }
  const std::vector<int64_t>& row_ptr() const { return row_ptr_; }
  const std::vector<int32_t>& col_idx() const { return col_idx_; }
  const std::vector<double>& values() const { return val_; }
  std::vector<Triplet> triplets_row_order() const;

 private:
  Index rows_ = 0;
  Index cols_ = 0;
  std::vector<int64_t> row_ptr_{0};
  std::vector<int32_t> col_idx_;
  std::vector<double> val_;
};

// inc/lp_model.hpp:27-37
struct StandardFormLP {
  SparseMatrix a;
  Vector b;
  Vector c;
  StandardFormLP(SparseMatrix a_in, Vector b_in, Vector c_in);
  Index num_rows() const { return a.rows(); }
  Index num_cols() const { return a.cols(); }
};

// inc/lp_model.hpp:39-74
enum class RowRelation { kLessEqual, kEqual, kGreaterEqual };

struct GeneralFormRow {
  std::string name;
  RowRelation relation = RowRelation::kEqual;
  double rhs = 0.0;
  std::optional<double> range;
};

struct GeneralFormColumn {
  std::string name;
  double lower = 0.0;
  double upper = std::numeric_limits<double>::infinity();
};

struct GeneralFormLP {
  std::string name;
  bool maximize = false;
  std::string objective_name;
  double objective_constant = 0.0;
  std::vector<GeneralFormRow> rows;
  std::vector<GeneralFormColumn> columns;
  std::vector<double> objective;
  std::vector<Triplet> entries;
  Index num_rows() const { return static_cast<Index>(rows.size()); }
  Index num_cols() const { return static_cast<Index>(columns.size()); }
};

// inc/lp_model.hpp:77-119
struct VariableRecovery {
  enum class Kind { kShifted, kMirrored, kSplit };
  Kind kind = Kind::kShifted;
  Index col = 0;
  Index neg_col = 0;
  double offset = 0;
};

struct RowConversion {
  double lower = 0.0;
  double upper = 0.0;
  std::optional<Index> slack_col;
  double slack_sign = 0.0;
};

struct BoundRow {
  Index row = 0;
  Index col = 0;
  Index slack_col = 0;
  double rhs = 0.0;
};

struct VariableMap {
  std::vector<VariableRecovery> recoveries;
  std::vector<RowConversion> row_conversions;
  std::vector<BoundRow> bound_rows;
  double objective_sign = 1.0;
  double objective_constant = 0.0;
  Index standard_rows = 0;
  Index standard_cols = 0;
  Vector recover_primal(const Vector& x_std) const;
  double recover_objective(double standard_objective) const {
    return objective_sign * standard_objective + objective_constant;
  }
};

// inc/lp_model.hpp:126; same row/column ordering as src/lp_model.cpp:155-325.
std::pair<StandardFormLP, VariableMap> to_standard_form(const GeneralFormLP& g);
// The same from the flat CSR-with-bounds description of include/hplp_types.h.
std::pair<StandardFormLP, VariableMap> to_standard_form(const hplp_general_t& g);

// inc/pdhg_core.hpp:23-30, :82-87
struct Iterate {
  Vector x;
  Vector y;
};

struct KktError {
  double primal_residual = 0.0;
  double dual_residual = 0.0;
  double gap_residual = 0.0;
  double max_relative = 0.0;
};

// inc/solver.hpp:32-58
struct RestartScheme {
  enum class Kind { kFixedFrequency, kAdaptiveResidualDecay, kNone };
  Kind kind = Kind::kAdaptiveResidualDecay;
  long k_star = 0;
  double beta = 0.36787944117144233;
  long tau0 = 32;
  static RestartScheme fixed(long k_star);
  static RestartScheme adaptive(double beta = 0.36787944117144233, long tau0 = 32);
  static RestartScheme none();
};

bool should_restart(const RestartScheme& scheme, long n, long k, double residual_now,
                    double residual_epoch_start);

enum class SolveStatus {
  kOptimal,
  kPrimalInfeasible,
  kDualInfeasible,
  kPrimalDualInfeasible,
  kIterationLimit,
  kTimeLimit,
};

const char* to_string(SolveStatus status);

enum class CandidateSource { kNormalizedIterate, kIterateDifference };
enum class Orientation { kAsIs, kNegated };

// inc/diagnostics.hpp:28-33 -- active-set partition of the primal
// coordinates: N reduced cost > tol*sigma, B1 |reduced cost| <= tol*sigma and
// x > tol, B2 the rest (src/diagnostics.cpp:26-43).
struct PartitionEstimate {
  std::vector<Index> n_set;
  std::vector<Index> b1_set;
  std::vector<Index> b2_set;
  double tol_active = 1e-6;
};

// partition_estimate_from_reduced_costs, src/diagnostics.cpp:26-43.
PartitionEstimate partition_estimate_from_reduced_costs(const Iterate& z, const Vector& reduced_costs,
                                                        double tol_active, double sigma_estimate);

// inc/diagnostics.hpp:72-84; filled as src/solver.cpp:271-290 does (the
// reduced costs come from a device A^T y of the traced iterate).
struct TraceRecord {
  long epoch = 0;
  long inner = 0;
  long iteration = 0;
  double fixed_point_residual = 0.0;
  KktError kkt;
  PartitionEstimate partition;
  double candidate_norm_normalized = std::numeric_limits<double>::quiet_NaN();
  double candidate_norm_difference = std::numeric_limits<double>::quiet_NaN();
  double wall_seconds = 0.0;
};

// inc/solver.hpp:62-80
struct SolverConfig {
  RestartScheme restart;
  double tolerance = 1e-8;
  long iteration_limit = 1000000;
  double time_limit_seconds = std::numeric_limits<double>::infinity();
  std::optional<double> eta_override;
  long infeasibility_check_period = 100;
  long trace_period = 0;
  double certificate_tolerance = 1e-6;
  double tol_active = 1e-6;
  long adaptive_stall_cap = 2000;
  std::uint64_t seed = 12345;
  std::optional<Iterate> initial_iterate;
  std::function<void(const TraceRecord&, const Iterate&)> trace_sink;
  int device = 0;  // B200 ordinal (extension; the reference has no device)
  // Extension (no reference counterpart): Ruiz rounds and a
  // Pock-Chambolle step applied on the device before the loop; the loop then
  // runs the reference's exact semantics on the scaled instance and the
  // result is mapped back (x = C x', y = R y', certificates re-normalised).
  // final_kkt is the KKT error of the scaled instance the loop terminated on.
  int precondition_ruiz_iters = 0;
  double precondition_pc_alpha = -1.0;  // < 0: no Pock-Chambolle step
  // Iteration scheme (HPLP_SCHEME_*): 0 = solve(); 1-3 = solve_baseline's
  // modes (set by solve_baseline, or directly through the C ABI).
  int scheme = 0;
  // Extension (C ABI): when both are set, the final iterate is read from the
  // device straight into these caller buffers (n and m doubles) and
  // SolveResult::final_iterate stays empty -- no host staging copy.
  double* out_x = nullptr;
  double* out_y = nullptr;
};

// inc/solver.hpp:82-116
struct EpochStats {
  long epoch = 0;
  long restart_length = 0;
  double residual_at_start = 0.0;
  KktError kkt_at_start;
};

struct Certificate {
  Vector vector;
  CandidateSource source = CandidateSource::kIterateDifference;
  long at_iteration = 0;
  Orientation orientation = Orientation::kAsIs;
  double residual = 0.0;
  double margin = 0.0;
};

struct SolveTotals {
  long iterations = 0;
  long spmv_count = 0;
  double wall_seconds = 0.0;
  double eta = 0.0;
  double sigma_estimate = 0.0;
};

struct SolveResult {
  SolveStatus status = SolveStatus::kIterationLimit;
  Iterate final_iterate;
  KktError final_kkt;
  std::optional<Certificate> primal_certificate;
  std::optional<Certificate> dual_certificate;
  std::vector<EpochStats> epochs;
  SolveTotals totals;
};

// The power iteration's random start (src/sparse_matrix.cpp:145-150): n
// normal draws from std::mt19937_64(seed), normalised, plus the generator
// state for a re-draw.  Sequential host work (~8 ms at n = 430k), so it is
// drawn on a host thread while the problem uploads and kept for later
// solves with the same seed.
struct PowerStart;
using PowerStartFuture = std::shared_future<std::shared_ptr<PowerStart>>;
PowerStartFuture draw_power_start_async(int64_t n, uint64_t seed);
// The normalised start vector itself (src/sparse_matrix.cpp:145-151), drawn as above.
std::vector<double> power_start(int64_t n, uint64_t seed);

// Box form (no reference counterpart, a flagged
// mode): the trailing bound rows x_j + s_j = u_j that to_standard_form
// appends (src/lp_model.cpp:232-252) become column upper bounds enforced by
// the primal projection, leaving the leading m x n block of the standard
// form.  Detected structurally: trailing rows with entries (j, s), both 1.0,
// where s is the matching trailing column, appears in no other row and has
// c_s = 0; rhs >= 0.
struct BoxForm {
  int64_t m = 0, n = 0;             // the box LP: leading rows / columns
  std::vector<int64_t> bound_col;   // per removed bound row t (row m + t, slack column n + t): column j
  Vector upper;                     // length n: u_j, +inf where unbounded
};
BoxForm detect_box_form(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                        const double* b, const double* c);

// A device-resident problem: upload once, solve many times (bench, warm
// starts).  Owns one hx context.
class Solver {
 public:
  struct BoxFormTag {};
  // The box form of a standard-form LP (detect_box_form): solve() runs rHPDHG
  // on it and maps the result back to the standard form's dimensions
  // (slack s_j = u_j - x_j; bound-row dual max(0, -(c + A^T y)_j)).  No
  // infeasibility scan; final_kkt is the box form's KKT error; trace iterates
  // are box-form vectors.
  Solver(BoxFormTag, int device, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
         const double* val, const double* b, const double* c);
  bool box_form() const { return box_.has_value(); }
  Solver(const StandardFormLP& lp, int device = 0);
  Solver(int device, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
         const double* b, const double* c);
  // Multi-GPU row partition: nranks contexts in this process,
  // rank r on devices[r % devices.size()], blocks from hplp_plan_partition.
  // Ranks sharing one device are emulated as CTA groups of one launch
  // (ctas_per_rank = 0 splits the device evenly).
  Solver(const std::vector<int>& devices, int nranks, int64_t m, int64_t n, const int64_t* row_ptr,
         const int32_t* col_idx, const double* val, const double* b, const double* c, int ctas_per_rank = 0);
  // One rank of a team spread over processes (one process per GPU): the
  // context owns block `rank` of hplp_plan_partition(nranks); the caller
  // exchanges team_export() blobs between the processes and hands every
  // rank's blob to team_import() before the first solve().
  Solver(int device, int nranks, int rank, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
         const double* val, const double* b, const double* c);
  std::vector<unsigned char> team_export() const;
  void team_import(const void* blob, std::size_t size);
  ~Solver();
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;
  SolveResult solve(const SolverConfig& config);
  ::hx_ctx* hx() const { return ctx_; }
  ::hx_ctx* rank_hx(int r) const {
    return ranks_.empty() ? (r == 0 ? ctx_ : nullptr)
                          : (r >= 0 && r < static_cast<int>(ranks_.size()) ? ranks_[r] : nullptr);
  }
  int nranks() const { return ranks_.empty() ? 1 : static_cast<int>(ranks_.size()); }
  int64_t rows() const { return box_ ? box_->m_std : m_; }  // the standard form's dimensions
  int64_t cols() const { return box_ ? box_->n_std : n_; }
  // a start vector drawn elsewhere (draw_power_start_async) for solves with `seed`
  void use_power_start(uint64_t seed, PowerStartFuture start) {
    start_seed_ = seed;
    start_ = std::move(start);
  }

 private:
  uint64_t start_seed_ = 0;
  PowerStartFuture start_;  // invalid until drawn
  struct BoxInfo {
    int64_t m_std = 0, n_std = 0;
    std::vector<int64_t> bound_col;
    Vector bound_upper;  // u of each removed bound row (unscaled)
  };
  std::optional<BoxInfo> box_;
  SolveResult solve_core(const SolverConfig& config);
  ::hx_ctx* ctx_ = nullptr;          // the context (a team: rank 0)
  std::vector<::hx_ctx*> ranks_;      // team in rank order; empty for one context
  int64_t m_ = 0, n_ = 0, nnz_ = 0;
  bool scaled_ = false;
  int ruiz_ = 0;
  double pc_alpha_ = -1.0;
  Vector row_scale_, col_scale_;  // R (m), C (n) when scaled_
};

// inc/solver.hpp:130 -- src/solver.cpp:206-342 on the GPU.
SolveResult solve(const StandardFormLP& lp, const SolverConfig& config);

// inc/solver.hpp:132-139 -- solve_baseline (src/solver.cpp:344-509) on the
// GPU: vanilla PDHG, its running average, and the average restarted.
enum class BaselineMode { kVanilla, kAveraged, kRestartedAverage };
SolveResult solve_baseline(const StandardFormLP& lp, const SolverConfig& config, BaselineMode mode);

// config <-> flat POD (include/hplp_types.h)
SolverConfig from_pod(const hplp_config_t& c);
hplp_config_t to_pod(const SolverConfig& c);

// ---- MPS ingestion and reports: inc/hplp/mps_io.hpp:29-94 (declared by the
// reference, implemented here in csrc/mps_io.cpp) --------------------------------
class MpsParseError : public std::runtime_error {
 public:
  MpsParseError(long line, const std::string& message)
      : std::runtime_error("line " + std::to_string(line) + ": " + message), line_(line) {}
  long line() const { return line_; }

 private:
  long line_;
};

struct MpsDocument {
  std::string problem_name;
  std::string objective_row_name;
  std::vector<std::string> warnings;
};

GeneralFormLP parse_mps(std::istream& in, MpsDocument* doc = nullptr);
GeneralFormLP parse_mps(const std::string& text, MpsDocument* doc = nullptr);
GeneralFormLP parse_mps_file(const std::string& path, MpsDocument* doc = nullptr);
std::string write_mps(const GeneralFormLP& g);

struct SolutionReport {
  std::string instance;
  SolveStatus status = SolveStatus::kIterationLimit;
  double primal_objective = std::numeric_limits<double>::quiet_NaN();
  double dual_objective = std::numeric_limits<double>::quiet_NaN();
  KktError kkt;
  long iterations = 0;
  long epochs = 0;
  long spmv_count = 0;
  double eta = 0.0;
  double sigma_estimate = 0.0;
  double solve_seconds = 0.0;
  std::optional<Vector> primal_solution;
  std::optional<Vector> dual_solution;
  std::optional<Certificate> primal_certificate;
  std::optional<Certificate> dual_certificate;
  std::vector<std::pair<std::string, std::string>> config_echo;
};

struct JsonWriteOptions {
  bool include_timing = true;
  Index vector_elision_threshold = 100000;
};

std::string write_solution_json(const SolutionReport& report, const JsonWriteOptions& options = {});
SolutionReport parse_solution_json(const std::string& text);
std::string write_trace_csv(const std::vector<TraceRecord>& trace);

}  // namespace hplp_gpu
