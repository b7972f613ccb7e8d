/*
 * Plain-old-data types shared by every C-ABI in this repo: the product
 * (include/hplp_gpu.h, include/hx.h) and the CPU checkers under oracle/.
 * Field meanings follow the reference C++ types one for one; each struct
 * cites the type it flattens.  No torch or C++ types cross this boundary.
 */
#ifndef HPLP_TYPES_H_
#define HPLP_TYPES_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes returned by every entry point (0 = success).  The C++ host
 * driver maps them back onto the reference's exception types. */
enum {
  HPLP_OK = 0,
  HPLP_EINVAL = 1,  /* std::invalid_argument in the reference            */
  HPLP_EDOMAIN = 2, /* std::domain_error (negative canonical form)       */
  HPLP_ECUDA = 3,   /* CUDA runtime / launch failure                     */
  HPLP_ENOMEM = 4,  /* device or host allocation failure                 */
  HPLP_ESTATE = 5,  /* call out of order (no problem uploaded, ...)      */
  HPLP_ETIMEOUT = 6, /* device watchdog fired inside a persistent kernel  */
  HPLP_EPARSE = 7    /* MpsParseError (message carries the line number)    */
};

/* RestartScheme::Kind, inc/solver.hpp:32-44 (same enumerator order). */
enum { HPLP_RESTART_FIXED = 0, HPLP_RESTART_ADAPTIVE = 1, HPLP_RESTART_NONE = 2 };

/* SolveStatus, inc/solver.hpp:51-58 (same enumerator order). */
enum {
  HPLP_STATUS_OPTIMAL = 0,
  HPLP_STATUS_PRIMAL_INFEASIBLE = 1,
  HPLP_STATUS_DUAL_INFEASIBLE = 2,
  HPLP_STATUS_PRIMAL_DUAL_INFEASIBLE = 3,
  HPLP_STATUS_ITERATION_LIMIT = 4,
  HPLP_STATUS_TIME_LIMIT = 5
};

/* CandidateSource / Orientation, inc/infeasibility.hpp:23,40. */
enum { HPLP_SOURCE_NORMALIZED_ITERATE = 0, HPLP_SOURCE_ITERATE_DIFFERENCE = 1 };
enum { HPLP_ORIENT_AS_IS = 0, HPLP_ORIENT_NEGATED = 1 };

/* RowRelation, inc/lp_model.hpp:39. */
enum { HPLP_ROW_LE = 0, HPLP_ROW_EQ = 1, HPLP_ROW_GE = 2 };

/* SolverConfig, inc/solver.hpp:62-80.  std::optional<double> eta_override is
 * (has_eta_override, eta_override); initial_iterate and trace_sink travel in
 * hplp_io_t below.  Use hplp_config_default() for the reference defaults. */
typedef struct hplp_config {
  int32_t restart_kind;
  int32_t has_eta_override;
  int64_t k_star;
  double beta;
  int64_t tau0;
  double tolerance;
  int64_t iteration_limit;
  double time_limit_seconds;
  double eta_override;
  int64_t infeasibility_check_period;
  int64_t trace_period;
  double certificate_tolerance;
  double tol_active;
  int64_t adaptive_stall_cap;
  uint64_t seed;
  /* Extension (no reference counterpart): diagonal
   * preconditioning applied to the instance before the loop.  0 / -1 = off,
   * i.e. the reference's own semantics. */
  int32_t precondition_ruiz_iters;
  /* Iteration scheme: HPLP_SCHEME_RHPDHG = solve() (src/solver.cpp:206-342);
   * the others are solve_baseline(mode) (src/solver.cpp:344-509). */
  int32_t scheme;
  double precondition_pc_alpha;
} hplp_config_t;

enum {
  HPLP_SCHEME_RHPDHG = 0,
  HPLP_SCHEME_VANILLA = 1,           /* BaselineMode::kVanilla */
  HPLP_SCHEME_AVERAGED = 2,          /* BaselineMode::kAveraged */
  HPLP_SCHEME_RESTARTED_AVERAGE = 3  /* BaselineMode::kRestartedAverage */
};

/* KktError, inc/pdhg_core.hpp:82-87. */
typedef struct hplp_kkt {
  double primal_residual;
  double dual_residual;
  double gap_residual;
  double max_relative;
} hplp_kkt_t;

/* EpochStats, inc/solver.hpp:82-87. */
typedef struct hplp_epoch {
  int64_t epoch;
  int64_t restart_length;
  double residual_at_start;
  hplp_kkt_t kkt_at_start;
} hplp_epoch_t;

/* Certificate metadata, inc/solver.hpp:91-98 (the vector itself is written
 * into hplp_io_t::primal_cert / dual_cert). */
typedef struct hplp_cert_meta {
  int32_t present;
  int32_t source;
  int32_t orientation;
  int32_t reserved;
  int64_t at_iteration;
  double residual;
  double margin;
} hplp_cert_meta_t;

/* SolveResult + SolveTotals, inc/solver.hpp:100-116. */
typedef struct hplp_result {
  int32_t status;
  int32_t reserved;
  int64_t iterations;
  int64_t spmv_count;
  double wall_seconds;
  double eta;
  double sigma_estimate;
  hplp_kkt_t final_kkt;
  int64_t n_epochs; /* total epochs; hplp_io_t::epochs holds the first cap */
  hplp_cert_meta_t primal_cert;
  hplp_cert_meta_t dual_cert;
} hplp_result_t;

/* TraceRecord (inc/diagnostics.hpp:72-84).  The partition estimate
 * (PartitionEstimate, :28-33) is given as its three set sizes and one array
 * holding the N, B1 and B2 index sets back to back (valid during the call). */
typedef struct hplp_trace {
  int64_t epoch;
  int64_t inner;
  int64_t iteration;
  double fixed_point_residual;
  hplp_kkt_t kkt;
  double candidate_norm_normalized; /* NaN at k == 0 */
  double candidate_norm_difference;
  double wall_seconds;
  int64_t partition_n, partition_b1, partition_b2;
  const int64_t* partition_sets;
} hplp_trace_t;

/* Synchronous trace sink: SolverConfig::trace_sink(rec, z), called on the
 * solving thread every trace_period iterations (src/solver.cpp:271-290). */
typedef void (*hplp_trace_fn)(const hplp_trace_t* rec, const double* x, int64_t n,
                              const double* y, int64_t m, void* user);

/* Caller-owned buffers for solve().  Any pointer may be NULL. */
typedef struct hplp_io {
  const double* init_x; /* SolverConfig::initial_iterate (n), with init_y (m) */
  const double* init_y;
  double* x;            /* final iterate x (n) */
  double* y;            /* final iterate y (m) */
  double* primal_cert;  /* certificate vector (m), when status says so */
  double* dual_cert;    /* certificate vector (n) */
  hplp_epoch_t* epochs; /* first epochs_capacity EpochStats */
  int64_t epochs_capacity;
  hplp_trace_fn trace_fn;
  void* trace_user;
} hplp_io_t;

/* General-form problem in CSR with row relations and column bounds: the
 * GeneralFormLP of inc/lp_model.hpp:60-74 with entries given as CSR.
 * row_range[i] is NaN when the row has no RANGES entry. */
typedef struct hplp_general {
  int64_t m;
  int64_t n;
  int64_t nnz;
  const int64_t* row_ptr; /* m+1 */
  const int32_t* col_idx; /* nnz */
  const double* val;      /* nnz */
  const int32_t* row_relation; /* m, HPLP_ROW_* */
  const double* row_rhs;       /* m */
  const double* row_range;     /* m or NULL (no ranges) */
  const double* col_lower;     /* n (-inf allowed) */
  const double* col_upper;     /* n (+inf allowed) */
  const double* objective;     /* n */
  int32_t maximize;
  int32_t reserved;
  double objective_constant;
} hplp_general_t;

static inline hplp_config_t hplp_config_default(void) {
  hplp_config_t c;
  c.restart_kind = HPLP_RESTART_ADAPTIVE;
  c.has_eta_override = 0;
  c.k_star = 0;
  c.beta = 0.36787944117144233;
  c.tau0 = 32;
  c.tolerance = 1e-8;
  c.iteration_limit = 1000000;
  c.time_limit_seconds = 1.0 / 0.0;
  c.eta_override = 0.0;
  c.infeasibility_check_period = 100;
  c.trace_period = 0;
  c.certificate_tolerance = 1e-6;
  c.tol_active = 1e-6;
  c.adaptive_stall_cap = 2000;
  c.seed = 12345u;
  c.precondition_ruiz_iters = 0;
  c.scheme = HPLP_SCHEME_RHPDHG;
  c.precondition_pc_alpha = -1.0;
  return c;
}

#ifdef __cplusplus
}
#endif

#endif /* HPLP_TYPES_H_ */
