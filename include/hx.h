/*
 * hx -- the thin C-ABI CUDA layer under the B200 rHPDHG host driver.
 *
 * One hx_ctx owns one device, its stream, the problem (A as CSR, an explicit
 * A^T built on the device, b, c), all iterate buffers and the device-side
 * controller state.  Plain pointers and sizes only; host pointers are copied.
 * Every entry point returns an HPLP_* code (include/hplp_types.h) and leaves
 * a message for hx_last_error().  One context per host thread; independent
 * contexts may be used concurrently.
 *
 * The reference has no FFI: each entry point below replaces a reference C++
 * function, cited in brackets.  include/hplp_gpu.h is the solve()-level
 * boundary built on top of this layer.
 */
#ifndef HX_H_
#define HX_H_

#include <stdint.h>

#include "hplp_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hx_ctx hx_ctx;

/* Progress snapshot returned by hx_run (the loop state of
 * src/solver.cpp:218-227 plus the last iteration's KKT/residual). */
typedef struct hx_progress {
  int64_t it;          /* iterations completed (reference `it`) */
  int64_t n;           /* epoch index (reference `n`) */
  int64_t k;           /* inner index (reference `k`) */
  int64_t spmv_count;  /* device-side SpMVs since hx_setup (excl. setup) */
  int32_t status;      /* -1 running, else HPLP_STATUS_* */
  int32_t error;       /* HPLP_OK or HPLP_EDOMAIN / HPLP_ETIMEOUT */
  int32_t paused;      /* 1: stopped at a trace point (trace_* valid) */
  int32_t best_valid;  /* best_kkt finite */
  double res_epoch_start;
  double best_kkt;
  hplp_kkt_t best_err;
  /* last completed iteration (trace record fields) */
  int64_t trace_it, trace_n, trace_k;
  double trace_res;
  hplp_kkt_t trace_kkt;
  hplp_kkt_t final_kkt; /* KKT of the returned iterate for terminal status */
  int64_t n_epochs;     /* epochs started since hx_setup */
  hplp_cert_meta_t primal_cert, dual_cert;
  double device_ms;     /* CUDA-event time of the hx_run call */
  int64_t launches;     /* kernels launched by this call */
  double trace_res_diff; /* ||T(z) - z|| of the last iteration (the candidate's residual differs for
                            the averaged baselines) */
} hx_progress_t;

int hx_create(int32_t device, hx_ctx** out);
void hx_destroy(hx_ctx* ctx);
const char* hx_last_error(hx_ctx* ctx); /* ctx may be NULL (creation errors) */
int hx_device_info(hx_ctx* ctx, int32_t* sm_count, int32_t* grid_ctas, int32_t* cta_threads);
/* cudaStream_t the context launches on (for event timing by the caller). */
void* hx_stream(hx_ctx* ctx);
int64_t hx_launch_count(hx_ctx* ctx);

/* [SparseMatrix(rows, cols, triplets), src/sparse_matrix.cpp:24-66;
 *  StandardFormLP ctor, src/lp_model.cpp:35-43]
 * Copies CSR A (validated: indices in range, finite values, ascending unique
 * columns per row), b and c to the device, builds the explicit A^T with
 * ascending row order per column (inc/sparse_matrix.hpp:61-62), and the
 * nnz-balanced warp schedules of both matrices. */
int hx_upload_csr(hx_ctx* ctx, int64_t m, int64_t n, const int64_t* row_ptr,
                  const int32_t* col_idx, const double* val, const double* b, const double* c);
/* [spmv / spmv_transpose summation order, src/sparse_matrix.cpp:108-115 and
 *  :127-134; SURVEY.md §8d "deterministic-reduction mode"]
 * HX_SUM_FAST (default): every row sum is deterministic (fixed order, run to
 * run bit-identical) but not the reference's order -- short rows as two
 * interleaved partial sums, long rows as lane-strided partials + trees.
 * HX_SUM_REFERENCE: every row of A and A^T is summed as ONE sequential chain
 * in ascending index order, `acc = 0; acc += a_ij * x_j`, bit-identical to
 * the reference's loops (products rounded once, no FMA); long rows become a
 * single run carried by one warp.  Iterates then differ from the reference
 * only through its norms/dots (restart tests, sigma): used for the full-size
 * parity tests on the Zipf instance (configs[4]).  Set before hx_upload_csr
 * (HPLP_ESTATE after). */
#define HX_SUM_FAST 0
#define HX_SUM_REFERENCE 1
int hx_set_sum_order(hx_ctx* ctx, int32_t order);
/* The order contexts created afterwards start with (all solver constructors
 * of include/hplp_gpu.h go through hx_create); -1 returns to the default,
 * HPLP_SUM_ORDER=reference in the environment, else HX_SUM_FAST. */
int hx_set_default_sum_order(int32_t order);
int32_t hx_sum_order(hx_ctx* ctx);
/* Nonzeros of A and of A^T this context stores on its device: nnz and nnz
 * for one GPU; for a rank of a team (hx_set_partition) only its row block of
 * A and its column block (= rows of A^T), about 2 nnz / nranks together --
 * the full matrix is never on a rank's device. */
int hx_stored_nonzeros(hx_ctx* ctx, int64_t* nnz_a, int64_t* nnz_t);
/* Same with device-resident inputs (no host copies; used by re-uploads). */
int hx_dims(hx_ctx* ctx, int64_t* m, int64_t* n, int64_t* nnz);
/* Host-only diagnostic (no GPU needed): the warp schedule hx_upload_csr
 * builds for a CSR row-pointer array of `rows` rows on `ctas` CTAs of the
 * loop kernel's width (lead: warp 0's starting load, as phase A uses).
 * Writes up to `capacity` tasks as 4 int32 each {row_begin, row_end | kind <<
 * 30, nz_begin, nz_end} in the kernels' layout (warp w's k-th task at k * W +
 * w, W = ctas * warps per CTA; empty slots are zeros) and the number of slots
 * to *n_tasks; stats (may be NULL) receives {W, max warp cost, mean warp
 * cost, max CTA cost, mean CTA cost} in the schedule's cost units.
 * HPLP_EINVAL on a capacity below the slot count (with *n_tasks set). */
int hx_schedule_info(const int32_t* row_ptr, int32_t rows, int32_t ctas, double lead, int32_t* tasks,
                     int64_t capacity, int64_t* n_tasks, double* stats);

/* Diagonal preconditioning of the uploaded problem in place (no reference
 * counterpart; SPEC.md:101,259 name Ruiz / Pock-Chambolle as extension
 * points): ruiz_iters rounds of Ruiz inf-norm equilibration, then one
 * Pock-Chambolle step (pc_alpha >= 0).  A' = R A C, b' = R b, c' = C c on both
 * stored copies; the accumulated scales R (m) and C (n) are returned when the
 * pointers are non-NULL.  Iterates of the transformed LP map back as
 * x = C x', y = R y'. */
int hx_precondition(hx_ctx* ctx, int32_t ruiz_iters, double pc_alpha, double* row_scale, double* col_scale);
/* [no reference counterpart: SURVEY.md §8f rank 4, the flagged box form]
 * Column upper bounds (length n, >= 0, +inf = none) enforced by the primal
 * projection x+ = clamp(x - eta (A^T y + c), 0, u) instead of bound rows;
 * the KKT dual residual counts only unbounded columns and the gap adds
 * sum_j u_j [-(c + A^T y)_j]^+ to b^T y.  upper = NULL returns to the
 * standard form.  Call after hx_upload_csr, before hx_precondition (which
 * rescales u) and hx_setup; rHPDHG only, without infeasibility scans. */
int hx_set_box(hx_ctx* ctx, const double* upper);
/* Which loop kernel hx_run launches: 0 loop_kernel, 1 loop_kernel_stream (the
 * matrix streams loaded L2 evict_first: the working set exceeds ~70% of L2;
 * HPLP_L2_STREAM=0/1 overrides), 2 loop_kernel_box, 3 loop_kernel_stream_cb
 * (the stream kernel with phase B swept in two column blocks: x+ far larger
 * than L2; HX_COLBLOCK=0/1 overrides), 4 loop_kernel_exact (the reference
 * summation order), 5 loop_kernel_team / 6 loop_kernel_team_stream (a rank of
 * a team); -1 before an upload.  With a trace period the trace-ring kernels
 * (loop_kernel_trace, loop_kernel_team_trace) run instead. */
int32_t hx_loop_variant(hx_ctx* ctx);
/* The device problem (after any preconditioning): CSR A, b, c (one GPU;
 * HPLP_EINVAL for a rank, which stores only its blocks). */
int hx_download_problem(hx_ctx* ctx, int64_t* row_ptr, int32_t* col_idx, double* val, double* b, double* c);

/* [spmv, src/sparse_matrix.cpp:101-117]  out = A x, host vectors.  A rank of
 * a team computes its own rows (columns for the transpose); the rest of out
 * is 0. */
int hx_spmv(hx_ctx* ctx, const double* x, double* out);
/* [spmv_transpose, src/sparse_matrix.cpp:119-136]  out = A^T y. */
int hx_spmv_transpose(hx_ctx* ctx, const double* y, double* out);

/* [power_iteration loop body, src/sparse_matrix.cpp:153-177]
 * Runs from the unit start vector x0 (host, length n; drawn by the caller's
 * std::mt19937_64 for parity) starting at iteration k0 with sigma_prev.
 * Stops on convergence, max_iters, or sigma == 0 (*need_redraw = 1: the
 * caller re-draws x from its generator and calls again with k0 = *iters). */
int hx_power_iteration(hx_ctx* ctx, const double* x0, double tol, int64_t k0, int64_t max_iters,
                       double sigma_prev, double* sigma, int64_t* iters, int32_t* converged,
                       int32_t* need_redraw);

/* [make_setup + initial_point + loop prologue, src/solver.cpp:67-87,208-216]
 * Binds the config (validated by the caller), sigma_used and eta, loads the
 * initial iterate (NULL = zeros), computes a_x = A x and sets the anchor.
 * Resets it/n/k, best tracking and the epoch log. */
int hx_setup(hx_ctx* ctx, const hplp_config_t* cfg, double sigma_used, double eta,
             const double* x0, const double* y0);

/* [the while(true) loop, src/solver.cpp:241-341]
 * Runs up to max_iters iterations on the device with the reference's exact
 * per-iteration semantics (termination, certificate scans, restarts, Halpern
 * combine, best tracking).  trace_period > 0 pauses after every traced
 * iteration.  One persistent cooperative kernel per call. */
int hx_run(hx_ctx* ctx, int64_t max_iters, hx_progress_t* progress);
int hx_progress(hx_ctx* ctx, hx_progress_t* progress);

/* ---- Multi-GPU row partition (north star "A is
 * row-partitioned across the 8 GPUs of a single box") ------------------------
 * A team of nranks contexts solves ONE LP: rank r owns rows [row0,row1) of A
 * (y, A x, b) and columns [col0,col1) (x, c) -- hplp_plan_partition gives
 * nnz-balanced blocks.  Each rank's loop kernel runs its blocks and pushes
 * every owned slice a peer gathers (x+, y+, the Halpern y combo, certificate
 * vectors) and its partial-sum records straight into the peers' device
 * memory (NVLink P2P stores), with a two-level cross-rank barrier; every rank
 * reduces all records in one fixed order, so the replicated controllers take
 * bit-identical decisions.  The reference has no counterpart (its solve() is
 * single-threaded); results equal the single-GPU solve within
 * reduction-order rounding.
 *
 * hx_set_partition  before hx_upload_csr, with every rank's blocks (row_bounds
 *                   and col_bounds, nranks + 1 entries: hplp_plan_partition's
 *                   output); the upload derives which peers read each owned
 *                   element, and pushes go only there.  hx_upload_csr still
 *                   takes the FULL problem:
 *                   setup, power iteration and the boundary SpMVs run whole on
 *                   every rank, deterministically identical).  ctas = CTAs of
 *                   this rank (0 = one per SM; emulation splits one device).
 * hx_team_bind      ranks living in one process: on one device the team is
 *                   emulated as CTA groups of one cooperative launch (the way
 *                   to exercise the protocol with one GPU); on several devices
 *                   peer access is enabled and each device runs its rank.
 *                   Then hx_team_run drives all of them.
 * hx_team_export /  one process per GPU: each rank exports CUDA IPC handles of
 * hx_team_import    its shared buffers, the blobs are exchanged by the caller
 *                   (torch.distributed all_gather_object in bench.py) and every
 *                   rank imports all blobs; then each rank calls hx_run, all
 *                   ranks concurrently (the barrier's 10 s watchdog turns a
 *                   missing rank into HPLP_ETIMEOUT).
 * Iterates and certificates read back from any rank are assembled from the
 * peers' blocks. */
int hx_set_partition(hx_ctx* ctx, int32_t nranks, int32_t rank, const int64_t* row_bounds,
                     const int64_t* col_bounds, int32_t ctas);
int hx_team_bind(hx_ctx** ctxs, int32_t count);
/* nranks of the context's team (1 for a plain context). */
int32_t hx_team_size(hx_ctx* ctx);
int hx_team_export(hx_ctx* ctx, void* blob, int64_t capacity, int64_t* size);
int hx_team_import(hx_ctx* ctx, const void* blob, int64_t size);
/* progress: count entries (one per ctxs[i]) or NULL. */
int hx_team_run(hx_ctx** ctxs, int32_t count, int64_t max_iters, hx_progress_t* progress);

/* Epoch log (EpochStats, inc/solver.hpp:82-87) entries [first, first+count). */
int hx_epochs(hx_ctx* ctx, int64_t first, int64_t count, hplp_epoch_t* out);

/* Iterates: which = 0 current z (as of the last completed iteration when
 * paused/terminated, else the next iterate), 1 best, 2 T(z) of the last
 * completed iteration. */
enum { HX_ITERATE_CURRENT = 0, HX_ITERATE_BEST = 1, HX_ITERATE_NEXT = 2, HX_ITERATE_LAST = 3 };
int hx_get_iterate(hx_ctx* ctx, int32_t which, double* x, double* y);

/* [make_certificate, src/solver.cpp:89-101] kind 0 primal (m), 1 dual (n). */
int hx_get_certificate(hx_ctx* ctx, int32_t kind, double* vec);

/* [TraceRecord fields, src/solver.cpp:279-287] for the last completed
 * iteration: aty (n) = A^T y and c_out (n) = c of the device problem (the
 * partition estimate's reduced costs are c + A^T y), and the canonical norm
 * of the normalized candidate (2/k)(z - anchor); NaN when undefined (k = 0,
 * multi-rank context).  Any output may be NULL.  A rank of a team stores
 * only its blocks: aty / c_out give HPLP_EINVAL there (its traces come from
 * the device trace ring, hx_trace_take). */
int hx_trace_extras(hx_ctx* ctx, double* aty, double* c_out, double* cand_norm_normalized);
/* [src/solver.cpp:278-279, partition_estimate_from_reduced_costs's input]
 * rc (n) = c + A^T y of the last traced iteration, on the device problem.  A
 * rank of a team takes it from the trace slots the loop kernel's phase A
 * fills (every rank its own columns; read back through CUDA IPC), so no
 * boundary SpMV over the whole matrix is needed. */
int hx_trace_reduced_costs(hx_ctx* ctx, double* rc);
/* [TraceRecord + trace_sink, src/solver.cpp:271-290; SURVEY.md §8f rank 3]
 * Device trace ring.  With a trace period (hx_setup) the rHPDHG loop of the
 * standard form -- one GPU or a team -- records every traced iteration on the
 * device: the record's scalars, the iterate z and the partition class of
 * every column (0 N, 1 B1, 2 B2: partition_estimate_from_reduced_costs,
 * src/diagnostics.cpp:26-43, on c + A^T y from phase A), with the normalized
 * candidate's canonical norm from the phases' partial sums -- no pause per
 * record; a launch stops early only when the ring is one slot from full.
 * hx_trace_pending: records not yet taken; hx_trace_take: the oldest one
 * (rec: scalars and the three set sizes, partition_sets NULL; x (n), y (m),
 * cls (n) may be NULL).  The box form and the baseline schemes keep the
 * pause-per-record path (hx_trace_extras). */
int32_t hx_trace_ring_capacity(hx_ctx* ctx);  /* slots of the ring set up by hx_setup; 0: none */
int64_t hx_trace_pending(hx_ctx* ctx);
int hx_trace_take(hx_ctx* ctx, hplp_trace_t* rec, double* x, double* y, unsigned char* cls);

/* [kkt_error, src/pdhg_core.cpp:70-73] at the current iterate with fresh
 * products (the limit path of src/solver.cpp:242-254 when no best exists). */
int hx_kkt_current(hx_ctx* ctx, hplp_kkt_t* out);

/* The warp task list of the fused SpMV (which: 0 rows of A, 1 rows of A^T),
 * 4 int32 per task {row_begin, row_end | kind << 30, nz_begin, nz_end}; warp w
 * of the grid runs tasks w, w + W, w + 2W, ... (W = grid * warps per CTA).
 * Diagnostics: the schedule's per-warp composition. */
int hx_sched_tasks(hx_ctx* ctx, int32_t which, int32_t* out, int64_t capacity, int64_t* count);

/* Diagnostics: per-CTA phase timers when the context was created with
 * HX_PROFILE=1 in the environment; out holds grid * (16 + 2 * warps per CTA)
 * counters (SM cycles): per CTA phase A, barrier 1, phase B, barrier 2,
 * controller, iterations, smid, scan/redo, controller totals / scalar; then
 * (builds with -DHX_WPROF only) per-warp SpMV cycles of phase A and B. */
int hx_profile(hx_ctx* ctx, unsigned long long* out, int32_t reset);

/* sizeof checks for the ABI tests. */
int64_t hx_sizeof(int32_t which);

#ifdef __cplusplus
}
#endif

#endif /* HX_H_ */
