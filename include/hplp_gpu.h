/*
 * hplp_gpu -- the solve()-level C ABI of the B200 rHPDHG solver.
 *
 * This is the drop-in boundary for the reference's public API
 * (/root/reference/proj/include/hplp): problem load (CSR with bounds, or a
 * standard-form CSR), SolverConfig, solve(), SolveStatus + KktError report.
 * The C++ mirror of the reference types lives in
 * paper_2407_16144_b200/csrc/hplp_gpu.hpp; INTEGRATION.md shows the ctypes
 * and C++ bindings a maintainer adds on the reference side.
 *
 * All pointers are host pointers, copied on entry.  Return value: HPLP_OK or
 * an HPLP_E* code with hplp_last_error() describing it; HPLP_EINVAL is the
 * reference's std::invalid_argument, HPLP_EDOMAIN its std::domain_error.
 */
#ifndef HPLP_GPU_H_
#define HPLP_GPU_H_

#include <stdint.h>

#include "hplp_types.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* hplp_last_error(void);

/* to_string(SolveStatus), src/solver.cpp:176-192. */
const char* hplp_status_string(int32_t status);

/* validate_config, src/solver.cpp:40-65 (HPLP_EINVAL + message). */
int hplp_validate_config(const hplp_config_t* cfg);

/* SolveResult solve(const StandardFormLP&, const SolverConfig&)
 * (inc/solver.hpp:130, src/solver.cpp:206-342) on a standard-form LP
 * min c'x s.t. Ax = b, x >= 0 given as CSR (StandardFormLP, inc/lp_model.hpp:27-37).
 * Rows may list columns in any order; duplicates are an error
 * (src/sparse_matrix.cpp:45-52). */
int hplp_solve_csr(int32_t device, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                   const double* val, const double* b, const double* c, const hplp_config_t* cfg,
                   hplp_io_t* io, hplp_result_t* result);

/* The unit start vector of power_iteration (src/sparse_matrix.cpp:145-151):
 * n draws of std::normal_distribution<double>(0, 1) from
 * std::mt19937_64(seed), normalised -- bit-identical to the reference's
 * sequential loop (libstdc++), computed with the uniform conversion and the
 * polar method's log/sqrt on host threads.  Host only; x has n entries. */
int hplp_power_start(int64_t n, uint64_t seed, double* x);

/* A device-resident problem for repeated solves (upload once). */
int hplp_solver_create(int32_t device, int64_t m, int64_t n, const int64_t* row_ptr,
                       const int32_t* col_idx, const double* val, const double* b, const double* c,
                       void** solver);
/* [no reference counterpart: SURVEY.md §8f rank 4, a flagged mode] The box
 * form of a standard-form LP: the trailing bound rows x_j + s_j = u_j that
 * to_standard_form appends (src/lp_model.cpp:232-252) are detected and
 * replaced by the projection x_j in [0, u_j] on the leading block (hx_set_box).
 * hplp_solver_solve then runs rHPDHG on it -- a different iteration from the
 * reference's, not iterate-comparable -- and returns x, y in the standard
 * form's dimensions (slack u_j - x_j; bound-row dual max(0, -(c + A^T y)_j)).
 * No infeasibility scan (the check period is ignored), final_kkt is the box
 * form's KKT error, trace iterates are box-form vectors. */
int hplp_solver_create_box(int32_t device, int64_t m, int64_t n, const int64_t* row_ptr,
                           const int32_t* col_idx, const double* val, const double* b, const double* c,
                           void** solver);
/* Dimensions (m_box, n_box) of that box form and its upper bounds (n_box
 * values, +inf = none; `upper` may be NULL or hold n values). Host only. */
int hplp_box_form_dims(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                       const double* b, const double* c, int64_t* m_box, int64_t* n_box, double* upper);
/* The same LP row-partitioned across nranks contexts of this process (SURVEY.md
 * §8e): rank r on devices[r % ndevices], nnz-balanced blocks from
 * hplp_plan_partition, bound with hx_team_bind.  Ranks sharing a device are
 * emulated as CTA groups of one launch (ctas_per_rank 0 = split evenly).
 * hplp_solver_solve then runs the partitioned loop. */
int hplp_solver_create_team(const int32_t* devices, int32_t ndevices, int32_t nranks, int32_t ctas_per_rank,
                            int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                            const double* b, const double* c, void** solver);
/* One rank of a team spread over processes (one process per GPU, e.g. under
 * torchrun): the solver owns block `rank` of hplp_plan_partition(nranks).
 * Every process exports its blob (CUDA IPC handles of the buffers peers write
 * into), the caller exchanges the blobs (any transport; bench.py uses
 * torch.distributed all_gather_object) and imports all of them; then all ranks
 * call hplp_solver_solve with the same config, concurrently. */
int hplp_solver_create_rank(int32_t device, int32_t nranks, int32_t rank, int64_t m, int64_t n,
                            const int64_t* row_ptr, const int32_t* col_idx, const double* val, const double* b,
                            const double* c, void** solver);
/* blob = NULL: *size = bytes needed. */
int hplp_solver_team_export(void* solver, void* blob, int64_t capacity, int64_t* size);
int hplp_solver_team_import(void* solver, const void* blob, int64_t size);
int hplp_solver_solve(void* solver, const hplp_config_t* cfg, hplp_io_t* io, hplp_result_t* result);
/* The underlying hx context (include/hx.h) for benchmarks and tests. */
void* hplp_solver_hx(void* solver);
/* hx context of rank `rank` of a team (rank 0 = hplp_solver_hx); NULL if none. */
void* hplp_solver_rank_hx(void* solver, int32_t rank);
void hplp_solver_free(void* solver);

/* to_standard_form (inc/lp_model.hpp:126, src/lp_model.cpp:155-325): general
 * form -> standard form with the reference's row/column ordering, plus the
 * VariableMap for recovery. */
int hplp_to_standard_form(const hplp_general_t* g, void** std_form, int64_t* m, int64_t* n, int64_t* nnz);
int hplp_std_export(void* std_form, int64_t* row_ptr, int32_t* col_idx, double* val, double* b, double* c);
/* VariableMap::recover_primal (src/lp_model.cpp:65-85) and recover_objective
 * (inc/lp_model.hpp:116-118).  Either output may be NULL. */
int hplp_std_recover(void* std_form, const double* x_std, double* x_orig, double std_objective,
                     double* objective);
void hplp_std_free(void* std_form);

/* "Problem load in CSR with bounds" + solve + recovery in one call: the
 * north-star entry point.  io holds standard-form buffers (may be NULL);
 * x_orig (n of the general form) and objective (original sense, with the
 * objective constant) may be NULL. */
int hplp_solve_general(int32_t device, const hplp_general_t* g, const hplp_config_t* cfg, hplp_io_t* io,
                       hplp_result_t* result, double* x_orig, double* objective);

/* ---- MPS ingestion and reports: the reference's declared (unimplemented)
 * inc/hplp/mps_io.hpp:29-94, SPEC.md [MODULE] mps_io / cli cmd_solve ------
 * hplp_mps_parse      parse_mps (fixed or free MPS) into a handle holding the
 *                     GeneralFormLP; HPLP_EPARSE + "line N: ..." on errors.
 * hplp_mps_view       its CSR-with-bounds view (pointers owned by the handle),
 *                     ready for hplp_solve_general / hplp_to_standard_form.
 * hplp_mps_names      0 problem name, 1 objective row, 2 warnings, 3 row
 *                     names, 4 column names (newline separated).
 * hplp_mps_write      write_mps: normalized free MPS, 17 significant digits.
 * hplp_mps_from_general  write_mps of a CSR-with-bounds problem.
 * hplp_solve_mps      cmd_solve: MPS text -> to_standard_form -> GPU solve ->
 *                     write_solution_json (elide_above < 0: default 100000)
 *                     and, with cfg->trace_period > 0, write_trace_csv.
 * hplp_json_normalize parse_solution_json then write_solution_json.
 * Text outputs: out == NULL -> *size = length; else cap >= length + 1. */
int hplp_mps_parse(const char* text, void** handle, int64_t* m, int64_t* n, int64_t* nnz);
int hplp_mps_view(void* handle, hplp_general_t* view);
int hplp_mps_names(void* handle, int32_t what, char* out, int64_t cap, int64_t* size);
int hplp_mps_write(void* handle, char* out, int64_t cap, int64_t* size);
int hplp_mps_from_general(const hplp_general_t* g, char* out, int64_t cap, int64_t* size);
void hplp_mps_free(void* handle);
int hplp_solve_mps(int32_t device, const char* mps_text, const hplp_config_t* cfg, const char* instance,
                   int64_t elide_above, char* json, int64_t json_cap, int64_t* json_size, char* trace_csv,
                   int64_t trace_cap, int64_t* trace_size, int32_t* status);
int hplp_json_normalize(const char* json, int32_t include_timing, char* out, int64_t cap, int64_t* size);

/* Multi-GPU row partition plan: rank p owns rows
 * [row_bounds[p], row_bounds[p+1]) of A and columns [col_bounds[p],
 * col_bounds[p+1]) (rows of A^T), each cut balanced by nnz + 3 per row.
 * row_bounds and col_bounds hold parts + 1 entries. */
int hplp_plan_partition(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int32_t parts,
                        int64_t* row_bounds, int64_t* col_bounds);

#ifdef __cplusplus
}
#endif

#endif /* HPLP_GPU_H_ */
