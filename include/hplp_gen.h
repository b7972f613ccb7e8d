/*
 * Seeded synthetic-instance generator for the BASELINE.json configurations
 * (SURVEY.md §8d).  The paper's MIPLIB relaxations are not in this container;
 * these planted / structured LPs stand in for them, with the shapes, sizes and
 * value distributions BASELINE.json states.  Output is a general-form LP
 * (hplp_general_t arrays) that both the product and the CPU checkers convert
 * with to_standard_form.  Pure host C++ (libhplp_gen.so).
 */
#ifndef HPLP_GEN_H_
#define HPLP_GEN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { HPLP_GEN_PLANTED = 0, HPLP_GEN_TRANSPORT = 1 };

typedef struct hplp_gen_params {
  int32_t kind;            /* HPLP_GEN_* */
  int32_t zipf;            /* planted: 1 = Zipf row lengths, 0 = fixed per row */
  int64_t m;               /* planted: general-form rows (before infeasible copies) */
  int64_t n;               /* planted: columns */
  int64_t nnz_per_row;     /* planted, zipf == 0: distinct uniform columns per row */
  double eq_frac;          /* planted: leading fraction of rows that are '=' (rest '>=') */
  double row_scale_log10;  /* planted: log10 r_i ~ U[-s, s] row scaling (0 = none) */
  double zipf_s;           /* zipf: exponent */
  int64_t zipf_cap;        /* zipf: max row length */
  int64_t zipf_target_nnz; /* zipf: total nnz the lengths are rescaled to */
  int64_t zipf_force_cap;  /* zipf: number of rows forced to zipf_cap */
  int64_t infeasible_rows; /* planted: appended copies of '=' rows with b += U[5,10] */
  double ub_lo, ub_hi;     /* planted: upper bounds u ~ U[ub_lo, ub_hi] */
  int64_t sources, sinks;  /* transport */
  uint64_t seed;
} hplp_gen_params_t;

/* Fill *p with BASELINE.json configs[cfg] (0..4); returns 0 or HPLP_EINVAL. */
int hplp_gen_preset(int32_t cfg, hplp_gen_params_t* p);

/* Generate; the handle owns the arrays until hplp_gen_free. */
int hplp_gen_create(const hplp_gen_params_t* p, void** handle);
void hplp_gen_dims(void* handle, int64_t* m, int64_t* n, int64_t* nnz);
/* Copy out the general form.  planted_objective = c^T x* in the original
 * space (NaN for transport, whose optimum is not known in closed form). */
int hplp_gen_export(void* handle, int64_t* row_ptr, int32_t* col_idx, double* val,
                    int32_t* row_relation, double* row_rhs, double* col_lower,
                    double* col_upper, double* objective, double* planted_objective);
/* Planted primal optimum x* (n), or NaN-filled for transport. */
int hplp_gen_planted_x(void* handle, double* x_star);
void hplp_gen_free(void* handle);
const char* hplp_gen_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* HPLP_GEN_H_ */
