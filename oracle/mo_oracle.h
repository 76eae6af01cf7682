/* mo_oracle.h — C restatement of the reference solver path (TEST
 * INFRASTRUCTURE ONLY; never linked into the product).
 *
 * A plain sequential CPU re-statement of minopt's hot path over the same
 * moplan interchange the product consumes:
 *   run_program  program.hpp:89-167     exec_grid  exec.hpp:151-214
 *   EvalEnv      eval.hpp:41-61         exec_graph exec.hpp:223-309 (sequential order)
 *   pow_eval     common.hpp:102-124     pcg        pcg.hpp:63-130
 *   Solver       solver.hpp:125-515 (refresh, cost, residuals, build_normal,
 *                apply_jtj, linearize + Materialize::kJ, solve GN/LM; no callbacks)
 *   SparseCSR    sparse.hpp (push checks, spmv, spmv_t)
 * Real is float or double per instance, like Solver<float>/Solver<double>.
 * Pinned against the unmodified reference's golden outputs by
 * tests/test_oracle_cpu.py.
 */
#ifndef MO_ORACLE_H_
#define MO_ORACLE_H_
#include <stddef.h>
#include <stdint.h>

typedef struct moo moo;

typedef struct {
  int method, nonlinear_iters, linear_iters, use_preconditioner;
  double pcg_rel_tol, pcg_abs_tol, lm_radius0, lm_radius_min, lm_radius_max;
  double lm_diag_min, lm_diag_max, lm_min_decrease, cost_stop_tol;
} moo_config;

typedef struct {
  double final_cost;
  int reason, nonfinite_kernels, indefinite, n_trace;
  int64_t unconstrained;
} moo_result;

/* returns 0 on success, else 1 + reference Err code; message via moo_error() */
int moo_create(const char* plan_text, size_t len, int f64, moo** out);
void moo_destroy(moo* o);
const char* moo_error(void);
int moo_set_dim(moo* o, const char* name, int64_t extent);
int moo_set_config(moo* o, const moo_config* c);
int64_t moo_num_cols(moo* o);
/* binds copy host data (Real = float or double per instance) */
int moo_bind_x(moo* o, const void* x, int64_t n);
int moo_bind_array(moo* o, int i, const void* a, int64_t n);
int moo_bind_params(moo* o, const double* p, int64_t n);
int moo_bind_graph(moo* o, int i, const uint64_t* v, int64_t n, int arity);
int moo_refresh(moo* o);
int64_t moo_num_rows(moo* o);
int moo_excluded(moo* o, uint8_t* out);
int moo_cost(moo* o, double* out);
int moo_residuals(moo* o, void* out);
int moo_build_normal(moo* o, void* b, void* m);
int moo_apply_jtj(moo* o, const void* v, void* out);
/* trace arrays sized >= 4096 rows by the caller */
int moo_solve(moo* o, moo_result* r, int* t_iter, double* t_cost, int* t_acc, double* t_radius, int* t_pcg);
int moo_get_x(moo* o, void* out);
/* linearize (solver.hpp:291-376) / jacobian() CSR; Materialize::kJ plans then
 * apply 2 J^T (J v) through spmv / spmv_t (sparse.hpp). */
int moo_linearize(moo* o);
int moo_jacobian(moo* o, int64_t* rows, int64_t* nnz, int64_t* offs, int64_t* col, void* val);
/* normal_matrix() (solver.hpp:383-387): H = 2 J^T J of a kJtJ plan, CSR */
int moo_normal_matrix(moo* o, int64_t* nnz, int64_t* offs, int64_t* col, void* val);

#endif
