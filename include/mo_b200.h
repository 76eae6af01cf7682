/* mo_b200.h — C ABI of the B200-native matrix-free GN/LM solver core.
 *
 * Drop-in boundary for the reference "minopt" solver path (arXiv 1604.06525,
 * /root/reference/proj/include/minopt).  The reference exposes header-only C++
 * templates; each entry point below replaces one of its public routines
 * (SURVEY.md §8b).  Plans are produced at plan time by the reference's own
 * front end (compile_source lower.hpp:619 -> plan plan.hpp:189) and handed
 * over through integration/minopt_b200_bridge.hpp; everything after that —
 * residual/cost evaluation, J^T F + Jacobi, matrix-free J^T J p, Jacobi PCG,
 * GN / LM control — runs on the GPU.  There is no CPU fallback: without a
 * CUDA device every compute entry point returns MO_ERR_NO_DEVICE.
 *
 * Conventions: every function returns 0 on success or 1 + the reference Err
 * code (common.hpp:13-32; MO_ERR_* below) and records a message retrievable
 * with mo_last_error() (thread local).  Host buffers use the reference layout:
 * the unknown vector is in plan column order col = ubase[f] + elem*C_f + ch
 * (plan.hpp:212-218), arrays are channel-interleaved row-major (problem.hpp:
 * 131-136), graphs are edge-major uint64 vertex tables (exec.hpp:36-43).
 * Real data is float when the session precision is MO_F32, double otherwise.
 */
#ifndef MO_B200_H_
#define MO_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: 1 + minopt::Err (common.hpp:13-32). */
enum {
  MO_OK = 0,
  MO_ERR_SYNTAX = 1,
  MO_ERR_UNDECLARED = 2,
  MO_ERR_ARITY = 3,
  MO_ERR_NONCONST_OFFSET = 4,
  MO_ERR_MIXED_DOMAIN = 5,
  MO_ERR_NONCONST_EXPONENT = 6,
  MO_ERR_DOMAIN_MISMATCH = 7,
  MO_ERR_NONBOOLEAN = 8,
  MO_ERR_CYCLIC_COMPUTED = 9,
  MO_ERR_SHAPE_MISMATCH = 10,
  MO_ERR_INDEX_OUT_OF_RANGE = 11,
  MO_ERR_FORMAT = 12,
  MO_ERR_TRUNCATED = 13,
  MO_ERR_GRAPH_DOMAIN = 14,
  MO_ERR_BIND = 15,
  MO_ERR_NONFINITE_COST = 16,
  MO_ERR_CYCLIC_IR = 17,
  MO_ERR_INTERNAL = 18,
  MO_ERR_CUDA = 101,      /* device/driver failure (no reference counterpart) */
  MO_ERR_NO_DEVICE = 102  /* no CUDA device: the product has no CPU fallback */
};

enum { MO_GAUSS_NEWTON = 0, MO_LEVENBERG_MARQUARDT = 1 }; /* plan.hpp:15 Method */
enum { MO_F32 = 0, MO_F64 = 1 };                         /* plan.hpp:16 Precision */

/* StopReason, solver.hpp:40-46 */
enum { MO_STOP_ITER_LIMIT = 0, MO_STOP_COST_TOL = 1, MO_STOP_STALLED = 2, MO_STOP_NONFINITE = 3 };

/* SolveConfig (plan.hpp:19-38).  exec/force_evalj have no device meaning and
 * are omitted; `materialize` is fixed at plan time (a Materialize::kJ plan
 * carries no matrix-free J^T J programs) and is reported by mo_plan_materialize. */
typedef struct mo_solve_config {
  int method;
  int precision;
  int nonlinear_iters;
  int linear_iters;
  double pcg_rel_tol; /* < 0: 1e-4 (f32) / 1e-8 (f64), plan.hpp:192-193 */
  double pcg_abs_tol;
  int use_preconditioner;
  double lm_radius0, lm_radius_min, lm_radius_max;
  double lm_diag_min, lm_diag_max;
  double lm_min_decrease;
  double cost_stop_tol;
} mo_solve_config;

/* IterRow (solver.hpp:31-38) */
typedef struct mo_iter_row {
  int iter;
  double cost;
  int accepted;
  double radius;
  int pcg_iters;
  double wall_ms;
} mo_iter_row;

/* SolveResult (solver.hpp:58-74).  `trace` is owned by the session and stays
 * valid until the next mo_solve or mo_session_destroy. */
typedef struct mo_solve_result {
  double final_cost;
  int reason;
  int nonfinite_kernels;
  int indefinite_operator;
  int64_t unconstrained;
  int n_trace;
  const mo_iter_row* trace;
} mo_solve_result;

typedef struct mo_plan_s* mo_plan;
typedef struct mo_session_s* mo_session;

/* Per-iteration callback (solver.hpp:503): may read/modify the bound data
 * through mo_get_x / mo_bind_* before the next nonlinear iteration. */
typedef void (*mo_iter_cb)(int iter, mo_session s, void* user);

const char* mo_last_error(void);
const char* mo_version(void);
int mo_device_count(int* n);

/* ---- plans: CompiledPlan (plan.hpp:125-137) ---------------------------- */
/* Parse the moplan v1 interchange (integration/minopt_b200_bridge.hpp). */
int mo_plan_parse(const char* text, size_t len, mo_plan* out);
/* Override a declared dim's extent (programs are shape independent; the
 * column layout is recomputed as plan.hpp:212-218 would). */
int mo_plan_set_dim(mo_plan p, const char* name, int64_t extent);
int mo_plan_get_config(mo_plan p, mo_solve_config* cfg);
int mo_plan_set_config(mo_plan p, const mo_solve_config* cfg); /* plan(spec, cfg) checks, plan.hpp:190-199 */
int mo_plan_num_cols(mo_plan p, int64_t* n);
/* Generate + NVRTC-compile the plan's sm_100a module into the kernel cache
 * (no GPU needed); sessions then load it without compiling. */
int mo_plan_precompile(mo_plan p, int precision);
/* exact != 0: compile the per-element kernels without FMA contraction so
 * their add/mul round exactly like the reference's CPU build (bitwise
 * per-element parity); default 0 lets nvcc contract a*b+c into FMA
 * (results within the fp32 1e-5 / fp64 1e-10 tolerances). */
int mo_plan_set_exact(mo_plan p, int exact);
/* Materialize (plan.hpp:17) the plan was compiled for: 0 kNone, 1 kJ, 2 kJtJ. */
int mo_plan_materialize(mo_plan p, int* mode);
int mo_plan_counts(mo_plan p, int* n_params, int* n_arrays, int* n_graphs, int* n_unknowns);
int mo_plan_array_size(mo_plan p, int i, int64_t* n_scalars);
int mo_plan_graph_arity(mo_plan p, int i, int* arity);
void mo_plan_destroy(mo_plan p);

/* ---- sessions: Solver<Real> (solver.hpp:84-635) ------------------------ */
/* Bind the plan to a device; precision comes from the plan config.  The
 * session owns one stream and every device vector (solver.hpp:616-632). */
int mo_session_create(mo_plan p, int device, mo_session* out);
void mo_session_destroy(mo_session s);

/* SolveData<Real> (solver.hpp:23-29), copied host -> device. */
int mo_bind_x(mo_session s, const void* x, int64_t n);
int mo_bind_array(mo_session s, int i, const void* data, int64_t n);
int mo_bind_params(mo_session s, const double* params, int64_t n);
int mo_bind_graph(mo_session s, int i, const uint64_t* verts, int64_t n_entries, int arity);
/* Device-resident variants (pointers on the session's device). */
int mo_bind_x_device(mo_session s, const void* x, int64_t n);
int mo_bind_array_device(mo_session s, int i, const void* data, int64_t n);

/* refresh (solver.hpp:125-168): validate binds, computed arrays, masks. */
int mo_refresh(mo_session s);
int mo_num_cols(mo_session s, int64_t* n);
int mo_num_rows(mo_session s, int64_t* n);
int mo_get_excluded(mo_session s, uint8_t* out, int64_t n);

int mo_cost(mo_session s, double* out);                    /* solver.hpp:174 */
int mo_residuals(mo_session s, void* out, int64_t n);      /* solver.hpp:196 */
int mo_build_normal(mo_session s);                         /* solver.hpp:220 */
int mo_get_rhs(mo_session s, void* out, int64_t n);        /* rhs()  :108 */
int mo_get_precond(mo_session s, void* out, int64_t n);    /* precond() :109 */
int mo_apply_jtj(mo_session s, const void* v, void* out, int64_t n); /* :255 */
int mo_apply_jtj_device(mo_session s, const void* v, void* out);
int mo_solve(mo_session s, mo_iter_cb cb, void* user, mo_solve_result* out); /* :389 */
int mo_get_x(mo_session s, void* out, int64_t n);
int mo_saw_nonfinite(mo_session s, int* out);               /* :110 */
/* linearize (solver.hpp:291-377): evaluate the Jacobian lanes at x on the
 * device (plans with Jacobian lanes: materialized or force_evalj).  In
 * Materialize::kJ sessions mo_apply_jtj then computes 2 J^T (J v) in the
 * reference's spmv / spmv_t order (solver.hpp:278-283), in kJtJ sessions
 * spmv(H, v) over the assembled H = 2 J^T J (solver.hpp:284); before the first
 * linearize after a refresh it fails with MO_ERR_INTERNAL like the reference. */
int mo_linearize(mo_session s);
/* jacobian() (solver.hpp:378-381): the reference's CSR (rows template-major,
 * columns ascending, repeated edge vertices merged).  Call mo_jacobian_size,
 * then mo_get_jacobian with offs[rows + 1], col[nnz], val[nnz] (Real). */
int mo_jacobian_size(mo_session s, int64_t* rows, int64_t* cols, int64_t* nnz);
int mo_get_jacobian(mo_session s, int64_t* offs, int64_t* col, void* val, int64_t nnz);
/* normal_matrix() (solver.hpp:383-387): H = 2 J^T J of a Materialize::kJtJ
 * session, assembled on the device by mo_linearize in the reference's
 * transpose + spgemm order (sparse.hpp); offs[num_cols + 1], col/val[nnz]. */
int mo_normal_matrix_size(mo_session s, int64_t* nnz);
int mo_get_normal_matrix(mo_session s, int64_t* offs, int64_t* col, void* val, int64_t nnz);

/* ---- strip sharding (multi-GPU; no reference counterpart) --
 * A grid plan (one grid domain, no graphs) is split into contiguous strips
 * of axis-0 rows, one session per strip.  Each strip stores its rows plus
 * mo_plan_halo_rows() halo rows on each side (clipped at the domain edge);
 * binds take the strip's LOCAL data [lo, hi) (mo_session_local_layout).
 * Per PCG iteration the p halo is exchanged and the two dot products are
 * reduced in fixed rank order, so every strip takes identical steps. */
typedef struct mo_comm_s* mo_comm;
typedef struct mo_world_s* mo_world;
int mo_plan_halo_rows(mo_plan p, int* rows);
/* NCCL transport, one process per GPU: rank 0 creates the id, every rank passes it. */
int mo_nccl_unique_id(void* out, size_t len /* >= 128 */);
int mo_comm_create_nccl(const void* id, size_t len, int rank, int world, int device, mo_comm* out);
/* Single-process transport: `world` strip sessions on one device, each driven
 * from its own host thread (halo copies + fixed-order gathers). */
int mo_world_create_local(int world, int device, mo_world* out);
int mo_comm_create_local(mo_world w, int rank, mo_comm* out);
void mo_world_destroy(mo_world w);
void mo_comm_destroy(mo_comm c);
int mo_session_create_shard(mo_plan p, int device, mo_comm c, int64_t row0, int64_t row1, mo_session* out);
/* Graph energies (vertices = the domain's elements) shard the same way: a
 * strip stores every edge with an endpoint in its rows, so `halo` must cover
 * the graph's row bandwidth (max row distance within an edge; refused with
 * MO_ERR_BIND otherwise).  halo <= mo_plan_halo_rows() means the plan's. */
int mo_session_create_shard_halo(mo_plan p, int device, mo_comm c, int64_t row0, int64_t row1, int halo,
                                 mo_session* out);
int mo_session_local_layout(mo_session s, int64_t* lo, int64_t* hi, int64_t* row0, int64_t* row1);

/* ---- standalone Jacobi PCG: pcg<Real>(apply_a, b, m, delta, opt, ws,
 * excluded) (pcg.hpp:59-130) with PcgOptions / PcgOutcome (pcg.hpp:12-24).
 * The operator is the caller's: `apply(x, y, stream, user)` gets DEVICE
 * pointers of n Reals and must leave y = A x complete on return or enqueued
 * on `stream` (a cudaStream_t).  b, m, delta (out) and excluded (uint8, may
 * be NULL) are host buffers.  Numerical failures are flags, never errors. */
typedef struct mo_pcg_options {
  int max_iters;
  double tol_rel, tol_abs;
  int use_preconditioner;
} mo_pcg_options;
typedef struct mo_pcg_outcome {
  int iterations, indefinite, nonfinite;
} mo_pcg_outcome;
typedef void (*mo_apply_fn)(const void* x, void* y, void* stream, void* user);
int mo_pcg(int device, int precision, int64_t n, mo_apply_fn apply, void* user, const void* b, const void* m,
           void* delta, const mo_pcg_options* opt, const uint8_t* excluded, mo_pcg_outcome* out);

/* ---- on-disk formats (io.hpp:97-192) ------------------------------------ */
/* .optd dense arrays: "OPTD", u32 version 1, u8 dtype (0 = f32, 1 = f64),
 * u8 ndims, u16 channels, ndims x u64 extents, channel-interleaved row-major
 * IEEE payload; all little-endian.  Errors as read_optd / write_optd:
 * MO_ERR_FORMAT (bad magic / version / dtype, implausible extents, payload
 * longer than promised), MO_ERR_TRUNCATED (file ends early). */
int mo_optd_stat(const char* path, int* dtype, int* channels, int* ndims, int64_t* extents, int max_dims); /* io.hpp:122 */
int mo_optd_read(const char* path, void* values, int64_t count, int dtype);                                /* io.hpp:122 */
int mo_optd_write(const char* path, int dtype, int channels, int ndims, const int64_t* extents,
                  const void* values);                                                                      /* io.hpp:97 */
/* .optg hyperedge lists: "OPTG", u32 version 1, u16 arity, u64 edges,
 * edges x arity u64 vertex ids (read_optg / write_optg, io.hpp:158-192). */
int mo_optg_stat(const char* path, int* arity, int64_t* edges);                /* io.hpp:171 */
int mo_optg_read(const char* path, uint64_t* verts, int64_t n);                /* io.hpp:171 */
int mo_optg_write(const char* path, int arity, int64_t edges, const uint64_t* verts); /* io.hpp:158 */

/* ---- measurement hooks (bench.py) -------------------------------------- */
/* When enabled, CUDA events bracket every J^T J p apply and PCG vector update
 * launched by mo_solve (on the session stream, also inside CUDA graphs). */
int mo_set_profiling(mo_session s, int enable);
/* kind: 0 = J^T J p apply, 1 = PCG vector update, 2 = build_normal, 3 = cost */
int mo_profile_read(mo_session s, int kind, double* total_ms, int64_t* launches);
int mo_profile_reset(mo_session s);
/* Unperturbed kernel time for the roofline: `reps` back-to-back launches of
 * the J^T J p apply (which = 0, the PCG's own launch on the session's p) or
 * of build_normal (which = 1) replayed as one CUDA graph, best of 3; writes
 * ms per launch.  Clobbers the PCG scratch vectors (x is untouched). */
int mo_bench_kernel(mo_session s, int which, int reps, double* ms_per_launch);
int mo_session_stream(mo_session s, void** stream); /* cudaStream_t */
/* Number of this library's kernels launched so far (host-side count). */
int mo_kernel_launches(mo_session s, int64_t* n);
/* Name of the J^T J p kernel gather set i runs (autotuned on first use;
 * MO_B200_JTJ=gather|twophase|stream|tma|warp|gprog|tma4 forces it). */
int mo_apply_kernel(mo_session s, int gather_set, char* name, size_t len);
/* Name of the build_normal (J^T F + Jacobi) kernel gather set i runs
 * (solver.hpp:220-251; tuned on first use like mo_apply_kernel). */
int mo_normal_kernel(mo_session s, int gather_set, char* name, size_t len);

#ifdef __cplusplus
}
#endif
#endif /* MO_B200_H_ */
