// mo_capi.cpp — extern "C" boundary (include/mo_b200.h).  Every entry point
// catches mo::Error and maps it to 1 + Err (common.hpp:13-32), recording the
// message for mo_last_error().
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "../../include/mo_b200.h"
#include "mo_codegen.hpp"
#include "mo_comm.hpp"
#include "mo_jit.hpp"
#include "mo_plan.hpp"
#include "mo_session.hpp"

namespace mo {
const char* device_prelude() {
  static const char* kPrelude =
#include "mo_device_cuh.inc"
      ;
  return kPrelude;
}
}  // namespace mo

struct mo_plan_s {
  mo::Plan plan;
};
struct mo_world_s {
  std::shared_ptr<mo::LocalWorld> w;
};
struct mo_comm_s {
  std::unique_ptr<mo::Comm> c;
};
struct mo_session_s {
  std::unique_ptr<mo::SessionBase> impl;
  std::vector<mo_iter_row> trace;
  mo_iter_cb cb = nullptr;
  void* user = nullptr;
  bool f32 = false;
};

namespace {

thread_local std::string g_err;

int code_of(mo::Err e) {
  if (e == mo::Err::kCuda) return MO_ERR_CUDA;
  if (e == mo::Err::kNoDevice) return MO_ERR_NO_DEVICE;
  return 1 + int(e);
}

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return MO_OK;
  } catch (const mo::Error& e) {
    g_err = e.what();
    return code_of(e.code);
  } catch (const std::exception& e) {
    g_err = e.what();
    return MO_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  mo::check(p != nullptr, mo::Err::kBindError, std::string("null ") + what);
}

mo::Config from_c(const mo_solve_config& c) {
  mo::Config k;
  k.method = c.method;
  k.precision = c.precision;
  k.nonlinear_iters = c.nonlinear_iters;
  k.linear_iters = c.linear_iters;
  k.pcg_rel_tol = c.pcg_rel_tol;
  k.pcg_abs_tol = c.pcg_abs_tol;
  k.use_preconditioner = c.use_preconditioner != 0;
  k.lm_radius0 = c.lm_radius0;
  k.lm_radius_min = c.lm_radius_min;
  k.lm_radius_max = c.lm_radius_max;
  k.lm_diag_min = c.lm_diag_min;
  k.lm_diag_max = c.lm_diag_max;
  k.lm_min_decrease = c.lm_min_decrease;
  k.cost_stop_tol = c.cost_stop_tol;
  return k;
}

void to_c(const mo::Config& k, mo_solve_config* c) {
  c->method = k.method;
  c->precision = k.precision;
  c->nonlinear_iters = k.nonlinear_iters;
  c->linear_iters = k.linear_iters;
  c->pcg_rel_tol = k.pcg_rel_tol;
  c->pcg_abs_tol = k.pcg_abs_tol;
  c->use_preconditioner = k.use_preconditioner ? 1 : 0;
  c->lm_radius0 = k.lm_radius0;
  c->lm_radius_min = k.lm_radius_min;
  c->lm_radius_max = k.lm_radius_max;
  c->lm_diag_min = k.lm_diag_min;
  c->lm_diag_max = k.lm_diag_max;
  c->lm_min_decrease = k.lm_min_decrease;
  c->cost_stop_tol = k.cost_stop_tol;
}

void trampoline(int iter, void* user) {
  auto* s = static_cast<mo_session_s*>(user);
  if (s->cb) s->cb(iter, s, s->user);
}

}  // namespace

namespace mo {
// (mo_io.cpp records its errors here too: one mo_last_error() per thread)
void set_last_error(const std::string& m) { g_err = m; }
}  // namespace mo

extern "C" {

const char* mo_last_error(void) { return g_err.c_str(); }
const char* mo_version(void) { return "mo_b200 0.1 (sm_100a)"; }

int mo_device_count(int* n) {
  return guard([&] {
    need(n, "output");
    int k = 0;
    if (cudaGetDeviceCount(&k) != cudaSuccess) {
      cudaGetLastError();
      k = 0;
    }
    *n = k;
  });
}

int mo_plan_parse(const char* text, size_t len, mo_plan* out) {
  return guard([&] {
    need(text, "plan text");
    need(out, "output");
    auto* p = new mo_plan_s{mo::parse_plan(std::string(text, len))};
    *out = p;
  });
}

int mo_plan_set_dim(mo_plan p, const char* name, int64_t extent) {
  return guard([&] {
    need(p, "plan");
    need(name, "dim name");
    mo::check(extent >= 0 && extent < (int64_t(1) << 31), mo::Err::kBindError, "dim extent out of range");
    bool found = false;
    for (auto& d : p->plan.dims)
      if (d.first == name) {
        d.second = extent;
        found = true;
      }
    mo::check(found, mo::Err::kUndeclaredIdentifier, std::string("no dim named ") + name);
    p->plan.relayout();
  });
}

int mo_plan_get_config(mo_plan p, mo_solve_config* cfg) {
  return guard([&] {
    need(p, "plan");
    need(cfg, "config");
    to_c(p->plan.cfg, cfg);
  });
}

// plan(spec, cfg) argument checks (plan.hpp:190-199).
int mo_plan_set_config(mo_plan p, const mo_solve_config* cfg) {
  return guard([&] {
    need(p, "plan");
    need(cfg, "config");
    mo::Config k = from_c(*cfg);
    mo::check(k.nonlinear_iters >= 1, mo::Err::kBindError, "nonlinear iteration count must be >= 1");
    mo::check(k.linear_iters >= 1, mo::Err::kBindError, "linear iteration count must be >= 1");
    mo::check(k.method == 0 || k.method == 1, mo::Err::kBindError, "unknown method");
    mo::check(k.precision == 0 || k.precision == 1, mo::Err::kBindError, "unknown precision");
    if (k.pcg_rel_tol < 0) k.pcg_rel_tol = k.precision == 0 ? 1e-4 : 1e-8;
    mo::check(k.pcg_abs_tol >= 0 && k.cost_stop_tol >= 0, mo::Err::kBindError, "tolerances must be non-negative");
    mo::check(k.lm_radius_min <= k.lm_radius0 && k.lm_radius0 <= k.lm_radius_max, mo::Err::kBindError,
              "trust-region radius bounds must bracket the initial radius");
    mo::check(k.lm_diag_min <= k.lm_diag_max && k.lm_diag_min >= 0, mo::Err::kBindError,
              "damping diagonal clamp must be an interval");
    k.materialize = p->plan.cfg.materialize;  // fixed at plan time
    p->plan.cfg = k;
  });
}

int mo_plan_precompile(mo_plan p, int precision) {
  return guard([&] {
    need(p, "plan");
    mo::compile_cubin(mo::generate_module(p->plan, precision != 0, mo::device_prelude()), "mo_plan.cu", p->plan.exact);
  });
}

int mo_plan_set_exact(mo_plan p, int exact) {
  return guard([&] {
    need(p, "plan");
    p->plan.exact = exact != 0;
  });
}

int mo_plan_materialize(mo_plan p, int* mode) {
  return guard([&] {
    need(p, "plan");
    need(mode, "output");
    *mode = p->plan.cfg.materialize;
  });
}
int mo_plan_num_cols(mo_plan p, int64_t* n) {
  return guard([&] {
    need(p, "plan");
    need(n, "output");
    *n = p->plan.num_cols;
  });
}

int mo_plan_counts(mo_plan p, int* np, int* na, int* ng, int* nu) {
  return guard([&] {
    need(p, "plan");
    if (np) *np = int(p->plan.params.size());
    if (na) *na = int(p->plan.arrays.size());
    if (ng) *ng = int(p->plan.graphs.size());
    if (nu) *nu = int(p->plan.unknowns.size());
  });
}

int mo_plan_array_size(mo_plan p, int i, int64_t* n) {
  return guard([&] {
    need(p, "plan");
    need(n, "output");
    mo::check(i >= 0 && size_t(i) < p->plan.arrays.size(), mo::Err::kBindError, "array index out of range");
    *n = p->plan.extent_of(p->plan.arrays[size_t(i)].dom) * p->plan.arrays[size_t(i)].channels;
  });
}

int mo_plan_graph_arity(mo_plan p, int i, int* arity) {
  return guard([&] {
    need(p, "plan");
    need(arity, "output");
    mo::check(i >= 0 && size_t(i) < p->plan.graphs.size(), mo::Err::kBindError, "graph index out of range");
    *arity = p->plan.graphs[size_t(i)].second;
  });
}

void mo_plan_destroy(mo_plan p) { delete p; }

int mo_session_create(mo_plan p, int device, mo_session* out) {
  return guard([&] {
    need(p, "plan");
    need(out, "output");
    auto s = std::make_unique<mo_session_s>();
    s->impl = mo::make_session(p->plan, device);
    s->f32 = p->plan.cfg.precision == 0;
    *out = s.release();
  });
}

void mo_session_destroy(mo_session s) { delete s; }

#define SESSION_CALL(...) \
  return guard([&] {      \
    need(s, "session");   \
    __VA_ARGS__;          \
  })

int mo_bind_x(mo_session s, const void* x, int64_t n) { SESSION_CALL(s->impl->bind_x(x, n, false)); }
int mo_bind_array(mo_session s, int i, const void* d, int64_t n) { SESSION_CALL(s->impl->bind_array(i, d, n, false)); }
int mo_bind_params(mo_session s, const double* p, int64_t n) { SESSION_CALL(s->impl->bind_params(p, n)); }
int mo_bind_graph(mo_session s, int i, const uint64_t* v, int64_t n, int arity) {
  SESSION_CALL(s->impl->bind_graph(i, v, n, arity));
}
int mo_bind_x_device(mo_session s, const void* x, int64_t n) { SESSION_CALL(s->impl->bind_x(x, n, true)); }
int mo_bind_array_device(mo_session s, int i, const void* d, int64_t n) {
  SESSION_CALL(s->impl->bind_array(i, d, n, true));
}
int mo_refresh(mo_session s) { SESSION_CALL(s->impl->refresh()); }
int mo_num_cols(mo_session s, int64_t* n) { SESSION_CALL(need(n, "output"); *n = s->impl->num_cols()); }
int mo_num_rows(mo_session s, int64_t* n) { SESSION_CALL(need(n, "output"); *n = s->impl->num_rows()); }
int mo_get_excluded(mo_session s, uint8_t* out, int64_t n) { SESSION_CALL(s->impl->excluded(out, n)); }
int mo_cost(mo_session s, double* out) { SESSION_CALL(need(out, "output"); *out = s->impl->cost()); }
int mo_residuals(mo_session s, void* out, int64_t n) { SESSION_CALL(s->impl->residuals(out, n)); }
int mo_build_normal(mo_session s) { SESSION_CALL(s->impl->build_normal()); }
int mo_get_rhs(mo_session s, void* out, int64_t n) { SESSION_CALL(s->impl->get_rhs(out, n)); }
int mo_get_precond(mo_session s, void* out, int64_t n) { SESSION_CALL(s->impl->get_precond(out, n)); }
int mo_apply_jtj(mo_session s, const void* v, void* out, int64_t n) {
  SESSION_CALL(s->impl->apply_jtj(v, out, n, false));
}
int mo_apply_jtj_device(mo_session s, const void* v, void* out) {
  SESSION_CALL(s->impl->apply_jtj(v, out, s->impl->num_cols(), true));
}
int mo_get_x(mo_session s, void* out, int64_t n) { SESSION_CALL(s->impl->get_x(out, n)); }
int mo_saw_nonfinite(mo_session s, int* out) { SESSION_CALL(need(out, "output"); *out = s->impl->saw_nonfinite()); }

int mo_solve(mo_session s, mo_iter_cb cb, void* user, mo_solve_result* out) {
  SESSION_CALL({
    need(out, "output");
    s->cb = cb;
    s->user = user;
    mo::SolveResult r = s->impl->solve(cb ? trampoline : nullptr, s);
    s->trace.clear();
    for (const mo::IterRow& row : r.trace)
      s->trace.push_back({row.iter, row.cost, row.accepted ? 1 : 0, row.radius, row.pcg_iters, row.wall_ms});
    out->final_cost = r.final_cost;
    out->reason = r.reason;
    out->nonfinite_kernels = r.nonfinite_kernels ? 1 : 0;
    out->indefinite_operator = r.indefinite_operator ? 1 : 0;
    out->unconstrained = r.unconstrained;
    out->n_trace = int(s->trace.size());
    out->trace = s->trace.data();
  });
}

int mo_plan_halo_rows(mo_plan p, int* rows) {
  return guard([&] {
    need(p, "plan");
    need(rows, "output");
    *rows = mo::halo_rows(p->plan);
  });
}

int mo_nccl_unique_id(void* out, size_t len) {
  return guard([&] {
    need(out, "output");
    mo::check(len >= 128, mo::Err::kBindError, "NCCL unique id needs 128 bytes");
    mo::nccl_unique_id(out);
  });
}

int mo_comm_create_nccl(const void* id, size_t len, int rank, int world, int device, mo_comm* out) {
  return guard([&] {
    need(id, "id");
    need(out, "output");
    mo::check(len >= 128, mo::Err::kBindError, "NCCL unique id needs 128 bytes");
    auto c = std::make_unique<mo_comm_s>();
    c->c = mo::make_nccl_comm(id, rank, world, device);
    *out = c.release();
  });
}

int mo_world_create_local(int world, int device, mo_world* out) {
  return guard([&] {
    need(out, "output");
    auto w = std::make_unique<mo_world_s>();
    w->w = mo::make_local_world(world, device);
    *out = w.release();
  });
}

int mo_comm_create_local(mo_world w, int rank, mo_comm* out) {
  return guard([&] {
    need(w, "world");
    need(out, "output");
    auto c = std::make_unique<mo_comm_s>();
    c->c = mo::make_local_comm(w->w, rank);
    *out = c.release();
  });
}

void mo_world_destroy(mo_world w) { delete w; }
void mo_comm_destroy(mo_comm c) { delete c; }

int mo_session_create_shard(mo_plan p, int device, mo_comm c, int64_t row0, int64_t row1, mo_session* out) {
  return guard([&] {
    need(p, "plan");
    need(c, "communicator");
    need(out, "output");
    auto s = std::make_unique<mo_session_s>();
    s->impl = mo::make_shard_session(p->plan, device, c->c.get(), row0, row1);
    s->f32 = p->plan.cfg.precision == 0;
    *out = s.release();
  });
}

int mo_session_create_shard_halo(mo_plan p, int device, mo_comm c, int64_t row0, int64_t row1, int halo,
                                 mo_session* out) {
  return guard([&] {
    need(p, "plan");
    need(c, "communicator");
    need(out, "output");
    auto s = std::make_unique<mo_session_s>();
    s->impl = mo::make_shard_session(p->plan, device, c->c.get(), row0, row1, halo);
    s->f32 = p->plan.cfg.precision == 0;
    *out = s.release();
  });
}

int mo_session_local_layout(mo_session s, int64_t* lo, int64_t* hi, int64_t* row0, int64_t* row1) {
  SESSION_CALL(need(lo, "output"); need(hi, "output"); need(row0, "output"); need(row1, "output");
               s->impl->local_layout(lo, hi, row0, row1));
}

int mo_set_profiling(mo_session s, int enable) { SESSION_CALL(s->impl->set_profiling(enable != 0)); }
int mo_profile_read(mo_session s, int kind, double* ms, int64_t* n) {
  SESSION_CALL(need(ms, "output"); need(n, "output"); s->impl->profile_read(kind, ms, n));
}
int mo_profile_reset(mo_session s) { SESSION_CALL(s->impl->profile_reset()); }
int mo_bench_kernel(mo_session s, int which, int reps, double* ms_per_launch) {
  SESSION_CALL(need(ms_per_launch, "output"); *ms_per_launch = s->impl->bench_kernel(which, reps));
}
int mo_session_stream(mo_session s, void** st) { SESSION_CALL(need(st, "output"); *st = s->impl->stream()); }
int mo_kernel_launches(mo_session s, int64_t* n) { SESSION_CALL(need(n, "output"); *n = s->impl->launches()); }
int mo_linearize(mo_session s) { SESSION_CALL(s->impl->linearize()); }
int mo_jacobian_size(mo_session s, int64_t* rows, int64_t* cols, int64_t* nnz) {
  SESSION_CALL({
    need(rows, "output");
    need(cols, "output");
    need(nnz, "output");
    std::vector<int64_t> offs;
    s->impl->jacobian(rows, cols, &offs, nullptr, nullptr);
    *nnz = offs.empty() ? 0 : offs.back();
  });
}
int mo_get_jacobian(mo_session s, int64_t* offs, int64_t* col, void* val, int64_t nnz) {
  SESSION_CALL({
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> o, c;
    std::vector<double> v;
    s->impl->jacobian(&rows, &cols, &o, &c, &v);
    mo::check(nnz == int64_t(c.size()), mo::Err::kShapeMismatch, "jacobian(): nnz does not match mo_jacobian_size");
    if (offs) std::memcpy(offs, o.data(), o.size() * sizeof(int64_t));
    if (col && !c.empty()) std::memcpy(col, c.data(), c.size() * sizeof(int64_t));
    if (val) {
      if (s->f32)
        for (size_t k = 0; k < v.size(); ++k) static_cast<float*>(val)[k] = float(v[k]);
      else if (!v.empty())
        std::memcpy(val, v.data(), v.size() * sizeof(double));
    }
  });
}

int mo_normal_matrix_size(mo_session s, int64_t* nnz) {
  SESSION_CALL({
    need(nnz, "output");
    std::vector<int64_t> o, c;
    std::vector<double> v;
    s->impl->normal_matrix(&o, &c, &v);
    *nnz = int64_t(c.size());
  });
}
int mo_get_normal_matrix(mo_session s, int64_t* offs, int64_t* col, void* val, int64_t nnz) {
  SESSION_CALL({
    std::vector<int64_t> o, c;
    std::vector<double> v;
    s->impl->normal_matrix(&o, &c, &v);
    mo::check(nnz == int64_t(c.size()), mo::Err::kShapeMismatch, "normal_matrix(): nnz does not match");
    if (offs) std::memcpy(offs, o.data(), o.size() * sizeof(int64_t));
    if (col && !c.empty()) std::memcpy(col, c.data(), c.size() * sizeof(int64_t));
    if (val) {
      if (s->f32)
        for (size_t k = 0; k < v.size(); ++k) static_cast<float*>(val)[k] = float(v[k]);
      else if (!v.empty())
        std::memcpy(val, v.data(), v.size() * sizeof(double));
    }
  });
}

int mo_pcg(int device, int precision, int64_t n, mo_apply_fn apply, void* user, const void* b, const void* m,
           void* delta, const mo_pcg_options* opt, const uint8_t* excluded, mo_pcg_outcome* out) {
  return guard([&] {
    need(opt, "options");
    need(out, "output");
    mo::PcgOpts o;
    o.max_iters = opt->max_iters;
    o.tol_rel = opt->tol_rel;
    o.tol_abs = opt->tol_abs;
    o.use_preconditioner = opt->use_preconditioner != 0;
    const mo::PcgOutcome r = mo::run_pcg(device, precision, n, apply, user, b, m, delta, o, excluded);
    out->iterations = r.iterations;
    out->indefinite = r.indefinite ? 1 : 0;
    out->nonfinite = r.nonfinite ? 1 : 0;
  });
}

int mo_apply_kernel(mo_session s, int gather_set, char* name, size_t len) {
  SESSION_CALL(need(name, "output"); const std::string k = s->impl->apply_kernel(gather_set);
               mo::check(len > k.size(), mo::Err::kShapeMismatch, "name buffer too small");
               std::memcpy(name, k.c_str(), k.size() + 1));
}

int mo_normal_kernel(mo_session s, int gather_set, char* name, size_t len) {
  SESSION_CALL(need(name, "output"); const std::string k = s->impl->normal_kernel(gather_set);
               mo::check(len > k.size(), mo::Err::kShapeMismatch, "name buffer too small");
               std::memcpy(name, k.c_str(), k.size() + 1));
}

}  // extern "C"
