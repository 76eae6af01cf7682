// mo_session.hpp — precision-erased interface of a bound solver session
// (the device counterpart of minopt::Solver<Real>, solver.hpp:80-635).
#pragma once
#include <string>

#include <cstdint>
#include <memory>
#include <vector>

#include "mo_plan.hpp"

namespace mo {

struct IterRow {
  int iter = 0;
  double cost = 0;
  bool accepted = true;
  double radius = 0;
  int pcg_iters = 0;
  double wall_ms = 0;
};

struct SolveResult {
  double final_cost = 0;
  int reason = 0;  // StopReason (solver.hpp:40-46)
  std::vector<IterRow> trace;
  bool nonfinite_kernels = false;
  bool indefinite_operator = false;
  int64_t unconstrained = 0;
};

using IterCallback = void (*)(int iter, void* user);

class SessionBase {
 public:
  virtual ~SessionBase() = default;
  virtual void bind_x(const void* x, int64_t n, bool device) = 0;
  virtual void bind_array(int i, const void* data, int64_t n, bool device) = 0;
  virtual void bind_params(const double* p, int64_t n) = 0;
  virtual void bind_graph(int i, const uint64_t* verts, int64_t n, int arity) = 0;
  virtual void refresh() = 0;
  virtual int64_t num_cols() const = 0;
  virtual int64_t num_rows() = 0;
  virtual void excluded(uint8_t* out, int64_t n) = 0;
  virtual double cost() = 0;
  virtual void residuals(void* out, int64_t n) = 0;
  virtual void build_normal() = 0;
  virtual void get_rhs(void* out, int64_t n) = 0;
  virtual void get_precond(void* out, int64_t n) = 0;
  virtual void apply_jtj(const void* v, void* out, int64_t n, bool device) = 0;
  virtual SolveResult solve(IterCallback cb, void* user) = 0;
  virtual void get_x(void* out, int64_t n) = 0;
  virtual bool saw_nonfinite() = 0;
  virtual void set_profiling(bool on) = 0;
  virtual void profile_read(int kind, double* ms, int64_t* n) = 0;
  virtual void profile_reset() = 0;
  virtual double bench_kernel(int which, int reps) = 0;
  virtual void* stream() = 0;
  virtual int64_t launches() const = 0;
  virtual std::string apply_kernel(int gather_set) = 0;
  virtual std::string normal_kernel(int gather_set) = 0;
  // linearize / jacobian (solver.hpp:291-382): evaluate the Jacobian lanes on
  // the device; jacobian() assembles the reference's CSR from them (host).
  virtual void linearize() = 0;
  virtual void jacobian(int64_t* rows, int64_t* cols, std::vector<int64_t>* offs, std::vector<int64_t>* col,
                        std::vector<double>* val) = 0;
  // normal_matrix() (solver.hpp:383-387) of a Materialize::kJtJ session, CSR.
  virtual void normal_matrix(std::vector<int64_t>* offs, std::vector<int64_t>* col, std::vector<double>* val) = 0;
  // Strip shards: stored rows [lo, hi), owned rows [row0, row1) (all 0 when unsharded).
  virtual void local_layout(int64_t* lo, int64_t* hi, int64_t* row0, int64_t* row1) const = 0;
};

// Standalone Jacobi PCG (pcg.hpp:12-130) over a caller's operator.
struct PcgOpts {  // PcgOptions defaults (pcg.hpp:12-17)
  int max_iters = 10;
  double tol_rel = 1e-3, tol_abs = 0.0;
  bool use_preconditioner = true;
};
struct PcgOutcome {
  int iterations = 0;
  bool indefinite = false, nonfinite = false;
};
using PcgApply = void (*)(const void* x, void* y, void* stream, void* user);
PcgOutcome run_pcg(int device, int precision, int64_t n, PcgApply apply, void* user, const void* b, const void* m,
                   void* delta, const PcgOpts& opt, const uint8_t* excluded);

class Comm;
std::unique_ptr<SessionBase> make_session(const Plan& plan, int device);
// Strip shard owning rows [row0, row1) of the plan's grid domain; `comm` must
// outlive the session.
std::unique_ptr<SessionBase> make_shard_session(const Plan& plan, int device, Comm* comm, int64_t row0,
                                                int64_t row1, int halo = 0);
// Halo rows a strip needs on each side (max axis-0 reach of every program +
// the two-phase apply's lane halo).
int halo_rows(const Plan& plan);

}  // namespace mo
