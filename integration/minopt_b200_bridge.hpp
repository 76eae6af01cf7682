// minopt_b200_bridge.hpp — the reference-side binding a minopt maintainer adds
// to hand a CompiledPlan to the B200 library.
//
// This header is compiled AGAINST the reference headers
// (/root/reference/proj/include/minopt); it is not part of the product
// library.  It serialises the plan-time output of the reference compiler —
// CompiledPlan (plan.hpp:125-137): the spec's domains/fields, the column layout
// `ubase` (plan.hpp:212-218), and every KernelProgram (program.hpp:74-82) of
// the matrix-free path — into the plain-text "moplan v1" interchange that
// mo_plan_parse() (include/mo_b200.h) consumes.  Nothing here runs on the hot
// path: the device executes its own CUDA translation of these programs.
//
// Format (whitespace separated, one record per line, doubles as C99 hexfloats
// so immediates round-trip bit-exactly):
//   moplan 1
//   cfg <method> <precision> <nl> <lin> <rel> <abs> <precond> <r0> <rmin> <rmax>
//       <dmin> <dmax> <eta> <cost_stop>
//   [materialize M]   (1 = Materialize::kJ, 2 = kJtJ; absent = matrix-free)
//   dims N            / dim NAME EXTENT
//   params N          / param NAME
//   unknowns N        / unknown NAME CH ND dims...
//   arrays N          / array NAME CH ND dims...
//   computed N        / computed NAME MODE TOTALCH ND dims...
//   graphs N          / graph NAME ARITY
//   residuals N       / residual grid ND dims... | residual graph G
//   ubase N cols... ; num_cols V
//   grid_sets N       / grid_set ND dims... NT t...   + programs cost, evalf
//                       [+ evalj NT / jtemplate T GUARD ORIGIN NL (out f c o0 o1 o2)...
//                          + program evalj]   (plans built with force_evalj)
//   gather_sets N     / gather_set ND dims... NCH (f c)...   + programs bm, jtj
//   graph_sets N      / graph_set G NT t... NS (slot f c)... + cost, evalf, bm, jtj
//                       [+ gevalj NT / gjtemplate T NL (out f c slot)... + program evalj]
//   computed_kernels N/ computed_kernel IDX ND dims...   + program prog
//   exclude_kernels N / exclude_kernel ND dims...        + program prog
//   end
// program NAME REGS NI NB NG NO, then NI `i` lines (op sub dst a b c gid field
// channel graph off0 off1 off2 slot imm pnum pden), NB `b` lines (gid begin
// end), NG `g` lines (guard register), NO `o` lines (nroots (gid reg)...).
#pragma once

#include <algorithm>
#include <array>
#include <cstdio>
#include <sstream>
#include <string>

#include "minopt/plan.hpp"

namespace minopt::b200 {

namespace bridge_detail {

inline std::string hexf(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", v);
  return buf;
}

inline void put_domain(std::ostream& os, const GridDomain& d) {
  os << d.dims.size();
  for (int di : d.dims) os << ' ' << di;
}

inline void put_program(std::ostream& os, const char* name, const KernelProgram& p) {
  os << "program " << name << ' ' << p.num_regs << ' ' << p.instrs.size() << ' '
     << p.blocks.size() << ' ' << p.guards.size() << ' ' << p.outputs.size() << '\n';
  for (const Instr& in : p.instrs)
    os << "i " << int(in.op) << ' ' << int(in.sub) << ' ' << in.dst << ' ' << in.a << ' '
       << in.b << ' ' << in.c << ' ' << in.gid << ' ' << in.field << ' ' << in.channel << ' '
       << int(in.acc.graph) << ' ' << in.acc.off[0] << ' ' << in.acc.off[1] << ' '
       << in.acc.off[2] << ' ' << in.acc.slot << ' ' << hexf(in.imm) << ' ' << in.pnum << ' '
       << in.pden << '\n';
  for (const Block& b : p.blocks) os << "b " << b.gid << ' ' << b.begin << ' ' << b.end << '\n';
  for (const GuardInfo& g : p.guards) os << "g " << g.reg << '\n';
  for (const KernelOutput& o : p.outputs) {
    os << "o " << o.roots.size();
    for (auto [gid, reg] : o.roots) os << ' ' << gid << ' ' << reg;
    os << '\n';
  }
}

}  // namespace bridge_detail

// Serialise a CompiledPlan.  Materialized plans (Materialize::kJ / kJtJ,
// plan.hpp:17) carry no gather J^T J programs (plan.hpp:210, 289, 331); the
// device then applies its J (or H = 2 J^T J) assembled from the evalj lanes.
inline std::string export_plan_text(const CompiledPlan& P) {
  using namespace bridge_detail;
  const ProblemSpec& s = P.spec;
  const SolveConfig& c = P.cfg;
  std::ostringstream os;
  os << "moplan 1\n";
  os << "cfg " << int(c.method) << ' ' << int(c.precision) << ' ' << c.nonlinear_iters << ' '
     << c.linear_iters << ' ' << hexf(c.pcg_rel_tol) << ' ' << hexf(c.pcg_abs_tol) << ' '
     << int(c.use_preconditioner) << ' ' << hexf(c.lm_radius0) << ' ' << hexf(c.lm_radius_min)
     << ' ' << hexf(c.lm_radius_max) << ' ' << hexf(c.lm_diag_min) << ' '
     << hexf(c.lm_diag_max) << ' ' << hexf(c.lm_min_decrease) << ' ' << hexf(c.cost_stop_tol)
     << '\n';
  if (c.materialize != Materialize::kNone) os << "materialize " << int(c.materialize) << '\n';
  os << "dims " << s.dims.size() << '\n';
  for (const DimDecl& d : s.dims) os << "dim " << d.name << ' ' << d.extent << '\n';
  os << "params " << s.params.size() << '\n';
  for (const std::string& p : s.params) os << "param " << p << '\n';
  os << "unknowns " << s.unknowns.size() << '\n';
  for (const UnknownField& u : s.unknowns) {
    os << "unknown " << u.name << ' ' << u.channels << ' ';
    put_domain(os, u.domain);
    os << '\n';
  }
  os << "arrays " << s.arrays.size() << '\n';
  for (const ArrayField& a : s.arrays) {
    os << "array " << a.name << ' ' << a.channels << ' ';
    put_domain(os, a.domain);
    os << '\n';
  }
  os << "computed " << s.computed.size() << '\n';
  for (const ComputedArray& ca : s.computed) {
    os << "computed " << ca.name << ' ' << int(ca.mode) << ' ' << ca.total_channels() << ' ';
    put_domain(os, ca.domain);
    os << '\n';
  }
  os << "graphs " << s.graphs.size() << '\n';
  for (const GraphDecl& g : s.graphs) os << "graph " << g.name << ' ' << g.arity() << '\n';
  os << "residuals " << P.transformed.residuals.size() << '\n';
  for (const ResidualTerm& r : P.transformed.residuals) {
    if (r.kind == DomainKind::kGrid) {
      os << "residual grid ";
      put_domain(os, r.domain);
    } else {
      os << "residual graph " << r.graph;
    }
    os << '\n';
  }
  os << "ubase " << P.ubase.size();
  for (int64_t u : P.ubase) os << ' ' << u;
  os << "\nnum_cols " << P.num_cols << '\n';

  os << "grid_sets " << P.grid_sets.size() << '\n';
  for (const GridKernels& g : P.grid_sets) {
    os << "grid_set ";
    put_domain(os, g.domain);
    os << ' ' << g.templates.size();
    for (int t : g.templates) os << ' ' << t;
    os << '\n';
    put_program(os, "cost", g.cost);
    put_program(os, "evalf", g.evalf);
    if (P.has_evalj) {
      // Per-template Jacobian lanes (plan.hpp:59-72, 244-264): the device's
      // two-phase J^T J p evaluates these once per element.
      os << "evalj " << g.jtemplates.size() << '\n';
      for (const auto& jt : g.jtemplates) {
        // ORIGIN: the template reads at its own pixel, so a shifted instance
        // whose centre leaves the domain is guarded off (transform.hpp:177-198);
        // the bound guard itself folds that test away at the origin.
        const auto& offs = P.transformed.residuals[size_t(jt.tmpl)].offsets;
        const bool origin = std::find(offs.begin(), offs.end(), std::array<int16_t, 3>{0, 0, 0}) != offs.end();
        os << "jtemplate " << jt.tmpl << ' ' << jt.guard_out << ' ' << int(origin) << ' ' << jt.lanes.size();
        for (const JLane& l : jt.lanes)
          os << ' ' << l.out << ' ' << l.field << ' ' << l.channel << ' ' << l.off[0] << ' ' << l.off[1]
             << ' ' << l.off[2];
        os << '\n';
      }
      put_program(os, "evalj", g.evalj);
    }
  }
  os << "gather_sets " << P.gather_sets.size() << '\n';
  for (const GatherKernels& g : P.gather_sets) {
    os << "gather_set ";
    put_domain(os, g.domain);
    os << ' ' << g.chans.size();
    for (const auto& ch : g.chans) os << ' ' << ch.field << ' ' << ch.channel;
    os << '\n';
    put_program(os, "bm", g.bm);
    put_program(os, "jtj", g.jtj);
  }
  os << "graph_sets " << P.graph_sets.size() << '\n';
  for (const GraphKernels& g : P.graph_sets) {
    os << "graph_set " << g.graph << ' ' << g.templates.size();
    for (int t : g.templates) os << ' ' << t;
    os << ' ' << g.scats.size();
    for (const auto& sc : g.scats) os << ' ' << sc.slot << ' ' << sc.field << ' ' << sc.channel;
    os << '\n';
    put_program(os, "cost", g.cost);
    put_program(os, "evalf", g.evalf);
    put_program(os, "bm", g.bm);
    put_program(os, "jtj", g.jtj);
    if (P.has_evalj) {
      // Per-template Jacobian lanes of the edge rows (plan.hpp:318-330).
      os << "gevalj " << g.jtemplates.size() << '\n';
      for (const auto& jt : g.jtemplates) {
        os << "gjtemplate " << jt.tmpl << ' ' << jt.lanes.size();
        for (const JLane& l : jt.lanes) os << ' ' << l.out << ' ' << l.field << ' ' << l.channel << ' ' << l.slot;
        os << '\n';
      }
      put_program(os, "evalj", g.evalj);
    }
  }
  os << "computed_kernels " << P.computed_kernels.size() << '\n';
  for (const ComputedKernels& ck : P.computed_kernels) {
    os << "computed_kernel " << ck.index << ' ';
    put_domain(os, s.computed[size_t(ck.index)].domain);
    os << '\n';
    put_program(os, "prog", ck.prog);
  }
  os << "exclude_kernels " << P.exclude_kernels.size() << '\n';
  for (const ExcludeKernels& ek : P.exclude_kernels) {
    os << "exclude_kernel ";
    put_domain(os, ek.domain);
    os << '\n';
    put_program(os, "prog", ek.prog);
  }
  os << "end\n";
  return os.str();
}

}  // namespace minopt::b200

#ifdef MINOPT_B200_WITH_SOLVER
// ---------------------------------------------------------------------------
// Drop-in device solver: same constructor and routine signatures as
// minopt::Solver<Real> (solver.hpp:80-635), executing on the GPU through the
// C ABI of libmo_b200.so.  Switching a caller from minopt::Solver<double> to
// minopt::b200::Solver<double> is the whole integration.
#include <cstring>
#include <functional>
#include <span>

#include "mo_b200.h"
#include "minopt/solver.hpp"
#include "minopt/sparse.hpp"

namespace minopt::b200 {

[[noreturn]] inline void rethrow(int rc) {
  Err code = Err::kInternal;
  if (rc >= 1 && rc <= int(Err::kInternal) + 1) code = Err(rc - 1);
  throw Error(code, std::string("mo_b200: ") + mo_last_error());
}
inline void ok(int rc) {
  if (rc != MO_OK) rethrow(rc);
}

template <class Real>
class Solver {
 public:
  Solver(const CompiledPlan& plan, SolveData<Real>& data, int device = 0) : data_(data) {
    // The device's two-phase J^T J p wants the per-template Jacobian lanes;
    // re-plan with force_evalj when the caller's plan lacks them (the other
    // programs are unchanged by it).
    std::string text;
    if (plan.has_evalj) {
      text = export_plan_text(plan);
    } else {
      SolveConfig c = plan.cfg;
      c.force_evalj = true;
      text = export_plan_text(minopt::plan(plan.spec, c));
    }
    ok(mo_plan_parse(text.data(), text.size(), &plan_));
    mo_solve_config c{};
    ok(mo_plan_get_config(plan_, &c));
    c.precision = sizeof(Real) == 4 ? MO_F32 : MO_F64;
    ok(mo_plan_set_config(plan_, &c));
    ok(mo_session_create(plan_, device, &s_));
    bind();
    ok(mo_refresh(s_));
  }
  ~Solver() {
    mo_session_destroy(s_);
    mo_plan_destroy(plan_);
  }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  int64_t num_cols() const {
    int64_t n = 0;
    ok(mo_num_cols(s_, &n));
    return n;
  }
  int64_t num_rows() const {
    int64_t n = 0;
    ok(mo_num_rows(s_, &n));
    return n;
  }
  std::span<const uint8_t> excluded() {
    excl_.resize(size_t(num_cols()));
    ok(mo_get_excluded(s_, excl_.data(), int64_t(excl_.size())));
    return excl_;
  }
  double cost() {
    double v = 0;
    ok(mo_cost(s_, &v));
    return v;
  }
  void residuals(std::span<Real> f) { ok(mo_residuals(s_, f.data(), int64_t(f.size()))); }
  void build_normal() {
    ok(mo_build_normal(s_));
    b_.resize(size_t(num_cols()));
    m_.resize(size_t(num_cols()));
    ok(mo_get_rhs(s_, b_.data(), int64_t(b_.size())));
    ok(mo_get_precond(s_, m_.data(), int64_t(m_.size())));
  }
  std::span<const Real> rhs() const { return b_; }
  std::span<const Real> precond() const { return m_; }
  void apply_jtj(std::span<const Real> v, std::span<Real> out) {
    check(v.size() == out.size(), Err::kShapeMismatch, "apply_jtj(): size mismatch");
    ok(mo_apply_jtj(s_, v.data(), out.data(), int64_t(v.size())));
  }
  bool saw_nonfinite_kernel() const {
    int v = 0;
    ok(mo_saw_nonfinite(s_, &v));
    return v != 0;
  }
  // linearize() / jacobian() (solver.hpp:291-382): lanes evaluated on the
  // device, the CSR assembled exactly as the reference assembles it.
  void linearize() { ok(mo_linearize(s_)); }
  // (fetched on every call: like the reference it throws kBindError once a
  // refresh - e.g. the end of solve() - has invalidated the linearization)
  const SparseCSR<Real>& jacobian() const {
    int64_t rows = 0, cols = 0, nnz = 0;
    ok(mo_jacobian_size(s_, &rows, &cols, &nnz));
    J_ = SparseCSR<Real>{};
    J_.rows = rows;
    J_.cols = cols;
    J_.offs.resize(size_t(rows) + 1);
    J_.col.resize(size_t(nnz));
    J_.val.resize(size_t(nnz));
    ok(mo_get_jacobian(s_, J_.offs.data(), J_.col.data(), J_.val.data(), nnz));
    return J_;
  }
  // normal_matrix() (solver.hpp:383-387): kJtJ sessions
  const SparseCSR<Real>& normal_matrix() const {
    int64_t nnz = 0;
    ok(mo_normal_matrix_size(s_, &nnz));
    H_ = SparseCSR<Real>{};
    H_.rows = H_.cols = num_cols();
    H_.offs.resize(size_t(H_.rows) + 1);
    H_.col.resize(size_t(nnz));
    H_.val.resize(size_t(nnz));
    ok(mo_get_normal_matrix(s_, H_.offs.data(), H_.col.data(), H_.val.data(), nnz));
    return H_;
  }

  SolveResult solve(const std::function<void(int, SolveData<Real>&)>& callback = {}) {
    cb_ = &callback;
    mo_solve_result r{};
    ok(mo_solve(s_, callback ? &Solver::trampoline : nullptr, this, &r));
    data_.x.resize(size_t(num_cols()));
    ok(mo_get_x(s_, data_.x.data(), int64_t(data_.x.size())));
    SolveResult out;
    out.final_cost = r.final_cost;
    out.reason = StopReason(r.reason);
    out.nonfinite_kernels = r.nonfinite_kernels != 0;
    out.indefinite_operator = r.indefinite_operator != 0;
    out.unconstrained = r.unconstrained;
    for (int i = 0; i < r.n_trace; ++i) {
      const mo_iter_row& t = r.trace[i];
      out.trace.push_back({t.iter, t.cost, t.accepted != 0, t.radius, t.pcg_iters, t.wall_ms});
    }
    return out;
  }

 private:
  void bind() {
    ok(mo_bind_x(s_, data_.x.data(), int64_t(data_.x.size())));
    for (size_t i = 0; i < data_.arrays.size(); ++i)
      ok(mo_bind_array(s_, int(i), data_.arrays[i].data(), int64_t(data_.arrays[i].size())));
    ok(mo_bind_params(s_, data_.params.data(), int64_t(data_.params.size())));
    for (size_t i = 0; i < data_.graphs.size(); ++i)
      ok(mo_bind_graph(s_, int(i), data_.graphs[i].verts.data(), int64_t(data_.graphs[i].verts.size()),
                       data_.graphs[i].arity));
  }
  // Callbacks observe and may mutate SolveData between iterations
  // (solver.hpp:503): download x, call, re-upload everything.
  static void trampoline(int iter, mo_session, void* user) {
    auto* self = static_cast<Solver*>(user);
    self->data_.x.resize(size_t(self->num_cols()));
    ok(mo_get_x(self->s_, self->data_.x.data(), int64_t(self->data_.x.size())));
    (*self->cb_)(iter, self->data_);
    self->bind();
  }

  SolveData<Real>& data_;
  mo_plan plan_ = nullptr;
  mo_session s_ = nullptr;
  std::vector<Real> b_, m_;
  std::vector<uint8_t> excl_;
  mutable SparseCSR<Real> J_, H_;
  const std::function<void(int, SolveData<Real>&)>* cb_ = nullptr;
};

}  // namespace minopt::b200
#endif  // MINOPT_B200_WITH_SOLVER
