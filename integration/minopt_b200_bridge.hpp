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
//   dims N            / dim NAME EXTENT
//   params N          / param NAME
//   unknowns N        / unknown NAME CH ND dims...
//   arrays N          / array NAME CH ND dims...
//   computed N        / computed NAME MODE TOTALCH ND dims...
//   graphs N          / graph NAME ARITY
//   residuals N       / residual grid ND dims... | residual graph G
//   ubase N cols... ; num_cols V
//   grid_sets N       / grid_set ND dims... NT t...   + programs cost, evalf
//   gather_sets N     / gather_set ND dims... NCH (f c)...   + programs bm, jtj
//   graph_sets N      / graph_set G NT t... NS (slot f c)... + cost, evalf, bm, jtj
//   computed_kernels N/ computed_kernel IDX ND dims...   + program prog
//   exclude_kernels N / exclude_kernel ND dims...        + program prog
//   end
// program NAME REGS NI NB NG NO, then NI `i` lines (op sub dst a b c gid field
// channel graph off0 off1 off2 slot imm pnum pden), NB `b` lines (gid begin
// end), NG `g` lines (guard register), NO `o` lines (nroots (gid reg)...).
#pragma once

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

// Serialise a matrix-free CompiledPlan.  Throws Err::kBindError for plans
// compiled for the materialized modes (out of scope for the device path).
inline std::string export_plan_text(const CompiledPlan& P) {
  using namespace bridge_detail;
  check(P.cfg.materialize == Materialize::kNone, Err::kBindError,
        "the B200 path executes matrix-free plans only");
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
