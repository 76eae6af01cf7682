// mo_plan.hpp — host-side, plain-data mirror of the reference CompiledPlan
// (plan.hpp:125-137) restricted to what the matrix-free device path executes:
// domains and fields (problem.hpp:13-127), the column layout ubase/num_cols
// (plan.hpp:212-218), and the KernelPrograms (program.hpp:74-82) of every
// grid/gather/graph/computed/exclude kernel set (plan.hpp:59-120).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mo {

// Error codes mirror the reference taxonomy (common.hpp:13-32); the C ABI
// returns 1 + code so that 0 means success.
enum class Err : int {
  kSyntax = 0, kUndeclaredIdentifier, kArityMismatch, kNonConstantOffset, kMixedDomain,
  kNonConstantExponent, kDomainMismatch, kNonBooleanPredicate, kCyclicComputedArray,
  kShapeMismatch, kIndexOutOfRange, kFormatError, kTruncatedFile, kGraphDomain, kBindError,
  kNonFiniteCost, kCyclicIR, kInternal,
  kCuda = 100,      // device / driver failure (no reference counterpart)
  kNoDevice = 101,  // no CUDA device: the product has no CPU fallback
};

struct Error : std::runtime_error {
  Err code;
  Error(Err c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(Err c, const std::string& m) { throw Error(c, m); }
inline void check(bool ok, Err c, const std::string& m) {
  if (!ok) fail(c, m);
}

// Opcodes: same numbering as the reference Op enum (program.hpp:21-39).
enum Op : uint8_t {
  kImm, kParam, kIndex, kLoadU, kLoadA, kLoadC, kLoadP, kInB, kAdd, kMul, kPow, kUn, kCmp,
  kAnd, kOr, kNot, kSel
};
enum Un : uint8_t { kSqrt, kSin, kCos, kExp, kLog, kAbs, kAtan };      // expr.hpp UnaryFn
enum Cmp : uint8_t { kEq, kNe, kLt, kLe, kGt, kGe };                 // expr.hpp CmpOp

struct Instr {
  uint8_t op = 0, sub = 0;
  uint16_t dst = 0, a = 0, b = 0, c = 0;
  uint32_t gid = 0;
  int32_t field = 0, channel = 0;
  bool graph = false;
  int16_t off[3] = {0, 0, 0};
  int16_t slot = 0;
  double imm = 0;
  long long pnum = 1, pden = 1;
};

struct Block {
  uint32_t gid = 0, begin = 0, end = 0;
};

struct Program {
  uint32_t num_regs = 0;
  std::vector<Instr> instrs;
  std::vector<Block> blocks;
  std::vector<uint16_t> guard_regs;  // guard table; entry 0 is "always"
  std::vector<std::vector<std::pair<uint32_t, uint16_t>>> outputs;  // (gid, reg) roots
};

struct Domain {
  std::vector<int> dims;  // indices into Plan::dims
  bool operator==(const Domain& o) const { return dims == o.dims; }
};

struct Field {
  std::string name;
  int channels = 1;
  Domain dom;
  int mode = 0;  // computed arrays: 0 freeze, 1 cache
};

struct Config {  // SolveConfig (plan.hpp:19-38), device-relevant members
  int method = 0;     // 0 GN, 1 LM
  int precision = 1;  // 0 f32, 1 f64
  int nonlinear_iters = 8, linear_iters = 100;
  double pcg_rel_tol = -1.0, pcg_abs_tol = 0.0;
  bool use_preconditioner = true;
  double lm_radius0 = 1e4, lm_radius_min = 1e-32, lm_radius_max = 1e16;
  double lm_diag_min = 1e-6, lm_diag_max = 1e32, lm_min_decrease = 1e-3;
  double cost_stop_tol = 0.0;
  int materialize = 0;  // Materialize (plan.hpp:17): 0 none, 1 kJ, 2 kJtJ
};

struct Residual {
  bool graph = false;
  Domain dom;
  int graph_idx = -1;
};

// One materialized-Jacobian lane (plan.hpp:50-56): evalj output `out` is
// d r_t / d x[field, channel](e + off).
struct Lane {
  int out = 0, field = 0, channel = 0;
  int off[3] = {0, 0, 0};
  int slot = -1;  // graph rows: edge slot of the column's vertex
};
struct JTemplate {
  int tmpl = 0, guard_out = 0;
  bool origin = true;  // template reads its own pixel: instances centred
                       // outside the domain are guarded off
  std::vector<Lane> lanes;
};

struct GridSet {
  Domain dom;
  std::vector<int> templates;
  Program cost, evalf;
  bool has_evalj = false;  // plan exported with force_evalj (two-phase apply)
  std::vector<JTemplate> jtemplates;
  Program evalj;
};
struct GatherSet {
  Domain dom;
  std::vector<std::pair<int, int>> chans;  // (field, channel)
  Program bm, jtj;
};
struct Scat {
  int slot = 0, field = 0, channel = 0;
};
struct GraphSet {
  int graph = 0;
  std::vector<int> templates;
  std::vector<Scat> scats;
  Program cost, evalf, bm, jtj;
  bool has_evalj = false;
  std::vector<JTemplate> jtemplates;  // lanes carry slots (plan.hpp:318-330)
  Program evalj;
};
struct ComputedKernel {
  int index = 0;
  Domain dom;
  Program prog;
};
struct ExcludeKernel {
  Domain dom;
  Program prog;
};

struct Plan {
  Config cfg;
  std::vector<std::pair<std::string, int64_t>> dims;
  std::vector<std::string> params;
  std::vector<Field> unknowns, arrays, computed;
  std::vector<std::pair<std::string, int>> graphs;  // (name, arity)
  std::vector<Residual> residuals;
  std::vector<int64_t> ubase;
  int64_t num_cols = 0;
  std::vector<GridSet> grid_sets;
  std::vector<GatherSet> gather_sets;
  std::vector<GraphSet> graph_sets;
  std::vector<ComputedKernel> computed_kernels;
  std::vector<ExcludeKernel> exclude_kernels;
  bool exact = false;  // compile without FMA contraction (bitwise-faithful mode)

  std::array<int64_t, 3> shape_of(const Domain& d) const {
    std::array<int64_t, 3> s{1, 1, 1};
    for (size_t i = 0; i < d.dims.size(); ++i) s[i] = dims[size_t(d.dims[i])].second;
    return s;
  }
  int64_t extent_of(const Domain& d) const {
    int64_t n = 1;
    for (int di : d.dims) n *= dims[size_t(di)].second;
    return n;
  }
  // Recompute ubase/num_cols from the (possibly overridden) dims (plan.hpp:212-218).
  void relayout();
};

Plan parse_plan(const std::string& text);

}  // namespace mo
