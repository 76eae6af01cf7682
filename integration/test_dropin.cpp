// test_dropin.cpp — the reference's own solver tests (proj/tests/test_solver.cpp)
// re-run with `minopt::b200::Solver` in place of `minopt::Solver`: same energy
// sources, same plan(), same SolveData, same checks.  Built against the
// reference headers + libmo_b200.so by integration/Makefile; run on a GPU by
// tests/test_dropin_gpu.py.  (Catch2 is absent here, so CHECK is a macro.)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#define MINOPT_B200_WITH_SOLVER
#include "minopt/lower.hpp"
#include "minopt_b200_bridge.hpp"

using namespace minopt;

namespace dropin {
// The one-line switch: this scope's `Solver` is the device implementation.
using minopt::b200::Solver;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    ++g_checks;                                                         \
    if (!(c)) {                                                         \
      ++g_fail;                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);          \
    }                                                                   \
  } while (0)
static bool approx(double a, double b, double eps) { return std::fabs(a - b) <= eps * std::max(std::fabs(a), std::fabs(b)) + 1e-300; }

static const char* kChain = R"(
dim W 2
unknown X [W]
array A [W]
energy X(0) - A(0)
energy X(0) - X(1)
)";

template <class Real>
SolveData<Real> chain_data(std::vector<Real> x, std::vector<Real> a) {
  SolveData<Real> d;
  d.x = std::move(x);
  d.arrays = {std::move(a)};
  return d;
}

// test_solver.cpp:39-77 (matrix-free part)
static void two_pixel_values() {
  CompiledPlan p = plan(compile_source(kChain), SolveConfig{});
  SolveData<double> data = chain_data<double>({0.0, 0.0}, {1.0, 0.0});
  Solver<double> s(p, data);
  CHECK(s.num_cols() == 2);
  CHECK(s.num_rows() == 4);
  CHECK(s.cost() == 1.0);
  std::vector<double> f(4, 99.0);
  s.residuals(f);
  CHECK((f == std::vector<double>{-1.0, 0.0, 0.0, 0.0}));
  s.build_normal();
  CHECK(s.rhs()[0] == 2.0 && s.rhs()[1] == 0.0);
  CHECK(s.precond()[0] == 4.0 && s.precond()[1] == 4.0);
  std::vector<double> v{1.0, 0.0}, out(2);
  s.apply_jtj(v, out);
  CHECK(out[0] == 4.0 && out[1] == -2.0);
}

// test_solver.cpp:39-77 (materialized part: force_evalj, linearize, jacobian)
static void two_pixel_jacobian() {
  SolveConfig cfg;
  cfg.force_evalj = true;
  CompiledPlan p = plan(compile_source(kChain), cfg);
  SolveData<double> data = chain_data<double>({0.0, 0.0}, {1.0, 0.0});
  Solver<double> s(p, data);
  s.build_normal();
  std::vector<double> v{1.0, 0.0}, out(2);
  s.apply_jtj(v, out);
  CHECK(out[0] == 4.0 && out[1] == -2.0);
  s.linearize();
  const SparseCSR<double>& j = s.jacobian();
  CHECK(j.rows == 4);
  CHECK(j.cols == 2);
  CHECK((j.offs == std::vector<int64_t>{0, 1, 2, 4, 4}));
  CHECK((j.col == std::vector<int64_t>{0, 1, 0, 1}));
  CHECK((j.val == std::vector<double>{1.0, 1.0, 1.0, -1.0}));
}

// test_solver.cpp:103-153: kJ, kJtJ and the matrix-free apply agree and
// deliver the same iterates
static void materialized_agrees() {
  const char* src = R"(
dim W 9
unknown X [W]
array A [W]
energy sin(X(0)) - A(0)
energy 0.5 * (X(0) - X(1))
)";
  std::mt19937 rng(41);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<double> x0(9), a0(9);
  for (auto& v : x0) v = u(rng);
  for (auto& v : a0) v = u(rng);
  auto make = [&](Materialize mode) {
    SolveConfig cfg;
    cfg.materialize = mode;
    return plan(compile_source(src), cfg);
  };
  CompiledPlan pn = make(Materialize::kNone), pj = make(Materialize::kJ), ph = make(Materialize::kJtJ);
  SolveData<double> dn = chain_data<double>(x0, a0), dj = chain_data<double>(x0, a0), dh = chain_data<double>(x0, a0);
  Solver<double> sn(pn, dn), sj(pj, dj), sh(ph, dh);
  bool threw = false;
  std::vector<double> probe(9, 1.0), pout(9);
  try {
    sj.apply_jtj(probe, pout);  // solver.hpp:278: apply before linearize()
  } catch (const Error&) {
    threw = true;
  }
  CHECK(threw);
  sj.linearize();
  sh.linearize();
  for (int trial = 0; trial < 10; ++trial) {
    std::vector<double> v(9), on(9), oj(9), oh(9);
    for (auto& e : v) e = u(rng);
    sn.apply_jtj(v, on);
    sj.apply_jtj(v, oj);
    sh.apply_jtj(v, oh);
    for (int i = 0; i < 9; ++i) {
      CHECK(std::fabs(oj[i] - on[i]) <= 1e-12);
      CHECK(std::fabs(oh[i] - on[i]) <= 1e-12);
    }
  }
  const SparseCSR<double>& h = sh.normal_matrix();
  CHECK(h.rows == 9 && h.offs.size() == 10 && h.nnz() == 25);  // tridiagonal 9x9
  SolveResult rn = sn.solve(), rj = sj.solve(), rh = sh.solve();
  bool stale = false;
  try {
    (void)sj.jacobian();  // solve() ends with refresh(): the linearization is gone (solver.hpp:167, 379)
  } catch (const Error& e) {
    stale = e.code() == Err::kBindError;
  }
  CHECK(stale);
  CHECK(approx(rn.final_cost, rj.final_cost, 1e-10));
  CHECK(approx(rn.final_cost, rh.final_cost, 1e-10));
  for (int i = 0; i < 9; ++i) {
    CHECK(std::fabs(dj.x[i] - dn.x[i]) <= 1e-8);
    CHECK(std::fabs(dh.x[i] - dn.x[i]) <= 1e-8);
  }
}

// test_solver.cpp:186-204
static void degenerate_hyperedge() {
  SolveConfig cfg;
  cfg.materialize = Materialize::kJ;
  CompiledPlan p = plan(compile_source("dim N 2\nunknown P [N]\ngraph G (a, b)\nenergy P(G.a) - P(G.b)"), cfg);
  SolveData<double> data;
  data.x = {5.0, 7.0};
  data.graphs = {EdgeTable{2, {0, 0}}};
  Solver<double> s(p, data);
  s.linearize();
  const SparseCSR<double>& j = s.jacobian();
  CHECK(j.rows == 1);
  CHECK((j.offs == std::vector<int64_t>{0, 1}));
  CHECK((j.col == std::vector<int64_t>{0}));
  CHECK(j.val.size() == 1 && j.val[0] == 0.0);
  std::vector<double> v{1.0, 2.0}, out(2, 9.0);
  s.apply_jtj(v, out);  // J = [0 0]: 2 J^T J v = 0
  CHECK(out[0] == 0.0 && out[1] == 0.0);
}

// test_solver.cpp:79-101
static void one_gn_step() {
  SolveConfig cfg;
  cfg.nonlinear_iters = 1;
  CompiledPlan p = plan(compile_source(kChain), cfg);
  SolveData<double> data = chain_data<double>({0.0, 0.0}, {1.0, 0.0});
  Solver<double> s(p, data);
  SolveResult r = s.solve();
  CHECK(approx(data.x[0], 2.0 / 3.0, 1e-12));
  CHECK(approx(data.x[1], 1.0 / 3.0, 1e-12));
  CHECK(approx(r.final_cost, 1.0 / 3.0, 1e-12));
  CHECK(r.reason == StopReason::kIterLimit);
  CHECK(r.trace.size() == 1 && r.trace[0].accepted && r.trace[0].radius == 0.0);
  CHECK(r.trace[0].pcg_iters <= 2);
  CHECK(r.trace_csv().substr(0, 43) == "iter,cost,accepted,radius,pcg_iters,wall_ms");
}

// test_solver.cpp:155-186
static void graph_scatter() {
  CompiledPlan p = plan(compile_source("dim N 2\nunknown P [N]\ngraph G (a, b)\nenergy P(G.a) - P(G.b)"), SolveConfig{});
  SolveData<double> data;
  data.x = {3.0, 1.0};
  data.graphs = {EdgeTable{2, {0, 1}}};
  Solver<double> s(p, data);
  CHECK(s.num_rows() == 1);
  CHECK(s.cost() == 4.0);
  s.build_normal();
  CHECK(s.rhs()[0] == -4.0 && s.rhs()[1] == 4.0);
  CHECK(s.precond()[0] == 2.0 && s.precond()[1] == 2.0);
  CHECK(s.solve().unconstrained == 0);
  std::vector<double> v{1.0, 0.0}, out(2);
  s.apply_jtj(v, out);
  CHECK(out[0] == 2.0 && out[1] == -2.0);
  CHECK(std::fabs(s.cost()) < 1e-20);
}

// test_solver.cpp:206-234
static void frozen_unknowns() {
  SolveConfig cfg;
  cfg.nonlinear_iters = 1;
  CompiledPlan p = plan(compile_source("dim W 2\nunknown X [W]\narray A [W]\nenergy X(0) - A(0)\n"
                                       "exclude less(index(0), 1)"),
                        cfg);
  SolveData<double> data = chain_data<double>({-0.0, 0.0}, {1.0, 2.0});
  Solver<double> s(p, data);
  CHECK(s.excluded()[0] == 1 && s.excluded()[1] == 0);
  CHECK(s.cost() == 5.0);
  s.build_normal();
  CHECK(s.rhs()[0] == 0.0 && s.precond()[0] == 1.0);
  CHECK(s.rhs()[1] == 4.0 && s.precond()[1] == 2.0);
  SolveResult r = s.solve();
  const double neg_zero = -0.0;
  CHECK(std::memcmp(&data.x[0], &neg_zero, sizeof(double)) == 0);
  CHECK(approx(data.x[1], 2.0, 1e-12));
  CHECK(approx(r.final_cost, 1.0, 1e-12));
}

// test_solver.cpp:298-321
static void lm_triples_radius() {
  SolveConfig cfg;
  cfg.method = Method::kLevenbergMarquardt;
  cfg.nonlinear_iters = 2;
  CompiledPlan p = plan(compile_source(kChain), cfg);
  SolveData<double> data = chain_data<double>({0.0, 0.0}, {1.0, 0.0});
  Solver<double> s(p, data);
  SolveResult r = s.solve();
  CHECK(r.trace.size() >= 2);
  CHECK(r.trace[0].accepted && r.trace[0].radius == 1e4);
  CHECK(approx(r.trace[1].radius, 3e4, 1e-10));
}

// test_solver.cpp:360-407
static void nonfinite_energies() {
  {
    CompiledPlan p = plan(compile_source("dim W 1\nunknown X [W]\nenergy log(X(0))"), SolveConfig{});
    SolveData<double> data;
    data.x = {-1.0};
    Solver<double> s(p, data);
    SolveResult r = s.solve();
    CHECK(r.reason == StopReason::kNonFiniteCost);
    CHECK(std::isnan(r.final_cost));
    CHECK(r.trace.size() == 1 && !r.trace[0].accepted);
  }
  {
    SolveConfig cfg;
    cfg.method = Method::kLevenbergMarquardt;
    cfg.lm_radius0 = 1e8;
    cfg.nonlinear_iters = 20;
    CompiledPlan p = plan(compile_source("dim W 1\nunknown X [W]\nenergy log(X(0))"), cfg);
    SolveData<double> data;
    data.x = {4.0};
    Solver<double> s(p, data);
    SolveResult r = s.solve();
    CHECK(r.reason == StopReason::kStalled);
    CHECK(approx(data.x[0], 1.0, 1e-6));
    CHECK(r.final_cost < 1e-10);
  }
}

// test_solver.cpp:409-430
static void callbacks_mutate() {
  SolveConfig cfg;
  cfg.nonlinear_iters = 2;
  CompiledPlan p = plan(compile_source("dim W 2\nunknown X [W]\narray A [W]\nenergy X(0) - A(0)"), cfg);
  SolveData<double> data = chain_data<double>({0.0, 0.0}, {1.0, 2.0});
  Solver<double> s(p, data);
  int calls = 0;
  SolveResult r = s.solve([&](int iter, SolveData<double>& d) {
    ++calls;
    if (iter == 0) {
      CHECK(approx(d.x[0], 1.0, 1e-12));
      d.arrays[0] = {5.0, 6.0};
    }
  });
  CHECK(calls == 2);
  CHECK(approx(data.x[0], 5.0, 1e-12) && approx(data.x[1], 6.0, 1e-12));
  CHECK(std::fabs(r.final_cost) < 1e-20);
}

// test_solver.cpp:432-453
static void callbacks_grow_graph() {
  SolveConfig cfg;
  cfg.nonlinear_iters = 2;
  CompiledPlan p = plan(compile_source("dim N 3\nunknown P [N]\ngraph G (a, b)\nenergy P(G.a) - P(G.b) - 1"), cfg);
  SolveData<double> data;
  data.x = {0.0, 0.0, 0.0};
  data.graphs = {EdgeTable{2, {0, 1}}};
  Solver<double> s(p, data);
  CHECK(s.num_rows() == 1);
  SolveResult r = s.solve([&](int iter, SolveData<double>& d) {
    if (iter == 0) d.graphs[0] = EdgeTable{2, {0, 1, 1, 2}};
  });
  CHECK(s.num_rows() == 2);
  CHECK(approx(data.x[0] - data.x[1], 1.0, 1e-10));
  CHECK(approx(data.x[1] - data.x[2], 1.0, 1e-10));
  CHECK(std::fabs(r.final_cost) < 1e-18);
}

// test_solver.cpp:488-507
static void single_precision() {
  SolveConfig cfg;
  cfg.precision = Precision::kF32;
  cfg.nonlinear_iters = 1;
  CompiledPlan p = plan(compile_source(kChain), cfg);
  SolveData<float> data;
  data.x = {0.0f, 0.0f};
  data.arrays = {{1.0f, 0.0f}};
  Solver<float> s(p, data);
  CHECK(s.cost() == 1.0);
  s.build_normal();
  CHECK(s.rhs()[0] == 2.0f && s.precond()[0] == 4.0f);
  SolveResult r = s.solve();
  CHECK(approx(data.x[0], 2.0 / 3.0, 1e-6) && approx(data.x[1], 1.0 / 3.0, 1e-6));
  CHECK(approx(r.final_cost, 1.0 / 3.0, 1e-6));
}

// test_solver.cpp:509-537
static void binding_mistakes() {
  CompiledPlan p = plan(compile_source(kChain), SolveConfig{});
  bool threw = false;
  try {
    SolveData<double> data = chain_data<double>({0.0}, {1.0, 0.0});
    Solver<double> s(p, data);
  } catch (const Error& e) {
    threw = e.code() == Err::kBindError;
  }
  CHECK(threw);
  threw = false;
  try {
    SolveData<double> data = chain_data<double>({0.0, 0.0}, {1.0});
    Solver<double> s(p, data);
  } catch (const Error& e) {
    threw = e.code() == Err::kBindError;
  }
  CHECK(threw);
}

// test_solver.cpp:539-552
static void no_energies() {
  SolveConfig cfg;
  cfg.nonlinear_iters = 1;
  CompiledPlan p = plan(compile_source("dim W 3\nunknown X [W]"), cfg);
  SolveData<double> data;
  data.x = {1.0, 2.0, 3.0};
  Solver<double> s(p, data);
  CHECK(s.num_rows() == 0);
  SolveResult r = s.solve();
  CHECK(r.final_cost == 0.0);
  CHECK((data.x == std::vector<double>{1.0, 2.0, 3.0}));
  CHECK(r.unconstrained == 3);
}

}  // namespace dropin

int main() {
  using namespace dropin;
  two_pixel_values();
  two_pixel_jacobian();
  materialized_agrees();
  degenerate_hyperedge();
  one_gn_step();
  graph_scatter();
  frozen_unknowns();
  lm_triples_radius();
  nonfinite_energies();
  callbacks_mutate();
  callbacks_grow_graph();
  single_precision();
  binding_mistakes();
  no_energies();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
