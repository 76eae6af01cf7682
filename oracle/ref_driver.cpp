// ref_driver.cpp — command-line harness around the UNMODIFIED reference solver
// (/root/reference/proj/include/minopt, header-only C++20).
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/ref_driver
// straight from the reference headers (never copied).  The pytest suite uses it
// to produce golden vectors, and bench.py's `--impl reference` arm uses it to
// time the reference's own CPU implementation of the path.
//
// It drives exactly the reference's public API:
//   compile_source (lower.hpp:619) -> plan (plan.hpp:189) -> Solver<Real>
//   (solver.hpp:84) -> cost (174) / residuals (196) / build_normal (220) /
//   apply_jtj (255) / solve (389).
//
// usage:
//   ref_driver --energy F.opt [--dim W=16 ...] --in IN.mob --out OUT.mob
//              [--prec f32|f64] [--method gn|lm] [--nl N] [--lin N] [--rel T]
//              [--abs T] [--noprecond] [--radius0 R] [--cost-stop T]
//              [--exec seq|par] [--repeat N] [--materialize none|j|jtj]
//              [--force-evalj] --do cmd[,cmd...]
//   cmds: cost residuals normal linearize jtj solve time routines
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "minopt/lower.hpp"
#include "minopt/solver.hpp"
#include "mob.h"

using namespace minopt;

namespace {

struct Args {
  std::string energy, in, out;
  std::vector<std::pair<std::string, long long>> dims;
  bool f32 = false;
  SolveConfig cfg;
  std::vector<std::string> cmds;
  int repeat = 1;
};

std::string read_text(const std::string& p) {
  std::ifstream f(p);
  if (!f) {
    std::fprintf(stderr, "cannot read %s\n", p.c_str());
    std::exit(2);
  }
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

// Rewrite `dim NAME <n>` lines so one energy file serves every grid size.
std::string with_dims(const std::string& src,
                      const std::vector<std::pair<std::string, long long>>& dims) {
  std::istringstream is(src);
  std::ostringstream os;
  std::string line;
  while (std::getline(is, line)) {
    std::istringstream ls(line);
    std::string kw, name;
    ls >> kw >> name;
    bool done = false;
    if (kw == "dim")
      for (auto& [n, v] : dims)
        if (n == name) {
          os << "dim " << name << " " << v << "\n";
          done = true;
        }
    if (!done) os << line << "\n";
  }
  return os.str();
}

Args parse_args(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "missing value for %s\n", k.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (k == "--energy") a.energy = next();
    else if (k == "--in") a.in = next();
    else if (k == "--out") a.out = next();
    else if (k == "--dim") {
      std::string v = next();
      auto eq = v.find('=');
      a.dims.push_back({v.substr(0, eq), std::atoll(v.c_str() + eq + 1)});
    } else if (k == "--prec") a.f32 = next() == "f32";
    else if (k == "--method") a.cfg.method = next() == "lm" ? Method::kLevenbergMarquardt : Method::kGaussNewton;
    else if (k == "--nl") a.cfg.nonlinear_iters = std::atoi(next().c_str());
    else if (k == "--lin") a.cfg.linear_iters = std::atoi(next().c_str());
    else if (k == "--rel") a.cfg.pcg_rel_tol = std::atof(next().c_str());
    else if (k == "--materialize") {
      std::string m = next();
      a.cfg.materialize = m == "j" ? Materialize::kJ : m == "jtj" ? Materialize::kJtJ : Materialize::kNone;
    } else if (k == "--force-evalj") a.cfg.force_evalj = true;
    else if (k == "--abs") a.cfg.pcg_abs_tol = std::atof(next().c_str());
    else if (k == "--noprecond") a.cfg.use_preconditioner = false;
    else if (k == "--radius0") a.cfg.lm_radius0 = std::atof(next().c_str());
    else if (k == "--cost-stop") a.cfg.cost_stop_tol = std::atof(next().c_str());
    else if (k == "--exec") a.cfg.exec = next() == "par" ? ExecMode::kParallel : ExecMode::kSequential;
    else if (k == "--repeat") a.repeat = std::atoi(next().c_str());
    else if (k == "--do") {
      std::string v = next();
      std::stringstream ss(v);
      std::string c;
      while (std::getline(ss, c, ',')) a.cmds.push_back(c);
    } else {
      std::fprintf(stderr, "unknown option %s\n", k.c_str());
      std::exit(2);
    }
  }
  a.cfg.precision = a.f32 ? Precision::kF32 : Precision::kF64;
  return a;
}

template <class Real>
std::vector<Real> get_real(const mob_file& m, const char* name) {
  const mob_rec* r = mob_find(&m, name);
  std::vector<Real> v;
  if (!r) return v;
  v.resize(r->n);
  for (uint64_t i = 0; i < r->n; ++i) {
    if (r->dtype == MOB_F32) v[i] = Real(((const float*)r->data)[i]);
    else if (r->dtype == MOB_F64) v[i] = Real(((const double*)r->data)[i]);
    else {
      std::fprintf(stderr, "record %s is not floating point\n", name);
      std::exit(2);
    }
  }
  return v;
}

template <class Real>
constexpr int real_dtype() {
  return sizeof(Real) == 4 ? MOB_F32 : MOB_F64;
}

template <class Real>
int run(const Args& a, const CompiledPlan& P) {
  mob_file in;
  if (mob_read(a.in.c_str(), &in) != 0) {
    std::fprintf(stderr, "cannot read %s\n", a.in.c_str());
    return 2;
  }
  SolveData<Real> data;
  data.x = get_real<Real>(in, "x");
  for (size_t i = 0; i < P.spec.arrays.size(); ++i)
    data.arrays.push_back(get_real<Real>(in, ("array" + std::to_string(i)).c_str()));
  data.params = get_real<double>(in, "params");
  for (size_t i = 0; i < P.spec.graphs.size(); ++i) {
    std::string g = "graph" + std::to_string(i);
    const mob_rec* ar = mob_find(&in, (g + "_arity").c_str());
    const mob_rec* vr = mob_find(&in, g.c_str());
    EdgeTable et;
    et.arity = ar ? int(((const int64_t*)ar->data)[0]) : P.spec.graphs[i].arity();
    if (vr) et.verts.assign((const uint64_t*)vr->data, (const uint64_t*)vr->data + vr->n);
    data.graphs.push_back(std::move(et));
  }
  const std::vector<Real> x0 = data.x;

  mob_writer w;
  if (mob_open_w(&w, a.out.c_str()) != 0) return 2;
  constexpr int RD = real_dtype<Real>();
  try {
    Solver<Real> s(P, data);
    int64_t ncols = s.num_cols(), nrows = s.num_rows();
    mob_put(&w, "num_cols", MOB_I64, &ncols, 1);
    mob_put(&w, "num_rows", MOB_I64, &nrows, 1);
    std::vector<uint8_t> exc(s.excluded().begin(), s.excluded().end());
    mob_put(&w, "excluded", MOB_U8, exc.data(), exc.size());
    for (const std::string& c : a.cmds) {
      if (c == "cost") {
        double v = s.cost();
        mob_put(&w, "cost", MOB_F64, &v, 1);
      } else if (c == "residuals") {
        std::vector<Real> f(static_cast<size_t>(s.num_rows()));
        s.residuals(f);
        mob_put(&w, "residuals", RD, f.data(), f.size());
      } else if (c == "normal") {
        s.build_normal();
        mob_put(&w, "b", RD, s.rhs().data(), s.rhs().size());
        mob_put(&w, "m", RD, s.precond().data(), s.precond().size());
      } else if (c == "linearize") {  // solver.hpp:291-381
        s.linearize();
        const SparseCSR<Real>& j = s.jacobian();
        mob_put(&w, "j_offs", MOB_I64, j.offs.data(), j.offs.size());
        mob_put(&w, "j_col", MOB_I64, j.col.data(), j.col.size());
        mob_put(&w, "j_val", RD, j.val.data(), j.val.size());
        if (a.cfg.materialize == Materialize::kJtJ) {
          const SparseCSR<Real>& h = s.normal_matrix();
          mob_put(&w, "h_offs", MOB_I64, h.offs.data(), h.offs.size());
          mob_put(&w, "h_col", MOB_I64, h.col.data(), h.col.size());
          mob_put(&w, "h_val", RD, h.val.data(), h.val.size());
        }
      } else if (c == "jtj") {
        std::vector<Real> v = get_real<Real>(in, "v");
        std::vector<Real> out(static_cast<size_t>(ncols));
        s.apply_jtj(v, out);
        mob_put(&w, "jtj", RD, out.data(), out.size());
      } else if (c == "solve" || c == "time") {
        int reps = c == "time" ? a.repeat : 1;
        std::vector<double> ms, row_ms;
        SolveResult r;
        for (int k = 0; k < reps; ++k) {
          data.x = x0;
          auto t0 = std::chrono::steady_clock::now();
          r = s.solve();
          auto t1 = std::chrono::steady_clock::now();
          ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
          for (const IterRow& row : r.trace) row_ms.push_back(row.wall_ms);  // one per trial
        }
        mob_put(&w, "time_row_ms", MOB_F64, row_ms.data(), row_ms.size());
        mob_put(&w, "x_final", RD, data.x.data(), data.x.size());
        mob_put(&w, "final_cost", MOB_F64, &r.final_cost, 1);
        int64_t reason = int64_t(r.reason), unc = r.unconstrained;
        int64_t nfk = r.nonfinite_kernels, ind = r.indefinite_operator;
        mob_put(&w, "reason", MOB_I64, &reason, 1);
        mob_put(&w, "unconstrained", MOB_I64, &unc, 1);
        mob_put(&w, "nonfinite_kernels", MOB_I64, &nfk, 1);
        mob_put(&w, "indefinite", MOB_I64, &ind, 1);
        std::vector<int64_t> it, acc, pcg;
        std::vector<double> cost, rad, wall;
        for (const IterRow& row : r.trace) {
          it.push_back(row.iter);
          acc.push_back(row.accepted);
          pcg.push_back(row.pcg_iters);
          cost.push_back(row.cost);
          rad.push_back(row.radius);
          wall.push_back(row.wall_ms);
        }
        mob_put(&w, "trace_iter", MOB_I64, it.data(), it.size());
        mob_put(&w, "trace_accepted", MOB_I64, acc.data(), acc.size());
        mob_put(&w, "trace_pcg", MOB_I64, pcg.data(), pcg.size());
        mob_put(&w, "trace_cost", MOB_F64, cost.data(), cost.size());
        mob_put(&w, "trace_radius", MOB_F64, rad.data(), rad.size());
        mob_put(&w, "trace_ms", MOB_F64, wall.data(), wall.size());
        mob_put(&w, c == "time" ? "time_ms" : "solve_ms", MOB_F64, ms.data(), ms.size());
        std::string csv = r.trace_csv();
        mob_put(&w, "trace_csv", MOB_U8, csv.data(), csv.size());
      } else if (c == "routines") {
        // Per-routine wall times of the generated CPU routines (median input).
        std::vector<double> tc, tn, tj;
        std::vector<Real> v(static_cast<size_t>(ncols), Real(0.5));
        std::vector<Real> out(static_cast<size_t>(ncols));
        for (int k = 0; k < a.repeat; ++k) {
          auto t0 = std::chrono::steady_clock::now();
          volatile double cc = s.cost();
          (void)cc;
          auto t1 = std::chrono::steady_clock::now();
          s.build_normal();
          auto t2 = std::chrono::steady_clock::now();
          s.apply_jtj(v, out);
          auto t3 = std::chrono::steady_clock::now();
          tc.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
          tn.push_back(std::chrono::duration<double, std::milli>(t2 - t1).count());
          tj.push_back(std::chrono::duration<double, std::milli>(t3 - t2).count());
        }
        mob_put(&w, "routine_cost_ms", MOB_F64, tc.data(), tc.size());
        mob_put(&w, "routine_normal_ms", MOB_F64, tn.data(), tn.size());
        mob_put(&w, "routine_jtj_ms", MOB_F64, tj.data(), tj.size());
      } else {
        std::fprintf(stderr, "unknown command %s\n", c.c_str());
        mob_close_w(&w);
        return 2;
      }
    }
  } catch (const Error& e) {
    int64_t code = int64_t(e.code());
    mob_put(&w, "error_code", MOB_I64, &code, 1);
    std::string msg = e.what();
    mob_put(&w, "error", MOB_U8, msg.data(), msg.size());
  }
  mob_close_w(&w);
  mob_free(&in);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Args a = parse_args(argc, argv);
  if (a.energy.empty() || a.in.empty() || a.out.empty()) {
    std::fprintf(stderr, "need --energy, --in, --out\n");
    return 2;
  }
  std::string src = with_dims(read_text(a.energy), a.dims);
  CompiledPlan P;
  try {
    P = plan(compile_source(src), a.cfg);
  } catch (const Error& e) {
    mob_writer w;
    if (mob_open_w(&w, a.out.c_str()) != 0) return 2;
    int64_t code = int64_t(e.code());
    mob_put(&w, "error_code", MOB_I64, &code, 1);
    std::string msg = e.what();
    mob_put(&w, "error", MOB_U8, msg.data(), msg.size());
    mob_close_w(&w);
    return 0;
  }
  return a.f32 ? run<float>(a, P) : run<double>(a, P);
}
