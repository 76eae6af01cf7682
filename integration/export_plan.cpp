// export_plan.cpp — compile an energy with the reference front end and write
// the moplan v1 interchange the B200 library executes.
//
//   export_plan --energy F.opt [--dim W=16 ...] [--prec f32|f64] [--method gn|lm]
//               [--nl N] [--lin N] [--rel T] [--materialize none|j|jtj]
//               [--out plan.moplan]
//
// Plan-time only (the reference's parse/lower/transform/schedule pipeline is
// out of scope for the device path); built by
// integration/Makefile against /root/reference/proj/include.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "minopt/lower.hpp"
#include "minopt_b200_bridge.hpp"

using namespace minopt;

int main(int argc, char** argv) {
  std::string energy, out;
  std::vector<std::pair<std::string, long long>> dims;
  SolveConfig cfg;
  cfg.force_evalj = true;  // ship per-template Jacobian lanes for the two-phase apply
  bool f32 = false;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&]() -> std::string { return i + 1 < argc ? argv[++i] : ""; };
    if (k == "--energy") energy = next();
    else if (k == "--out") out = next();
    else if (k == "--dim") {
      std::string v = next();
      auto eq = v.find('=');
      dims.push_back({v.substr(0, eq), std::atoll(v.c_str() + eq + 1)});
    } else if (k == "--prec") f32 = next() == "f32";
    else if (k == "--method") cfg.method = next() == "lm" ? Method::kLevenbergMarquardt : Method::kGaussNewton;
    else if (k == "--nl") cfg.nonlinear_iters = std::atoi(next().c_str());
    else if (k == "--lin") cfg.linear_iters = std::atoi(next().c_str());
    else if (k == "--rel") cfg.pcg_rel_tol = std::atof(next().c_str());
    else if (k == "--materialize") {
      std::string m = next();
      cfg.materialize = m == "j" ? Materialize::kJ : m == "jtj" ? Materialize::kJtJ : Materialize::kNone;
    } else if (k == "--force-evalj") cfg.force_evalj = true;
    else {
      std::fprintf(stderr, "unknown option %s\n", k.c_str());
      return 2;
    }
  }
  cfg.precision = f32 ? Precision::kF32 : Precision::kF64;
  std::ifstream f(energy);
  if (!f) {
    std::fprintf(stderr, "cannot read %s\n", energy.c_str());
    return 2;
  }
  std::stringstream ss;
  ss << f.rdbuf();
  std::istringstream is(ss.str());
  std::ostringstream src;
  std::string line;
  while (std::getline(is, line)) {
    std::istringstream ls(line);
    std::string kw, name;
    ls >> kw >> name;
    bool done = false;
    if (kw == "dim")
      for (auto& [n, v] : dims)
        if (n == name) {
          src << "dim " << name << ' ' << v << '\n';
          done = true;
        }
    if (!done) src << line << '\n';
  }
  try {
    CompiledPlan P = plan(compile_source(src.str()), cfg);
    std::string text = b200::export_plan_text(P);
    if (out.empty()) {
      std::cout << text;
    } else {
      std::ofstream o(out);
      o << text;
    }
  } catch (const Error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
  return 0;
}
