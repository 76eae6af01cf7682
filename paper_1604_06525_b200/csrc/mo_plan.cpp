// mo_plan.cpp — parser for the moplan v1 interchange written by
// integration/minopt_b200_bridge.hpp (format documented there).
#include "mo_plan.hpp"

#include <cstdlib>
#include <sstream>

namespace mo {

namespace {

struct Lexer {
  std::istringstream is;
  explicit Lexer(const std::string& t) : is(t) {}
  std::string word() {
    std::string w;
    if (!(is >> w)) fail(Err::kTruncatedFile, "moplan: unexpected end of input");
    return w;
  }
  std::string peek() {
    auto pos = is.tellg();
    std::string w;
    is >> w;
    is.clear();
    is.seekg(pos);
    return w;
  }
  void expect(const char* kw) {
    std::string w = word();
    check(w == kw, Err::kFormatError, std::string("moplan: expected '") + kw + "', got '" + w + "'");
  }
  long long integer() {
    std::string w = word();
    char* end = nullptr;
    long long v = std::strtoll(w.c_str(), &end, 10);
    check(end && *end == 0, Err::kFormatError, "moplan: bad integer '" + w + "'");
    return v;
  }
  double real() {
    std::string w = word();
    char* end = nullptr;
    double v = std::strtod(w.c_str(), &end);  // accepts C99 hexfloats
    check(end && *end == 0, Err::kFormatError, "moplan: bad number '" + w + "'");
    return v;
  }
  Domain domain(int ndims) {
    Domain d;
    long long nd = integer();
    check(nd >= 0 && nd <= 3, Err::kFormatError, "moplan: domain rank out of range");
    for (long long i = 0; i < nd; ++i) {
      long long di = integer();
      check(di >= 0 && di < ndims, Err::kFormatError, "moplan: domain dim index out of range");
      d.dims.push_back(int(di));
    }
    return d;
  }
  Program program(const char* name) {
    expect("program");
    expect(name);
    Program p;
    p.num_regs = uint32_t(integer());
    long long ni = integer(), nb = integer(), ng = integer(), no = integer();
    // (a program the plan did not compile - e.g. the gather J^T J of a
    // materialized plan - is exported empty, without even the "always" guard)
    check(ni >= 0 && nb >= 0 && no >= 0 && (ng >= 1 || (ni == 0 && nb == 0 && no == 0)), Err::kFormatError,
          "moplan: bad program header");
    p.instrs.resize(size_t(ni));
    for (Instr& in : p.instrs) {
      expect("i");
      in.op = uint8_t(integer());
      in.sub = uint8_t(integer());
      in.dst = uint16_t(integer());
      in.a = uint16_t(integer());
      in.b = uint16_t(integer());
      in.c = uint16_t(integer());
      in.gid = uint32_t(integer());
      in.field = int32_t(integer());
      in.channel = int32_t(integer());
      in.graph = integer() != 0;
      for (int k = 0; k < 3; ++k) in.off[k] = int16_t(integer());
      in.slot = int16_t(integer());
      in.imm = real();
      in.pnum = integer();
      in.pden = integer();
      check(in.op <= kSel, Err::kFormatError, "moplan: unknown opcode");
      check(in.dst < p.num_regs && in.a < p.num_regs + 1 && in.b < p.num_regs + 1, Err::kFormatError,
            "moplan: register out of range");
    }
    p.blocks.resize(size_t(nb));
    for (Block& b : p.blocks) {
      expect("b");
      b.gid = uint32_t(integer());
      b.begin = uint32_t(integer());
      b.end = uint32_t(integer());
      check(b.begin <= b.end && b.end <= p.instrs.size() && b.gid < uint32_t(ng), Err::kFormatError,
            "moplan: bad block");
    }
    p.guard_regs.resize(size_t(ng));
    for (uint16_t& g : p.guard_regs) {
      expect("g");
      g = uint16_t(integer());
    }
    p.outputs.resize(size_t(no));
    for (auto& o : p.outputs) {
      expect("o");
      long long nr = integer();
      for (long long r = 0; r < nr; ++r) {
        uint32_t gid = uint32_t(integer());
        uint16_t reg = uint16_t(integer());
        check(gid < uint32_t(ng) && reg < p.num_regs, Err::kFormatError, "moplan: bad output root");
        o.push_back({gid, reg});
      }
    }
    return p;
  }
};

}  // namespace

void Plan::relayout() {
  ubase.assign(unknowns.size(), 0);
  int64_t col = 0;
  for (size_t f = 0; f < unknowns.size(); ++f) {
    ubase[f] = col;
    col += extent_of(unknowns[f].dom) * unknowns[f].channels;
  }
  num_cols = col;
}

Plan parse_plan(const std::string& text) {
  Lexer L(text);
  Plan P;
  L.expect("moplan");
  check(L.integer() == 1, Err::kFormatError, "moplan: unsupported version");
  L.expect("cfg");
  Config& c = P.cfg;
  c.method = int(L.integer());
  c.precision = int(L.integer());
  c.nonlinear_iters = int(L.integer());
  c.linear_iters = int(L.integer());
  c.pcg_rel_tol = L.real();
  c.pcg_abs_tol = L.real();
  c.use_preconditioner = L.integer() != 0;
  c.lm_radius0 = L.real();
  c.lm_radius_min = L.real();
  c.lm_radius_max = L.real();
  c.lm_diag_min = L.real();
  c.lm_diag_max = L.real();
  c.lm_min_decrease = L.real();
  c.cost_stop_tol = L.real();
  if (L.peek() == "materialize") {
    L.expect("materialize");
    c.materialize = int(L.integer());
    check(c.materialize >= 0 && c.materialize <= 2, Err::kFormatError, "moplan: bad materialize mode");
  }

  L.expect("dims");
  long long nd = L.integer();
  for (long long i = 0; i < nd; ++i) {
    L.expect("dim");
    std::string n = L.word();
    P.dims.push_back({n, L.integer()});
  }
  const int ndims = int(P.dims.size());
  L.expect("params");
  long long np = L.integer();
  for (long long i = 0; i < np; ++i) {
    L.expect("param");
    P.params.push_back(L.word());
  }
  auto fields = [&](const char* hdr, const char* kw, std::vector<Field>& out, bool computed) {
    L.expect(hdr);
    long long n = L.integer();
    for (long long i = 0; i < n; ++i) {
      L.expect(kw);
      Field f;
      f.name = L.word();
      if (computed) f.mode = int(L.integer());
      f.channels = int(L.integer());
      f.dom = L.domain(ndims);
      out.push_back(f);
    }
  };
  fields("unknowns", "unknown", P.unknowns, false);
  fields("arrays", "array", P.arrays, false);
  fields("computed", "computed", P.computed, true);
  L.expect("graphs");
  long long ng = L.integer();
  for (long long i = 0; i < ng; ++i) {
    L.expect("graph");
    std::string n = L.word();
    P.graphs.push_back({n, int(L.integer())});
  }
  L.expect("residuals");
  long long nr = L.integer();
  for (long long i = 0; i < nr; ++i) {
    L.expect("residual");
    Residual r;
    std::string k = L.word();
    if (k == "grid") {
      r.dom = L.domain(ndims);
    } else {
      check(k == "graph", Err::kFormatError, "moplan: bad residual kind");
      r.graph = true;
      r.graph_idx = int(L.integer());
    }
    P.residuals.push_back(r);
  }
  L.expect("ubase");
  long long nu = L.integer();
  for (long long i = 0; i < nu; ++i) P.ubase.push_back(L.integer());
  L.expect("num_cols");
  P.num_cols = L.integer();

  L.expect("grid_sets");
  long long n = L.integer();
  for (long long i = 0; i < n; ++i) {
    L.expect("grid_set");
    GridSet g;
    g.dom = L.domain(ndims);
    long long nt = L.integer();
    for (long long t = 0; t < nt; ++t) g.templates.push_back(int(L.integer()));
    g.cost = L.program("cost");
    g.evalf = L.program("evalf");
    if (L.peek() == "evalj") {
      L.expect("evalj");
      long long njt = L.integer();
      for (long long k = 0; k < njt; ++k) {
        L.expect("jtemplate");
        JTemplate jt;
        jt.tmpl = int(L.integer());
        jt.guard_out = int(L.integer());
        jt.origin = L.integer() != 0;
        long long nl = L.integer();
        for (long long l = 0; l < nl; ++l) {
          Lane ln;
          ln.out = int(L.integer());
          ln.field = int(L.integer());
          ln.channel = int(L.integer());
          for (int a = 0; a < 3; ++a) ln.off[a] = int(L.integer());
          jt.lanes.push_back(ln);
        }
        g.jtemplates.push_back(std::move(jt));
      }
      g.evalj = L.program("evalj");
      g.has_evalj = true;
      for (const JTemplate& jt : g.jtemplates)
        for (const Lane& ln : jt.lanes)
          check(ln.out >= 0 && size_t(ln.out) < g.evalj.outputs.size() && ln.field >= 0 &&
                    size_t(ln.field) < P.unknowns.size(),
                Err::kFormatError, "moplan: bad Jacobian lane");
    }
    P.grid_sets.push_back(std::move(g));
  }
  L.expect("gather_sets");
  n = L.integer();
  for (long long i = 0; i < n; ++i) {
    L.expect("gather_set");
    GatherSet g;
    g.dom = L.domain(ndims);
    long long nc = L.integer();
    for (long long t = 0; t < nc; ++t) {
      int f = int(L.integer());
      g.chans.push_back({f, int(L.integer())});
    }
    g.bm = L.program("bm");
    g.jtj = L.program("jtj");
    P.gather_sets.push_back(std::move(g));
  }
  L.expect("graph_sets");
  n = L.integer();
  for (long long i = 0; i < n; ++i) {
    L.expect("graph_set");
    GraphSet g;
    g.graph = int(L.integer());
    long long nt = L.integer();
    for (long long t = 0; t < nt; ++t) g.templates.push_back(int(L.integer()));
    long long ns = L.integer();
    for (long long t = 0; t < ns; ++t) {
      Scat s;
      s.slot = int(L.integer());
      s.field = int(L.integer());
      s.channel = int(L.integer());
      g.scats.push_back(s);
    }
    g.cost = L.program("cost");
    g.evalf = L.program("evalf");
    g.bm = L.program("bm");
    g.jtj = L.program("jtj");
    if (L.peek() == "gevalj") {
      L.expect("gevalj");
      long long njt = L.integer();
      for (long long k = 0; k < njt; ++k) {
        L.expect("gjtemplate");
        JTemplate jt;
        jt.tmpl = int(L.integer());
        jt.guard_out = -1;
        long long nl = L.integer();
        for (long long l = 0; l < nl; ++l) {
          Lane ln;
          ln.out = int(L.integer());
          ln.field = int(L.integer());
          ln.channel = int(L.integer());
          ln.slot = int(L.integer());
          jt.lanes.push_back(ln);
        }
        g.jtemplates.push_back(std::move(jt));
      }
      g.evalj = L.program("evalj");
      g.has_evalj = true;
      for (const JTemplate& jt : g.jtemplates)
        for (const Lane& ln : jt.lanes)
          check(ln.out >= 0 && size_t(ln.out) < g.evalj.outputs.size() && ln.field >= 0 &&
                    size_t(ln.field) < P.unknowns.size() && ln.slot >= 0 &&
                    ln.slot < P.graphs[size_t(g.graph)].second,
                Err::kFormatError, "moplan: bad graph Jacobian lane");
    }
    P.graph_sets.push_back(std::move(g));
  }
  L.expect("computed_kernels");
  n = L.integer();
  for (long long i = 0; i < n; ++i) {
    L.expect("computed_kernel");
    ComputedKernel ck;
    ck.index = int(L.integer());
    ck.dom = L.domain(ndims);
    ck.prog = L.program("prog");
    P.computed_kernels.push_back(std::move(ck));
  }
  L.expect("exclude_kernels");
  n = L.integer();
  for (long long i = 0; i < n; ++i) {
    L.expect("exclude_kernel");
    ExcludeKernel ek;
    ek.dom = L.domain(ndims);
    ek.prog = L.program("prog");
    P.exclude_kernels.push_back(std::move(ek));
  }
  L.expect("end");

  // Structural checks the device path relies on.
  check(P.ubase.size() == P.unknowns.size(), Err::kFormatError, "moplan: ubase size");
  check(P.unknowns.size() <= 16, Err::kInternal, "moplan: more than 16 unknown fields");
  check(2 * P.unknowns.size() + P.arrays.size() + P.computed.size() <= 32, Err::kInternal,
        "moplan: more than 32 bound fields");
  // (materialized plans compile no J^T J gather programs, plan.hpp:210)
  const bool free = P.cfg.materialize == 0;
  for (const GatherSet& g : P.gather_sets) {
    check(g.bm.outputs.size() == 2 * g.chans.size(), Err::kFormatError, "moplan: bm outputs");
    check(!free || g.jtj.outputs.size() == g.chans.size(), Err::kFormatError, "moplan: jtj outputs");
  }
  for (const GraphSet& g : P.graph_sets) {
    check(g.bm.outputs.size() == 2 * g.scats.size(), Err::kFormatError, "moplan: graph bm outputs");
    check(!free || g.jtj.outputs.size() == g.scats.size(), Err::kFormatError, "moplan: graph jtj outputs");
    check(g.graph >= 0 && size_t(g.graph) < P.graphs.size(), Err::kFormatError, "moplan: graph index");
  }
  int64_t saved = P.num_cols;
  std::vector<int64_t> sb = P.ubase;
  P.relayout();
  check(saved == P.num_cols && sb == P.ubase, Err::kFormatError, "moplan: column layout mismatch");
  return P;
}

}  // namespace mo
