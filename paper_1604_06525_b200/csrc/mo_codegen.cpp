// mo_codegen.cpp — plan-time translation of the reference's guarded register
// programs (program.hpp:21-167) into CUDA C++ for NVRTC (sm_100a).
//
// Semantics reproduced per element exactly as run_program (program.hpp:89-167):
//  * every register starts at 0 (regs.assign, :92);
//  * a block whose guard register is 0 is skipped wholesale (:94-95);
//  * loads follow EvalEnv::read (eval.hpp:41-55): grid reads outside the
//    field's own shape return 0, slot reads index edge[slot];
//  * InBounds tests the iteration domain (eval.hpp:57-61);
//  * pow uses the shared pow_eval rounding rule (common.hpp:116-124);
//  * each output is Real(0) plus its guarded roots in listed order (:159-166).
// Modules are compiled with --fmad=false so add/mul round exactly like the
// reference's x86 build (no contraction), which makes per-element outputs of
// add/mul/select programs bitwise equal to the CPU reference.
//
// The per-element bodies are wrapped in hand-written kernel skeletons: 32x8
// tiles with a grid-stride tile loop (grid sized to the SM count), fused
// epilogues (PCG p'Ap reduction, LM damping, identity patch of build_normal),
// and deterministic last-block reductions.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>

#include "mo_codegen.hpp"

namespace mo {

namespace {

constexpr int kTileX = 32, kTileY = 8, kThreads = 256;  // = MO_TILE_X/Y, MO_THREADS

std::string hexd(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", v);
  std::string s = buf;
  if (s == "inf") return "(1.0/0.0)";
  if (s == "-inf") return "(-1.0/0.0)";
  if (s == "nan" || s == "-nan") return "(0.0/0.0)";
  return s;
}

struct Gen {
  // Merged-lane (field, channel, o0, o1) and lane lists shared by the
  // two-phase apply generators.
  struct MLane {
    int f, c, o0, o1;
  };
  struct LaneG {
    int t, out, f, c, o0, o1;
  };
  const Plan& P;
  bool f64;
  std::ostringstream os;
  int nprog = 0;

  Gen(const Plan& p, bool d) : P(p), f64(d) {}

  int slot_of(int op, int field) const {
    const int U = int(P.unknowns.size()), A = int(P.arrays.size());
    switch (op) {
      case kLoadU: return field;
      case kLoadP: return U + field;
      case kLoadA: return 2 * U + field;
      case kLoadC: return 2 * U + A + field;
    }
    return -1;
  }
  const Field& field_of(int op, int field) const {
    check(field >= 0, Err::kShapeMismatch, "kernel reads a field that is not bound");
    switch (op) {
      case kLoadU:
      case kLoadP:
        check(size_t(field) < P.unknowns.size(), Err::kShapeMismatch, "kernel reads a field that is not bound");
        return P.unknowns[size_t(field)];
      case kLoadA:
        check(size_t(field) < P.arrays.size(), Err::kShapeMismatch, "kernel reads a field that is not bound");
        return P.arrays[size_t(field)];
      default:
        check(size_t(field) < P.computed.size(), Err::kShapeMismatch, "kernel reads a field that is not bound");
        return P.computed[size_t(field)];
    }
  }

  const char* fn(int sub) const {
    static const char* f32n[] = {"sqrtf", "sinf", "cosf", "expf", "logf", "fabsf", "atanf"};
    static const char* f64n[] = {"sqrt", "sin", "cos", "exp", "log", "fabs", "atan"};
    check(sub <= kAtan, Err::kFormatError, "codegen: unknown unary function");
    return f64 ? f64n[sub] : f32n[sub];
  }

  // Emit `template <bool I> __device__ void NAME(P, p0, p1, p2, vs, out)`.
  // I = true is the interior-tile variant: reads of fields living on the
  // iteration domain skip the OOB test and InBounds folds to 1, valid when
  // the tile is at least `reach` elements from every border; the compiler
  // then drops the guards and can hoist every load (same values, bit for bit).
  const Domain* iter_dom = nullptr;
  int reach = 0;
  // Shared-memory staged fields (TMA apply): slot -> (byte offset of the
  // field's row ring in dynamic smem, channels).  In sm_mode, reads of these
  // fields come from the ring: row ri[o0 + st_rx], column lx + o1.
  bool sm_mode = false;
  int st_rx = 0, st_win = 0;
  std::vector<std::pair<int, std::pair<long long, int>>> staged;
  const std::pair<long long, int>* staged_of(int sl) const {
    for (auto& x : staged)
      if (x.first == sl) return &x.second;
    return nullptr;
  }
  int reach_of(const Program& pg, const Domain* dom) {
    int r = 0;
    for (const Instr& in : pg.instrs) {
      bool counts = in.op == kInB;
      if ((in.op == kLoadU || in.op == kLoadA || in.op == kLoadC || in.op == kLoadP) && !in.graph)
        counts = dom && field_of(in.op, in.field).dom == *dom;
      if (counts)
        for (int a = 0; a < 3; ++a) r = std::max(r, std::abs(int(in.off[a])));
    }
    return r;
  }
  static constexpr int MO_MAX_TMAPS_HOST = 16;  // = MO_MAX_TMAPS (mo_device.cuh)
  // ---- lane cache: the x-dependent part of evalj, evaluated once per
  // linearisation.  Every evalj instruction is either UNIFORM (built from
  // immediates and parameters only, through uniform registers) or VARYING
  // (reads a field, an index or InBounds, or a varying register written
  // earlier in program order).  A lane whose roots are all uniform is a
  // function of the parameters and of guard outcomes only; the others are
  // cached by value.  Re-running the uniform instructions under the cached
  // guard outcomes (block-entry guards, final output guards) reproduces
  // every lane bit for bit, so an apply that reads the cache computes
  // exactly what the full evalj would have.
  struct LaneSplit {
    bool ok = false;
    std::vector<char> u;       // per instruction: uniform
    std::vector<int> blk_bit;  // per block: bit of its entry guard outcome (-1: not needed)
    std::vector<int> out_bit;  // per gid: bit of its final guard outcome (-1: not needed)
    std::vector<int> varying;  // evalj outputs cached by value, in order
    int nbits = 0;
  };
  static LaneSplit split_lanes(const Program& pg) {
    LaneSplit ls;
    std::vector<char> v(pg.num_regs, 0);  // register holds (or may hold) a varying value here
    ls.u.assign(pg.instrs.size(), 0);
    ls.blk_bit.assign(pg.blocks.size(), -1);
    ls.out_bit.assign(pg.guard_regs.size(), -1);
    for (size_t bi = 0; bi < pg.blocks.size(); ++bi) {
      const Block& b = pg.blocks[bi];
      bool any_u = false;
      for (uint32_t i = b.begin; i < b.end; ++i) {
        const Instr& in = pg.instrs[i];
        bool var = false;
        switch (in.op) {
          case kImm: case kParam: break;
          case kAdd: case kMul: case kCmp: case kAnd: case kOr: var = v[in.a] || v[in.b]; break;
          case kPow: case kUn: case kNot: var = v[in.a]; break;
          case kSel: var = v[in.a] || v[in.b] || v[in.c]; break;
          default: var = true;  // loads, index, InBounds
        }
        ls.u[i] = !var;
        // an unconditional write replaces the register's value; a guarded one
        // may leave the old (possibly varying) value in place
        if (b.gid == 0) v[in.dst] = var;
        else if (var) v[in.dst] = 1;
        any_u |= !var;
      }
      if (b.gid != 0 && any_u) ls.blk_bit[bi] = ls.nbits++;
    }
    // A root whose last write is a uniform instruction in a block guarded by
    // the root's own guard (and that guard register is not rewritten after
    // the block starts) always holds that uniform value when the root counts:
    // the usual shape of generated code (guarded block computes, guarded
    // root reads), even when the register held varying values earlier.
    std::vector<int> last_w(pg.num_regs, -1), blk_of(pg.instrs.size(), -1);
    for (size_t bi = 0; bi < pg.blocks.size(); ++bi)
      for (uint32_t i = pg.blocks[bi].begin; i < pg.blocks[bi].end; ++i) {
        last_w[pg.instrs[i].dst] = int(i);
        blk_of[i] = int(bi);
      }
    auto root_var = [&](uint32_t gid, uint16_t reg) {
      if (!v[reg]) return false;
      const int w = last_w[reg];
      if (w < 0 || !ls.u[size_t(w)] || gid == 0) return true;
      const Block& b = pg.blocks[size_t(blk_of[size_t(w)])];
      if (b.gid != gid) return true;
      const uint16_t g = pg.guard_regs[gid];
      for (size_t i = b.begin; i < pg.instrs.size(); ++i)
        if (pg.instrs[i].dst == g) return true;
      return false;
    };
    for (size_t o = 0; o < pg.outputs.size(); ++o) {
      bool var = false;
      for (auto [gid, reg] : pg.outputs[o]) var |= root_var(gid, reg);
      if (var) {
        ls.varying.push_back(int(o));
        continue;
      }
      for (auto [gid, reg] : pg.outputs[o])
        if (gid != 0 && ls.out_bit[gid] < 0) ls.out_bit[gid] = ls.nbits++;
    }
    ls.ok = ls.nbits <= 32;
    return ls;
  }
  // split_mode 1: program() also returns the guard outcomes (`*bits_out`);
  // split_mode 2: program() is the cache READER: uniform instructions only,
  // guards from `bits`, varying outputs from `cv[]`.
  const LaneSplit* cur_split = nullptr;
  int split_mode = 0;

  std::string program(const Program& pg, bool graph, const Domain* dom = nullptr, bool sm = false) {
    std::string name = "mo_prog_" + std::to_string(nprog++);
    iter_dom = graph ? nullptr : dom;
    sm_mode = sm && !graph;
    reach = reach_of(pg, iter_dom);
    const LaneSplit* ls = split_mode ? cur_split : nullptr;
    if (ls && split_mode == 2) {
      os << "__device__ __forceinline__ void " << name
         << "(const mo_kparams& P, unsigned bits, const Real* cv, Real* out) {\n  (void)P; (void)bits; (void)cv;\n";
      std::vector<char> used(pg.num_regs, 0);  // every register the uniform slice touches
      for (size_t i = 0; i < pg.instrs.size(); ++i)
        if (ls->u[i]) {
          const Instr& in = pg.instrs[i];
          used[in.dst] = 1;
          if (in.op != kImm && in.op != kParam) used[in.a] = 1;
          if (in.op == kAdd || in.op == kMul || in.op == kCmp || in.op == kAnd || in.op == kOr || in.op == kSel)
            used[in.b] = 1;
          if (in.op == kSel) used[in.c] = 1;
        }
      for (const auto& o : pg.outputs)
        for (auto [gid, reg] : o) used[reg] = 1;
      for (uint32_t r = 0; r < pg.num_regs; ++r)
        if (used[r]) os << "  Real r" << r << " = (Real)0;\n";
      for (size_t bi = 0; bi < pg.blocks.size(); ++bi) {
        const Block& b = pg.blocks[bi];
        bool any = false;
        for (uint32_t i = b.begin; i < b.end; ++i) any |= ls->u[i] != 0;
        if (!any) continue;
        std::string ind = "  ";
        if (b.gid != 0) {
          os << "  if ((bits >> " << ls->blk_bit[bi] << ") & 1u) {\n";
          ind = "    ";
        }
        for (uint32_t i = b.begin; i < b.end; ++i)
          if (ls->u[i]) os << ind << instr(pg.instrs[i], graph) << "\n";
        if (b.gid != 0) os << "  }\n";
      }
      size_t vi = 0;
      for (size_t o = 0; o < pg.outputs.size(); ++o) {
        if (vi < ls->varying.size() && ls->varying[vi] == int(o)) {
          os << "  out[" << o << "] = cv[" << vi++ << "];\n";
          continue;
        }
        os << "  { Real acc = (Real)0;";
        for (auto [gid, reg] : pg.outputs[o]) {
          if (gid != 0)
            os << " if ((bits >> " << ls->out_bit[gid] << ") & 1u) acc += r" << reg << ";";
          else
            os << " acc += r" << reg << ";";
        }
        os << " out[" << o << "] = acc; }\n";
      }
      os << "}\n";
      return name;
    }
    if (sm_mode)
      os << "template <bool I> __device__ __forceinline__ void " << name
         << "(const mo_kparams& P, int p0, int p1, int p2, const int* ri, int lx, Real* out"
         << (ls ? ", unsigned* bits_out" : "") << ") {\n"
         << "  (void)P; (void)p0; (void)p1; (void)p2; (void)ri; (void)lx; const int eb = 0; (void)eb;\n";
    else
      os << "template <bool I> __device__ __forceinline__ void " << name
         << "(const mo_kparams& P, int p0, int p1, int p2, int eb, const int* vs, Real* out"
         << (ls ? ", unsigned* bits_out" : "") << ") {\n"
         << "  (void)P; (void)p0; (void)p1; (void)p2; (void)eb; (void)vs;\n";
    if (ls) os << "  unsigned bits = 0u;\n";
    if (iter_dom) {
      // Strides of the iteration domain are plan constants (the plan fixes the
      // global dims), so every interior stencil read is base + immediate.
      const auto sh = P.shape_of(*iter_dom);
      const size_t nd = iter_dom->dims.size();
      const long long m0 = nd == 3 ? sh[1] * sh[2] : (nd == 2 ? sh[1] : 1), m1 = nd == 3 ? sh[2] : 1;
      os << "  constexpr int ms0 = " << m0 << ", ms1 = " << m1 << ";\n  (void)ms0; (void)ms1;\n";
    } else {
      os << "  const int ms0 = P.dnd == 3 ? P.d1 * P.d2 : (P.dnd == 2 ? P.d1 : 1), ms1 = P.dnd == 3 ? P.d2 : 1;\n"
         << "  (void)ms0; (void)ms1;\n";
    }
    {
      std::vector<std::pair<int, int>> slots;
      for (const Instr& in : pg.instrs) {
        if (!(in.op == kLoadU || in.op == kLoadA || in.op == kLoadC || in.op == kLoadP) || in.graph) continue;
        const Field& f = field_of(in.op, in.field);
        if (!iter_dom || !(f.dom == *iter_dom)) continue;
        std::pair<int, int> sc{slot_of(in.op, in.field), f.channels};
        if (std::find(slots.begin(), slots.end(), sc) == slots.end()) slots.push_back(sc);
      }
      if (!sm_mode) os << ldi_bases(slots);
    }
    for (uint32_t r = 0; r < pg.num_regs; ++r) os << "  Real r" << r << " = (Real)0;\n";
    for (size_t bi = 0; bi < pg.blocks.size(); ++bi) {
      const Block& b = pg.blocks[bi];
      std::string ind = "  ";
      if (ls && ls->blk_bit[bi] >= 0)
        os << "  bits |= (r" << pg.guard_regs[b.gid] << " != (Real)0 ? 1u : 0u) << " << ls->blk_bit[bi] << ";\n";
      if (b.gid != 0) {
        os << "  if (r" << pg.guard_regs[b.gid] << " != (Real)0) {\n";
        ind = "    ";
      }
      for (uint32_t i = b.begin; i < b.end; ++i) {
        // sin(x) next to cos(x) of the same register: one sincos call shares
        // the argument reduction (rotate2d/rotate3d emit exactly this pair).
        const Instr& a = pg.instrs[i];
        if (i + 1 < b.end && a.op == kUn && (a.sub == kSin || a.sub == kCos) && a.dst != a.a) {
          const Instr& c = pg.instrs[i + 1];
          if (c.op == kUn && c.a == a.a && (c.sub == kSin || c.sub == kCos) && c.sub != a.sub) {
            const Instr& si = a.sub == kSin ? a : c;
            const Instr& co = a.sub == kSin ? c : a;
            os << ind << "{ Real s_, c_; " << (f64 ? "sincos" : "sincosf") << "(" << reg(a.a) << ", &s_, &c_); "
               << reg(si.dst) << " = s_; " << reg(co.dst) << " = c_; }\n";
            ++i;
            continue;
          }
        }
        os << ind << instr(a, graph) << "\n";
      }
      if (b.gid != 0) os << "  }\n";
    }
    for (size_t o = 0; o < pg.outputs.size(); ++o) {
      os << "  { Real acc = (Real)0;";
      for (auto [gid, reg] : pg.outputs[o]) {
        if (gid != 0)
          os << " if (r" << pg.guard_regs[gid] << " != (Real)0) acc += r" << reg << ";";
        else
          os << " acc += r" << reg << ";";
      }
      os << " out[" << o << "] = acc; }\n";
    }
    if (ls) {
      for (size_t gid = 0; gid < ls->out_bit.size(); ++gid)
        if (ls->out_bit[gid] >= 0)
          os << "  bits |= (r" << pg.guard_regs[gid] << " != (Real)0 ? 1u : 0u) << " << ls->out_bit[gid] << ";\n";
      os << "  *bits_out = bits;\n";
    }
    os << "}\n";
    return name;
  }

  std::string reg(int r) const { return "r" + std::to_string(r); }

  // Interior-tile read of a field on the iteration domain: one shared element
  // index `eb` plus a constant stencil offset (strides ms0/ms1 are uniform).
  static std::string ldi(int C, int sl, int o0, int o1, int o2, int ch) {
    std::ostringstream s;
    (void)C;
    s << "__ldg(b" << sl << " + ((" << o0 << ") * ms0 + (" << o1 << ") * ms1 + (" << o2 << ")) * " << C << " + " << ch
      << ")";
    return s.str();
  }
  // Staged read: field ring in dynamic smem, row ri[o0 + rx], column lx + o1.
  std::string smx(int sl, int o0, int o1, int ch) const {
    const auto* st = staged_of(sl);
    std::ostringstream s;
    const int C = st->second;
    s << "reinterpret_cast<const Real*>(mo_dsm + " << st->first << ")[ri[" << o0 + st_rx << "] * " << st_win * C
      << " + (lx + (" << o1 << ")) * " << C << " + " << ch << "]";
    return s.str();
  }
  // Per-field interior base pointers (field start + eb*C): each stencil load
  // is then base + (row offset) + immediate.
  static std::string ldi_bases(const std::vector<std::pair<int, int>>& slots) {
    std::ostringstream s;
    for (auto [sl, C] : slots)
      s << "  const Real* __restrict__ b" << sl << " = I ? reinterpret_cast<const Real*>(P.v[" << sl
        << "].p) + (long long)eb * " << C << " : nullptr; (void)b" << sl << ";\n";
    return s.str();
  }
  static std::string ldi_unused(int C, int sl, int o0, int o1, int o2, int ch) {
    std::ostringstream s;
    s << "mo_ldi<Real, " << C << ">(P.v[" << sl << "], eb + (" << o0 << ") * ms0 + (" << o1 << ") * ms1 + (" << o2
      << "), " << ch << ")";
    return s.str();
  }

  std::string instr(const Instr& in, bool graph) {
    std::ostringstream s;
    s << reg(in.dst) << " = ";
    switch (in.op) {
      case kImm: s << "(Real)(" << hexd(in.imm) << ")"; break;
      case kParam:
        check(in.field >= 0 && size_t(in.field) < P.params.size(), Err::kShapeMismatch,
              "kernel reads a parameter that is not declared");
        if (in.field < 16) s << "(Real)P.pv[" << in.field << "]";  // MO_MAX_PARAMS
        else s << "(Real)P.params[" << in.field << "]";
        break;
      case kIndex:
        if (graph || in.field > 2) s << "(Real)0";  // graph env pix = {0,0,0}
        else s << "(Real)p" << in.field;
        break;
      case kLoadU:
      case kLoadA:
      case kLoadC:
      case kLoadP: {
        const Field& f = field_of(in.op, in.field);
        check(in.channel >= 0 && in.channel < f.channels, Err::kShapeMismatch,
              "kernel reads past the bound channel count");
        int sl = slot_of(in.op, in.field);
        if (in.graph) {
          s << "mo_ldv<Real, " << f.channels << ">(P.v[" << sl << "], vs[" << in.slot << "], "
            << in.channel << ")";
        } else {
          int nd = int(f.dom.dims.size());
          const bool same = iter_dom && f.dom == *iter_dom;
          if (same && sm_mode && staged_of(sl)) {
            s << smx(sl, in.off[0], in.off[1], in.channel);
            break;
          }
          if (same && !sm_mode) s << "(I ? " << ldi(f.channels, sl, in.off[0], in.off[1], in.off[2], in.channel) << " : ";
          s << "mo_ld<Real, " << (nd ? nd : 1) << ", " << f.channels << ", false>(P.v[" << sl << "], p0 + ("
            << in.off[0] << "), p1 + (" << in.off[1] << "), p2 + (" << in.off[2] << "), " << in.channel << ")";
          if (same && !sm_mode) s << ")";
        }
        break;
      }
      case kInB:
        if (graph) s << "(Real)(" << (in.off[0] == 0 ? 1 : 0) << ")";
        else
          s << "((I || mo_inb(P, p0 + (" << in.off[0] << "), p1 + (" << in.off[1] << "), p2 + ("
            << in.off[2] << "))) ? (Real)1 : (Real)0)";
        break;
      case kAdd: s << reg(in.a) << " + " << reg(in.b); break;
      case kMul: s << reg(in.a) << " * " << reg(in.b); break;
      case kPow: s << "mo_pow_eval<Real>(" << reg(in.a) << ", " << in.pnum << "LL, " << in.pden << "LL)"; break;
      case kUn: s << fn(in.sub) << "(" << reg(in.a) << ")"; break;
      case kCmp: {
        static const char* ops[] = {"==", "!=", "<", "<=", ">", ">="};
        check(in.sub <= kGe, Err::kFormatError, "codegen: unknown comparison");
        s << "((" << reg(in.a) << " " << ops[in.sub] << " " << reg(in.b) << ") ? (Real)1 : (Real)0)";
        break;
      }
      case kAnd:
        s << "((" << reg(in.a) << " != (Real)0 && " << reg(in.b) << " != (Real)0) ? (Real)1 : (Real)0)";
        break;
      case kOr:
        s << "((" << reg(in.a) << " != (Real)0 || " << reg(in.b) << " != (Real)0) ? (Real)1 : (Real)0)";
        break;
      case kNot: s << "((" << reg(in.a) << " == (Real)0) ? (Real)1 : (Real)0)"; break;
      case kSel: s << "((" << reg(in.a) << " != (Real)0) ? " << reg(in.b) << " : " << reg(in.c) << ")"; break;
      default: fail(Err::kFormatError, "codegen: unknown opcode");
    }
    s << ";";
    return s.str();
  }

  static std::string call(const std::string& pn) {
    return "if (it) " + pn + "<true>(P, p0, p1, p2, mo_local_elem(P, p0, p1, p2), nullptr, o); else " + pn +
           "<false>(P, p0, p1, p2, 0, nullptr, o);";
  }

  static std::string kbegin(const std::string& kname) {
    return "extern \"C\" __global__ void __launch_bounds__(MO_THREADS) " + kname +
           "(const __grid_constant__ mo_kparams P) {\n  MO_PDL_ENTRY();\n";
  }

  // --------------------------------------------------------- grid kernels
  void grid_cost(const std::string& pn, const std::string& kn) {
    os << kbegin(kn)
       << "  double acc = 0; bool bad = false;\n"
          "  const int nt = mo_num_tiles(P);\n"
          "  for (int t = blockIdx.x; t < nt; t += gridDim.x) {\n"
       << "    const mo_tile T = mo_tile_at(P, t);\n"
       << "    const bool it = mo_tile_in(P, T, " << reach << ");\n"
          "    int p0, p1, p2;\n"
          "    if (mo_tile_elem(P, T, p0, p1, p2)) {\n"
          "      Real o[1];\n      "
       << call(pn) << "\n"
          "      if (!mo_finite((double)o[0])) bad = true;\n"
          "      acc += (double)o[0];\n"
          "    }\n"
          "  }\n"
          "  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n"
          "  mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n"
          "}\n";
  }

  void grid_evalf(const std::string& pn, const std::string& kn, size_t nout) {
    os << kbegin(kn) << "  bool bad = false;\n"
       << "  const int nt = mo_num_tiles(P);\n"
          "  for (int t = blockIdx.x; t < nt; t += gridDim.x) {\n"
       << "    const mo_tile T = mo_tile_at(P, t);\n"
       << "    const bool it = mo_tile_in(P, T, " << reach << ");\n"
          "    int p0, p1, p2;\n"
          "    if (mo_tile_elem(P, T, p0, p1, p2)) {\n"
          "      const int e = mo_local_elem(P, p0, p1, p2);\n"
          "      Real o["
       << (nout ? nout : 1) << "];\n      " << call(pn) << "\n";
    for (size_t k = 0; k < nout; ++k)
      os << "      if (!mo_finite((double)o[" << k << "])) bad = true;\n"
         << "      ((Real*)P.out0)[P.rowbase[" << k << "] + e] = o[" << k << "];\n";
    os << "    }\n  }\n  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n}\n";
  }

  // Per-element writes of `nout` outputs into strided buffers (computed arrays).
  void grid_store(const std::string& pn, const std::string& kn, size_t nout) {
    os << kbegin(kn) << "  bool bad = false;\n"
       << "  const int nt = mo_num_tiles(P);\n"
          "  for (int t = blockIdx.x; t < nt; t += gridDim.x) {\n"
       << "    const mo_tile T = mo_tile_at(P, t);\n"
       << "    const bool it = mo_tile_in(P, T, " << reach << ");\n"
          "    int p0, p1, p2;\n"
          "    if (mo_tile_elem(P, T, p0, p1, p2)) {\n"
          "      const long long e = mo_local_elem(P, p0, p1, p2);\n"
          "      Real o["
       << (nout ? nout : 1) << "];\n      " << call(pn) << "\n";
    for (size_t k = 0; k < nout; ++k)
      os << "      if (!mo_finite((double)o[" << k << "])) bad = true;\n"
         << "      ((Real*)P.out0)[e * " << nout << " + " << k << "] = o[" << k << "];\n";
    os << "    }\n  }\n  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n}\n";
  }

  void grid_exclude(const std::string& pn, const std::string& kn) {
    os << kbegin(kn)
       << "  const int nt = mo_num_tiles(P);\n"
          "  for (int t = blockIdx.x; t < nt; t += gridDim.x) {\n"
       << "    const mo_tile T = mo_tile_at(P, t);\n"
       << "    const bool it = mo_tile_in(P, T, " << reach << ");\n"
          "    int p0, p1, p2;\n"
          "    if (mo_tile_elem(P, T, p0, p1, p2)) {\n"
          "      const int e = mo_local_elem(P, p0, p1, p2);\n"
          "      Real o[1];\n      "
       << call(pn) << "\n"
          "      ((unsigned char*)P.out0)[e] = (o[0] != (Real)0) ? 1 : 0;\n"
          "    }\n  }\n}\n";
  }

  // build_normal gather (solver.hpp:221-230) + fused identity patch (241-250).
  void gather_bm(const GatherSet& g, const std::string& pn, const std::string& kn) {
    const size_t K = g.chans.size();
    os << kbegin(kn) << "  double cnt = 0, rz = 0; bool bad = false;\n"
       << "  Real* B = (Real*)P.out0; Real* M = (Real*)P.out1;\n"
       << "  Real* PP = (Real*)P.out2; Real* DL = (Real*)P.out3; Real* RR = (Real*)P.out4;\n"
       << "  const bool pinit = (P.flags & MO_F_PCGINIT) != 0;\n"
       << "  const int pre = P.state->use_precond;\n"
       << "  if (pinit && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) {\n"
       << "    P.state->done = 0; P.state->iters = 0; P.state->indefinite = 0; P.state->nonfinite = 0; P.state->stop_code = 0x7fffffff;\n"
       << "  }\n"
          "  const int nt = mo_num_tiles(P);\n"
          "  for (int t = blockIdx.x; t < nt; t += gridDim.x) {\n"
       << "    const mo_tile T = mo_tile_at(P, t);\n"
       << "    const bool it = mo_tile_in(P, T, " << reach << ");\n"
          "    int p0, p1, p2;\n"
          "    if (mo_tile_elem(P, T, p0, p1, p2)) {\n"
          "      const long long e = mo_local_elem(P, p0, p1, p2);\n"
          "      Real o["
       << (K ? 2 * K : 1)
       << "];\n"
          "      const bool ex = P.mask && P.mask[e];\n"
          "      if (ex) {\n"
       << "        for (int k = 0; k < " << 2 * K << "; ++k) o[k] = (Real)0;\n"
       << "      } else {\n        " << call(pn) << "\n"
       << "        for (int k = 0; k < " << 2 * K << "; ++k) if (!mo_finite((double)o[k])) bad = true;\n"
       << "      }\n";
    for (size_t k = 0; k < K; ++k) {
      int f = g.chans[k].first, ch = g.chans[k].second;
      int C = P.unknowns[size_t(f)].channels;
      os << "      { const long long col = P.ubase[" << f << "] + e * " << C << " + " << ch << ";\n"
         << "        Real b = o[" << 2 * k << "], m = o[" << 2 * k + 1 << "];\n"
         << "        if (P.flags & MO_F_PATCH) {\n"
         << "          if (ex) { b = (Real)0; m = (Real)1; }\n"
         << "          else if (m == (Real)0) { m = (Real)1; cnt += 1.0; }\n"
         << "        }\n"
         << "        B[col] = b; M[col] = m;\n"
         << "        if (pinit) {  // k_pcg_init (pcg.hpp:75-97) on the patched b, m\n"
         << "          const bool xc = P.colmask && (P.colmask[col] & 1);\n"
         << "          const Real ri = xc ? (Real)0 : b;\n"
         << "          const Real zi = xc ? (Real)0 : (pre ? ((ri == (Real)0 && m > (Real)0) ? ri : ri / m) : ri);\n"
         << "          DL[col] = (Real)0; RR[col] = ri; PP[col] = zi; rz += (double)(ri * zi);\n"
         << "        } }\n";
    }
    os << "    }\n  }\n  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n"
       << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, cnt, rz, pinit);\n}\n";
  }

  // Matrix-free normal apply gather (solver.hpp:257-265), with optional fused
  // LM damping (401-405), excluded zeroing and p'Ap reduction (pcg.hpp:100-102).
  void gather_jtj(const GatherSet& g, const std::string& pn, const std::string& kn) {
    const size_t K = g.chans.size();
    // Inside the PCG (MO_F_EXSKIP) with an active-tile list in in3 ([count,
    // tile ids ascending]): fully excluded tiles store nothing, so only the
    // listed tiles are visited (Poisson: 1/4 of them).
    os << kbegin(kn) << "  if ((P.flags & MO_F_SKIPDONE) && P.state->done) return;\n"
       << "  double acc = 0; bool bad = false;\n"
       << "  Real* OUT = (Real*)P.out0; const Real* PV = (const Real*)P.in0; const Real* DAMP = (const Real*)P.in1;\n"
          "  const int* const TL = (P.flags & MO_F_EXSKIP) ? (const int*)P.in3 : nullptr;\n"
          "  const int nt = TL ? __ldg(TL) : mo_num_tiles(P);\n"
          "  for (int ti = blockIdx.x; ti < nt; ti += gridDim.x) {\n"
          "    const int t = TL ? __ldg(TL + 1 + ti) : ti;\n"
       << "    const mo_tile T = mo_tile_at(P, t);\n"
       << "    const bool it = mo_tile_in(P, T, " << reach << ");\n"
          "    int p0, p1, p2;\n"
          "    if (mo_tile_elem(P, T, p0, p1, p2)) {\n"
          "      const long long e = mo_local_elem(P, p0, p1, p2);\n"
          "      Real o["
       << (K ? K : 1)
       << "];\n"
          "      const bool ex = P.mask && P.mask[e];\n"
          "      if (ex) {\n"
       << "        for (int k = 0; k < " << K << "; ++k) o[k] = (Real)0;\n"
       << "      } else {\n        " << call(pn) << "\n"
       << "        for (int k = 0; k < " << K << "; ++k) if (!mo_finite((double)o[k])) bad = true;\n"
       << "      }\n";
    // An excluded element's outputs are 0 and so are its p'Ap terms (p is
    // pinned to 0 on excluded columns, pcg.hpp:50-55): unless an undamped-
    // then-unzeroed LM apply asks for damp * p there, nothing is read for it.
    // The column mask of a field on the gather's domain is the element mask
    // (k_colmask), so ZEROEXCL tests `ex`.  Inside the PCG (MO_F_EXSKIP) an
    // excluded element stores nothing at all: the update reads the column
    // mask first and never the Ap of an excluded column (pcg_update1 /
    // pcg_update_r1), so the zeros are dead writes (Poisson 8192^2: 3/4 of
    // the elements, 600 of the 1020 MB a launch moved).
    os << "      const bool ez = ex && (!(P.flags & MO_F_DAMP) || (P.flags & MO_F_ZEROEXCL));\n";
    for (size_t k = 0; k < K; ++k) {
      int f = g.chans[k].first, ch = g.chans[k].second;
      int C = P.unknowns[size_t(f)].channels;
      os << "      { const long long col = P.ubase[" << f << "] + e * " << C << " + " << ch << ";\n"
         << "        if (ez) { if (!(P.flags & MO_F_EXSKIP)) OUT[col] = (Real)0; }\n"
         << "        else {\n"
         << "          Real v = o[" << k << "];\n"
         << "          if (P.flags & MO_F_DAMP) v = v + DAMP[col] * PV[col];\n"
         << "          if ((P.flags & MO_F_ZEROEXCL) && ex) v = (Real)0;\n"
         << "          OUT[col] = v;\n"
         << "          if (P.flags & MO_F_REDUCE) acc += (double)(PV[col] * v);\n"
         << "        } }\n";
    }
    os << "    }\n  }\n  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n"
       << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n}\n";
  }

  // Two-phase matrix-free normal apply (the fast path; exact mode keeps the
  // gather program above).  Mathematically identical to the reference gather
  // (transform.hpp:238-260): jtj_c(q) = 2 sum_t sum_{lanes l of t on (f,c)}
  // d_l(q - o_l) * Jp_t(q - o_l) with Jp_t(e) = sum_{l in t} d_l(e) p(e + o_l)
  // and d_l the per-template partials of the reference's evalj program
  // (plan.hpp:244-264; already guarded by the implicit bound guard).
  // Phase 1 evaluates evalj ONCE per element of the tile plus an H-halo and
  // stores c_l(e) = d_l(e) Jp_t(e) in shared memory; phase 2 gathers.  This
  // removes the gather program's per-neighbour recomputation of every shifted
  // residual instance (ARAP: 114 vs 386 instructions per element).
  // Returns false (no kernel) when the domain is 3-D or no lanes exist.
  struct TwoPhase {
    bool ok = false;
    int H = 0, reach = 0, nlanes = 0;
    size_t smem = 0;
  };

  TwoPhase gather_jtj2(const GatherSet& g, int gi) {
    TwoPhase tp;
    const GridSet* S = nullptr;
    for (const GridSet& s : P.grid_sets)
      if (s.dom == g.dom && s.has_evalj) S = &s;
    const int nd = int(g.dom.dims.size());
    if (!S || nd < 1 || nd > 2) return tp;
    struct L {
      int t, out, f, c, o0, o1;
    };
    std::vector<L> lanes;
    for (size_t t = 0; t < S->jtemplates.size(); ++t)
      for (const Lane& ln : S->jtemplates[t].lanes) {
        if (ln.off[2] != 0 || (nd == 1 && ln.off[1] != 0)) return tp;
        lanes.push_back({int(t), ln.out, ln.field, ln.channel, ln.off[0], ln.off[1]});
      }
    if (lanes.empty()) return tp;
    int H = 0;
    for (const L& l : lanes) H = std::max({H, std::abs(l.o0), std::abs(l.o1)});
    const std::string pe = program(S->evalj, false, &g.dom);
    const int R = H + std::max(reach, H);
    const int NO = int(S->evalj.outputs.size());
    const int WX = nd == 2 ? kTileX + 2 * H : kThreads + 2 * H;
    const int WY = nd == 2 ? kTileY + 2 * H : 1;
    const int NE = WX * WY;
    const int SY = nd == 2 ? WX : 1;  // shared-memory stride of axis 0
    const int U = int(P.unknowns.size());
    // Merge lanes that land on the same (field, channel, offset): phase 1
    // pre-sums their contributions, phase 2 gathers one value per offset.
    struct M {
      int f, c, o0, o1;
    };
    std::vector<M> merged;
    std::vector<int> lane_slot(lanes.size());
    for (size_t li = 0; li < lanes.size(); ++li) {
      const L& l = lanes[li];
      int s = -1;
      for (size_t k = 0; k < merged.size(); ++k)
        if (merged[k].f == l.f && merged[k].c == l.c && merged[k].o0 == l.o0 && merged[k].o1 == l.o1) s = int(k);
      if (s < 0) {
        s = int(merged.size());
        merged.push_back({l.f, l.c, l.o0, l.o1});
      }
      lane_slot[li] = s;
    }
    const int NM = int(merged.size());
    const std::string sfx = std::to_string(gi);
    // Phase-1 body for one haloed element k at (p0, p1).
    os << "template <bool I> __device__ __forceinline__ void mo_lanes_" << sfx
       << "(const mo_kparams& P, int p0, int p1, int k, Real* CL, int ls) {\n"
       << "  constexpr int ms0 = " << (nd == 2 ? P.shape_of(g.dom)[1] : 1) << ", ms1 = 1; (void)ms1;\n"
       << "  const int eb = I ? mo_local_elem(P, p0, p1, 0) : 0;\n"
       << "  const bool inside = I || mo_inb(P, p0, p1, 0);\n";
    {
      std::vector<std::pair<int, int>> slots;
      for (const L& l : lanes) {
        std::pair<int, int> sc{U + l.f, P.unknowns[size_t(l.f)].channels};
        if (std::find(slots.begin(), slots.end(), sc) == slots.end()) slots.push_back(sc);
      }
      os << ldi_bases(slots);
    }
    os << "  Real d[" << NO << "];\n  " << pe << "<I>(P, p0, p1, 0, eb, nullptr, d);\n";
    for (int s = 0; s < NM; ++s) os << "  Real m" << s << " = (Real)0;\n";
    for (size_t t = 0; t < S->jtemplates.size(); ++t) {
      os << "  { Real jp = (Real)0;\n";
      for (const L& l : lanes) {
        if (l.t != int(t)) continue;
        const Field& f = P.unknowns[size_t(l.f)];
        os << "    jp += d[" << l.out << "] * (I ? " << ldi(f.channels, U + l.f, l.o0, l.o1, 0, l.c) << " : mo_ld<Real, "
           << nd << ", " << f.channels << ", false>(P.v[" << U + l.f << "], p0 + (" << l.o0 << "), p1 + (" << l.o1
           << "), 0, " << l.c << "));\n";
      }
      // An instance centred outside the domain exists only for templates that
      // never read their own pixel (transform.hpp:177-198 shifted guard).
      const bool origin = S->jtemplates[t].origin;
      if (origin) os << "    if (inside) {\n";
      for (size_t li = 0; li < lanes.size(); ++li)
        if (lanes[li].t == int(t)) os << "    m" << lane_slot[li] << " += d[" << lanes[li].out << "] * jp;\n";
      if (origin) os << "    }\n";
      os << "  }\n";
    }
    for (int s = 0; s < NM; ++s) os << "  CL[" << s << " * ls + k] = m" << s << ";\n";
    os << "}\n";
    const std::string kn = "mo_gather_jtj2_" + sfx;
    // Occupancy knob (blocks/SM the register allocator must allow) and
    // phase-1 unroll; MO_B200_JTJ2_MINB / MO_B200_JTJ2_UNROLL override.
    const char* mb = std::getenv("MO_B200_JTJ2_MINB");
    const char* ur = std::getenv("MO_B200_JTJ2_UNROLL");
    // Measured on B200 (ARAP 1024^2/8192^2, Poisson 8192^2, SFS): 5 resident
    // blocks (<= 48 registers) is the best single setting; unrolling hurts.
    const int minb = mb ? std::atoi(mb) : 5, unroll = ur ? std::atoi(ur) : 1;
    os << "extern \"C\" __global__ void __launch_bounds__(MO_THREADS" << (minb > 0 ? ", " + std::to_string(minb) : "")
       << ") " << kn
       << "(const __grid_constant__ mo_kparams P) {\n"
       << "  MO_PDL_ENTRY();\n"
       << "  if ((P.flags & MO_F_SKIPDONE) && P.state->done) return;\n"
       << "  extern __shared__ __align__(16) unsigned char mo_smem[];\n"
       << "  Real* CL = reinterpret_cast<Real*>(mo_smem);  // [" << NM << " merged lanes][" << NE << " elements]\n"
       << "  double acc = 0; bool bad = false;\n"
       << "  Real* OUT = (Real*)P.out0; const Real* PV = (const Real*)P.in0; const Real* DAMP = (const Real*)P.in1;\n"
       << "  const int tid = threadIdx.x + threadIdx.y * blockDim.x;\n"
       << "  const int nt = mo_num_tiles(P);\n"
       << "  for (int t = blockIdx.x; t < nt; t += gridDim.x) {\n"
       << "    const mo_tile T = mo_tile_at(P, t);\n"
       << "    const bool it = mo_tile_in(P, T, " << R << ");\n";
    const std::string pragma = unroll > 1 ? "    #pragma unroll " + std::to_string(unroll) + "\n" : "";
    if (nd == 2)
      os << "    const int r0 = T.o0 - " << H << ", c0 = T.o1 - " << H
         << ";\n"
         << pragma << "    for (int k = tid; k < " << NE << "; k += MO_THREADS) {\n"
         << "      const int q0 = r0 + k / " << WX << ", q1 = c0 + k % " << WX << ";\n";
    else
      os << "    const int r0 = T.o0 - " << H << ", c0 = 0; (void)c0;\n"
         << "    for (int k = tid; k < " << NE << "; k += MO_THREADS) {\n"
         << "      const int q0 = r0 + k, q1 = 0;\n";
    // (a strip stores rows [row0 - R, row1 + R): elements no owned output
    // needs are not evaluated, so no read leaves the strip's storage)
    os << "      if (q0 < P.row0 - " << H << " || q0 >= P.row1 + " << H << ") {\n"
       << "        for (int s = 0; s < " << NM << "; ++s) CL[s * " << NE << " + k] = (Real)0;\n"
       << "        continue;\n      }\n"
       << "      if (it) mo_lanes_" << sfx << "<true>(P, q0, q1, k, CL, " << NE << "); else mo_lanes_" << sfx
       << "<false>(P, q0, q1, k, CL, " << NE << ");\n"
       << "    }\n    __syncthreads();\n"
       << "    int p0, p1, p2;\n"
       << "    if (mo_tile_elem(P, T, p0, p1, p2)) {\n"
       << "      const long long e = mo_local_elem(P, p0, p1, p2);\n"
       << "      const int hb = (p0 - r0) * " << SY << (nd == 2 ? " + (p1 - c0)" : "") << ";\n"
       << "      const bool ex = P.mask && P.mask[e];\n";
    for (size_t k = 0; k < g.chans.size(); ++k) {
      const int f = g.chans[k].first, ch = g.chans[k].second;
      const int C = P.unknowns[size_t(f)].channels;
      os << "      { Real s = (Real)0;\n";
      for (int s = 0; s < NM; ++s) {
        const M& m = merged[size_t(s)];
        if (m.f != f || m.c != ch) continue;
        os << "        s += CL[" << s * NE << " + hb - (" << m.o0 * SY + (nd == 2 ? m.o1 : 0) << ")];\n";
      }
      os << "        Real v = ex ? (Real)0 : (Real)2 * s;\n"
         << "        if (!mo_finite((double)v)) bad = true;\n"
         << "        const long long col = P.ubase[" << f << "] + e * " << C << " + " << ch << ";\n"
         << "        if (P.flags & MO_F_DAMP) v = v + DAMP[col] * PV[col];\n"
         << "        if ((P.flags & MO_F_ZEROEXCL) && P.colmask && P.colmask[col]) v = (Real)0;\n"
         << "        OUT[col] = v;\n"
         << "        if (P.flags & MO_F_REDUCE) acc += (double)(PV[col] * v); }\n";
    }
    os << "    }\n    __syncthreads();\n  }\n"
       << "  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n"
       << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n}\n";
    tp.ok = true;
    tp.H = H;
    tp.reach = R;
    tp.nlanes = NM;
    tp.smem = size_t(NM) * size_t(NE) * (f64 ? 8 : 4);
    if (nd == 2) {
      gather_jtj3(g, gi, H, std::max(reach, H), NM, merged_off(merged));
      std::vector<LaneG> lg;
      for (const L& l : lanes) lg.push_back({l.t, l.out, l.f, l.c, l.o0, l.o1});
      gather_jtj4(g, gi, *S, lg, lane_slot, merged_off(merged), H);
      gather_jtj4(g, gi, *S, lg, lane_slot, merged_off(merged), H, 4);
      gather_jtj4(g, gi, *S, lg, lane_slot, merged_off(merged), H, 8, true);
      gather_jtj5(g, gi, *S, lg, lane_slot, merged_off(merged), H);
      gather_jtj8(g, gi, *S, lg, lane_slot, merged_off(merged), H, 0);
      gather_jtj8(g, gi, *S, lg, lane_slot, merged_off(merged), H, 1);
      lane_cache(g, gi, *S, H);
      if (lc_info.ok) gather_jtj8(g, gi, *S, lg, lane_slot, merged_off(merged), H, 2);
      if (lc_info.ok) gather_jtj8(g, gi, *S, lg, lane_slot, merged_off(merged), H, 4);
      // build_normal that also writes the lane cache (mo_gather_bm8c_<gi>)
      if (lc_info.ok) gather_jtj8(g, gi, *S, lg, lane_slot, merged_off(merged), H, 3);
    }
    return tp;
  }

  // TMA-staged row-streaming apply (2-D domains): gather_jtj3's band/ring
  // schedule, with every field the phase-1 body reads (x, arrays, computed on
  // the iteration domain and p) streamed into shared-memory row rings by TMA
  // 8 rows at a time, NBUF blocks deep, completion tracked by mbarriers.
  // Phase 1 then reads only shared memory (immediate offsets, no 64-bit
  // address arithmetic, no L1TEX misses on its critical path) and the loads
  // of the next rows overlap the current rows' arithmetic.  TMA zero-fills
  // out-of-bounds box elements, which is the reference's OOB->0 read rule
  // (eval.hpp:47-51), so border bands run the same code.
  // RS = rows per step = warps per block (8: mo_gather_jtj4_<gi>, 4:
  // mo_gather_jtj7_<gi>, twice the resident blocks for small grids).
  // bm = true: the same schedule for build_normal (solver.hpp:220-251):
  // phase 1 evaluates evalj AND evalf (residual values, one per template,
  // plan.hpp:236-239) once per element and forms per merged lane the J^T F
  // terms d_l r_t and the Jacobi terms d_l^2 (two contribution planes);
  // phase 2 gathers b = -2 sum, m = 2 sum with the identity patch, the
  // unconstrained count and the fused PCG start (mo_gather_bm4_<gi>).
  void gather_jtj4(const GatherSet& g, int gi, const GridSet& S, const std::vector<LaneG>& lanes,
                   const std::vector<int>& lane_slot, const std::vector<MLane>& merged, int H, int RS = 8,
                   bool bm = false) {
    const int LRS = RS == 8 ? 3 : 2;
    const std::string LN = bm ? "mo_lanesbm_" : RS == 8 ? "mo_lanes4_" : "mo_lanes7_";
    if (bm && S.evalf.outputs.size() != S.jtemplates.size()) return;
    if (f64_disabled_tma()) return;
    const std::string sfx = std::to_string(gi);
    const auto sh = P.shape_of(g.dom);
    const long long D0 = sh[0], D1 = sh[1];
    const int BW = 32 - 2 * H;
    if (BW < 8) return;
    const int U = int(P.unknowns.size());
    const int RX = std::max(std::max(reach_of(S.evalj, &g.dom), bm ? reach_of(S.evalf, &g.dom) : 0), H);
    if (2 * RX > RS) return;  // two RS-row blocks cover one step's input rows
    // TMA needs a 16-byte aligned box start: the window starts at the
    // aligned column cs <= c0 - H - RX (shift sh = c0 - H - RX - cs < AU).
    const int AU = f64 ? 2 : 4;
    const int WIN = (32 + 2 * RX + AU - 1 + AU - 1) / AU * AU;
    const int NBUF = std::getenv("MO_B200_JTJ4_NBUF") ? std::max(3, std::atoi(std::getenv("MO_B200_JTJ4_NBUF"))) : 3;
    const int NEED = 1 + (2 * RX + RS - 1) / RS;
    const int RING = RS + 2 * H;  // two barriers per step
    const int LS = RING * 32;
    const int NM = int(merged.size());
    const int RB = f64 ? 8 : 4;
    // Staged slots: same-domain fields evalj reads + the lanes' p fields.
    std::vector<std::pair<int, int>> slots;  // (slot, channels)
    auto add = [&](int sl, int C) {
      for (auto& x : slots)
        if (x.first == sl) return;
      slots.push_back({sl, C});
    };
    for (const Instr& in : S.evalj.instrs) {
      if (!(in.op == kLoadU || in.op == kLoadA || in.op == kLoadC || in.op == kLoadP) || in.graph) continue;
      const Field& f = field_of(in.op, in.field);
      if (f.dom == g.dom) add(slot_of(in.op, in.field), f.channels);
    }
    if (bm) {
      for (const Instr& in : S.evalf.instrs) {
        if (!(in.op == kLoadU || in.op == kLoadA || in.op == kLoadC || in.op == kLoadP) || in.graph) continue;
        const Field& f = field_of(in.op, in.field);
        if (f.dom == g.dom) add(slot_of(in.op, in.field), f.channels);
      }
    } else {
      for (const LaneG& l : lanes) add(U + l.f, P.unknowns[size_t(l.f)].channels);
    }
    if (slots.empty() || int(slots.size()) > MO_MAX_TMAPS_HOST) return;
    for (auto& x : slots)
      if (WIN * x.second > 256) return;  // TMA box inner extent limit
    // Dynamic smem layout: CL ring | field rings (128-B aligned) | mbarriers.
    const int NPL = bm ? 2 * NM : NM;  // contribution planes
    long long off = (long long)NPL * LS * RB;
    off = (off + 127) / 128 * 128;
    staged.clear();
    long long tx = 0;
    std::vector<long long> boxbytes;
    for (auto& x : slots) {
      staged.push_back({x.first, {off, x.second}});
      const long long bb = (long long)RS * WIN * x.second * RB;
      if (bb % 128) return;  // ring rows are contiguous across 128-byte aligned slots
      boxbytes.push_back(bb);
      tx += bb;
      off += (long long)NBUF * bb;
    }
    const long long mbar_off = off;
    off += 8LL * NBUF;
    st_rx = RX;
    st_win = WIN;
    const std::string pe = program(S.evalj, false, &g.dom, true);
    const std::string pf = bm ? program(S.evalf, false, &g.dom, true) : std::string();
    const int NO = int(S.evalj.outputs.size());
    const int NT = int(S.jtemplates.size());
    // Phase-1 body from shared memory.
    os << "template <bool I> __device__ __forceinline__ void " << LN << sfx
       << "(const mo_kparams& P, int p0, int p1, int k, Real* CL, const int* ri, int lx) {\n"
       << "  const bool inside = I || mo_inb(P, p0, p1, 0);\n"
       << "  Real d[" << NO << "];\n  " << pe << "<I>(P, p0, p1, 0, ri, lx, d);\n";
    if (bm) {
      os << "  Real fv[" << NT << "];\n  " << pf << "<I>(P, p0, p1, 0, ri, lx, fv);\n";
      for (int si = 0; si < NM; ++si) os << "  Real mb" << si << " = (Real)0, mm" << si << " = (Real)0;\n";
      for (int t = 0; t < NT; ++t) {
        const bool origin = S.jtemplates[size_t(t)].origin;
        os << "  {" << (origin ? " if (inside) {" : "") << "\n";
        for (size_t li = 0; li < lanes.size(); ++li)
          if (lanes[li].t == t)
            os << "    mb" << lane_slot[li] << " += d[" << lanes[li].out << "] * fv[" << t << "]; mm" << lane_slot[li]
               << " += d[" << lanes[li].out << "] * d[" << lanes[li].out << "];\n";
        os << "  }" << (origin ? " }" : "") << "\n";
      }
      for (int si = 0; si < NM; ++si)
        os << "  CL[" << si * LS << " + k] = mb" << si << "; CL[" << (NM + si) * LS << " + k] = mm" << si << ";\n";
      os << "}\n";
    }
    if (!bm) {
    for (int si = 0; si < NM; ++si) os << "  Real m" << si << " = (Real)0;\n";
    for (size_t t = 0; t < S.jtemplates.size(); ++t) {
      os << "  { Real jp = (Real)0;\n";
      for (const LaneG& l : lanes)
        if (l.t == int(t)) os << "    jp += d[" << l.out << "] * " << smx(U + l.f, l.o0, l.o1, l.c) << ";\n";
      const bool origin = S.jtemplates[t].origin;
      if (origin) os << "    if (inside) {\n";
      for (size_t li = 0; li < lanes.size(); ++li)
        if (lanes[li].t == int(t)) os << "    m" << lane_slot[li] << " += d[" << lanes[li].out << "] * jp;\n";
      if (origin) os << "    }\n";
      os << "  }\n";
    }
    for (int si = 0; si < NM; ++si) os << "  CL[" << si * LS << " + k] = m" << si << ";\n";
    os << "}\n";
    }
    sm_mode = false;

    const std::string kn = (bm ? "mo_gather_bm4_" : RS == 8 ? "mo_gather_jtj4_" : "mo_gather_jtj7_") + sfx;
    const char* mb = std::getenv("MO_B200_JTJ4_MINB");
    const int minb = mb ? std::atoi(mb) : 32 / RS;
    os << "extern \"C\" __global__ void __launch_bounds__(" << 32 * RS << (minb > 0 ? ", " + std::to_string(minb) : "")
       << ") " << kn << "(const __grid_constant__ mo_kparams P, const __grid_constant__ mo_tmaps T) {\n"
       << "  MO_PDL_ENTRY();\n"
       << "  if ((P.flags & MO_F_SKIPDONE) && P.state->done) return;\n"
       << "  Real* CL = reinterpret_cast<Real*>(mo_dsm);  // [" << NPL << " planes][" << RING << " rows][32]\n"
       << "  double cnt = 0, rz = 0; (void)cnt; (void)rz;\n";
    if (bm)
      os << "  if ((P.flags & MO_F_PCGINIT) && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) {\n"
         << "    P.state->done = 0; P.state->iters = 0; P.state->indefinite = 0; P.state->nonfinite = 0; P.state->stop_code = 0x7fffffff;\n"
         << "  }\n";
    os << "  unsigned long long* MB = reinterpret_cast<unsigned long long*>(mo_dsm + " << mbar_off << ");\n"
       << "  double acc = 0;\n"
       << "  unsigned em = 0;  // max exponent field of the outputs: all ones <=> a non-finite output\n"
       << "  const int tid = threadIdx.x + threadIdx.y * blockDim.x;\n"
       << "  const int w = tid >> 5, l = tid & 31;\n"
       << "  constexpr int NB = " << NB(D1, BW) << ", BW = " << BW << ", H = " << H << ", RX = " << RX << ";\n"
       << "  constexpr int D0 = " << D0 << ", D1 = " << D1 << ", RING = " << RING << ", NBUF = " << NBUF
       << ", NEED = " << NEED << ";\n"
       << "  if (tid == 0) {\n"
       << "    for (int i = 0; i < NBUF; ++i) mo_mbar_init(MB + i, 1);\n"
       << "    mo_mbar_fence_init();\n"
       << "  }\n"
       << "  __syncthreads();\n"
       << "  const int CH = P.chunk;\n"
       << "  const int nch = (P.row1 - P.row0 + CH - 1) / CH;\n"
       << "  const int items = NB * nch;\n"
       << "  int slot0 = 0;        // ring slot of the item's input block 0\n"
       << "  unsigned ph = 0;      // per-slot mbarrier phase parity (bit per slot)\n"
       << "  // input row block j of an item = global rows [y0 - H - RX + 8j, +8), window columns from cs\n";
    // Issue code is emitted inline at both sites: the tensor maps must be
    // addressed in kernel-parameter space (a helper that is not inlined
    // would see a local copy, which TMA rejects).
    std::ostringstream is;
    is << "{ int slot_ = slot0 + (JJ); while (slot_ >= NBUF) slot_ -= NBUF;\n"
       << "  mo_mbar_expect_tx(MB + slot_, " << tx << "u);\n"
       << "  const int r_ = y0 - H - RX + " << RS << " * (JJ) - P.row_lo;\n";
    for (size_t i = 0; i < slots.size(); ++i)
      is << "  mo_tma_load_2d(mo_dsm + " << staged[i].second.first << " + slot_ * " << boxbytes[i] << ", &T.m[" << i
         << "], cs * " << slots[i].second << ", r_, MB + slot_);\n";
    is << "}\n";
    auto issue = [&](const std::string& j) {
      std::string t = is.str();
      for (size_t p = t.find("JJ"); p != std::string::npos; p = t.find("JJ", p)) t.replace(p, 2, j);
      return t;
    };
    os << "  for (int t = blockIdx.x; t < items; t += gridDim.x) {\n"
       << "    const int ci = t / NB, c0 = (t - ci * NB) * BW;\n"
       << "    const int y0 = P.row0 + ci * CH, y1 = min(y0 + CH, P.row1);\n"
       << "    const bool it = y0 - H - RX >= 0 && y1 + H - 1 + RX < D0 && c0 - H - RX >= 0 && c0 - H + 31 + RX < D1;\n"
       << "    const int q1 = c0 - H + l;\n"
       << "    const int sh = (c0 - H - RX) & " << AU - 1 << ", cs = c0 - H - RX - sh;  // 16-byte aligned window start\n"
       << "    const int nsteps = (y1 - y0 + 2 * H + " << RS - 1 << ") >> " << LRS << ";\n"
       << "    const int nblk = (y1 - y0 + 2 * H + 2 * RX + " << RS - 1 << ") >> " << LRS << ";\n"
       << "    if (tid == 0) {\n"
       << "      mo_fence_proxy_async();\n"
       << "      for (int j = 0; j < NBUF && j < nblk; ++j) " << issue("j")
       << "    }\n"
       << "    // Per-warp ring bookkeeping, advanced incrementally (no divisions):\n"
       << "    // ss = ring slot of input block s; cr = CL ring row of phase-1 row 8s + w.\n"
       << "    int ss = slot0, cr = w;\n"
       << "    // Output columns of this lane (phase 2): 32-bit column indices.\n"
       << "    const bool lane_out = l >= H && l < 32 - H && q1 < D1;\n"
       << "    for (int s = 0; s < nsteps; ++s) {\n"
       << "      // Wait for the newest input block this step needs (each block is\n"
       << "      // waited exactly once; earlier ones were waited by earlier steps).\n"
       << "      if (s == 0) {\n"
       << "        for (int j = 0; j < NEED - 1 && j < nblk; ++j) {\n"
       << "          int q = ss + j; if (q >= NBUF) q -= NBUF;\n"
       << "          mo_mbar_wait(MB + q, (ph >> q) & 1u);\n"
       << "          ph ^= 1u << q;\n"
       << "        }\n"
       << "      }\n"
       << "      if (s + NEED - 1 < nblk) {\n"
       << "        int q = ss + NEED - 1; if (q >= NBUF) q -= NBUF;\n"
       << "        mo_mbar_wait(MB + q, (ph >> q) & 1u);\n"
       << "        ph ^= 1u << q;\n"
       << "      }\n"
       << "      const int rr = " << RS << " * s + w;  // phase-1 row relative to y0 - H\n"
       << "      const int q0 = y0 - H + rr;\n"
       << "      if (q0 < y1 + H) {\n"
       << "        int ri[" << 2 * RX + 1 << "];\n"
       << "        #pragma unroll\n"
       << "        for (int o = 0; o < " << 2 * RX + 1 << "; ++o) {\n"
       << "          const int rel = w + o;  // input row q0 + o - RX, relative to block s\n"
       << "          int b = ss + (rel >> " << LRS << "); if (b >= NBUF) b -= NBUF;\n"
       << "          ri[o] = b * " << RS << " + (rel & " << RS - 1 << ");\n"
       << "        }\n"
       << "        const int k = cr * 32 + l;\n"
       << "        if (it) " << LN << sfx << "<true>(P, q0, q1, k, CL, ri, l + RX + sh); else " << LN << sfx
       << "<false>(P, q0, q1, k, CL, ri, l + RX + sh);\n"
       << "      }\n"
       << "      __syncthreads();\n"
       << "      const int y = q0 - H;\n"
       << "      if (y >= y0 && y < y1 && lane_out) {\n"
       << "        const int e = (y - P.row_lo) * D1 + q1;\n"
       << "        const bool ex = P.mask && P.mask[e];\n";
    // CL ring row of output-row minus o0, for o0 in [-H, H]: cr - H - o0 (mod RING).
    for (int o = -H; o <= H; ++o)
      os << "        int sl" << (o < 0 ? "m" : "p") << std::abs(o) << " = cr - " << H + o << "; if (sl"
         << (o < 0 ? "m" : "p") << std::abs(o) << " < 0) sl" << (o < 0 ? "m" : "p") << std::abs(o) << " += RING; sl"
         << (o < 0 ? "m" : "p") << std::abs(o) << " = sl" << (o < 0 ? "m" : "p") << std::abs(o) << " * 32 + l;\n";
    if (bm) epilogue_bm4(g, merged, LS, NM, "        ", RS);
    else epilogue4(g, merged, LS, "        ", RS);
    os << "      }\n"
       << "      __syncthreads();  // CL ring rows are rewritten by the next step's phase 1\n"
       << "      // Input block s (read by phase 1 and, for p, by phase 2) is free now.\n"
       << "      if (tid == 0 && s + NBUF < nblk) {\n"
       << "        mo_fence_proxy_async();\n"
       << "        " << issue("s + NBUF")
       << "      }\n"
       << "      ss = ss + 1 == NBUF ? 0 : ss + 1;\n"
       << "      cr += " << RS << "; if (cr >= RING) cr -= RING;\n"
       << "    }\n"
       << "    slot0 += nblk; slot0 %= NBUF;\n"
       << "  }\n"
       << "  if (em == MO_EXP_MASK) atomicOr(&P.state->nonfinite_kernel, 1);\n";
    if (bm)
      os << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, cnt, rz, (P.flags & MO_F_PCGINIT) != 0);\n}\n";
    else
      os << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n}\n";
    ModuleInfo::Tma ti;
    ti.ok = true;
    ti.smem = size_t(off);
    ti.halo = H;
    ti.band = BW;
    ti.rx = RX;
    ti.win = WIN;
    ti.rows = RS;
    ti.threads = 32 * RS;
    for (auto& x : slots) ti.slots.push_back({x.first, x.second});
    (bm ? tmabm_info : RS == 8 ? tma_info : tma7_info) = ti;
    staged.clear();
  }
  // Warp-streaming TMA apply (2-D domains).  A block is NW warps side by
  // side: warp w owns the band of BW = 32 - 2H output columns starting at
  // c0 + w*BW and walks a chunk of rows on its own.  Per phase-1 row every lane
  // evaluates the evalj template partials of its element ONCE (from the
  // TMA-fed shared-memory input ring), forms the NM merged-lane contributions
  // and routes them to their output pixels without shared memory: the column
  // offset o1 through a warp shuffle, the row offset o0 into one of 2H+1
  // rolling register accumulators (out(q) = sum_s c_s(q - o_s), gather_jtj2's
  // sum).  Row q0 - H is complete after row q0 and is written at once.  No
  // block barrier per row: input blocks of R rows are refilled by whichever
  // warp releases a slot last (shared-memory arrival counter), consumers wait
  // on the slot's mbarrier.  One TMA box per field and input block, so the
  // block window (NW*BW + 2H + 2RX, aligned) must fit 256/C columns.
  void gather_jtj5(const GatherSet& g, int gi, const GridSet& S, const std::vector<LaneG>& lanes,
                   const std::vector<int>& lane_slot, const std::vector<MLane>& merged, int H) {
    if (f64_disabled_tma()) return;
    const std::string sfx = std::to_string(gi);
    const auto sh = P.shape_of(g.dom);
    const long long D0 = sh[0], D1 = sh[1];
    const int BW = 32 - 2 * H;
    if (BW < 8) return;
    const int U = int(P.unknowns.size());
    const int RX = std::max(reach_of(S.evalj, &g.dom), H);
    const int AU = f64 ? 2 : 4;
    const int R = 1;  // rows per input block (TMA box); the ring holds NBUF rows
    int NBUF = 1;
    while (NBUF < 2 * RX + 2) NBUF *= 2;  // rows a phase-1 row reads + one in flight, power of two
    const int NM = int(merged.size());
    const int RB = f64 ? 8 : 4;
    std::vector<std::pair<int, int>> slots;  // (slot, channels)
    auto add = [&](int sl, int C) {
      for (auto& x : slots)
        if (x.first == sl) return;
      slots.push_back({sl, C});
    };
    for (const Instr& in : S.evalj.instrs) {
      if (!(in.op == kLoadU || in.op == kLoadA || in.op == kLoadC || in.op == kLoadP) || in.graph) continue;
      const Field& f = field_of(in.op, in.field);
      if (f.dom == g.dom) add(slot_of(in.op, in.field), f.channels);
    }
    for (const LaneG& l : lanes) add(U + l.f, P.unknowns[size_t(l.f)].channels);
    for (auto& fc : g.chans) add(U + fc.first, P.unknowns[size_t(fc.first)].channels);
    if (slots.empty() || int(slots.size()) > MO_MAX_TMAPS_HOST) return;
    int cmax = 1;
    for (auto& x : slots) cmax = std::max(cmax, x.second);
    // widest block whose window fits one TMA box row (<= 256 elements)
    int NW = 0, WIN = 0;
    // WIN unit: 16-byte aligned box starts (AU) and R-row slots that are
    // whole multiples of 128 bytes (R * WIN * RB % 128 == 0 for any C).
    const int WU = std::max(AU, 128 / (R * RB));
    for (int nw = 4; nw >= 1; --nw) {
      const int win = (nw * BW + 2 * H + 2 * RX + AU - 1 + WU - 1) / WU * WU;
      if (win * cmax <= 256) {
        NW = nw;
        WIN = win;
        break;
      }
    }
    if (!NW) return;
    // Dynamic smem: field rings [NBUF*R rows][WIN*C] (128-B aligned) | mbarriers | counters.
    long long off = 0;
    staged.clear();
    long long tx = 0;
    std::vector<long long> boxbytes;
    for (auto& x : slots) {
      staged.push_back({x.first, {off, x.second}});
      const long long bb = (long long)R * WIN * x.second * RB;
      boxbytes.push_back(bb);  // a multiple of 128 bytes (WIN rounding): TMA destinations are 128-byte aligned
      tx += bb;
      off += (long long)NBUF * bb;
    }
    const long long mbar_off = off;
    off += 8LL * NBUF;
    const long long cnt_off = off;
    off += 4LL * NBUF;
    st_rx = RX;
    st_win = WIN;
    const std::string pe = program(S.evalj, false, &g.dom, true);
    const int NO = int(S.evalj.outputs.size());
    os << "template <bool I> __device__ __forceinline__ void mo_lanes5_" << sfx
       << "(const mo_kparams& P, int p0, int p1, const int* ri, int lx, Real* c) {\n"
       << "  const bool inside = I || mo_inb(P, p0, p1, 0);\n"
       << "  Real d[" << NO << "];\n  " << pe << "<I>(P, p0, p1, 0, ri, lx, d);\n";
    for (int si = 0; si < NM; ++si) os << "  Real m" << si << " = (Real)0;\n";
    for (size_t t = 0; t < S.jtemplates.size(); ++t) {
      os << "  { Real jp = (Real)0;\n";
      for (const LaneG& l : lanes)
        if (l.t == int(t)) os << "    jp += d[" << l.out << "] * " << smx(U + l.f, l.o0, l.o1, l.c) << ";\n";
      const bool origin = S.jtemplates[t].origin;
      if (origin) os << "    if (inside) {\n";
      for (size_t li = 0; li < lanes.size(); ++li)
        if (lanes[li].t == int(t)) os << "    m" << lane_slot[li] << " += d[" << lanes[li].out << "] * jp;\n";
      if (origin) os << "    }\n";
      os << "  }\n";
    }
    for (int si = 0; si < NM; ++si) os << "  c[" << si << "] = m" << si << ";\n";
    os << "}\n";
    sm_mode = false;

    const int K = int(g.chans.size());
    const int NA = 2 * H + 1;
    const std::string kn = "mo_gather_jtj5_" + sfx;
    const char* mb = std::getenv("MO_B200_JTJ5_MINB");
    const int minb = mb ? std::atoi(mb) : 0;
    std::ostringstream is;  // TMA issue of input block JJ (inline: tensor maps in param space)
    is << "{ const int slot_ = (slot0 + (JJ)) & (NBUF - 1);\n"
       << "  mo_mbar_expect_tx(MB + slot_, " << tx << "u);\n"
       << "  const int r_ = y0 - H - RX + R * (JJ) - P.row_lo;\n";
    for (size_t i = 0; i < slots.size(); ++i)
      is << "  mo_tma_load_2d(mo_dsm + " << staged[i].second.first << " + slot_ * " << boxbytes[i] << ", &T.m[" << i
         << "], cs * " << slots[i].second << ", r_, MB + slot_);\n";
    is << "}\n";
    auto issue = [&](const std::string& j) {
      std::string t = is.str();
      for (size_t p = t.find("JJ"); p != std::string::npos; p = t.find("JJ", p)) t.replace(p, 2, j);
      return t;
    };
    os << "extern \"C\" __global__ void __launch_bounds__(" << 32 * NW << (minb > 0 ? ", " + std::to_string(minb) : "")
       << ") " << kn << "(const __grid_constant__ mo_kparams P, const __grid_constant__ mo_tmaps T) {\n"
       << "  MO_PDL_ENTRY();\n"
       << "  if ((P.flags & MO_F_SKIPDONE) && P.state->done) return;\n"
       << "  unsigned long long* MB = reinterpret_cast<unsigned long long*>(mo_dsm + " << mbar_off << ");\n"
       << "  unsigned* CNT = reinterpret_cast<unsigned*>(mo_dsm + " << cnt_off << ");\n"
       << "  double acc = 0;\n"
       << "  unsigned em = 0;\n"
       << "  const int tid = threadIdx.x + threadIdx.y * blockDim.x;\n"
       << "  const int w = tid >> 5, l = tid & 31;\n"
       << "  constexpr int NW = " << NW << ", BW = " << BW << ", H = " << H << ", RX = " << RX << ", R = " << R
       << ", NBUF = " << NBUF << ";\n"
       << "  constexpr int D0 = " << D0 << ", D1 = " << D1 << ", NBG = " << (D1 + NW * BW - 1) / (NW * BW) << ";\n"
       << "  if (tid == 0) {\n"
       << "    for (int i = 0; i < NBUF; ++i) { mo_mbar_init(MB + i, 1); CNT[i] = 0u; }\n"
       << "    mo_mbar_fence_init();\n"
       << "  }\n"
       << "  __syncthreads();\n"
       << "  Real* const OUT = (Real*)P.out0; const Real* const DAMP = (const Real*)P.in1; (void)DAMP;\n"
       << "  const int fl = P.flags;\n"
       << "  const int CH = P.chunk;\n"
       << "  const int nch = (P.row1 - P.row0 + CH - 1) / CH;\n"
       << "  const int items = NBG * nch;\n"
       << "  int slot0 = 0;    // ring slot of the item's input block 0\n"
       << "  unsigned ph = 0;  // per-slot mbarrier parity\n"
       << "  for (int t = blockIdx.x; t < items; t += gridDim.x) {\n"
       << "    const int ci = t / NBG, c0 = (t - ci * NBG) * (NW * BW);\n"
       << "    const int y0 = P.row0 + ci * CH, y1 = min(y0 + CH, P.row1);\n"
       << "    const bool it = y0 - H - RX >= 0 && y1 + H - 1 + RX < D0 && c0 - H - RX >= 0 && c0 + NW * BW + H - 1 + RX < D1;\n"
       << "    const int sh = (c0 - H - RX) & " << AU - 1 << ", cs = c0 - H - RX - sh;\n"
       << "    const int nrows = y1 - y0 + 2 * H;              // phase-1 rows\n"
       << "    const int nblk = (nrows + 2 * RX + R - 1) / R;  // input blocks\n"
       << "    if (tid == 0) {\n"
       << "      mo_fence_proxy_async();\n"
       << "      for (int j = 0; j < NBUF && j < nblk; ++j) " << issue("j")
       << "    }\n"
       << "    const int q1 = c0 + w * BW - H + l;\n"
       << "    const int lx = w * BW + l + RX + sh;  // window column of this lane's element\n"
       << "    const bool lane_out = l >= H && l < 32 - H && q1 < D1;\n";
    for (int k = 0; k < K; ++k)
      for (int a = 0; a < NA; ++a) os << "    Real A" << k << "_" << a << " = (Real)0;\n";
    os << "    int sb = slot0;  // ring slot of input row k (one row per block)\n"
       << "    int e = (y0 - 2 * H - P.row_lo) * D1 + q1;  // element of output row y0 - 2H + k\n"
       << "    for (int k = 0; k < nrows; ++k, e += D1) {\n"
       << "      // newest input row this phase-1 row needs: k + 2RX (each waited once)\n"
       << "      if (k == 0) {\n"
       << "        for (int j = 0; j <= 2 * RX && j < nblk; ++j) {\n"
       << "          const int q = (sb + j) & (NBUF - 1);\n"
       << "          mo_mbar_wait(MB + q, (ph >> q) & 1u); ph ^= 1u << q;\n"
       << "        }\n"
       << "      } else if (k + 2 * RX < nblk) {\n"
       << "        const int q = (sb + 2 * RX) & (NBUF - 1);\n"
       << "        mo_mbar_wait(MB + q, (ph >> q) & 1u); ph ^= 1u << q;\n"
       << "      }\n"
       << "      int ri[" << 2 * RX + 1 << "];\n"
       << "      #pragma unroll\n"
       << "      for (int o = 0; o < " << 2 * RX + 1 << "; ++o) ri[o] = (sb + o) & (NBUF - 1);\n"
       << "      const int q0 = y0 - H + k;\n"
       << "      Real c[" << NM << "];\n"
       << "      if (it) mo_lanes5_" << sfx << "<true>(P, q0, q1, ri, lx, c); else mo_lanes5_" << sfx
       << "<false>(P, q0, q1, ri, lx, c);\n";
    // route contributions: value from lane l - o1, into accumulator of row q0 + o0 (slot H + o0)
    for (int si = 0; si < NM; ++si) {
      const MLane& m = merged[size_t(si)];
      int kk = -1;
      for (int k = 0; k < K; ++k)
        if (g.chans[size_t(k)].first == m.f && g.chans[size_t(k)].second == m.c) kk = k;
      if (kk < 0) continue;
      std::string v = "c[" + std::to_string(si) + "]";
      if (m.o1 > 0) v = "__shfl_up_sync(0xffffffffu, " + v + ", " + std::to_string(m.o1) + ")";
      if (m.o1 < 0) v = "__shfl_down_sync(0xffffffffu, " + v + ", " + std::to_string(-m.o1) + ")";
      os << "      A" << kk << "_" << H + m.o0 << " += " << v << ";\n";
    }
    // output row q0 - H is complete
    os << "      const int y = q0 - H;\n"
       << "      if (k >= 2 * H && y < y1 && lane_out) {\n"
       << "        const bool ex = P.mask && P.mask[e];\n"
       << "        const int rp = (sb + RX - H) & (NBUF - 1);  // staged p of the output pixel: input row k - H + RX\n"
       << "        Real pa = (Real)0;  // this pixel's p'Ap terms (products in Real, as pcg.hpp:43)\n";
    {
      std::vector<int> fields;
      for (auto& fc : g.chans)
        if (std::find(fields.begin(), fields.end(), fc.first) == fields.end()) fields.push_back(fc.first);
      for (int f : fields) {
        const int C = P.unknowns[size_t(f)].channels;
        os << "        const int cb" << f << " = (int)P.ubase[" << f << "] + e * " << C << ";\n"
           << "        Real* const o" << f << " = OUT + cb" << f << ";\n";
      }
      for (int k = 0; k < K; ++k) {
        const int f = g.chans[size_t(k)].first, ch = g.chans[size_t(k)].second;
        const int C = P.unknowns[size_t(f)].channels;
        const auto* st = staged_of(U + f);
        os << "        { Real v = ex ? (Real)0 : (Real)2 * A" << k << "_0;\n"
           << "          em = max(em, MO_EXP_BITS(v));\n"
           << "          const Real pc = reinterpret_cast<const Real*>(mo_dsm + " << st->first << ")[rp * " << WIN * C
           << " + lx * " << C << " + " << ch << "];\n"
           << "          if (fl & MO_F_DAMP) v = v + DAMP[cb" << f << " + " << ch << "] * pc;\n"
           << "          if ((fl & MO_F_ZEROEXCL) && ex) v = (Real)0;\n"
           << "          o" << f << "[" << ch << "] = v;\n"
           << "          pa += pc * v; }\n";
      }
      os << "        if (fl & MO_F_REDUCE) acc += (double)pa;\n";
    }
    os << "      }\n";
    for (int k = 0; k < K; ++k) {
      for (int a = 0; a + 1 < NA; ++a) os << "      A" << k << "_" << a << " = A" << k << "_" << a + 1 << ";\n";
      os << "      A" << k << "_" << NA - 1 << " = (Real)0;\n";
    }
    os << "      // release input row k (and every remaining row after the last one)\n"
       << "      const int jhi = k + 1 == nrows ? nblk - 1 : k;\n"
       << "      __syncwarp();\n"
       << "      if (l == 0) {\n"
       << "        __threadfence_block();\n"
       << "        for (int j = k; j <= jhi; ++j) {\n"
       << "          const int q = (slot0 + j) & (NBUF - 1);\n"
       << "          if (atomicAdd(CNT + q, 1u) == NW - 1) {\n"
       << "            CNT[q] = 0u;\n"
       << "            if (j + NBUF < nblk) {\n"
       << "              mo_fence_proxy_async();\n"
       << "              " << issue("j + NBUF")
       << "            }\n"
       << "          }\n"
       << "        }\n"
       << "      }\n"
       << "      sb = (sb + 1) & (NBUF - 1);\n"
       << "    }\n"
       << "    __syncthreads();  // every warp is done with this item's ring slots\n"
       << "    slot0 = (slot0 + nblk) & (NBUF - 1);\n"
       << "  }\n"
       << "  if (em == MO_EXP_MASK) atomicOr(&P.state->nonfinite_kernel, 1);\n"
       << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n}\n";
    ModuleInfo::Tma ti;
    ti.ok = true;
    ti.smem = size_t(off);
    ti.halo = H;
    ti.band = NW * BW;
    ti.rx = RX;
    ti.win = WIN;
    ti.rows = R;
    ti.threads = 32 * NW;
    for (auto& x : slots) ti.slots.push_back({x.first, x.second});
    tma5_info = ti;
    staged.clear();
  }
  ModuleInfo::Tma tma5_info;

  // Warp-specialised streaming apply / build_normal (2-D domains),
  // mo_gather_jtj8_<gi> / mo_gather_bm8_<gi>.  gather_jtj5's dataflow (every
  // lane evaluates evalj of its element once per phase-1 row, routes the NM
  // merged-lane contributions through warp shuffles (column offset) into
  // 2H+1 rolling register accumulators (row offset), and writes output row
  // q0 - H as soon as it is complete) with a producer/consumer pipeline:
  //  * warps 0..NW-1 are consumers, each walking its own band of BW output
  //    columns down the chunk; warp NW is the producer, whose lane 0 streams
  //    R-row input blocks of every staged field into an NBUF-slot ring by TMA;
  //  * FULL[s] (TMA transaction bytes) and EMPTY[s] (one arrival per consumer
  //    warp) mbarriers per slot: consumers never meet at a block barrier and
  //    never issue copies, the producer runs ahead across work items, so the
  //    next item's first rows are in flight while the current one drains;
  //  * the ring is a power of two rows deep, so a row's slot is one mask;
  //  * the output pixel's exclusion mask is loaded two rows ahead (loaded in
  //    the row itself, its use stalled every consumer warp: 27% of the stall
  //    samples of jtj9t at 8192^2) and 2- / 4-channel outputs are
  //    stored as one vector per pixel.
  // Sums are formed per output pixel in row-arrival order (tolerance parity
  // with the other fast variants, deterministic run to run).  bm = true:
  // build_normal (solver.hpp:220-251) on the same schedule: phase 1 adds
  // evalf, forms d_l r_t and d_l^2 per merged lane, two accumulator sets,
  // and the epilogue applies the identity patch, unconstrained count and the
  // fused PCG start exactly as mo_gather_bm4.
  // Lane cache of a gather set (see LaneSplit): planes [NV varying lanes |
  // guard bits] over the domain extended by H on every side (the phase-1
  // elements of the border items), element (y, x) at (y + H) * PW + x + HX,
  // HX = H rounded up to 16 bytes so TMA windows of the planes stay aligned.
  // mo_lanecache_<gi> writes it once per linearisation (full evalj, global
  // loads); mo_gather_jtj9_<gi> is gather_jtj8 with phase 1 fed from it.
  struct LcInfo {
    bool ok = false;
    int nv = 0, H = 0, HX = 0, PW = 0, rows = 0, slot0 = 0;
  } lc_info;
  LaneSplit lc_split;
  void lane_cache(const GatherSet& g, int gi, const GridSet& S, int H) {
    lc_info = LcInfo{};
    if (std::getenv("MO_B200_NO_LANECACHE") || f64_disabled_tma()) return;
    if (g.dom.dims.size() != 2) return;
    lc_split = split_lanes(S.evalj);
    if (std::getenv("MO_B200_LC_LOG"))
      fprintf(stderr, "[mo lanecache] gather set %d: %zu lanes, %zu varying, %d guard bits%s\n", gi,
              S.evalj.outputs.size(), lc_split.varying.size(), lc_split.nbits, lc_split.ok ? "" : " (too many: off)");
    if (!lc_split.ok) return;
    const int U = int(P.unknowns.size()), A = int(P.arrays.size());
    const int slot0 = 2 * U + A + int(P.computed.size());
    const int nv = int(lc_split.varying.size());
    // (the apply reads the planes straight from global memory: no view or
    // tensor-map slot per plane, so the lane count is not bounded by them;
    // past 48 varying lanes the cache costs more than the evalj it saves)
    if (nv > 48) return;
    const auto sh = P.shape_of(g.dom);
    const int AU = f64 ? 2 : 4;
    LcInfo li;
    li.nv = nv;
    li.H = H;
    li.HX = (H + AU - 1) / AU * AU;
    li.PW = int((sh[1] + li.HX + H + AU - 1) / AU * AU);
    li.rows = int(sh[0] + 2 * H);
    li.slot0 = slot0;
    const std::string sfx = std::to_string(gi);
    cur_split = &lc_split;
    split_mode = 1;
    const std::string pw = program(S.evalj, false, &g.dom);
    split_mode = 0;
    cur_split = nullptr;
    const int NO = int(S.evalj.outputs.size());
    const int R = reach_of(S.evalj, &g.dom);
    os << "extern \"C\" __global__ void __launch_bounds__(MO_THREADS) mo_lanecache_" << sfx
       << "(const __grid_constant__ mo_kparams P) {\n"
       << "  MO_PDL_ENTRY();\n"
       << "  constexpr int H = " << H << ", HX = " << li.HX << ", PW = " << li.PW << ", D0 = " << sh[0] << ", D1 = "
       << sh[1] << ", RR = " << R << ";\n"
       << "  constexpr long long S = (long long)PW * (D0 + 2 * H);  // plane stride\n"
       << "  constexpr long long N = (long long)(D0 + 2 * H) * (D1 + 2 * H);\n"
       << "  Real* const CC = (Real*)P.out0;\n"
       << "  bool bad = false;\n"
       << "  for (long long i = blockIdx.x * (long long)MO_THREADS + threadIdx.x + threadIdx.y * blockDim.x; i < N;\n"
       << "       i += (long long)gridDim.x * MO_THREADS) {\n"
       << "    const int y = int(i / (D1 + 2 * H)) - H, x = int(i % (D1 + 2 * H)) - H;\n"
       << "    const bool it = y >= RR && y < D0 - RR && x >= RR && x < D1 - RR;\n"
       << "    Real d[" << std::max(NO, 1) << "];\n"
       << "    unsigned bits = 0u;\n"
       << "    if (it) " << pw << "<true>(P, y, x, 0, y * D1 + x, nullptr, d, &bits); else " << pw
       << "<false>(P, y, x, 0, 0, nullptr, d, &bits);\n"
       << "    const long long c = (long long)(y + H) * PW + (x + HX);\n";
    for (int j = 0; j < nv; ++j)
      os << "    CC[" << j << " * S + c] = d[" << lc_split.varying[size_t(j)] << "];\n";
    os << "    CC[" << nv << " * S + c] = " << (f64 ? "__longlong_as_double((long long)bits)" : "__uint_as_float(bits)")
       << ";\n";
    os << "  }\n  (void)bad;\n}\n";
    li.ok = true;
    lc_info = li;
  }

  void gather_jtj8(const GatherSet& g, int gi, const GridSet& S, const std::vector<LaneG>& lanes,
                   const std::vector<int>& lane_slot, const std::vector<MLane>& merged, int H, int mode) {
    const bool bm = mode == 1 || mode == 3, cached = mode == 2 || mode == 4, lcw = mode == 3;
    if (f64_disabled_tma()) return;
    if (bm && S.evalf.outputs.size() != S.jtemplates.size()) return;
    auto envi = [](const char* n, int d) { const char* v = std::getenv(n); return v ? std::atoi(v) : d; };
    const std::string sfx = std::to_string(gi);
    const auto sh = P.shape_of(g.dom);
    const long long D0 = sh[0], D1 = sh[1];
    const int BW = 32 - 2 * H;
    if (BW < 8) return;
    const int U = int(P.unknowns.size());
    const int RX = cached ? H : std::max(std::max(reach_of(S.evalj, &g.dom), bm ? reach_of(S.evalf, &g.dom) : 0), H);
    const int AU = f64 ? 2 : 4;
    const int RB = f64 ? 8 : 4;
    // Lane cache staged by the producer warp too (MO_B200_JTJ9_TMA=1): its
    // planes ride the TMA ring (one-row boxes, NBUF deep) instead of the
    // consumers' row-ahead global loads.
    const bool lc_tma = mode == 4;
    int R = 1;
    while (R < envi("MO_B200_JTJ8_R", 2)) R *= 2;  // rows per TMA box (power of two)
    int NBUF = 1;
    // No deadlock: the block a consumer releases last must not wait for a
    // slot it still holds: NBUF >= 2 + ceil(2RX / R).
    while (NBUF < std::max(envi("MO_B200_JTJ8_NBUF", 4), 2 + (2 * RX + R - 1) / R)) NBUF *= 2;
    const int NR = NBUF * R;
    const int NM = int(merged.size());
    std::vector<std::pair<int, int>> slots;  // (slot, channels)
    auto add = [&](int sl, int C) {
      for (auto& x : slots)
        if (x.first == sl) return;
      slots.push_back({sl, C});
    };
    auto add_prog = [&](const Program& pg) {
      for (const Instr& in : pg.instrs) {
        if (!(in.op == kLoadU || in.op == kLoadA || in.op == kLoadC || in.op == kLoadP) || in.graph) continue;
        const Field& f = field_of(in.op, in.field);
        if (f.dom == g.dom) add(slot_of(in.op, in.field), f.channels);
      }
    };
    if (!cached) add_prog(S.evalj);
    if (bm) add_prog(S.evalf);
    else {
      for (const LaneG& l : lanes) add(U + l.f, P.unknowns[size_t(l.f)].channels);
      for (auto& fc : g.chans) add(U + fc.first, P.unknowns[size_t(fc.first)].channels);
    }
    if (lc_tma)
      for (int j = 0; j <= lc_info.nv; ++j) add(lc_info.slot0 + j, 1);
    if (slots.empty() || int(slots.size()) > MO_MAX_TMAPS_HOST) return;
    int cmax = 1;
    for (auto& x : slots) cmax = std::max(cmax, x.second);
    // Widest block whose window fits one TMA box row (<= 256 elements); the
    // window unit keeps 16-byte aligned box starts and 128-byte slots.
    const int WU = std::max(AU, 128 / (R * RB));
    int NW = 0, WIN = 0;
    for (int nw = std::min(4, std::max(1, envi("MO_B200_JTJ8_NW", 4))); nw >= 1; --nw) {
      const int win = (nw * BW + 2 * H + 2 * RX + AU - 1 + WU - 1) / WU * WU;
      if (win * cmax <= 256) {
        NW = nw;
        WIN = win;
        break;
      }
    }
    if (!NW) return;
    long long off = 0;
    staged.clear();
    long long tx = 0;
    std::vector<long long> boxbytes;
    for (auto& x : slots) {
      staged.push_back({x.first, {off, x.second}});
      const long long bb = (long long)R * WIN * x.second * RB;
      boxbytes.push_back(bb);
      tx += bb;
      off += (long long)NBUF * bb;
    }
    const long long mbar_off = off;
    off += 16LL * NBUF;
    st_rx = RX;
    st_win = WIN;
    if (cached || lcw) {
      cur_split = &lc_split;
      split_mode = cached ? 2 : 1;
    }
    const std::string pe = program(S.evalj, false, &g.dom, true);
    split_mode = 0;
    cur_split = nullptr;
    sm_mode = true;  // (smx below reads the staged rings)
    const std::string pf = bm ? program(S.evalf, false, &g.dom, true) : std::string();
    const int NO = int(S.evalj.outputs.size());
    const int NT = int(S.jtemplates.size());
    const std::string LN =
        (lcw ? "mo_lanesbm8c_" : bm ? "mo_lanesbm8_" : lc_tma ? "mo_lanes9t_" : cached ? "mo_lanes9_" : "mo_lanes8_") + sfx;
    os << "template <bool I> __device__ __forceinline__ void " << LN
       << "(const mo_kparams& P, int p0, int p1, const int* ri, int lx, Real* c" << (bm ? ", Real* cm" : "")
       << (cached ? ", const Real* cv, unsigned bits" : "") << ") {\n"
       << "  const bool inside = I || mo_inb(P, p0, p1, 0); (void)inside;\n"
       << "  Real d[" << NO << "];\n";
    if (lc_tma) {
      const int nv = lc_info.nv;
      os << "  (void)cv; (void)bits;\n  Real cs_[" << std::max(nv, 1) << "];\n";
      for (int j = 0; j < nv; ++j) os << "  cs_[" << j << "] = " << smx(lc_info.slot0 + j, 0, 0, 0) << ";\n";
      const std::string bv = smx(lc_info.slot0 + nv, 0, 0, 0);
      os << "  " << pe << "(P, " << (f64 ? "(unsigned)__double_as_longlong(" + bv + ")" : "__float_as_uint(" + bv + ")")
         << ", cs_, d);\n";
    } else if (cached) {
      os << "  " << pe << "(P, bits, cv, d);\n";
    } else if (lcw) {
      // evalj once, also the lane cache of the apply (its varying lanes and
      // guard outcomes) for this phase-1 element of the extended domain;
      // elements several items evaluate are written with identical values
      os << "  unsigned bits_ = 0u;\n  " << pe << "<I>(P, p0, p1, 0, ri, lx, d, &bits_);\n"
         << "  if ((P.flags & MO_F_LCACHE) && p1 < " << sh[1] + lc_info.H << ") {\n"
         << "    Real* const CC = (Real*)P.in2 + (long long)(p0 + " << lc_info.H << ") * " << lc_info.PW << " + (p1 + "
         << lc_info.HX << ");\n"
         << "    constexpr long long LSTR = (long long)" << lc_info.PW << " * " << lc_info.rows << ";\n";
      for (int j = 0; j < lc_info.nv; ++j)
        os << "    CC[" << j << " * LSTR] = d[" << lc_split.varying[size_t(j)] << "];\n";
      os << "    CC[" << lc_info.nv << " * LSTR] = "
         << (f64 ? "__longlong_as_double((long long)bits_)" : "__uint_as_float(bits_)") << ";\n  }\n";
    } else {
      os << "  " << pe << "<I>(P, p0, p1, 0, ri, lx, d);\n";
    }
    if (bm) {
      os << "  Real fv[" << NT << "];\n  " << pf << "<I>(P, p0, p1, 0, ri, lx, fv);\n";
      for (int si = 0; si < NM; ++si) os << "  Real mb" << si << " = (Real)0, mm" << si << " = (Real)0;\n";
      for (int t = 0; t < NT; ++t) {
        const bool origin = S.jtemplates[size_t(t)].origin;
        os << "  {" << (origin ? " if (inside) {" : "") << "\n";
        for (size_t li = 0; li < lanes.size(); ++li)
          if (lanes[li].t == t)
            os << "    mb" << lane_slot[li] << " += d[" << lanes[li].out << "] * fv[" << t << "]; mm" << lane_slot[li]
               << " += d[" << lanes[li].out << "] * d[" << lanes[li].out << "];\n";
        os << "  }" << (origin ? " }" : "") << "\n";
      }
      for (int si = 0; si < NM; ++si) os << "  c[" << si << "] = mb" << si << "; cm[" << si << "] = mm" << si << ";\n";
    } else {
      for (int si = 0; si < NM; ++si) os << "  Real m" << si << " = (Real)0;\n";
      for (int t = 0; t < NT; ++t) {
        os << "  { Real jp = (Real)0;\n";
        for (const LaneG& l : lanes)
          if (l.t == t) os << "    jp += d[" << l.out << "] * " << smx(U + l.f, l.o0, l.o1, l.c) << ";\n";
        const bool origin = S.jtemplates[size_t(t)].origin;
        if (origin) os << "    if (inside) {\n";
        for (size_t li = 0; li < lanes.size(); ++li)
          if (lanes[li].t == t) os << "    m" << lane_slot[li] << " += d[" << lanes[li].out << "] * jp;\n";
        if (origin) os << "    }\n";
        os << "  }\n";
      }
      for (int si = 0; si < NM; ++si) os << "  c[" << si << "] = m" << si << ";\n";
    }
    os << "}\n";
    sm_mode = false;

    const int K = int(g.chans.size());
    const int NA = 2 * H + 1;
    const std::string kn = (lcw      ? "mo_gather_bm8c_"
                            : bm     ? "mo_gather_bm8_"
                            : lc_tma ? "mo_gather_jtj9t_"
                            : cached ? "mo_gather_jtj9_"
                                     : "mo_gather_jtj8_") +
                           sfx;
    // resident blocks the register allocator must allow (0: unconstrained);
    // the lane-cache applies gain from 6 (jtj9, ARAP 8192^2: 966 vs 976 us)
    // and 4 (jtj9t with 2-row boxes: 751 vs 766 us; 1-row boxes 854 us)
    const int minb = envi(bm ? "MO_B200_BM8_MINB" : cached ? "MO_B200_JTJ9_MINB" : "MO_B200_JTJ8_MINB",
                          lc_tma ? 4 : cached ? 6 : 0);
    std::ostringstream is;  // TMA issue of input block j (inline: tensor maps in param space)
    is << "{ const int s_ = gb & (NBUF - 1);\n"
       << "          if (gb >= NBUF) mo_mbar_wait(EMPTY + s_, ((gb >> LNB) - 1) & 1);\n"
       << "          mo_fence_proxy_async();\n"
       << "          mo_mbar_expect_tx(FULL + s_, " << tx << "u);\n"
       << "          const int r_ = y0 - H - RX + R * j - P.row_lo;\n";
    // Lane-cache planes read with an L2 evict_first hint where the PCG's
    // working set could otherwise stay in L2 (cache <= 48 MB: ARAP 1024^2
    // 1.028 -> 1.001 ms per GN iteration); on HBM-sized grids the hint
    // costs the apply 2% (8192^2: 769 vs 751 us).  MO_B200_LC_EVICT=0/1.
    const double lc_bytes = lc_tma ? double(lc_info.nv + 1) * lc_info.PW * lc_info.rows * (f64 ? 8 : 4) : 0.0;
    const bool evict = envi("MO_B200_LC_EVICT", lc_bytes <= 48e6 ? 1 : 0) != 0;
    for (size_t i = 0; i < slots.size(); ++i) {
      const bool cp = cached && slots[i].first >= lc_info.slot0;  // lane-cache plane: extended-domain coordinates
      is << "          mo_tma_load_2d" << (cp && evict ? "_hint" : "") << "(mo_dsm + " << staged[i].second.first
         << " + s_ * " << boxbytes[i] << ", &T.m[" << i << "], "
         << (cp ? "cs + " + std::to_string(lc_info.HX) : "cs * " + std::to_string(slots[i].second)) << ", r_"
         << (cp ? " + P.row_lo + " + std::to_string(lc_info.H) : std::string()) << ", FULL + s_"
         << (cp && evict ? ", pol" : "") << ");\n";
    }
    is << "        }\n";
    int LNB = 0;
    while ((1 << LNB) < NBUF) ++LNB;
    int LR = 0;
    while ((1 << LR) < R) ++LR;
    os << "extern \"C\" __global__ void __launch_bounds__(" << 32 * (NW + 1) << (minb > 0 ? ", " + std::to_string(minb) : "")
       << ") " << kn << "(const __grid_constant__ mo_kparams P, const __grid_constant__ mo_tmaps T) {\n"
       << "  MO_PDL_ENTRY();\n"
       << "  if ((P.flags & MO_F_SKIPDONE) && P.state->done) return;\n";
    if (bm)
      os << "  if ((P.flags & MO_F_PCGINIT) && blockIdx.x == 0 && threadIdx.x == 0) {\n"
         << "    P.state->done = 0; P.state->iters = 0; P.state->indefinite = 0; P.state->nonfinite = 0; P.state->stop_code = 0x7fffffff;\n"
         << "  }\n";
    os << "  unsigned long long* const FULL = reinterpret_cast<unsigned long long*>(mo_dsm + " << mbar_off << ");\n"
       << "  unsigned long long* const EMPTY = FULL + " << NBUF << ";\n"
       << "  double acc = 0, cnt = 0, rz = 0; (void)cnt; (void)rz;\n"
       << "  unsigned em = 0;  // max exponent field of the outputs: all ones <=> a non-finite output\n"
       << "  const int tid = threadIdx.x;\n"
       << "  const int w = tid >> 5, l = tid & 31;\n"
       << "  constexpr int NW = " << NW << ", BW = " << BW << ", H = " << H << ", RX = " << RX << ", R = " << R
       << ", LR = " << LR << ", NBUF = " << NBUF << ", LNB = " << LNB << ", NR = " << NR << ";\n"
       << "  constexpr int D0 = " << D0 << ", D1 = " << D1 << ", NBG = " << (D1 + NW * BW - 1) / (NW * BW) << ";\n"
       << "  (void)D0; (void)LR;\n"
       << "  if (tid == 0) {\n"
       << "    for (int i = 0; i < NBUF; ++i) { mo_mbar_init(FULL + i, 1); mo_mbar_init(EMPTY + i, NW); }\n"
       << "    mo_mbar_fence_init();\n"
       << "  }\n"
       << "  __syncthreads();\n"
       << "  const int CH = P.chunk;\n"
       << "  const int nch = (P.row1 - P.row0 + CH - 1) / CH;\n"
       << "  const int items = NBG * nch;\n"
       << "  if (w == NW) {  // producer warp: lane 0 streams every item's input blocks\n"
       << "    if (l == 0) {\n"
       << "      int gb = 0;  // global input-block counter (slot gb % NBUF, use gb / NBUF)\n"
       << (lc_tma && evict ? "      const unsigned long long pol = mo_l2_evict_first();\n" : "")
       << "      for (int t = blockIdx.x; t < items; t += gridDim.x) {\n"
       << "        const int ci = t / NBG, c0 = (t - ci * NBG) * (NW * BW);\n"
       << "        const int y0 = P.row0 + ci * CH, y1 = min(y0 + CH, P.row1);\n"
       << "        const int cs = (c0 - H - RX) - ((c0 - H - RX) & " << AU - 1 << ");\n"
       << "        const int nblk = (y1 - y0 + 2 * H + 2 * RX + R - 1) >> LR;\n"
       << "        for (int j = 0; j < nblk; ++j, ++gb) " << is.str()
       << "      }\n"
       << "    }\n"
       << "    __syncwarp();\n"
       << "  } else {\n"
       << "    const int fl = P.flags; (void)fl;\n";
    if (bm)
      os << "    Real* const B = (Real*)P.out0; Real* const M = (Real*)P.out1;\n"
         << "    Real* const PP = (Real*)P.out2; Real* const DL = (Real*)P.out3; Real* const RR = (Real*)P.out4;\n"
         << "    const int pre = P.state->use_precond;\n";
    else
      os << "    Real* const OUT = (Real*)P.out0; const Real* const DAMP = (const Real*)P.in1; (void)DAMP;\n"
         << "    const bool vec_ok = (reinterpret_cast<unsigned long long>(OUT) & 15) == 0; (void)vec_ok;\n";
    os << "    int gb = 0;  // global index of the item's input block 0\n"
       << "    for (int t = blockIdx.x; t < items; t += gridDim.x) {\n"
       << "      const int ci = t / NBG, c0 = (t - ci * NBG) * (NW * BW);\n"
       << "      const int y0 = P.row0 + ci * CH, y1 = min(y0 + CH, P.row1);\n"
       << "      const bool it = y0 - H - RX >= 0 && y1 + H - 1 + RX < D0 && c0 - H - RX >= 0 && c0 + NW * BW + H - 1 + RX < D1;\n"
       << "      const int sh = (c0 - H - RX) & " << AU - 1 << ";\n"
       << "      const int nrows = y1 - y0 + 2 * H;  // phase-1 rows\n"
       << "      const int nblk = (nrows + 2 * RX + R - 1) >> LR;\n"
       << "      const int rb = (gb << LR) & (NR - 1);  // ring row of the item's input row 0\n"
       << "      const int q1 = c0 + w * BW - H + l;\n"
       << "      const int lx = w * BW + l + RX + sh;  // window column of this lane's element\n"
       << "      const bool lane_out = l >= H && l < 32 - H && q1 < D1;\n"
       << "      int nwt = 0;  // input blocks of this item waited so far\n";
    for (int k = 0; k < K; ++k)
      for (int a = 0; a < NA; ++a) {
        os << "      Real A" << k << "_" << a << " = (Real)0;\n";
        if (bm) os << "      Real Q" << k << "_" << a << " = (Real)0;\n";
      }
    // Mask two rows ahead: jtj9t 884 -> 854 us and bm8c 2144 -> 1882 us on
    // ARAP 8192^2; the direct-load lane-cache apply of SFS (26 cached lanes,
    // register-bound) loses 10% with it, so jtj8 / bm8 / jtj9 keep the
    // in-row load.  MO_B200_MASK_PF=0/1 forces either.
    const bool mask_pf = envi("MO_B200_MASK_PF", mode == 3 || mode == 4 ? 1 : 0) != 0;
    os << "      int e = (y0 - 2 * H - P.row_lo) * D1 + q1;  // element of output row y0 - 2H + k\n";
    if (mask_pf)
      os << "      // exclusion mask of phase-1 row k's output pixel, loaded two rows ahead\n"
         << "      const unsigned char* const MK = P.mask;\n"
         << "      const int e0 = e;\n"
         << "      auto mrow = [&](int kk) -> unsigned {\n"
         << "        return (MK && kk >= 2 * H && kk < nrows && lane_out) ? (unsigned)MK[e0 + kk * D1] : 0u;\n"
         << "      };\n"
         << "      unsigned mq0 = mrow(0), mq1 = mrow(1);\n";
    const int NVC = cached ? lc_info.nv + 1 : 0;
    if (lc_tma) {
      os << "      for (int k = 0; k < nrows; ++k, e += D1) {\n"
         << "        const Real* const cc = nullptr; const unsigned cbits = 0u;\n";
    } else if (cached) {
      // Lane cache of this lane's phase-1 element, read straight from global
      // memory (coalesced along the row, never a halo), PF rows ahead.
      // PF rows in flight per lane (MO_B200_JTJ9_PF; measured on ARAP
      // 8192^2: 1 row 976 us, 2 rows 1165 us, 3 rows 1127 us: the extra
      // registers cost more resident warps than the deeper prefetch gains).
      const int PF = std::max(1, std::min(4, envi("MO_B200_JTJ9_PF", 1)));
      os << "      constexpr long long LSTR = (long long)" << lc_info.PW << " * " << lc_info.rows << ";\n"
         << "      const Real* __restrict__ cp = (const Real*)P.in2 + (long long)y0 * " << lc_info.PW
         << " + min(q1, D1 + H - 1) + " << lc_info.HX << ";  // row q0 + H of phase-1 row k = 0\n"
         << "      Real cn[" << PF << "][" << NVC << "];\n"
         << "      #pragma unroll\n"
         << "      for (int a = 0; a < " << PF << "; ++a) {\n"
         << "        #pragma unroll\n"
         << "        for (int j = 0; j < " << NVC << "; ++j) cn[a][j] = a < nrows ? __ldg(cp + a * " << lc_info.PW
         << " + j * LSTR) : (Real)0;\n"
         << "      }\n"
         << "      cp += " << PF << " * " << lc_info.PW << ";\n";
      os << "      for (int k = 0; k < nrows; ++k, e += D1) {\n"
         << "        Real cc[" << NVC << "];\n"
         << "        #pragma unroll\n"
         << "        for (int j = 0; j < " << NVC << "; ++j) cc[j] = cn[0][j];\n"
         << "        #pragma unroll\n"
         << "        for (int a = 0; a + 1 < " << PF << "; ++a) {\n"
         << "          #pragma unroll\n"
         << "          for (int j = 0; j < " << NVC << "; ++j) cn[a][j] = cn[a + 1][j];\n"
         << "        }\n"
         << "        if (k + " << PF << " < nrows) {\n"
         << "          #pragma unroll\n"
         << "          for (int j = 0; j < " << NVC << "; ++j) cn[" << PF - 1 << "][j] = __ldg(cp + j * LSTR);\n"
         << "          cp += " << lc_info.PW << ";\n"
         << "        }\n"
         << "        const unsigned cbits = " << (f64 ? "(unsigned)__double_as_longlong(cc[" : "__float_as_uint(cc[")
         << NVC - 1 << "]);\n";
    } else {
      os << "      for (int k = 0; k < nrows; ++k, e += D1) {\n";
    }
    os << "        const int need = min(nblk - 1, (k + 2 * RX) >> LR);\n"
       << "        while (nwt <= need) {\n"
       << "          const int b = gb + nwt;\n"
       << "          mo_mbar_wait(FULL + (b & (NBUF - 1)), (b >> LNB) & 1);\n"
       << "          ++nwt;\n"
       << "        }\n"
       << "        const int q0 = y0 - H + k;\n"
       << "        const int y = q0 - H;\n"
       << "        const bool orow = k >= 2 * H && y < y1 && lane_out;\n"
       << (mask_pf ? "        const bool ex = orow && mq0 != 0u;\n        mq0 = mq1;\n        mq1 = mrow(k + 2);\n"
                   : "        const bool ex = orow && P.mask && P.mask[e];\n")
       << "        int ri[" << 2 * RX + 1 << "];\n"
       << "        #pragma unroll\n"
       << "        for (int o = 0; o < " << 2 * RX + 1 << "; ++o) ri[o] = (rb + k + o) & (NR - 1);\n"
       << "        Real c[" << NM << "];\n";
    if (bm)
      os << "        Real cm[" << NM << "];\n"
         << "        if (it) " << LN << "<true>(P, q0, q1, ri, lx, c, cm); else " << LN << "<false>(P, q0, q1, ri, lx, c, cm);\n";
    else if (cached)
      os << "        if (it) " << LN << "<true>(P, q0, q1, ri, lx, c, cc, cbits); else " << LN
         << "<false>(P, q0, q1, ri, lx, c, cc, cbits);\n";
    else
      os << "        if (it) " << LN << "<true>(P, q0, q1, ri, lx, c); else " << LN << "<false>(P, q0, q1, ri, lx, c);\n";
    for (int si = 0; si < NM; ++si) {
      const MLane& m = merged[size_t(si)];
      int kk = -1;
      for (int k = 0; k < K; ++k)
        if (g.chans[size_t(k)].first == m.f && g.chans[size_t(k)].second == m.c) kk = k;
      if (kk < 0) continue;
      auto route = [&](const std::string& acc, const std::string& arr) {
        std::string v = arr + "[" + std::to_string(si) + "]";
        if (m.o1 > 0) v = "__shfl_up_sync(0xffffffffu, " + v + ", " + std::to_string(m.o1) + ")";
        if (m.o1 < 0) v = "__shfl_down_sync(0xffffffffu, " + v + ", " + std::to_string(-m.o1) + ")";
        os << "        " << acc << kk << "_" << H + m.o0 << " += " << v << ";\n";
      };
      route("A", "c");
      if (bm) route("Q", "cm");
    }
    os << "        if (orow) {\n";
    if (bm) {
      for (int k = 0; k < K; ++k) {
        const int f = g.chans[size_t(k)].first, ch = g.chans[size_t(k)].second;
        const int C = P.unknowns[size_t(f)].channels;
        os << "          { Real b = ex ? (Real)0 : (Real)-2 * A" << k << "_0, m = ex ? (Real)0 : (Real)2 * Q" << k << "_0;\n"
           << "            em = max(em, max(MO_EXP_BITS(b), MO_EXP_BITS(m)));\n"
           << "            if (fl & MO_F_PATCH) {\n"
           << "              if (ex) { b = (Real)0; m = (Real)1; }\n"
           << "              else if (m == (Real)0) { m = (Real)1; cnt += 1.0; }\n"
           << "            }\n"
           << "            const int col = (int)P.ubase[" << f << "] + e * " << C << " + " << ch << ";\n"
           << "            B[col] = b; M[col] = m;\n"
           << "            if (fl & MO_F_PCGINIT) {\n"
           << "              const Real zi = ex ? (Real)0 : (pre ? ((b == (Real)0 && m > (Real)0) ? b : b / m) : b);\n"
           << "              DL[col] = (Real)0; RR[col] = b; PP[col] = zi; rz += (double)(b * zi);\n"
           << "            } }\n";
      }
    } else {
      os << "          const int rp = (rb + k - H + RX) & (NR - 1);  // staged p of the output pixel\n"
         << "          Real pa = (Real)0;  // this pixel's p'Ap terms (products in Real, as pcg.hpp:43)\n";
      std::vector<int> fields;
      for (auto& fc : g.chans)
        if (std::find(fields.begin(), fields.end(), fc.first) == fields.end()) fields.push_back(fc.first);
      for (int f : fields) {
        const int C = P.unknowns[size_t(f)].channels;
        os << "          const int cb" << f << " = (int)P.ubase[" << f << "] + e * " << C << ";\n";
        std::vector<int> ks;  // this field's output channels, channel order
        for (int c = 0; c < C; ++c)
          for (int k = 0; k < K; ++k)
            if (g.chans[size_t(k)].first == f && g.chans[size_t(k)].second == c) ks.push_back(k);
        for (int k : ks) {
          const int ch = g.chans[size_t(k)].second;
          const auto* st = staged_of(U + f);
          os << "          Real v" << k << " = ex ? (Real)0 : (Real)2 * A" << k << "_0;\n"
             << "          em = max(em, MO_EXP_BITS(v" << k << "));\n"
             << "          { const Real pc = reinterpret_cast<const Real*>(mo_dsm + " << st->first << ")[rp * " << WIN * C
             << " + lx * " << C << " + " << ch << "];\n"
             << "            if (fl & MO_F_DAMP) v" << k << " = v" << k << " + DAMP[cb" << f << " + " << ch << "] * pc;\n"
             << "            if ((fl & MO_F_ZEROEXCL) && ex) v" << k << " = (Real)0;\n"
             << "            pa += pc * v" << k << "; }\n";
        }
        // one vector store per pixel when the field's channels are all outputs
        const bool whole = int(ks.size()) == C;
        const long long ub = P.ubase[size_t(f)];
        const std::string vt = f64 ? (C == 2 ? "double2" : "") : (C == 2 ? "float2" : C == 4 ? "float4" : "");
        if (whole && !vt.empty() && (ub % C) == 0) {
          os << "          if (vec_ok) *reinterpret_cast<" << vt << "*>(OUT + cb" << f << ") = make_" << vt << "(";
          for (int c = 0; c < C; ++c) os << (c ? ", " : "") << "v" << ks[size_t(c)];
          os << ");\n          else {";
          for (int c = 0; c < C; ++c) os << " OUT[cb" << f << " + " << c << "] = v" << ks[size_t(c)] << ";";
          os << " }\n";
        } else {
          for (int k : ks) os << "          OUT[cb" << f << " + " << g.chans[size_t(k)].second << "] = v" << k << ";\n";
        }
      }
      os << "          if (fl & MO_F_REDUCE) acc += (double)pa;\n";
    }
    os << "        }\n";
    for (int k = 0; k < K; ++k)
      for (const char* A : {"A", "Q"}) {
        if (*A == 'Q' && !bm) continue;
        for (int a = 0; a + 1 < NA; ++a) os << "        " << A << k << "_" << a << " = " << A << k << "_" << a + 1 << ";\n";
        os << "        " << A << k << "_" << NA - 1 << " = (Real)0;\n";
      }
    os << "        if ((k & (R - 1)) == R - 1) {  // input block k / R: its last row as a phase-1 centre row\n"
       << "          __syncwarp();\n"
       << "          if (l == 0) mo_mbar_arrive(EMPTY + ((gb + (k >> LR)) & (NBUF - 1)));\n"
       << "        }\n"
       << "      }\n"
       << "      // release the item's remaining input blocks (each waited first)\n"
       << "      for (int j = nrows >> LR; j < nblk; ++j) {\n"
       << "        while (nwt <= j) {\n"
       << "          const int b = gb + nwt;\n"
       << "          mo_mbar_wait(FULL + (b & (NBUF - 1)), (b >> LNB) & 1);\n"
       << "          ++nwt;\n"
       << "        }\n"
       << "        __syncwarp();\n"
       << "        if (l == 0) mo_mbar_arrive(EMPTY + ((gb + j) & (NBUF - 1)));\n"
       << "      }\n"
       << "      gb += nblk;\n"
       << "    }\n"
       << "  }\n"
       << "  if (em == MO_EXP_MASK) atomicOr(&P.state->nonfinite_kernel, 1);\n";
    if (bm)
      os << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, cnt, rz, (P.flags & MO_F_PCGINIT) != 0);\n}\n";
    else
      os << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n}\n";
    ModuleInfo::Tma ti;
    ti.ok = true;
    ti.smem = size_t(off);
    ti.halo = H;
    ti.band = NW * BW;
    ti.rx = RX;
    ti.win = WIN;
    ti.rows = R;
    ti.threads = 32 * (NW + 1);
    for (auto& x : slots) ti.slots.push_back({x.first, x.second});
    if (cached) {
      ti.cache_tma = lc_tma;
      ti.cache_planes = lc_info.nv + 1;
      ti.cache_slot0 = lc_info.slot0;
      ti.cache_hx = lc_info.HX;
      ti.cache_pw = lc_info.PW;
      ti.cache_rows = lc_info.rows;
    }
    (lcw ? tmabm8c_info : bm ? tmabm8_info : lc_tma ? tma9t_info : cached ? tma9_info : tma8_info) = ti;
    staged.clear();
  }
  ModuleInfo::Tma tma8_info, tmabm8_info, tma9_info, tma9t_info, tmabm8c_info;

  // TMA-staged gather program (2-D domains): the reference's own J^T J p
  // gather program (transform.hpp:238-260, run_program semantics) per output
  // pixel, with every field it reads streamed into shared-memory row rings by
  // TMA (8-row blocks, NBUF deep, mbarrier completion) instead of read through
  // L1.  For cheap stencils (Poisson) this beats the two-phase schemes: no
  // phase-1 halo, no contribution ring, one barrier per 8-row step.  Work
  // item: a band of 32 output columns (one per lane) by `chunk` rows; each of
  // the 8 warps owns one output row per step.
  void gather_jtj6(const GatherSet& g, int gi) {
    if (f64_disabled_tma()) return;
    const auto sh = P.shape_of(g.dom);
    if (g.dom.dims.size() != 2) return;
    const long long D0 = sh[0], D1 = sh[1];
    const int U = int(P.unknowns.size());
    const int RG = reach_of(g.jtj, &g.dom);
    if (RG > 4) return;
    const int AU = f64 ? 2 : 4;
    const int WIN = (32 + 2 * RG + AU - 1 + AU - 1) / AU * AU;
    // (3 to 8 ring slots measured the same on Poisson 512^2 / 8192^2: the
    // kernel is instruction-bound, not waiting on TMA.)
    const int NBUF = std::getenv("MO_B200_JTJ6_NBUF") ? std::max(3, std::atoi(std::getenv("MO_B200_JTJ6_NBUF"))) : 3;
    const int NEED = 1 + (2 * RG + 7) / 8;
    const int RB = f64 ? 8 : 4;
    std::vector<std::pair<int, int>> slots;
    auto add = [&](int sl, int C) {
      for (auto& x : slots)
        if (x.first == sl) return;
      slots.push_back({sl, C});
    };
    for (const Instr& in : g.jtj.instrs) {
      if (!(in.op == kLoadU || in.op == kLoadA || in.op == kLoadC || in.op == kLoadP) || in.graph) continue;
      const Field& f = field_of(in.op, in.field);
      if (f.dom == g.dom) add(slot_of(in.op, in.field), f.channels);
    }
    for (auto& fc : g.chans) add(U + fc.first, P.unknowns[size_t(fc.first)].channels);
    if (slots.empty() || int(slots.size()) > MO_MAX_TMAPS_HOST) return;
    for (auto& x : slots)
      if (WIN * x.second > 256) return;
    long long off = 0;
    staged.clear();
    long long tx = 0;
    std::vector<long long> boxbytes;
    for (auto& x : slots) {
      staged.push_back({x.first, {off, x.second}});
      const long long bb = 8LL * WIN * x.second * RB;
      boxbytes.push_back(bb);
      tx += bb;
      off += ((long long)NBUF * bb + 127) / 128 * 128;
    }
    const long long mbar_off = off;
    off += 8LL * NBUF;
    st_rx = RG;
    st_win = WIN;
    const std::string pn = program(g.jtj, false, &g.dom, true);
    sm_mode = false;
    const std::string sfx = std::to_string(gi);
    const std::string kn = "mo_gather_jtj6_" + sfx;
    std::ostringstream is;
    is << "{ int slot_ = slot0 + (JJ); while (slot_ >= NBUF) slot_ -= NBUF;\n"
       << "  mo_mbar_expect_tx(MB + slot_, " << tx << "u);\n"
       << "  const int r_ = y0 - RG + 8 * (JJ) - P.row_lo;\n";
    for (size_t i = 0; i < slots.size(); ++i)
      is << "  mo_tma_load_2d(mo_dsm + " << staged[i].second.first << " + slot_ * " << boxbytes[i] << ", &T.m[" << i
         << "], cs * " << slots[i].second << ", r_, MB + slot_);\n";
    is << "}\n";
    auto issue = [&](const std::string& j) {
      std::string t = is.str();
      for (size_t p = t.find("JJ"); p != std::string::npos; p = t.find("JJ", p)) t.replace(p, 2, j);
      return t;
    };
    const size_t K = g.chans.size();
    os << "extern \"C\" __global__ void __launch_bounds__(MO_THREADS) " << kn
       << "(const __grid_constant__ mo_kparams P, const __grid_constant__ mo_tmaps T) {\n"
       << "  MO_PDL_ENTRY();\n"
       << "  if ((P.flags & MO_F_SKIPDONE) && P.state->done) return;\n"
       << "  unsigned long long* MB = reinterpret_cast<unsigned long long*>(mo_dsm + " << mbar_off << ");\n"
       << "  double acc = 0;\n"
       << "  bool bad = false;\n"
       << "  const int tid = threadIdx.x + threadIdx.y * blockDim.x;\n"
       << "  const int w = tid >> 5, l = tid & 31;\n"
       << "  constexpr int RG = " << RG << ", NBUF = " << NBUF << ", NEED = " << NEED << ";\n"
       << "  constexpr int D0 = " << D0 << ", D1 = " << D1 << ", NB = " << (D1 + 31) / 32 << ";\n"
       << "  if (tid == 0) {\n"
       << "    for (int i = 0; i < NBUF; ++i) mo_mbar_init(MB + i, 1);\n"
       << "    mo_mbar_fence_init();\n"
       << "  }\n"
       << "  __syncthreads();\n"
       << "  Real* const OUT = (Real*)P.out0; const Real* const DAMP = (const Real*)P.in1; (void)DAMP;\n"
       << "  const int fl = P.flags;\n"
       << "  const int CH = P.chunk;\n"
       << "  const int nch = (P.row1 - P.row0 + CH - 1) / CH;\n"
       << "  const int items = NB * nch;\n"
       << "  int slot0 = 0;\n"
       << "  unsigned ph = 0;\n"
       << "  for (int t = blockIdx.x; t < items; t += gridDim.x) {\n"
       << "    const int ci = t / NB, c0 = (t - ci * NB) * 32;\n"
       << "    const int y0 = P.row0 + ci * CH, y1 = min(y0 + CH, P.row1);\n"
       << "    const bool it = y0 - RG >= 0 && y1 - 1 + RG < D0 && c0 - RG >= 0 && c0 + 31 + RG < D1;\n"
       << "    const int sh = (c0 - RG) & " << AU - 1 << ", cs = c0 - RG - sh;\n"
       << "    const int nsteps = (y1 - y0 + 7) >> 3;\n"
       << "    const int nblk = (y1 - y0 + 2 * RG + 7) >> 3;\n"
       << "    if (tid == 0) {\n"
       << "      mo_fence_proxy_async();\n"
       << "      for (int j = 0; j < NBUF && j < nblk; ++j) " << issue("j")
       << "    }\n"
       << "    const int q1 = c0 + l;\n"
       << "    const int lx = l + RG + sh;\n"
       << "    int ss = slot0;\n"
       << "    for (int s = 0; s < nsteps; ++s) {\n"
       << "      if (s == 0) {\n"
       << "        for (int j = 0; j < NEED - 1 && j < nblk; ++j) { int q = ss + j; while (q >= NBUF) q -= NBUF;"
          " mo_mbar_wait(MB + q, (ph >> q) & 1u); ph ^= 1u << q; }\n"
       << "      }\n"
       << "      if (s + NEED - 1 < nblk) { int q = ss + NEED - 1; while (q >= NBUF) q -= NBUF;"
          " mo_mbar_wait(MB + q, (ph >> q) & 1u); ph ^= 1u << q; }\n"
       << "      const int y = y0 + 8 * s + w;\n"
       << "      if (y < y1 && q1 < D1) {\n"
       << "        int ri[" << 2 * RG + 1 << "];\n"
       << "        #pragma unroll\n"
       << "        for (int o = 0; o < " << 2 * RG + 1 << "; ++o) {\n"
       << "          const int rel = w + o;  // input row y + o - RG, relative to block s\n"
       << "          int b = ss + (rel >> 3); if (b >= NBUF) b -= NBUF;\n"
       << "          ri[o] = b * 8 + (rel & 7);\n"
       << "        }\n"
       << "        const int e = (y - P.row_lo) * D1 + q1;\n"
       << "        const bool ex = P.mask && P.mask[e];\n"
       << "        Real o[" << (K ? K : 1) << "];\n"
       << "        if (ex) { for (int k = 0; k < " << K << "; ++k) o[k] = (Real)0; }\n"
       << "        else { if (it) " << pn << "<true>(P, y, q1, 0, ri, lx, o); else " << pn
       << "<false>(P, y, q1, 0, ri, lx, o);\n"
       << "          for (int k = 0; k < " << K << "; ++k) if (!mo_finite((double)o[k])) bad = true; }\n"
       << "        Real pa = (Real)0;\n";
    for (size_t k = 0; k < K; ++k) {
      const int f = g.chans[k].first, ch = g.chans[k].second;
      const int C = P.unknowns[size_t(f)].channels;
      const auto* st = staged_of(U + f);
      os << "        { const int col = (int)P.ubase[" << f << "] + e * " << C << " + " << ch << ";\n"
         << "          Real v = o[" << k << "];\n"
         << "          const Real pc = reinterpret_cast<const Real*>(mo_dsm + " << st->first << ")[ri[" << RG << "] * "
         << WIN * C << " + lx * " << C << " + " << ch << "];\n"
         << "          if (fl & MO_F_DAMP) v = v + DAMP[col] * pc;\n"
         << "          if ((fl & MO_F_ZEROEXCL) && P.colmask && (P.colmask[col] & 1)) v = (Real)0;\n"
         << "          OUT[col] = v;\n"
         << "          pa += pc * v; }\n";
    }
    os << "        if (fl & MO_F_REDUCE) acc += (double)pa;\n"
       << "      }\n"
       << "      __syncthreads();  // every warp is done with input block s\n"
       << "      if (tid == 0 && s + NBUF < nblk) {\n"
       << "        mo_fence_proxy_async();\n"
       << "        " << issue("s + NBUF")
       << "      }\n"
       << "      ss = ss + 1 == NBUF ? 0 : ss + 1;\n"
       << "    }\n"
       << "    slot0 = (slot0 + nblk) % NBUF;\n"
       << "  }\n"
       << "  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n"
       << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n}\n";
    ModuleInfo::Tma ti;
    ti.ok = true;
    ti.smem = size_t(off);
    ti.halo = 0;
    ti.band = 32;
    ti.rx = RG;
    ti.win = WIN;
    for (auto& x : slots) ti.slots.push_back({x.first, x.second});
    tma6_info = ti;
    staged.clear();
  }
  ModuleInfo::Tma tma6_info;

  static long long NB(long long D1, int BW) { return (D1 + BW - 1) / BW; }
  bool f64_disabled_tma() const { return std::getenv("MO_B200_NO_TMA") != nullptr; }
  ModuleInfo::Tma tma_info, tma7_info, tmabm_info;

  // Phase-2 epilogue of the TMA kernel.  Columns are 32-bit (num_cols < 2^31
  // is checked on the host).  The per-column exclusion mask of a column of a
  // field on this domain equals the element mask (k_colmask), so ZEROEXCL
  // reuses `ex` instead of re-reading colmask.
  void epilogue4(const GatherSet& g, const std::vector<MLane>& merged, int LS, const std::string& ind, int RS = 8) {
    const int LRS = RS == 8 ? 3 : 2;
    const int U = int(P.unknowns.size());
    os << ind << "Real* const OUT = (Real*)P.out0; const Real* const PV = (const Real*)P.in0; (void)PV;\n"
       << ind << "const Real* const DAMP = (const Real*)P.in1; (void)DAMP;\n"
       << ind << "const int fl = P.flags;\n"
       << ind << "// staged p of the output row (input row y = block s row w - H + RX)\n"
       << ind << "int rp = ss + ((w - H + RX) >> " << LRS << "); if (rp >= NBUF) rp -= NBUF; rp = rp * " << RS
       << " + ((w - H + RX) & " << RS - 1 << ");\n"
       << ind << "const int lx = l + RX + sh; (void)lx;\n"
       << ind << "Real pa = (Real)0;  // this pixel's p'Ap terms (products in Real, as pcg.hpp:43)\n";
    std::vector<int> fields;
    for (auto& fc : g.chans)
      if (std::find(fields.begin(), fields.end(), fc.first) == fields.end()) fields.push_back(fc.first);
    for (int f : fields) {
      const int C = P.unknowns[size_t(f)].channels;
      os << ind << "const int cb" << f << " = (int)P.ubase[" << f << "] + e * " << C << ";\n"
         << ind << "Real* const o" << f << " = OUT + cb" << f << ";\n";
    }
    for (size_t k = 0; k < g.chans.size(); ++k) {
      const int f = g.chans[k].first, ch = g.chans[k].second;
      const int C = P.unknowns[size_t(f)].channels;
      os << ind << "{ Real s = (Real)0;\n";
      for (size_t si = 0; si < merged.size(); ++si) {
        const MLane& m = merged[si];
        if (m.f != f || m.c != ch) continue;
        os << ind << "  s += CL[" << si * LS << " + sl" << (m.o0 < 0 ? "m" : "p") << std::abs(m.o0) << " - (" << m.o1
           << ")];\n";
      }
      os << ind << "  Real v = ex ? (Real)0 : (Real)2 * s;\n"
         << ind << "  em = max(em, MO_EXP_BITS(v));\n";
      if (const auto* st = staged_of(U + f))
        os << ind << "  const Real pc = reinterpret_cast<const Real*>(mo_dsm + " << st->first << ")[rp * " << st_win * C
           << " + lx * " << C << " + " << ch << "];\n";
      else
        os << ind << "  const Real pc = PV[cb" << f << " + " << ch << "];\n";
      os << ind << "  if (fl & MO_F_DAMP) v = v + DAMP[cb" << f << " + " << ch << "] * pc;\n"
         << ind << "  if ((fl & MO_F_ZEROEXCL) && ex) v = (Real)0;\n"
         << ind << "  o" << f << "[" << ch << "] = v;\n"
         << ind << "  pa += pc * v; }\n";
    }
    os << ind << "if (fl & MO_F_REDUCE) acc += (double)pa;\n";
  }

  // Phase-2 epilogue of mo_gather_bm4: b = -2 sum_s cb_s(q - o_s),
  // m = 2 sum_s cm_s(q - o_s); excluded -> b = m = 0, then the identity
  // patch / unconstrained count (solver.hpp:241-250) and the fused PCG start
  // (k_pcg_init on the patched b, m).
  void epilogue_bm4(const GatherSet& g, const std::vector<MLane>& merged, int LS, int NM, const std::string& ind,
                    int RS) {
    (void)RS;
    os << ind << "Real* const B = (Real*)P.out0; Real* const M = (Real*)P.out1;\n"
       << ind << "Real* const PP = (Real*)P.out2; Real* const DL = (Real*)P.out3; Real* const RR = (Real*)P.out4;\n"
       << ind << "const int fl = P.flags; const int pre = P.state->use_precond;\n";
    for (size_t k = 0; k < g.chans.size(); ++k) {
      const int f = g.chans[k].first, ch = g.chans[k].second;
      const int C = P.unknowns[size_t(f)].channels;
      os << ind << "{ Real sb = (Real)0, sm = (Real)0;\n";
      for (size_t si = 0; si < merged.size(); ++si) {
        const MLane& m = merged[si];
        if (m.f != f || m.c != ch) continue;
        const std::string sl = std::string("sl") + (m.o0 < 0 ? "m" : "p") + std::to_string(std::abs(m.o0));
        os << ind << "  sb += CL[" << si * LS << " + " << sl << " - (" << m.o1 << ")]; sm += CL[" << (NM + si) * LS
           << " + " << sl << " - (" << m.o1 << ")];\n";
      }
      os << ind << "  Real b = ex ? (Real)0 : (Real)-2 * sb, m = ex ? (Real)0 : (Real)2 * sm;\n"
         << ind << "  em = max(em, max(MO_EXP_BITS(b), MO_EXP_BITS(m)));\n"
         << ind << "  if (fl & MO_F_PATCH) {\n"
         << ind << "    if (ex) { b = (Real)0; m = (Real)1; }\n"
         << ind << "    else if (m == (Real)0) { m = (Real)1; cnt += 1.0; }\n"
         << ind << "  }\n"
         << ind << "  const int col = (int)P.ubase[" << f << "] + e * " << C << " + " << ch << ";\n"
         << ind << "  B[col] = b; M[col] = m;\n"
         << ind << "  if (fl & MO_F_PCGINIT) {\n"
         << ind << "    const Real zi = ex ? (Real)0 : (pre ? ((b == (Real)0 && m > (Real)0) ? b : b / m) : b);\n"
         << ind << "    DL[col] = (Real)0; RR[col] = b; PP[col] = zi; rz += (double)(b * zi);\n"
         << ind << "  } }\n";
    }
  }

  // Phase-2 gather + apply epilogue of the streaming kernels: out(f,c)(q) =
  // 2 sum_s CL[s][q - o_s], LM damping, excluded zeroing, p'Ap partial.
  void epilogue(const GatherSet& g, const std::vector<MLane>& merged, int LS, const std::string& ind) {
    for (size_t k = 0; k < g.chans.size(); ++k) {
      const int f = g.chans[k].first, ch = g.chans[k].second;
      const int C = P.unknowns[size_t(f)].channels;
      os << ind << "{ Real s = (Real)0;\n";
      for (size_t si = 0; si < merged.size(); ++si) {
        const MLane& m = merged[si];
        if (m.f != f || m.c != ch) continue;
        os << ind << "  s += CL[" << si * LS << " + sl" << (m.o0 < 0 ? "m" : "p") << std::abs(m.o0) << " - (" << m.o1
           << ")];\n";
      }
      os << ind << "  Real v = ex ? (Real)0 : (Real)2 * s;\n"
         << ind << "  if (!(v == v && (v < (Real)0 ? -v : v) <= (Real)MO_REAL_MAX)) bad = true;\n"
         << ind << "  const long long col = P.ubase[" << f << "] + e * " << C << " + " << ch << ";\n"
         << ind << "  const Real pc = PV[col];\n"
         << ind << "  if (P.flags & MO_F_DAMP) v = v + DAMP[col] * pc;\n"
         << ind << "  if ((P.flags & MO_F_ZEROEXCL) && P.colmask && P.colmask[col]) v = (Real)0;\n"
         << ind << "  OUT[col] = v;\n"
         << ind << "  if (P.flags & MO_F_REDUCE) acc += (double)(pc * v); }\n";
    }
  }

  template <class V>
  static std::vector<MLane> merged_off(const V& m) {
    std::vector<MLane> r;
    for (const auto& x : m) r.push_back({x.f, x.c, x.o0, x.o1});
    return r;
  }

  // Row-streaming two-phase apply for 2-D domains (same mathematics as
  // gather_jtj2, transform.hpp:238-260).  A work item is a band of
  // BW = 32 - 2H output columns by `P.chunk` output rows.  Each warp owns one
  // row of 32 phase-1 elements (columns c0-H .. c0-H+31) per step of 8 rows;
  // the block walks down the band and keeps the last RING = 16 + 2H phase-1
  // rows of merged-lane contributions in a shared-memory ring, so every
  // residual instance is evaluated once per item except the 2H halo rows at
  // the chunk ends and the 2H halo columns of the band (vs. the 32x8 tile's
  // 1.33x for H = 1).  One barrier per step: phase 1 of step s+1 writes ring
  // rows [8s+8, 8s+16) while lagging warps may still read [8s-2H, 8s+8).
  void gather_jtj3(const GatherSet& g, int gi, int H, int RR, int NM, const std::vector<MLane>& merged) {
    const std::string sfx = std::to_string(gi);
    const auto sh = P.shape_of(g.dom);
    const long long D0 = sh[0], D1 = sh[1];
    const int BW = 32 - 2 * H;
    if (BW < 8) return;
    const int RING = 16 + 2 * H;
    const long long NB = (D1 + BW - 1) / BW;
    const int LS = RING * 32;
    const std::string kn = "mo_gather_jtj3_" + sfx;
    const char* mb = std::getenv("MO_B200_JTJ3_MINB");
    const int minb = mb ? std::atoi(mb) : 4;
    os << "extern \"C\" __global__ void __launch_bounds__(MO_THREADS" << (minb > 0 ? ", " + std::to_string(minb) : "")
       << ") " << kn << "(const __grid_constant__ mo_kparams P) {\n"
       << "  MO_PDL_ENTRY();\n"
       << "  if ((P.flags & MO_F_SKIPDONE) && P.state->done) return;\n"
       << "  extern __shared__ __align__(16) unsigned char mo_smem[];\n"
       << "  Real* CL = reinterpret_cast<Real*>(mo_smem);  // [" << NM << " merged lanes][" << RING << " rows][32]\n"
       << "  double acc = 0; bool bad = false;\n"
       << "  Real* OUT = (Real*)P.out0; const Real* PV = (const Real*)P.in0; const Real* DAMP = (const Real*)P.in1;\n"
       << "  const int tid = threadIdx.x + threadIdx.y * blockDim.x;\n"
       << "  const int w = tid >> 5, l = tid & 31;\n"
       << "  constexpr int NB = " << NB << ", BW = " << BW << ", H = " << H << ", RR = " << RR << ";\n"
       << "  constexpr int D0 = " << D0 << ", D1 = " << D1 << ", RING = " << RING << ";\n"
       << "  const int CH = P.chunk;\n"
       << "  const int nch = (P.row1 - P.row0 + CH - 1) / CH;\n"
       << "  const int items = NB * nch;\n"
       << "  for (int t = blockIdx.x; t < items; t += gridDim.x) {\n"
       << "    const int ci = t / NB, c0 = (t - ci * NB) * BW;\n"
       << "    const int y0 = P.row0 + ci * CH, y1 = min(y0 + CH, P.row1);\n"
       << "    const bool it = y0 - H - RR >= 0 && y1 + H - 1 + RR < D0 && c0 - H - RR >= 0 && c0 - H + 31 + RR < D1;\n"
       << "    const int q1 = c0 - H + l;\n"
       << "    const int nsteps = (y1 - y0 + 2 * H + 7) >> 3;\n"
       << "    for (int s = 0; s < nsteps; ++s) {\n"
       << "      const int rr = 8 * s + w;  // phase-1 row relative to y0 - H\n"
       << "      const int q0 = y0 - H + rr;\n"
       << "      if (q0 < y1 + H) {\n"
       << "        const int k = (rr % RING) * 32 + l;\n"
       << "        if (it) mo_lanes_" << sfx << "<true>(P, q0, q1, k, CL, " << LS << "); else mo_lanes_" << sfx
       << "<false>(P, q0, q1, k, CL, " << LS << ");\n"
       << "      }\n"
       << "      __syncthreads();\n"
       << "      const int y = q0 - H;\n"
       << "      if (y >= y0 && y < y1 && l >= H && l < 32 - H && q1 < D1) {\n"
       << "        const int rrel = rr - H;\n"
       << "        const long long e = (long long)(y - P.row_lo) * D1 + q1;\n"
       << "        const bool ex = P.mask && P.mask[e];\n";
    // ring row slot of output row minus o0, for every o0 in [-H, H]
    for (int o = -H; o <= H; ++o)
      os << "        const int sl" << (o < 0 ? "m" : "p") << std::abs(o) << " = ((rrel - (" << o << ")) % RING) * 32 + l;\n";
    for (size_t k = 0; k < g.chans.size(); ++k) {
      const int f = g.chans[k].first, ch = g.chans[k].second;
      const int C = P.unknowns[size_t(f)].channels;
      os << "        { Real s = (Real)0;\n";
      for (int si = 0; si < NM; ++si) {
        const MLane& m = merged[size_t(si)];
        if (m.f != f || m.c != ch) continue;
        os << "          s += CL[" << si * LS << " + sl" << (m.o0 < 0 ? "m" : "p") << std::abs(m.o0) << " - (" << m.o1
           << ")];\n";
      }
      os << "          Real v = ex ? (Real)0 : (Real)2 * s;\n"
         << "          if (!mo_finite((double)v)) bad = true;\n"
         << "          const long long col = P.ubase[" << f << "] + e * " << C << " + " << ch << ";\n"
         << "          if (P.flags & MO_F_DAMP) v = v + DAMP[col] * PV[col];\n"
         << "          if ((P.flags & MO_F_ZEROEXCL) && P.colmask && P.colmask[col]) v = (Real)0;\n"
         << "          OUT[col] = v;\n"
         << "          if (P.flags & MO_F_REDUCE) acc += (double)(PV[col] * v); }\n";
    }
    os << "      }\n    }\n    __syncthreads();\n  }\n"
       << "  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n"
       << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n}\n";
    ModuleInfo::Stream st;
    st.ok = true;
    st.smem = size_t(NM) * size_t(LS) * (f64 ? 8 : 4);
    st.halo = H;
    st.ring = RING;
    st.band = BW;
    stream_info = st;
    stream_gi = gi;
  }
  ModuleInfo::Stream stream_info;
  int stream_gi = -1;

  // --------------------------------------------------------- graph kernels
  // One thread per hyperedge (exec.hpp:223-309); scatter outputs go to a
  // per-edge contribution buffer that the deterministic vertex gather folds
  // in edge order (mo_kernels.cu: mo_graph_gather).
  // Deterministic vertex-centric scatter (replaces exec_graph's sequential
  // `+=` / parallel atomics, exec.hpp:265-282): one thread per target vertex
  // v re-evaluates the edge program of every incident edge (CSR, ascending
  // edge order) and accumulates, in registers, the outputs whose slot is v.
  // Per column that is the grid-written value followed by the edges in order
  // and the outputs in program order: the reference's sequential order.
  // fused != nullptr (J^T J p only): the kernel also evaluates the grid gather
  // program `fused` of the same (1-D vertex) domain for its vertex first -
  // exactly what exec_grid writes before the graph scatters add
  // (solver.hpp:257-265) - and finishes the apply in the same pass: LM
  // damping, excluded zeroing and the p'Ap partial (the k_apply_finish
  // epilogue), so one launch replaces gather + vertex gather + finish.
  void vertex_kernel(const GraphSet& g, const Domain& dom, const std::string& pn, const std::string& kn, int arity,
                     bool bm, const GatherSet* gs = nullptr, const std::string& fused = "") {
    const size_t K = g.scats.size();
    const size_t NO = bm ? 2 * K : K;
    struct Col {
      int vec, f, ch;
    };
    std::vector<Col> cols;
    std::vector<int> cidx(NO, -1);
    for (size_t o = 0; o < NO; ++o) {
      const Scat& sc = g.scats[bm ? o / 2 : o];
      if (!(P.unknowns[size_t(sc.field)].dom == dom)) continue;
      Col c{bm ? int(o % 2) : 0, sc.field, sc.channel};
      int k = -1;
      for (size_t j = 0; j < cols.size(); ++j)
        if (cols[j].vec == c.vec && cols[j].f == c.f && cols[j].ch == c.ch) k = int(j);
      if (k < 0) {
        k = int(cols.size());
        cols.push_back(c);
      }
      cidx[o] = k;
    }
    os << kbegin(kn) << "  if ((P.flags & MO_F_SKIPDONE) && P.state->done) return;\n"
       << "  bool bad = false; double acc = 0; (void)acc;\n"
       << "  Real* D0 = (Real*)P.out0; Real* D1 = (Real*)P.out1; (void)D1;\n"
       << "  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < P.nverts;"
          " v += (long long)gridDim.x * blockDim.x) {\n";
    auto colexpr = [&](const Col& c) {
      return std::string(c.vec ? "D1" : "D0") + "[P.ubase[" + std::to_string(c.f) + "] + v * " +
             std::to_string(P.unknowns[size_t(c.f)].channels) + " + " + std::to_string(c.ch) + "]";
    };
    if (gs) {
      // grid gather outputs of this vertex (element v of the 1-D domain)
      const size_t K = gs->chans.size();
      os << "    const bool gex = P.mask && P.mask[v];\n"
         << "    Real go[" << (K ? K : 1) << "];\n"
         << "    if (gex) { for (int k = 0; k < " << K << "; ++k) go[k] = (Real)0; }\n"
         << "    else { " << fused << "<false>(P, (int)v, 0, 0, 0, nullptr, go);\n"
         << "      for (int k = 0; k < " << K << "; ++k) if (!mo_finite((double)go[k])) bad = true; }\n";
      for (size_t j = 0; j < cols.size(); ++j) {
        int k = -1;
        for (size_t q = 0; q < K; ++q)
          if (gs->chans[q].first == cols[j].f && gs->chans[q].second == cols[j].ch) k = int(q);
        os << "    Real a" << j << " = " << (k >= 0 ? "go[" + std::to_string(k) + "]" : std::string("(Real)0")) << ";\n";
      }
    } else {
      for (size_t j = 0; j < cols.size(); ++j) os << "    Real a" << j << " = " << colexpr(cols[j]) << ";\n";
    }
    os << "    const int j1 = P.vptr[v + 1];\n"
       << "    for (int j = P.vptr[v]; j < j1; ++j) {\n"
       << "      const long long e = P.vedge[j];\n"
       << "      int vs[" << (arity ? arity : 1) << "];\n";
    for (int s2 = 0; s2 < arity; ++s2) os << "      vs[" << s2 << "] = P.verts[e * " << arity << " + " << s2 << "];\n";
    os << "      Real o[" << (NO ? NO : 1) << "];\n      " << pn << "<false>(P, 0, 0, 0, 0, vs, o);\n";
    for (size_t o = 0; o < NO; ++o) {
      os << "      if (!mo_finite((double)o[" << o << "])) bad = true;\n";
      if (cidx[o] < 0) continue;
      const Scat& sc = g.scats[bm ? o / 2 : o];
      os << "      if (vs[" << sc.slot << "] == (int)v) a" << cidx[o] << " += o[" << o << "];\n";
    }
    os << "    }\n";
    if (gs) {
      // k_apply_finish epilogue per owned column (solver.hpp:401-405, pcg.hpp:100-102)
      os << "    const Real* PV = (const Real*)P.in0; const Real* DAMP = (const Real*)P.in1;\n";
      for (size_t j = 0; j < cols.size(); ++j) {
        const std::string col = "P.ubase[" + std::to_string(cols[j].f) + "] + v * " +
                                std::to_string(P.unknowns[size_t(cols[j].f)].channels) + " + " +
                                std::to_string(cols[j].ch);
        os << "    { const long long col = " << col << "; Real x = a" << j << ";\n"
           << "      if (P.flags & MO_F_DAMP) x = x + DAMP[col] * PV[col];\n"
           << "      if ((P.flags & MO_F_ZEROEXCL) && P.colmask && (P.colmask[col] & 1)) x = (Real)0;\n"
           << "      D0[col] = x;\n"
           << "      if (P.flags & MO_F_REDUCE) acc += (double)(PV[col] * x); }\n";
      }
      os << "  }\n  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n"
         << "  if (P.flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n}\n";
      return;
    }
    for (size_t j = 0; j < cols.size(); ++j) os << "    " << colexpr(cols[j]) << " = a" << j << ";\n";
    os << "  }\n  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n}\n";
  }

  void graph_kernel(const std::string& pn, const std::string& kn, size_t nout, int arity, int mode) {
    // mode 0 = cost (reduce), 1 = evalf (row writes), 2 = contributions
    os << kbegin(kn) << "  if ((P.flags & MO_F_SKIPDONE) && P.state->done) return;\n"
       << "  double acc = 0; bool bad = false; (void)acc;\n"
       << "  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P.nedges;"
          " e += (long long)gridDim.x * blockDim.x) {\n"
       << "    int vs[" << (arity ? arity : 1) << "];\n";
    for (int s = 0; s < arity; ++s) os << "    vs[" << s << "] = P.verts[e * " << arity << " + " << s << "];\n";
    os << "    Real o[" << (nout ? nout : 1) << "];\n    " << pn << "<false>(P, 0, 0, 0, 0, vs, o);\n";
    for (size_t k = 0; k < nout; ++k) {
      os << "    if (!mo_finite((double)o[" << k << "])) bad = true;\n";
      if (mode == 0) os << "    acc += (double)o[0];\n";
      else if (mode == 1) os << "    ((Real*)P.out0)[P.rowbase[" << k << "] + e] = o[" << k << "];\n";
      else os << "    ((Real*)P.out0)[e * " << nout << " + " << k << "] = o[" << k << "];\n";
    }
    os << "  }\n  if (bad) atomicOr(&P.state->nonfinite_kernel, 1);\n";
    if (mode == 0) os << "  mo_reduce_epilogue<Real>(P.red, acc, 0.0, false);\n";
    os << "}\n";
  }

  ModuleInfo info;

  // linearize (solver.hpp:291-322): evalj per element / edge, output l of
  // element e -> out0[rowbase[l] + e] with rowbase[l] = l * extent (the
  // reference's jlanes buffers), no exclusion mask (exec_grid(..., nullptr)).
  void evalj_kernels() {
    for (size_t i = 0; i < P.grid_sets.size(); ++i) {
      const GridSet& g = P.grid_sets[i];
      if (g.has_evalj)
        grid_evalf(program(g.evalj, false, &g.dom), "mo_grid_evalj_" + std::to_string(i), g.evalj.outputs.size());
    }
    for (size_t i = 0; i < P.graph_sets.size(); ++i) {
      const GraphSet& g = P.graph_sets[i];
      if (g.has_evalj)
        graph_kernel(program(g.evalj, true), "mo_graph_evalj_" + std::to_string(i), g.evalj.outputs.size(),
                     P.graphs[size_t(g.graph)].second, 1);
    }
  }

  void run() {
    const bool mat = P.cfg.materialize != 0;
    for (size_t i = 0; i < P.grid_sets.size(); ++i) {
      const GridSet& g = P.grid_sets[i];
      grid_cost(program(g.cost, false, &g.dom), "mo_grid_cost_" + std::to_string(i));
      grid_evalf(program(g.evalf, false, &g.dom), "mo_grid_evalf_" + std::to_string(i), g.evalf.outputs.size());
    }
    if (mat) evalj_kernels();
    for (size_t i = 0; i < P.gather_sets.size(); ++i) {
      const GatherSet& g = P.gather_sets[i];
      gather_bm(g, program(g.bm, false, &g.dom), "mo_gather_bm_" + std::to_string(i));
      if (mat) {  // no gather J^T J program: the apply runs from the materialized J
        info.jtj2.push_back({});
        info.jtj3.push_back({});
        info.jtj4.push_back({});
        info.jtj5.push_back({});
        info.jtj6.push_back({});
        info.jtj7.push_back({});
        info.bm4.push_back({});
        info.jtj8.push_back({});
        info.bm8.push_back({});
        info.jtj9.push_back({});
        info.jtj9t.push_back({});
        info.bm8c.push_back({});
        continue;
      }
      gather_jtj(g, program(g.jtj, false, &g.dom), "mo_gather_jtj_" + std::to_string(i));
      tma6_info = ModuleInfo::Tma{};
      gather_jtj6(g, int(i));
      stream_info = ModuleInfo::Stream{};
      tma_info = ModuleInfo::Tma{};
      tma7_info = ModuleInfo::Tma{};
      tmabm_info = ModuleInfo::Tma{};
      tma5_info = ModuleInfo::Tma{};
      tma8_info = ModuleInfo::Tma{};
      tmabm8_info = ModuleInfo::Tma{};
      tma9_info = ModuleInfo::Tma{};
      tma9t_info = ModuleInfo::Tma{};
      tmabm8c_info = ModuleInfo::Tma{};
      TwoPhase tp = gather_jtj2(g, int(i));
      info.jtj2.push_back({tp.ok, tp.smem, tp.nlanes, tp.H});
      info.jtj3.push_back(stream_info);
      info.jtj4.push_back(tma_info);
      info.jtj5.push_back(tma5_info);
      info.jtj6.push_back(tma6_info);
      info.jtj7.push_back(tma7_info);
      info.bm4.push_back(tmabm_info);
      info.jtj8.push_back(tma8_info);
      info.bm8.push_back(tmabm8_info);
      info.jtj9.push_back(tma9_info);
      info.jtj9t.push_back(tma9t_info);
      info.bm8c.push_back(tmabm8c_info);
    }
    for (size_t i = 0; i < P.graph_sets.size(); ++i) {
      const GraphSet& g = P.graph_sets[i];
      int ar = P.graphs[size_t(g.graph)].second;
      std::string s = std::to_string(i);
      graph_kernel(program(g.cost, true), "mo_graph_cost_" + s, g.cost.outputs.size(), ar, 0);
      graph_kernel(program(g.evalf, true), "mo_graph_evalf_" + s, g.evalf.outputs.size(), ar, 1);
      graph_kernel(program(g.bm, true), "mo_graph_bm_" + s, g.bm.outputs.size(), ar, 2);
      if (!mat) graph_kernel(program(g.jtj, true), "mo_graph_jtj_" + s, g.jtj.outputs.size(), ar, 2);
      // Vertex-centric recompute kernels, one per scatter-target domain (in
      // the session's GatherDom order: first appearance over the scats).
      std::vector<Domain> doms;
      for (const Scat& sc : g.scats) {
        const Domain& d = P.unknowns[size_t(sc.field)].dom;
        if (std::find(doms.begin(), doms.end(), d) == doms.end()) doms.push_back(d);
      }
      const std::string pj = mat ? std::string() : program(g.jtj, true), pb = program(g.bm, true);
      for (size_t di = 0; di < doms.size(); ++di) {
        if (!mat) vertex_kernel(g, doms[di], pj, "mo_graph_vjtj_" + s + "_" + std::to_string(di), ar, false);
        vertex_kernel(g, doms[di], pb, "mo_graph_vbm_" + s + "_" + std::to_string(di), ar, true);
      }
      info.vertex_kernels.push_back(true);
      if (mat) continue;
      // One-pass apply: a single graph set scattering into one 1-D domain that
      // also holds the only gather set and every unknown column.
      bool one = P.graph_sets.size() == 1 && doms.size() == 1 && P.gather_sets.size() == 1 &&
                 P.gather_sets[0].dom == doms[0] && doms[0].dims.size() == 1;
      for (const Field& f : P.unknowns) one = one && f.dom == doms[0];
      if (one) {
        std::vector<std::pair<int, int>> need;
        for (size_t f = 0; f < P.unknowns.size(); ++f)
          for (int c = 0; c < P.unknowns[f].channels; ++c) need.push_back({int(f), c});
        for (auto fc : need) {  // every unknown column is a scatter target, so the kernel owns it
          bool hit = false;
          for (const Scat& sc : g.scats) hit = hit || (sc.field == fc.first && sc.channel == fc.second);
          one = one && hit;
        }
      }
      if (one) {
        const GatherSet& gs0 = P.gather_sets[0];
        const std::string pgj = program(gs0.jtj, false, &gs0.dom);
        vertex_kernel(g, doms[0], pj, "mo_graph_vjtjf_" + s, ar, false, &gs0, pgj);
        info.fused_vertex_apply = true;
      }
    }
    for (size_t i = 0; i < P.computed_kernels.size(); ++i) {
      const ComputedKernel& ck = P.computed_kernels[i];
      grid_store(program(ck.prog, false, &ck.dom), "mo_computed_" + std::to_string(i), ck.prog.outputs.size());
    }
    for (size_t i = 0; i < P.exclude_kernels.size(); ++i)
      grid_exclude(program(P.exclude_kernels[i].prog, false, &P.exclude_kernels[i].dom), "mo_exclude_" + std::to_string(i));
  }
};

}  // namespace

std::string generate_module(const Plan& P, bool f64, const std::string& prelude, ModuleInfo* info,
                            bool evalj_only) {
  Gen g(P, f64);
  g.os << "// generated by mo_codegen.cpp — do not edit\n";
  g.os << "typedef " << (f64 ? "double" : "float") << " Real;\n";
  g.os << "#define MO_REAL_MAX " << (f64 ? "1.7976931348623157e308" : "3.40282347e38f") << "\n";
  // Exponent field of a Real (as unsigned): all ones <=> inf or nan.
  if (f64)
    g.os << "#define MO_EXP_BITS(v) ((unsigned)(__double_as_longlong(v) >> 32) & 0x7ff00000u)\n#define MO_EXP_MASK 0x7ff00000u\n";
  else
    g.os << "#define MO_EXP_BITS(v) (__float_as_uint(v) & 0x7f800000u)\n#define MO_EXP_MASK 0x7f800000u\n";
  g.os << prelude << "\n";
  g.os << "extern __shared__ __align__(128) unsigned char mo_dsm[];\n";
  if (evalj_only)
    g.evalj_kernels();
  else
    g.run();
  if (info) *info = g.info;
  return g.os.str();
}

}  // namespace mo
