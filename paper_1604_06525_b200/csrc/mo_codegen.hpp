// mo_codegen.hpp — plan -> CUDA C++ module (see mo_codegen.cpp).
#pragma once
#include <string>

#include "mo_plan.hpp"

#include <vector>

namespace mo {

// What the generated module offers beyond the 1:1 program kernels.
struct ModuleInfo {
  struct TwoPhase {
    bool ok = false;       // mo_gather_jtj2_<i> exists
    size_t smem = 0;       // dynamic shared memory per block (bytes)
    int nlanes = 0, halo = 0;
  };
  // Row-streaming two-phase apply (mo_gather_jtj3_<i>, 2-D domains): one
  // block walks a band of 32 - 2*halo columns down `chunk` rows, keeping a
  // ring of `ring` phase-1 rows in shared memory.
  struct Stream {
    bool ok = false;
    size_t smem = 0;
    int halo = 0, ring = 0, band = 0;
  };
  // TMA-staged streaming apply (mo_gather_jtj4_<i>): kernel parameter 2 is a
  // mo_tmaps with one 2-D tensor map per staged slot, in `slots` order, over
  // the field as [rows][D1 * C] with box [8][win * C].
  struct Tma {
    bool ok = false;
    size_t smem = 0;
    int halo = 0, band = 0, rx = 0, win = 0;
    int rows = 8, threads = 256;             // box rows; block size
    std::vector<std::pair<int, int>> slots;  // (view slot, channels)
    // lane-cache apply (mo_gather_jtj9): planes, their first view slot and the
    // extended-domain plane geometry (column origin HX, pitch PW, rows)
    int cache_planes = 0, cache_slot0 = 0, cache_hx = 0, cache_pw = 0, cache_rows = 0;
    bool cache_tma = false;  // planes staged by TMA (views cache_slot0 + j) instead of direct loads
  };
  std::vector<TwoPhase> jtj2;  // per gather set
  std::vector<Stream> jtj3;    // per gather set
  std::vector<Tma> jtj4;       // per gather set
  std::vector<Tma> jtj5;       // per gather set: warp-streaming (box rows = rows)
  std::vector<Tma> jtj6;       // per gather set: TMA-staged gather program
  std::vector<Tma> jtj7;       // per gather set: variant 3 with 4-row steps (128 threads)
  std::vector<Tma> bm4;        // per gather set: TMA two-phase build_normal (mo_gather_bm4_<i>)
  std::vector<Tma> jtj8;       // per gather set: warp-specialised streaming apply (mo_gather_jtj8_<i>)
  std::vector<Tma> bm8;        // per gather set: warp-specialised streaming build_normal (mo_gather_bm8_<i>)
  std::vector<Tma> jtj9;       // per gather set: lane-cache streaming apply (mo_gather_jtj9_<i>, mo_lanecache_<i>)
  std::vector<Tma> bm8c;       // per gather set: mo_gather_bm8 that also writes jtj9's lane cache
  std::vector<Tma> jtj9t;      // per gather set: jtj9 with the lane-cache planes TMA-staged (mo_gather_jtj9t_<i>)
  std::vector<bool> vertex_kernels;  // per graph set: mo_graph_v{jtj,bm}_<g>_<dom> exist
  bool fused_vertex_apply = false;   // mo_graph_vjtjf_0: grid gather + graph gather + finish in one pass
};

// Full NVRTC translation unit for one plan and precision.  `prelude` is the
// text of mo_device.cuh.  evalj_only: just the linearize kernels
// (mo_grid_evalj_<i>, mo_graph_evalj_<g>), compiled on demand for matrix-free
// plans that also carry Jacobian lanes (force_evalj).
std::string generate_module(const Plan& P, bool f64, const std::string& prelude,
                            ModuleInfo* info = nullptr, bool evalj_only = false);
}  // namespace mo
