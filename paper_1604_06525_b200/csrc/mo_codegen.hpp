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
  std::vector<TwoPhase> jtj2;  // per gather set
  std::vector<bool> vertex_kernels;  // per graph set: mo_graph_v{jtj,bm}_<g>_<dom> exist
};

// Full NVRTC translation unit for one plan and precision.  `prelude` is the
// text of mo_device.cuh.
std::string generate_module(const Plan& P, bool f64, const std::string& prelude,
                            ModuleInfo* info = nullptr);
}  // namespace mo
