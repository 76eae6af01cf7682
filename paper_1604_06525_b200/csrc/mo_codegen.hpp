// mo_codegen.hpp — plan -> CUDA C++ module (see mo_codegen.cpp).
#pragma once
#include <string>

#include "mo_plan.hpp"

namespace mo {
// Full NVRTC translation unit for one plan and precision.  `prelude` is the
// text of mo_device.cuh.
std::string generate_module(const Plan& P, bool f64, const std::string& prelude);
}  // namespace mo
