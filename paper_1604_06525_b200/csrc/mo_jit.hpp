// mo_jit.hpp — NVRTC + cudaLibrary loading of generated plan modules.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "mo_plan.hpp"

namespace mo {

// Compile CUDA C++ to an sm_100a cubin (cached on disk under $MO_B200_CACHE or
// ~/.cache/mo_b200).  Works without a GPU.
// exact = true compiles with --fmad=false (no FMA contraction: add/mul round
// exactly like the reference's x86 build); false allows contraction.
std::vector<char> compile_cubin(const std::string& src, const std::string& name, bool exact,
                                std::string* log = nullptr);

class Module {
 public:
  Module() = default;
  ~Module();
  Module(const Module&) = delete;
  Module& operator=(const Module&) = delete;
  void load(const std::vector<char>& cubin);
  const void* kernel(const std::string& name);  // usable with cudaLaunchKernel
  bool loaded() const { return lib_ != nullptr; }

 private:
  void* lib_ = nullptr;
  std::map<std::string, const void*> kernels_;
};

}  // namespace mo
