// mo_jit.cpp — NVRTC compilation of generated plan modules for sm_100a and
// loading through the CUDA runtime library API (cudaLibraryLoadData /
// cudaLibraryGetKernel, CUDA >= 12.0), with an on-disk cubin cache keyed by a
// hash of the source and options.
#include "mo_jit.hpp"

#include <algorithm>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <mutex>
#include <sstream>
#include <sys/stat.h>
#include <unistd.h>
#include <vector>

namespace mo {

namespace {

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

// $MO_B200_CACHE, else <directory of libmo_b200.so>/_kcache (travels with the
// in-tree build), else ~/.cache/mo_b200.
std::string cache_dir() {
  if (const char* d = std::getenv("MO_B200_CACHE")) return d;
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&compile_cubin), &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    auto slash = p.rfind('/');
    if (slash != std::string::npos) return p.substr(0, slash) + "/_kcache";
  }
  if (const char* h = std::getenv("HOME")) return std::string(h) + "/.cache/mo_b200";
  return "/tmp/mo_b200_cache";
}

void mkdirs(const std::string& path) {
  std::string cur;
  std::stringstream ss(path);
  std::string part;
  if (!path.empty() && path[0] == '/') cur = "/";
  while (std::getline(ss, part, '/')) {
    if (part.empty()) continue;
    cur += part + "/";
    ::mkdir(cur.c_str(), 0755);
  }
}

const char* kOpts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo",
                       "-default-device", "--extra-device-vectorization"};

}  // namespace

std::vector<char> compile_cubin(const std::string& src, const std::string& name, bool exact, std::string* log_out) {
  std::vector<const char*> opts(std::begin(kOpts), std::end(kOpts));
  opts.push_back(exact ? "--fmad=false" : "--fmad=true");
  int maj = 0, min = 0;
  nvrtcVersion(&maj, &min);
  std::string key = src;
  for (const char* o : opts) key += o;
  key += std::to_string(maj) + "." + std::to_string(min);
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx", (unsigned long long)fnv1a(key));
  const std::string dir = cache_dir();
  const std::string path = dir + "/" + hex + ".cubin";
  if (!std::getenv("MO_B200_NOCACHE")) {
    std::ifstream f(path, std::ios::binary);
    if (f) {
      std::vector<char> buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
      if (!buf.empty()) return buf;
    }
  }
  nvrtcProgram prog;
  // The generated source is kept beside its cubin and named by that path so
  // -lineinfo maps SASS back to it (ncu --import-source, compute-sanitizer).
  std::string srcname = name;
  if (!std::getenv("MO_B200_NOCACHE")) {
    mkdirs(dir);
    srcname = dir + "/" + hex + ".cu";
    std::ofstream(srcname) << src;
  }
  check(nvrtcCreateProgram(&prog, src.c_str(), srcname.c_str(), 0, nullptr, nullptr) == NVRTC_SUCCESS,
        Err::kInternal, "nvrtcCreateProgram failed");
  nvrtcResult r = nvrtcCompileProgram(prog, int(opts.size()), opts.data());
  size_t logsz = 0;
  nvrtcGetProgramLogSize(prog, &logsz);
  std::string log(logsz, '\0');
  if (logsz) nvrtcGetProgramLog(prog, log.data());
  if (log_out) *log_out = log;
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    fail(Err::kInternal, std::string("NVRTC compilation of the plan module failed: ") +
                             nvrtcGetErrorString(r) + "\n" + log.substr(0, 4000));
  }
  size_t sz = 0;
  nvrtcGetCUBINSize(prog, &sz);
  std::vector<char> cubin(sz);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  if (!std::getenv("MO_B200_NOCACHE")) {
    mkdirs(dir);
    std::string tmp = path + ".tmp" + std::to_string(::getpid());
    std::ofstream o(tmp, std::ios::binary);
    o.write(cubin.data(), std::streamsize(cubin.size()));
    o.close();
    std::rename(tmp.c_str(), path.c_str());
  }
  return cubin;
}

Module::~Module() {
  if (lib_) cudaLibraryUnload(static_cast<cudaLibrary_t>(lib_));
}

void Module::load(const std::vector<char>& cubin) {
  cudaLibrary_t lib = nullptr;
  cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  check(e == cudaSuccess, Err::kCuda, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e));
  lib_ = lib;
  // Large generated programs (f64 division / sqrt subroutine calls) can need
  // a per-thread stack frame beyond the default 1 KiB limit: raise the
  // device limit here, at load time, never inside a stream capture.
  unsigned n = 0;
  if (cudaLibraryGetKernelCount(&n, lib) == cudaSuccess && n) {
    std::vector<cudaKernel_t> ks(n);
    if (cudaLibraryEnumerateKernels(ks.data(), n, lib) == cudaSuccess) {
      size_t need = 0;
      for (cudaKernel_t k : ks) {
        cudaFuncAttributes a{};
        if (cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k)) == cudaSuccess)
          need = std::max(need, size_t(a.localSizeBytes));
      }
      size_t cur = 0;
      cudaDeviceGetLimit(&cur, cudaLimitStackSize);
      if (need + 1024 > cur) cudaDeviceSetLimit(cudaLimitStackSize, (need + 1024 + 255) / 256 * 256);
    }
  }
  cudaGetLastError();
}

const void* Module::kernel(const std::string& name) {
  auto it = kernels_.find(name);
  if (it != kernels_.end()) return it->second;
  cudaKernel_t k = nullptr;
  cudaError_t e = cudaLibraryGetKernel(&k, static_cast<cudaLibrary_t>(lib_), name.c_str());
  check(e == cudaSuccess, Err::kCuda, "cudaLibraryGetKernel(" + name + "): " + cudaGetErrorString(e));
  kernels_[name] = reinterpret_cast<const void*>(k);
  return kernels_[name];
}

}  // namespace mo
