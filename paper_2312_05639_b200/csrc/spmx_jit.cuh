// spmx_jit.cuh — run-time instantiation of the SpMM kernel for one dense width d.
//
// The reference specialises its row kernel on d by emitting x86 code at run time
// (src/plan.cpp:80-93, src/jit.cpp:136-154). Here the same step compiles the CUDA kernel
// template of spmx_kernels.cuh for exactly (d, lanes per row, tiles per lane) with NVRTC for
// sm_100a: d becomes a compile-time constant (row strides fold into immediates, the tile
// loops unroll fully, ragged-column checks disappear when d divides evenly). Kernels are
// cached per (device, d, vector width). NVRTC is loaded with dlopen on first use, so the
// library itself has no link-time dependency on it.
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <chrono>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace spmx_jit {

static const char* kKernelSource =
#include "spmx_kernels_src.inc"
    ;

struct Nvrtc {
  void* handle = nullptr;
  decltype(&nvrtcCreateProgram) CreateProgram = nullptr;
  decltype(&nvrtcDestroyProgram) DestroyProgram = nullptr;
  decltype(&nvrtcAddNameExpression) AddNameExpression = nullptr;
  decltype(&nvrtcCompileProgram) CompileProgram = nullptr;
  decltype(&nvrtcGetLoweredName) GetLoweredName = nullptr;
  decltype(&nvrtcGetCUBINSize) GetCUBINSize = nullptr;
  decltype(&nvrtcGetCUBIN) GetCUBIN = nullptr;
  decltype(&nvrtcGetProgramLogSize) GetProgramLogSize = nullptr;
  decltype(&nvrtcGetProgramLog) GetProgramLog = nullptr;
  decltype(&nvrtcGetErrorString) GetErrorString = nullptr;

  static Nvrtc& get() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
      const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
      for (const char* nm : names)
        if ((n.handle = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
      if (!n.handle) return;
#define SPMX_SYM(f) n.f = reinterpret_cast<decltype(n.f)>(dlsym(n.handle, "nvrtc" #f))
      SPMX_SYM(CreateProgram); SPMX_SYM(DestroyProgram); SPMX_SYM(AddNameExpression);
      SPMX_SYM(CompileProgram); SPMX_SYM(GetLoweredName); SPMX_SYM(GetCUBINSize);
      SPMX_SYM(GetCUBIN); SPMX_SYM(GetProgramLogSize); SPMX_SYM(GetProgramLog);
      SPMX_SYM(GetErrorString);
#undef SPMX_SYM
    });
    return n;
  }
  bool ok() const { return handle && CreateProgram && CompileProgram && GetCUBIN && GetLoweredName; }
};

struct Shape {
  int g, vec, nt;
  bool ragged;
};

// Column vector per lane for width d: the widest of {4, 2, 1} floats that the alignment allows
// (vec_max) and that still spreads a row over at least five lanes, i.e. an 8-lane group with
// eight positions in flight (see run_kernels); rows of fewer than five columns use scalars.
inline int narrow_vec(int d, int vec_max) {
  for (int v = vec_max; v > 1; v >>= 1)
    if (d % v == 0 && d / v >= 5) return v;
  return 1;
}

// lanes per row and tiles per lane for width d: eight lanes whenever the row fits four tiles per
// lane (a row of fewer than five vectors: the next power of two), else 16, else all 32 lanes with
// up to eight tiles. Eight-lane groups measured best at every width they can hold (four chunk
// streams per warp, eight positions per batch, column/value broadcast through shared memory):
// d = 48 runs 8 x 2 (ragged) instead of 4 x 3, d = 20 8 x 1 instead of 4 x 2. d beyond 32 x 8
// vectors is slabbed by the caller.
inline Shape choose_shape(int d, int vec_max) {
  const int vec = narrow_vec(d, vec_max);
  const int lanes = (d + vec - 1) / vec;
  int g = 1;
  while (g < 8 && g < lanes) g <<= 1;
  for (; g <= 32; g <<= 1) {
    const int nt = (lanes + g - 1) / g;
    if (nt <= (g < 32 ? 4 : 8)) return {g, vec, nt, g * nt * vec != d};
  }
  return {32, vec, 8, true};
}
// widest d compiled as one kernel (wider ones run as slabs of the precompiled shapes)
inline int max_width(int vec) { return vec == 4 ? 128 : 32 * 8 * vec; }

struct Kernel {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t chunk = nullptr;
  Shape shape{};
  double compile_s = 0.0;
};

struct Stats {
  uint64_t compiled = 0;
  double seconds = 0.0;
};

inline std::mutex& mu() { static std::mutex m; return m; }
inline Stats& stats() { static Stats s; return s; }
inline std::map<std::tuple<int, int, int>, Kernel>& cache() {
  static std::map<std::tuple<int, int, int>, Kernel> c;
  return c;
}

// Returns the kernel specialised for (d, vec) on `device`, compiling it on first use.
inline const Kernel& get(int device, int d, int vec) {
  std::lock_guard<std::mutex> lock(mu());
  auto key = std::make_tuple(device, d, vec);
  auto it = cache().find(key);
  if (it != cache().end()) return it->second;

  Nvrtc& rt = Nvrtc::get();
  if (!rt.ok()) throw std::runtime_error("SPMX_JIT_WIDTH: NVRTC (libnvrtc.so.12) is not available");
  const auto t0 = std::chrono::steady_clock::now();
  const Shape sh = choose_shape(d, vec);
  const std::string name = "spmx_dev::spmm_chunk_kernel<" + std::to_string(d) + ", " +
                           std::to_string(sh.g) + ", " + std::to_string(sh.vec) + ", " +
                           std::to_string(sh.nt) + ", " + (sh.ragged ? "true" : "false") + ">";
  nvrtcProgram prog = nullptr;
  auto fail = [&](const std::string& what, nvrtcResult r) {
    std::string log;
    size_t n = 0;
    if (prog && rt.GetProgramLogSize && rt.GetProgramLogSize(prog, &n) == NVRTC_SUCCESS && n > 1) {
      log.resize(n);
      rt.GetProgramLog(prog, log.data());
    }
    if (prog) rt.DestroyProgram(&prog);
    throw std::runtime_error("NVRTC " + what + " failed for " + name + ": " +
                             (rt.GetErrorString ? rt.GetErrorString(r) : "?") + "\n" + log.substr(0, 2000));
  };
  nvrtcResult r = rt.CreateProgram(&prog, kKernelSource, "spmx_kernels.cuh", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) fail("program creation", r);
  r = rt.AddNameExpression(prog, name.c_str());
  if (r != NVRTC_SUCCESS) fail("name expression", r);
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "-DSPMX_JIT=1"};
  r = rt.CompileProgram(prog, 4, opts);
  if (r != NVRTC_SUCCESS) fail("compilation", r);
  const char* lowered = nullptr;
  r = rt.GetLoweredName(prog, name.c_str(), &lowered);
  if (r != NVRTC_SUCCESS) fail("name lookup", r);
  size_t size = 0;
  r = rt.GetCUBINSize(prog, &size);
  if (r != NVRTC_SUCCESS) fail("cubin size", r);
  std::vector<char> cubin(size);
  r = rt.GetCUBIN(prog, cubin.data());
  if (r != NVRTC_SUCCESS) fail("cubin", r);

  Kernel k;
  k.shape = sh;
  cudaError_t e = cudaLibraryLoadData(&k.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&k.chunk, k.lib, lowered);
  rt.DestroyProgram(&prog);
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("loading the compiled kernel failed: ") + cudaGetErrorString(e));
  cudaFuncSetAttribute((const void*)k.chunk, cudaFuncAttributePreferredSharedMemoryCarveout, 30);
  k.compile_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  stats().compiled += 1;
  stats().seconds += k.compile_s;
  return cache().emplace(key, k).first->second;
}

}  // namespace spmx_jit
