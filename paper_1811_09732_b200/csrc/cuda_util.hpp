// cuda_util.hpp — error plumbing between the CUDA runtime and trims::Error.
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>

#include <string>
#include <utility>

#include "errc.hpp"

#define TRIMS_CUDA(expr)                                                                        \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess) {                                                                    \
      ::trims::raise(_e == cudaErrorMemoryAllocation ? ::trims::Errc::OutOfDeviceMemory         \
                                                     : ::trims::Errc::CudaError,                \
                     std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" __FILE__ ":" + \
                         std::to_string(__LINE__) + ")");                                       \
    }                                                                                           \
  } while (0)

namespace trims {

// RAII device guard: the C-ABI may be entered from any host thread.
// nothrow=true for destructors (teardown may run after driver shutdown).
struct DeviceGuard {
  int prev{-1};
  explicit DeviceGuard(int dev, bool nothrow = false) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    if (prev != dev) {
      cudaError_t e = cudaSetDevice(dev);
      if (e != cudaSuccess && !nothrow) TRIMS_CUDA(e);
      if (e != cudaSuccess) cudaGetLastError();
    }
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Programmatic dependent launch (PDL): the forward-pass kernels are launched
// with programmatic stream serialisation, so a kernel's prologue (barrier
// init, TMEM alloc, tensor-map prefetch, weight loads) overlaps the tail of
// the kernel before it. Every such kernel calls pdl_wait() before it reads
// anything the previous kernel wrote (griddepcontrol.wait returns once the
// prerequisite grid has completed and its writes are visible), and
// pdl_trigger() to let the next kernel launch early.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// TRIMS_PDL=0 launches without the attribute (kernels still call
// griddepcontrol, which is then a no-op): under MPS many clients share the
// SMs, and CTAs launched early only to sit in griddepcontrol.wait hold SMs
// another client's kernel could run on.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  TRIMS_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}
#endif

}  // namespace trims
