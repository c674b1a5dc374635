// cuda_util.hpp — error plumbing between the CUDA runtime and trims::Error.
#pragma once

#include <cuda_runtime.h>

#include <string>

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

}  // namespace trims
