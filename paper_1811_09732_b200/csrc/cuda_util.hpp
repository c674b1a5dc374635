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
struct DeviceGuard {
  int prev{-1};
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) TRIMS_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace trims
