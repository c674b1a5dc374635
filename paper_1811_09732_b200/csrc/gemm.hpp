// gemm.hpp — host interface of the tcgen05 GEMM (K7).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace trims::gemm {

// A K-major bf16 operand: `rows` rows of `k` elements, row stride `ld`
// elements (ld*2 must be a multiple of 16 bytes; TMA zero-fills k..ceil64(k)).
struct Operand {
  const void* ptr;
  uint64_t rows, k, ld;
};

// out[m, n] = relu?(acc * scale[n] + bias[n] + residual[m, n]) as bf16.
struct Epilogue {
  uint16_t* out;
  uint64_t ldo;
  const float* scale{nullptr};
  const float* bias{nullptr};
  const uint16_t* residual{nullptr};
  uint64_t ldr{0};
  bool relu{false};
};

CUtensorMap make_tmap(const void* ptr, uint64_t rows, uint64_t k, uint64_t ld, uint32_t box_rows);
int pick_bn(uint64_t M, uint64_t N, int sms);

// A GEMM with its tensor maps encoded once (the executor builds these at
// bind time so a forward pass costs only kernel launches).
struct Prepared {
  CUtensorMap ta, tb;
  uint64_t M{0}, N{0}, K{0};
  int bn{128};
  Epilogue e;
  // Split-K (grid.z = splits): fp32 partial tiles in `ws`, one arrival
  // counter per output tile in `ctr` (zeroed once; the last split re-arms it).
  int splits{1};
  float* ws{nullptr};
  unsigned int* ctr{nullptr};
};
Prepared prepare(const Operand& A, const Operand& B, const Epilogue& e, int bn = 0);
void run(const Prepared& p, cudaStream_t stream);
// Split count for a GEMM shape on `sms` SMs, and the workspace it needs.
int pick_splits(uint64_t M, uint64_t N, uint64_t K, int bn, int sms);
uint64_t workspace_bytes(const Prepared& p);
uint64_t counter_count(const Prepared& p);
// D = epi(A . B^T); bn = 0 picks the tile width.
void launch(const Operand& A, const Operand& B, const Epilogue& e, cudaStream_t stream, int bn = 0);

}  // namespace trims::gemm
