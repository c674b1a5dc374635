// gemm.cu — K7: the conv/FC contraction on the 5th-gen tensor cores.
//
// D[M,N] = epi(A[M,K] . B[N,K]^T): A = activations (NHWC rows, or an im2col
// matrix), B = resident KRSC weights (row n = output channel n, K-major),
// bf16 operands, fp32 accumulation in TMEM, fused epilogue
//   out = relu?( acc * scale[n] + bias[n] + residual[m,n] )  -> bf16.
// One CTA per 128 x BN output tile: warp 0 issues TMA (SWIZZLE_128B boxes
// of 64 x rows) into a STAGES-deep mbarrier ring, warp 1 allocates TMEM and a
// single lane issues tcgen05.mma (M=128, N=BN, K=16 per instruction), warps
// 4-7 drain TMEM with tcgen05.ld and run the epilogue.
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "cuda_util.hpp"
#include "device_mem.hpp"
#include "gemm.cuh"
#include "gemm.hpp"

namespace trims::gemm {

using namespace trims::sm100;

namespace {

constexpr int BM = 128, BK = 64, kThreads = 256;

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, uint16_t* D,
                   int M, int N, int K, int ldd, const float* __restrict__ scale, const float* __restrict__ bias,
                   const uint16_t* __restrict__ res, int ldr, int relu) {
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = BN;  // 64 / 128 / 256: powers of two >= 32
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], accum_full;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kblocks = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&accum_full, 1);
    fence_barrier_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        uint8_t* sa = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        tma_load_2d(sa, &tmA, kb * BK, m0, &full[s]);
        tma_load_2d(sa + A_BYTES, &tmB, kb * BK, n0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&full[s], (kb / STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * STAGE_BYTES), sb = sa + A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          mma_bf16(tmem, smem_desc_sw128(sa + k * 32), smem_desc_sw128(sb + k * 32), idesc, (kb | k) != 0);
        mma_commit(&empty[s]);  // the stage is free once these MMAs have read it
      }
      mma_commit(&accum_full);
    }
  } else if (warp >= 4) {  // ---- epilogue: TMEM -> registers -> bf16 global
    mbar_wait(&accum_full, 0);
    tc_fence_after();
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = m0 + q * 32 + lane;
    uint16_t* drow = D + size_t(row) * ldd;
    const uint16_t* rrow = res ? res + size_t(row) * ldr : nullptr;
    const bool vec_ok = (ldd % 8 == 0) && (!res || ldr % 8 == 0);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(c0), r);
      const int n = n0 + c0;
      if (row >= M || n >= N) continue;
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int nj = n + j;
        float x = __uint_as_float(r[j]);
        if (nj < N) {
          if (scale) x *= __ldg(scale + nj);
          if (bias) x += __ldg(bias + nj);
        }
        v[j] = x;
      }
      if (vec_ok && n + 16 <= N) {
        if (rrow) {
          const uint4* rp = reinterpret_cast<const uint4*>(rrow + n);
          uint4 a = rp[0], b = rp[1];
          const uint32_t rw[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            v[2 * j] += bf16_lo(rw[j]);
            v[2 * j + 1] += bf16_hi(rw[j]);
          }
        }
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float a = v[2 * j], b = v[2 * j + 1];
          if (relu) {
            a = fmaxf(a, 0.f);
            b = fmaxf(b, 0.f);
          }
          o[j] = pack_bf16x2(a, b);
        }
        uint4* dp = reinterpret_cast<uint4*>(drow + n);
        dp[0] = make_uint4(o[0], o[1], o[2], o[3]);
        dp[1] = make_uint4(o[4], o[5], o[6], o[7]);
      } else {
        for (int j = 0; j < 16 && n + j < N; ++j) {
          float x = v[j];
          if (rrow) x += __uint_as_float(uint32_t(rrow[n + j]) << 16);
          if (relu) x = fmaxf(x, 0.f);
          drow[n + j] = uint16_t(pack_bf16x2(x, 0.f) & 0xffffu);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<TMEM_COLS>(tmem);
  }
}

using EncodeTiled = decltype(&cuTensorMapEncodeTiled);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      raise(Errc::NoDevice, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

template <int BN, int STAGES>
void run_bn(const Prepared& p, cudaStream_t stream) {
  constexpr size_t smem = size_t(STAGES) * (BM * BK * 2 + BN * BK * 2) + 1024;
  static bool attr = false;
  if (!attr) {
    TRIMS_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem)));
    attr = true;
  }
  const Epilogue& e = p.e;
  dim3 grid(unsigned((p.M + BM - 1) / BM), unsigned((p.N + BN - 1) / BN));
  gemm_tc_kernel<BN, STAGES><<<grid, kThreads, smem, stream>>>(p.ta, p.tb, e.out, int(p.M), int(p.N), int(p.K),
                                                                int(e.ldo), e.scale, e.bias, e.residual, int(e.ldr),
                                                                e.relu ? 1 : 0);
  TRIMS_CUDA(cudaGetLastError());
}

}  // namespace

CUtensorMap make_tmap(const void* ptr, uint64_t rows, uint64_t k, uint64_t ld, uint32_t box_rows) {
  if ((ld * 2) % 16 || reinterpret_cast<uintptr_t>(ptr) % 16)
    raise(Errc::InvalidArgument, "TMA operand rows must be 16-byte aligned (pad K)");
  CUtensorMap m;
  cuuint64_t dims[2] = {k, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {uint32_t(BK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cu_check(r, "cuTensorMapEncodeTiled");
  return m;
}

int pick_bn(uint64_t M, uint64_t N, int sms) {
  // Enough CTAs to cover the SMs first, then the widest tile.
  const uint64_t mt = (M + BM - 1) / BM;
  if (N <= 64) return 64;
  if (mt * ((N + 255) / 256) >= uint64_t(sms) && N % 256 == 0) return 256;
  if (mt * ((N + 127) / 128) >= uint64_t(sms) / 2 || N <= 128) return 128;
  return 64;
}

Prepared prepare(const Operand& A, const Operand& B, const Epilogue& e, int bn) {
  if (A.k != B.k) raise(Errc::InvalidArgument, "GEMM K mismatch");
  if (!bn) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    bn = pick_bn(A.rows, B.rows, sms);
  }
  if (bn != 64 && bn != 128 && bn != 256) raise(Errc::InvalidArgument, "BN must be 64, 128 or 256");
  Prepared p;
  p.ta = make_tmap(A.ptr, A.rows, A.k, A.ld, BM);
  p.tb = make_tmap(B.ptr, B.rows, B.k, B.ld, uint32_t(bn));
  p.M = A.rows;
  p.N = B.rows;
  p.K = A.k;
  p.bn = bn;
  p.e = e;
  return p;
}

void run(const Prepared& p, cudaStream_t stream) {
  switch (p.bn) {
    case 64: run_bn<64, 6>(p, stream); break;
    case 128: run_bn<128, 5>(p, stream); break;
    default: run_bn<256, 4>(p, stream); break;
  }
}

void launch(const Operand& A, const Operand& B, const Epilogue& e, cudaStream_t stream, int bn) {
  run(prepare(A, B, e, bn), stream);
}

}  // namespace trims::gemm
