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
#include <cstdlib>
#include <type_traits>
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

constexpr int BM = 128, BK = 64, kThreads = 256, kMaxSplits = 8;

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// Shared-memory plan of one CTA: the TMA ring, then the epilogue operands
// (residual tile, folded-BN scale and bias) prefetched during the mainloop.
template <int BN, int STAGES>
struct Smem {
  static constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t RES_LD = BN + 8;  // bf16 elements per residual row (+16 B: spreads banks)
  static constexpr uint32_t RING = STAGES * STAGE_BYTES;
  static constexpr uint32_t RES = RING, RES_BYTES = BM * RES_LD * 2;
  static constexpr uint32_t SCALE = RES + RES_BYTES, BIAS = SCALE + BN * 4;
  static constexpr uint32_t TOTAL = BIAS + BN * 4 + 1024;  // + 1 KiB realignment slack
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, uint16_t* D,
                   int M, int N, int K, int ldd, const float* __restrict__ scale, const float* __restrict__ bias,
                   const uint16_t* __restrict__ res, int ldr, int relu, int kper, const ConvGeom cg) {
  using L = Smem<BN, STAGES>;
  constexpr uint32_t TMEM_COLS = BN;  // 64 / 128 / 256: powers of two >= 32
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], accum_full;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint16_t* s_res = reinterpret_cast<uint16_t*>(smem + L::RES);
  float* s_scale = reinterpret_cast<float*>(smem + L::SCALE);
  float* s_bias = reinterpret_cast<float*>(smem + L::BIAS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int splits = gridDim.z, z = blockIdx.z;
  const int kblocks = (K + BK - 1) / BK;
  const int kb0 = z * kper, kb1 = min(kblocks, kb0 + kper);  // this split's k-blocks
  // Implicit conv: this tile = image ti, output rows [th*hbox, +hbox), cols [tw*wbox, +wbox).
  int ti = 0, th = 0, tw = 0;
  if (cg.impl) {
    tw = blockIdx.x % cg.tiles_w;
    th = (blockIdx.x / cg.tiles_w) % cg.tiles_h;
    ti = blockIdx.x / (cg.tiles_w * cg.tiles_h);
  }
  const int wbox = 1 << cg.wbox_log2;
  // Global output row of tile row rl, or -1 outside the output.
  auto row_of = [&](int rl) -> int {
    if (!cg.impl) return m0 + rl < M ? m0 + rl : -1;
    const int h = th * cg.hbox + (rl >> cg.wbox_log2), w = tw * wbox + (rl & (wbox - 1));
    return (h < cg.P && w < cg.Q) ? (ti * cg.P + h) * cg.Q + w : -1;
  };
  // Epilogue of tile columns [c_begin, c_end) for tile row rl: fetch(c0, v)
  // yields the 16 fp32 accumulators of columns c0..c0+15; then scale, bias,
  // residual (smem), ReLU, bf16, 32-byte stores.
  // Epilogue of tile columns [c_begin, c_end) for tile row rl, CW (16 or 8)
  // columns at a time: fetch(c0, v) yields the CW fp32 accumulators of
  // columns c0..c0+CW-1; then scale, bias, residual (smem), ReLU, bf16,
  // 16-byte stores.
  auto store_cols = [&](auto cw_tag, int c_begin, int c_end, int rl, auto&& fetch) {
    constexpr int CW = decltype(cw_tag)::value;
    const int row = row_of(rl);
    uint16_t* drow = D + size_t(row < 0 ? 0 : row) * ldd;
    const bool vec_ok = (ldd % 8 == 0);
#pragma unroll 1
    for (int c0 = c_begin; c0 < c_end; c0 += CW) {
      float v[CW];
      fetch(c0, v);
      const int n = n0 + c0;
      if (row < 0 || n >= N) continue;
      uint32_t rw[CW / 2];
#pragma unroll
      for (int q = 0; q < CW / 8; ++q) {
        const uint4 r4 = res ? reinterpret_cast<const uint4*>(s_res + rl * L::RES_LD + c0)[q] : make_uint4(0, 0, 0, 0);
        rw[4 * q] = r4.x, rw[4 * q + 1] = r4.y, rw[4 * q + 2] = r4.z, rw[4 * q + 3] = r4.w;
      }
      uint32_t o[CW / 2];
#pragma unroll
      for (int j = 0; j < CW / 2; ++j) {
        float a = v[2 * j] * s_scale[c0 + 2 * j] + s_bias[c0 + 2 * j];
        float b = v[2 * j + 1] * s_scale[c0 + 2 * j + 1] + s_bias[c0 + 2 * j + 1];
        if (res) {
          a += bf16_lo(rw[j]);
          b += bf16_hi(rw[j]);
        }
        if (relu) {
          a = fmaxf(a, 0.f);
          b = fmaxf(b, 0.f);
        }
        o[j] = pack_bf16x2(a, b);
      }
      if (vec_ok && n + CW <= N) {
        uint4* dp = reinterpret_cast<uint4*>(drow + n);
#pragma unroll
        for (int q = 0; q < CW / 8; ++q) dp[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < CW; ++j)
          if (n + j < N) drow[n + j] = uint16_t(o[j >> 1] >> (16 * (j & 1)));
      }
    }
  };
  auto load_a = [&](void* dst, int kb, uint64_t* bar) {
    if (cg.impl) {
      const int rs = kb / cg.cblocks, cb = kb - rs * cg.cblocks, r = rs / cg.S, s = rs - r * cg.S;
      tma_load_4d(dst, &tmA, cg.c_off + cb * BK, tw * wbox * cg.stride - cg.pad + s, th * cg.hbox * cg.stride - cg.pad + r, ti,
                  bar);
    } else {
      tma_load_2d(dst, &tmA, kb * BK, m0, bar);
    }
  };

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
  pdl_trigger();  // the next layer's CTAs may start their prologue now
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      // Weights (B) do not depend on the previous kernel: the first stages'
      // B tiles are requested before waiting on it, the activations after.
      const int pre = min(STAGES, kb1 - kb0);
      for (int i = 0; i < pre; ++i) {
        uint8_t* sa = smem + i * L::STAGE_BYTES;
        mbar_expect_tx(&full[i], L::STAGE_BYTES);
        tma_load_2d(sa + L::A_BYTES, &tmB, (kb0 + i) * BK, n0, &full[i]);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) load_a(smem + i * L::STAGE_BYTES, kb0 + i, &full[i]);
      for (int kb = kb0 + pre, i = pre; kb < kb1; ++kb, ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        uint8_t* sa = smem + s * L::STAGE_BYTES;
        mbar_expect_tx(&full[s], L::STAGE_BYTES);
        load_a(sa, kb, &full[s]);
        tma_load_2d(sa + L::A_BYTES, &tmB, kb * BK, n0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (i / STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES), sb = sa + L::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          mma_bf16(tmem, smem_desc_sw128(sa + k * 32), smem_desc_sw128(sb + k * 32), idesc, (i | k) != 0);
        mma_commit(&empty[s]);  // the stage is free once these MMAs have read it
      }
      mma_commit(&accum_full);
    }
  } else if (warp < 4) {  // ---- epilogue operands -> smem, during the mainloop
    const int t = threadIdx.x - 64;  // 64 threads
#pragma unroll
    for (int j = t; j < BN; j += 64) {
      const int n = n0 + j;
      s_scale[j] = (scale && n < N) ? __ldg(scale + n) : 1.f;
      s_bias[j] = (bias && n < N) ? __ldg(bias + n) : 0.f;
    }
    pdl_wait();
    if (res) {  // residual tile, 16-byte pieces (ldr % 8 == 0 checked on the host), 8 loads in flight
      constexpr int PR = BN / 8, PIECES = BM * PR / 64, BATCH = PIECES < 8 ? PIECES : 8;
#pragma unroll 1
      for (int b = 0; b < PIECES; b += BATCH) {
        uint4 v[BATCH];
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
          const int i = t + (b + u) * 64, r = i / PR, c = (i - r * PR) * 8, gr = row_of(r);
          v[u] = make_uint4(0, 0, 0, 0);
          if (gr >= 0 && n0 + c + 8 <= N) {
            v[u] = *reinterpret_cast<const uint4*>(res + size_t(gr) * ldr + n0 + c);
          } else if (gr >= 0) {
            for (int q = 0; q < 8 && n0 + c + q < N; ++q)
              reinterpret_cast<uint16_t*>(&v[u])[q] = res[size_t(gr) * ldr + n0 + c + q];
          }
        }
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
          const int i = t + (b + u) * 64, r = i / PR, c = (i - r * PR) * 8;
          *reinterpret_cast<uint4*>(s_res + r * L::RES_LD + c) = v[u];
        }
      }
    }
    asm volatile("bar.arrive 1, 192;" ::: "memory");  // operands ready for warps 4-7
  } else {  // ---- epilogue: TMEM -> registers -> bf16 global
    pdl_wait();
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int rl = q * 32 + lane;
    const uint32_t tq = tmem + (uint32_t(q * 32) << 16);
    mbar_wait(&accum_full, 0);
    tc_fence_after();
    if (splits > 1) {
      // Split-K: park this split's fp32 partial tile in the (now idle) ring,
      // column-major so a warp's accesses are contiguous.
      float* part = reinterpret_cast<float*>(smem);
      // A split can own no k-blocks (ceil(kblocks / splits) * (splits - 1)
      // >= kblocks): no MMA wrote its accumulator, so its partial is zero.
      const bool no_k = kb0 >= kb1;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        if (no_k) {
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = 0u;
        } else {
          tmem_ld16(tq + uint32_t(c0), r);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) part[(c0 + j) * BM + rl] = __uint_as_float(r[j]);
      }
    } else {
      asm volatile("bar.sync 1, 192;" ::: "memory");  // residual / scale / bias in smem
      store_cols(std::integral_constant<int, 16>{}, 0, BN, rl, [&](int c0, float (&v)[16]) {
        uint32_t r[16];
        tmem_ld16(tq + uint32_t(c0), r);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
      });
    }
  }
  if (splits > 1) {
    // The splits of a tile form one thread-block cluster. After a cluster
    // barrier, split z reduces columns [z*BN/S, (z+1)*BN/S) of the tile by
    // reading every split's partial from distributed shared memory in split
    // order (deterministic), and runs the epilogue for that slice.
    cluster_sync();
    if (warp >= 4) {
      const int rl = (warp & 3) * 32 + lane, cols = BN / splits, cbeg = z * cols;
      const uint32_t local = smem_u32(smem);
      asm volatile("bar.sync 1, 192;" ::: "memory");
      auto reduce = [&](auto cw_tag) {
        constexpr int CW = decltype(cw_tag)::value;
        store_cols(cw_tag, cbeg, cbeg + cols, rl, [&](int c0, float (&v)[CW]) {
          float pv[kMaxSplits][CW];
#pragma unroll
          for (int zz = 0; zz < kMaxSplits; ++zz) {
            if (zz < splits) {
              const uint32_t base = map_shared_rank(local, uint32_t(zz));
#pragma unroll
              for (int j = 0; j < CW; ++j) pv[zz][j] = ld_dsmem_f32(base + uint32_t(((c0 + j) * BM + rl) * 4));
            }
          }
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            v[j] = pv[0][j];
#pragma unroll
            for (int zz = 1; zz < kMaxSplits; ++zz)
              if (zz < splits) v[j] += pv[zz][j];
          }
        });
      };
      if (cols % 16 == 0) reduce(std::integral_constant<int, 16>{});
      else reduce(std::integral_constant<int, 8>{});
    }
    cluster_sync();  // no split leaves while its partial may still be read
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
  constexpr size_t smem = Smem<BN, STAGES>::TOTAL;
  static_assert(smem <= 227 * 1024, "GEMM shared memory");
  static bool smem_set = false;
  if (!smem_set) {
    TRIMS_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem)));
    smem_set = true;
  }
  const Epilogue& e = p.e;
  const int kblocks = int((p.K + BK - 1) / BK);
  const int kper = (kblocks + p.splits - 1) / p.splits;
  dim3 grid(unsigned(tile_rows(p) / BM), unsigned((p.N + BN - 1) / BN), unsigned(p.splits));
  // PDL always; split-K launches the splits of a tile as one (1, 1, S) cluster
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = unsigned(p.splits);
  cfg.attrs = attr;
  cfg.numAttrs = p.splits > 1 ? 2 : 1;
  TRIMS_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, STAGES>, p.ta, p.tb, e.out, int(p.M), int(p.N), int(p.K),
                                int(e.ldo), e.scale, e.bias, e.residual, int(e.ldr), e.relu ? 1 : 0, kper, p.g));
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
  if (e.residual && (e.ldr % 8 || reinterpret_cast<uintptr_t>(e.residual) % 16))
    raise(Errc::InvalidArgument, "GEMM residual rows must be 16-byte aligned");
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
  if (p.splits < 1 || p.splits > kMaxSplits || (p.bn / p.splits) % 8)
    raise(Errc::InvalidArgument, "GEMM split count");
  switch (p.bn) {
    case 64: run_bn<64, 6>(p, stream); break;
    case 128: run_bn<128, 5>(p, stream); break;
    default: run_bn<256, 3>(p, stream); break;
  }
}

int pick_splits(uint64_t M, uint64_t N, uint64_t K, int bn, int sms) {
  // Split K only while the output tiles leave most SMs idle, each split keeps
  // >= 4 k-blocks and every split's column slice of the tile is >= 8 wide.
  const uint64_t tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn), kb = (K + BK - 1) / BK;
  int s = 1;
  // 8 splits only for the tiniest tile counts (<= 8 tiles, e.g. ResNet-50
  // layer3/4 3x3 convs at batch 1); measured slower for 16 tiles (VGG-16
  // conv5), profiles/r03d_split.log.
  const int max_s = tiles <= 8 ? kMaxSplits : 4;
  static const uint64_t min_kb = [] {  // k-blocks each split keeps at least (A/B: TRIMS_SPLIT_MINKB)
    const char* e = std::getenv("TRIMS_SPLIT_MINKB");
    return e ? uint64_t(std::max(1, std::atoi(e))) : uint64_t(4);
  }();
  while (s < max_s && bn / (s * 2) >= 8 && tiles * uint64_t(s * 2) <= uint64_t(sms) && kb / uint64_t(s * 2) >= min_kb)
    s *= 2;
  return s;
}

uint64_t tile_rows(const Prepared& p) {
  if (p.g.impl) return uint64_t(p.g.N) * p.g.tiles_h * p.g.tiles_w * BM;
  return (p.M + BM - 1) / BM * BM;
}

ConvGeom conv_geom(int N, int H, int W, int C, int R, int S, int stride, int pad, int P, int Q, int cgroup,
                   int c_off) {
  ConvGeom g;
  g.impl = 1;
  g.N = N, g.H = H, g.W = W, g.C = C, g.R = R, g.S = S, g.stride = stride, g.pad = pad, g.P = P, g.Q = Q;
  int wl = 0;
  while ((1 << wl) < Q && wl < 7) ++wl;   // Wbox = next power of two >= Q, at most 128
  while ((1 << wl) * stride > 256) --wl;  // TMA box dims are <= 256 elements
  while ((BM >> wl) * stride > 256) ++wl;
  g.wbox_log2 = wl;
  g.hbox = BM >> wl;
  g.tiles_w = (Q + (1 << wl) - 1) >> wl;
  g.tiles_h = (P + g.hbox - 1) / g.hbox;
  g.cblocks = (cgroup ? cgroup : C) / BK;
  g.c_off = c_off;
  return g;
}

Prepared prepare_conv(const void* act, const ConvGeom& g, const Operand& B, const Epilogue& e, int bn) {
  if (!g.impl || g.C % 8 || g.c_off % BK || g.c_off + g.cblocks * BK > g.C || g.hbox * g.stride > 256)
    raise(Errc::InvalidArgument, "implicit conv geometry");
  if (B.k != uint64_t(g.R) * g.S * g.cblocks * BK) raise(Errc::InvalidArgument, "implicit conv K mismatch");
  const uint64_t M = uint64_t(g.N) * g.P * g.Q;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  Prepared p = prepare({act, M, B.k, B.k}, B, e, bn ? bn : pick_bn(uint64_t(g.N) * g.tiles_h * g.tiles_w * BM, B.rows,
                                                                     sms));
  // replace the A map: 4-D NHWC, box {64 ch, Wbox, Hbox, 1} at element strides {1, st, st, 1}
  CUtensorMap m;
  cuuint64_t dims[4] = {cuuint64_t(g.C), cuuint64_t(g.W), cuuint64_t(g.H), cuuint64_t(g.N)};
  cuuint64_t strides[3] = {cuuint64_t(g.C) * 2, cuuint64_t(g.W) * g.C * 2, cuuint64_t(g.H) * g.W * g.C * 2};
  cuuint32_t box[4] = {uint32_t(BK), uint32_t((1 << g.wbox_log2) * g.stride), uint32_t(g.hbox * g.stride), 1};
  cuuint32_t estr[4] = {1, uint32_t(g.stride), uint32_t(g.stride), 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(act), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cu_check(r, "cuTensorMapEncodeTiled (conv)");
  p.ta = m;
  p.g = g;
  return p;
}

void launch(const Operand& A, const Operand& B, const Epilogue& e, cudaStream_t stream, int bn) {
  run(prepare(A, B, e, bn), stream);
}

}  // namespace trims::gemm
