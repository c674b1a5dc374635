// gemm.cu — K7: the conv/FC contraction on the 5th-gen tensor cores.
//
// D[M,N] = epi(A[M,K] . B[N,K]^T): A = activations (NHWC rows, or an im2col
// matrix), B = resident KRSC weights (row n = output channel n, K-major),
// bf16 operands, fp32 accumulation in TMEM, fused epilogue
//   out = relu?( acc * scale[n] + bias[n] + residual[m,n] )  -> bf16.
// One CTA per 128 x BN output tile: warp 0 issues TMA (SWIZZLE_128B boxes
// of 64 x rows) into a STAGES-deep mbarrier ring, warp 1 allocates TMEM and a
// single lane issues tcgen05.mma (M=128, N=BN, K=16 per instruction), warps
// 2-3 stage folded-BN scale/bias, warps 4-11 drain TMEM with tcgen05.ld and
// run the epilogue; the staged bf16 tile leaves by TMA store. Variants (all
// template parameters): split-K over an (1,1,S) cluster reducing through
// DSMEM bulk copies; 2-SM pairs (cta_group::2, M = 256 over a (2,1,1)
// cluster); weight multicast across M-tiles (off by default); a job table
// that runs two independent GEMMs in one launch; lean 2-CTA/SM variants.
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "cuda_util.hpp"
#include "device_mem.hpp"
#include "gemm.cuh"
#include "gemm.hpp"

namespace trims::gemm {

using namespace trims::sm100;

namespace {

// 12 warps: 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2-3 folded-BN
// scale/bias, 4-11 epilogue (two warps per TMEM lane quarter, each taking
// half of the tile's columns: at batch 1 the epilogue is latency-bound, so a
// second warp per scheduler halves it).
constexpr int BM = 128, BK = 64, kThreads = 384, kMaxSplits = 8;

#ifdef TRIMS_GEMM_TRACE
// Diagnostic build only (make EXTRA=-DTRIMS_GEMM_TRACE ...; scripts/gemm_trace.py):
// per CTA [M<<32|N, K<<32|z<<16|y, start, producer past pdl_wait, first stage
// full (MMA), accumulator full (epilogue), end, smid | x<<32, operand warps
// done, epilogue operands ready, epilogue stores done, split-K: partial
// parked, past the first cluster barrier, reduction done] (%globaltimer ns).
constexpr int kGTW = 16, kGTCap = 16384;
__device__ unsigned long long g_gtrace[kGTCap * kGTW];
__device__ unsigned int g_gtrace_n;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GT_SET(slot, i, v) \
  do {                     \
    if ((slot) < kGTCap) g_gtrace[(slot) * kGTW + (i)] = (v); \
  } while (0)
#endif

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// Packed fp32 pairs (sm_100 FFMA2 / FADD2).
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
        "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// Shared-memory plan of one CTA: the TMA ring, the residual tile (staged by
// TMA in SWIZZLE_128B boxes of 64 channels x 128 rows), for split-K launches
// the receive buffer (S partial blocks of this CTA's column slice), then
// folded-BN scale/bias.
template <int BN, int STAGES, int S, bool PAIR = false>
struct Smem {
  // PAIR (2-SM MMA): this CTA holds half of every B stage (BN/2 rows)
  static constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2,
                            STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t RING = STAGES * STAGE_BYTES;
  // split-K: only the 64-channel box holding this CTA's slice
  static constexpr uint32_t RES = RING, RES_BYTES = S > 1 ? BM * 128 : BM * BN * 2;
  // split z's partial of slice j (<= 128 rows x BN/S fp32) lands in block z of CTA j
  static constexpr uint32_t RECV = RES + RES_BYTES, RECV_BYTES = S > 1 ? BM * BN * 4 : 0;
  static constexpr uint32_t SCALE = RECV + RECV_BYTES, BIAS = SCALE + BN * 4;
  static constexpr uint32_t TOTAL = BIAS + BN * 4 + 1024;  // + 1 KiB realignment slack
  // split-K: the idle ring holds the outgoing partial blocks
  static_assert(S == 1 || RING >= BM * BN * 4, "split-K outgoing blocks exceed the ring");
};

// Fused 2x2 / stride-2 max pool of a staged bf16 tile (128 rows = Hbox x
// Wbox pixels, row hr * Wbox + wc; BN channels in SWIZZLE_128B boxes of 64
// channels x 128 rows): pooled row ph * Wbox/2 + pw = the max of rows
// 2ph * Wbox + 2pw + {0, 1, Wbox, Wbox + 1}, written in place to rows
// [0, 32) of the same boxes (every thread's reads precede every write). The
// max of bf16 values is one of them: bit-identical to pooling the stored
// tile. 256 threads (t), named barrier 2.
// 8 bf16 channels: the max of four pixels' 16-byte chunks
__device__ __forceinline__ uint4 max4_bf16x8(uint4 a, uint4 b, uint4 c, uint4 d) {
  auto mx = [](uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    const float lo = fmaxf(fmaxf(bf16_lo(a), bf16_lo(b)), fmaxf(bf16_lo(c), bf16_lo(d)));
    const float hi = fmaxf(fmaxf(bf16_hi(a), bf16_hi(b)), fmaxf(bf16_hi(c), bf16_hi(d)));
    return pack_bf16x2(lo, hi);
  };
  return make_uint4(mx(a.x, b.x, c.x, d.x), mx(a.y, b.y, c.y, d.y), mx(a.z, b.z, c.z, d.z), mx(a.w, b.w, c.w, d.w));
}

template <int BN>
__device__ __forceinline__ void pool_staged_tile(uint16_t* s_out, int t, int wl) {
  constexpr int CPR = BN / 8, PER = BN / 64;  // 16-byte chunks per row; pooled chunks per thread
  auto at = [&](int r, int c) {
    return reinterpret_cast<uint4*>(s_out + (c >> 6) * BM * 64 + r * 64 + ((((c & 63) >> 3) ^ (r & 7)) << 3));
  };
  uint4 v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = t + k * 256, pr = i / CPR, c = (i % CPR) * 8;
    const int ph = pr >> (wl - 1), pw = pr & ((1 << (wl - 1)) - 1);
    const int r = ((2 * ph) << wl) + 2 * pw;
    v[k] = max4_bf16x8(*at(r, c), *at(r + 1, c), *at(r + (1 << wl), c), *at(r + (1 << wl) + 1, c));
  }
  asm volatile("bar.sync 2, 256;" ::: "memory");  // every window read before any pooled row is written
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = t + k * 256;
    *at(i / CPR, (i % CPR) * 8) = v[k];
  }
}

// S = 1: one CTA per output tile. S > 1: grid.z = S splits of K, the S CTAs
// of a tile form one (1, 1, S) cluster and split z owns output columns
// [z*CW, (z+1)*CW), CW = BN / S. Measured building blocks in one 8-CTA
// cluster (scripts/dsmem_bench.cu, profiles/r3/dsmem_bench.jsonl): a relaxed
// cluster barrier 124 cycles, a release/acquire one after global stores
// ~1000 (it drains the stores), tcgen05.ld x16 x2 25 cycles, per-thread
// remote stores (st.async) ~245 cycles EACH (serialised), per-thread remote
// loads worse, and bulk DSMEM copies the cheapest way to move a block. So:
// every split parks its partial of each owner's slice in its (idle) ring as
// one compact block (only the tile's valid rows, chunk-major: [CW/4][rows][4]
// floats, conflict-free for both sides), S-1 warps each ship one block with
// one bulk copy completing bytes on the owner's mbarrier, the owner sums the
// S partials in split order (deterministic) and stores its slice to global
// straight from registers. A relaxed cluster barrier (arrive once my inputs
// have landed, wait at exit) keeps every source alive until its blocks are
// read.
//
// A launch runs one GEMM, or two independent GEMMs of the same tile width
// and split count side by side (a job table in the kernel parameters: blocks
// [0, t0) run job 0, the rest job 1) -- ResNet's downsample and the first
// 1x1 conv of a stage read the same input, so they share one launch instead
// of adding a dependent step to the chain.
struct alignas(64) Job {
  CUtensorMap ta, tb, tr, td;  // A, B, residual, output tile maps
  uint16_t* D;
  const float* scale;
  const float* bias;
  int M, N, K, ldd, has_res, relu, kper, tma_out, tiles_m;
  ConvGeom cg;
};
struct Jobs {
  Job j[2];
  int t0;  // output tiles of job 0 (blocks >= t0 belong to job 1)
};

// MC > 1: the MC CTAs of consecutive M-tiles (same N-tile, same split) form
// the cluster's x dimension and share every B (weight) stage by TMA
// multicast: each loads BN/MC rows of it into all MC CTAs, so L2 serves each
// weight tile once per MC tiles. A stage is refilled only when all MC CTAs'
// MMAs released it (multicast commits). Off by default (pick_mc): at batch 1
// it measured slower.
// Lean variants (BN <= 128, <= 3 stages, no split) must fit two CTAs per SM:
// registers capped at 65536 / (2 x 384) = 85 per thread.
template <int BN, int STAGES, int S>
constexpr int min_ctas() { return (BN <= 128 && STAGES <= 3 && S == 1) ? 2 : 1; }

template <int BN, int STAGES, int S, int MC>
__global__ void __launch_bounds__(kThreads, min_ctas<BN, STAGES, S>()) gemm_tc_kernel(const __grid_constant__ Jobs jobs) {
  // MC < 0: a 2-SM pair (tcgen05 cta_group::2): the two CTAs of consecutive
  // M-tiles form a (2, 1, 1) cluster; the leader issues M = 256 MMAs over both
  // CTAs' A tiles and B halves, each CTA's TMEM holds its 128 rows of D.
  constexpr bool PAIR = MC < 0;
  constexpr int CX = PAIR ? -MC : MC;  // cluster x extent
  static_assert(!PAIR || (S == 1 && MC == -2 && BN >= 128), "2-SM pairs: unsplit, BN >= 128");
  const int jb = int(blockIdx.x) < jobs.t0 ? 0 : 1;
  const Job& J = jobs.j[jb];
  const int tile = int(blockIdx.x) - (jb ? jobs.t0 : 0);  // this job's output tile: M-tile fastest
  const CUtensorMap& tmA = J.ta;
  const CUtensorMap& tmB = J.tb;
  const CUtensorMap& tmR = J.tr;
  const CUtensorMap& tmD = J.td;
  uint16_t* const D = J.D;
  const float* __restrict__ scale = J.scale;
  const float* __restrict__ bias = J.bias;
  const int M = J.M, N = J.N, K = J.K, ldd = J.ldd, has_res = J.has_res, relu = J.relu, kper = J.kper,
            tma_out = J.tma_out;
  // by value: the producer's per-k-block address math reads these from
  // registers (a reference into the runtime-indexed job made each an indexed
  // constant load in that loop: VGG-16 +4.5 %)
  const ConvGeom cg = J.cg;
  const int mt = tile % J.tiles_m, nt = tile / J.tiles_m;
  const uint32_t cx = uint32_t(mt % CX);  // rank along the cluster's x dimension (multicast group / pair)
  // cluster ranks: x (multicast group) fastest, then the split z
  auto crank = [&](uint32_t x, uint32_t zz) { return x + uint32_t(CX) * zz; };
  constexpr bool SPLIT = S > 1;
  constexpr int CW = BN / S;  // split-K: columns of the slice this CTA owns
  static_assert(CW % 8 == 0, "split slices are >= 8 columns");
  using L = Smem<BN, STAGES, S, PAIR>;
  constexpr uint32_t TMEM_COLS = BN;  // 64 / 128 / 256: powers of two >= 32
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], accum_full, res_full, recv_full;
  __shared__ uint32_t tmem_base;
  // 1 KiB-aligned base for the SWIZZLE_128B tiles, derived from smem_raw by
  // pointer arithmetic (an integer round trip would drop the shared address
  // space and turn every epilogue smem access into a generic load)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* s_scale = reinterpret_cast<float*>(smem + L::SCALE);
  float* s_bias = reinterpret_cast<float*>(smem + L::BIAS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = mt * BM, n0 = nt * BN;
  const int z = SPLIT ? int(blockIdx.z) : 0;
  const int kblocks = (K + BK - 1) / BK;
  const int kb0 = z * kper, kb1 = min(kblocks, kb0 + kper);  // this split's k-blocks
  // residual boxes staged: all BN/64 of the tile, or the one holding the slice
  const int rbox0 = SPLIT ? (z * CW) / 64 : 0, rboxes = SPLIT ? 1 : (BN + 63) / 64;
  // Implicit conv: this tile = image ti, output rows [th*hbox, +hbox), cols [tw*wbox, +wbox).
  int ti = 0, th = 0, tw = 0;
  if (cg.impl) {
    tw = mt % cg.tiles_w;
    th = (mt / cg.tiles_w) % cg.tiles_h;
    ti = mt / (cg.tiles_w * cg.tiles_h);
  }
  const int wbox = 1 << cg.wbox_log2;
  // Global output row of tile row rl, or -1 outside the output.
  auto row_of = [&](int rl) -> int {
    if (!cg.impl) return m0 + rl < M ? m0 + rl : -1;
    const int h = th * cg.hbox + (rl >> cg.wbox_log2), w = tw * wbox + (rl & (wbox - 1));
    return (h < cg.P && w < cg.Q) ? (ti * cg.P + h) * cg.Q + w : -1;
  };
  // Valid rows of the tile (hv x qv box of the output; qv = 1 for a plain
  // GEMM) and tile row -> compact index among them (-1 if outside).
  // (a padding tile of a multicast group has none)
  const int hv = max(0, cg.impl ? min(cg.hbox, cg.P - th * cg.hbox) : min(BM, M - m0));
  const int qv = max(0, cg.impl ? min(wbox, cg.Q - tw * wbox) : 1);
  const int nvalid = hv * qv;
  auto cidx = [&](int rl) -> int {
    if (!cg.impl) return rl < hv ? rl : -1;
    const int hr = rl >> cg.wbox_log2, wc = rl & (wbox - 1);
    return (hr < hv && wc < qv) ? hr * qv + wc : -1;
  };
  // Epilogue of CW (8 or 16) tile columns c0.. of tile row rl: scale, bias,
  // residual, ReLU, bf16 -> back into the staging tile (the residual's
  // swizzled smem box, in place: each 16-byte chunk is read and rewritten by
  // the same thread). copy_out then writes the tile rows to global memory
  // whole: a thread per row storing its own 16-byte chunks puts every chunk
  // of a warp store in a different line (one L1 wavefront per 16 bytes, ~1
  // cycle each: ~1000 cycles for a 128 x 64 tile); row-major copy-out packs
  // a warp store into 128-byte row segments.
  uint16_t* s_out = reinterpret_cast<uint16_t*>(smem + L::RES);
  auto stage_at = [&](int rl, int c) {  // staging address of tile (row rl, column c), c % 8 == 0
    const int box = c / 64 - rbox0, chunk = ((c & 63) >> 3) ^ (rl & 7);
    return s_out + box * BM * 64 + rl * 64 + chunk * 8;
  };
  // scale, bias, residual (r4: its 8 bf16 values), ReLU of 8 values at tile
  // column c of row rl -> 4 bf16 pairs. Scale/bias are read with loads the
  // compiler may hoist above earlier shared-memory stores (they are never
  // written in the epilogue): C++ loads would each wait behind the previous
  // chunk's staging store (possible aliasing), a serial chain of round trips.
  // HR / RL: compile-time residual / ReLU (the unsplit epilogue runs a
  // specialised copy: predicated-off adds and max still cost issue slots,
  // and with two warps per scheduler the epilogue is issue-bound)
  auto epi8t = [&](int c, const float* v, uint32_t* o, const uint4 r4, auto hr_tag, auto rl_tag) {
    constexpr bool HR = decltype(hr_tag)::value, RL = decltype(rl_tag)::value;
    const uint32_t rw[4] = {r4.x, r4.y, r4.z, r4.w};
    const float4 sc0 = lds_f4(s_scale + c), sc1 = lds_f4(s_scale + c + 4);
    const float4 bi0 = lds_f4(s_bias + c), bi1 = lds_f4(s_bias + c + 4);
    const float sc[8] = {sc0.x, sc0.y, sc0.z, sc0.w, sc1.x, sc1.y, sc1.z, sc1.w};
    const float bi[8] = {bi0.x, bi0.y, bi0.z, bi0.w, bi1.x, bi1.y, bi1.z, bi1.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // packed pairs (FFMA2 / FADD2: two independent round-to-nearest fp32
      // ops, bit-identical to the scalar fma + add, half the issue slots)
      float2 ab = fma2(make_float2(v[2 * j], v[2 * j + 1]), make_float2(sc[2 * j], sc[2 * j + 1]),
                       make_float2(bi[2 * j], bi[2 * j + 1]));
      if constexpr (HR) ab = add2(ab, make_float2(bf16_lo(rw[j]), bf16_hi(rw[j])));
      if constexpr (RL) {
        ab.x = fmaxf(ab.x, 0.f);
        ab.y = fmaxf(ab.y, 0.f);
      }
      o[j] = pack_bf16x2(ab.x, ab.y);
    }
  };
  auto epi8r = [&](int c, const float* v, uint32_t* o, const uint4 r4) {  // runtime flags (split path)
    using T = std::true_type;
    using F = std::false_type;
    if (has_res) {
      if (relu) epi8t(c, v, o, r4, T{}, T{});
      else epi8t(c, v, o, r4, T{}, F{});
    } else {
      if (relu) epi8t(c, v, o, r4, F{}, T{});
      else epi8t(c, v, o, r4, F{}, F{});
    }
  };
  auto epi8 = [&](int rl, int c, const float* v, uint32_t* o) {
    epi8r(c, v, o, has_res ? *reinterpret_cast<const uint4*>(stage_at(rl, c)) : make_uint4(0, 0, 0, 0));
  };
  // W staged columns: every residual chunk is read before the first
  // in-place store, then converted and stored chunk by chunk
  auto finish_t = [&](int rl, int c0, auto cw_tag, const float* v, auto hr_tag, auto rl_tag) {
    constexpr int W = decltype(cw_tag)::value;
    constexpr bool HR = decltype(hr_tag)::value;
    // the row's staging address once; chunk q of the 16-byte chunks at (chunk0 + q) ^ (rl & 7)
    uint16_t* srow = s_out + (c0 / 64 - rbox0) * BM * 64 + rl * 64;
    const int chunk0 = (c0 & 63) >> 3, sw = rl & 7;
    uint4 res[W / 8];
#pragma unroll
    for (int q = 0; q < W / 8; ++q)
      res[q] = HR ? *reinterpret_cast<const uint4*>(srow + (((chunk0 + q) ^ sw) << 3)) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int q = 0; q < W / 8; ++q) {
      uint32_t o[4];
      epi8t(c0 + 8 * q, v + 8 * q, o, res[q], hr_tag, rl_tag);
      *reinterpret_cast<uint4*>(srow + (((chunk0 + q) ^ sw) << 3)) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  };
  // 8 finished columns of tile row rl -> D (one 16-byte store when aligned)
  auto store8 = [&](int row, int n, const uint32_t* o) {
    uint16_t* dp = D + size_t(row) * ldd + n;
    if (ldd % 8 == 0 && n + 8 <= N) {
      *reinterpret_cast<uint4*>(dp) = make_uint4(o[0], o[1], o[2], o[3]);
    } else {
      for (int j = 0; j < 8 && n + j < N; ++j) dp[j] = uint16_t(o[j >> 1] >> (16 * (j & 1)));
    }
  };
  // Staged tile columns [cbeg, cbeg + W) -> D, row-major: consecutive
  // threads take consecutive 16-byte chunks of a row. 256 epilogue threads.
  auto copy_out = [&](int t, int cbeg, int W) {
    const int lg = __ffs(W / 8) - 1;  // chunks per row = W / 8, a power of two
#pragma unroll 4
    for (int k = t; k < (BM << lg); k += 256) {
      const int rl = k >> lg, c = cbeg + (k & ((1 << lg) - 1)) * 8;
      const int row = row_of(rl), n = n0 + c;
      if (row < 0 || n >= N) continue;
      const uint4 v = *reinterpret_cast<const uint4*>(stage_at(rl, c));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      store8(row, n, w);
    }
  };
  auto load_a = [&](void* dst, int kb, uint64_t* bar) {
    if (cg.impl) {
      const int rs = kb / cg.cblocks, cb = kb - rs * cg.cblocks, r = rs / cg.S, s = rs - r * cg.S;
      const int c0 = cg.c_off + cb * BK, c1 = tw * wbox * cg.stride - cg.pad + s,
                c2 = th * cg.hbox * cg.stride - cg.pad + r;
      if constexpr (MC < 0) {
        tma_load_4d_pair(dst, &tmA, c0, c1, c2, ti, map_shared_rank(smem_u32(bar), 0u));  // leader = rank 0
      } else {
        tma_load_4d(dst, &tmA, c0, c1, c2, ti, bar);
      }
    } else {
      if constexpr (MC < 0) tma_load_2d_pair(dst, &tmA, kb * BK, m0, map_shared_rank(smem_u32(bar), 0u));
      else tma_load_2d(dst, &tmA, kb * BK, m0, bar);
    }
  };

#ifdef TRIMS_GEMM_TRACE
  __shared__ unsigned int gt_slot;
  if (threadIdx.x == 0) {
    gt_slot = atomicAdd(&g_gtrace_n, 1u);
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    GT_SET(gt_slot, 0, (uint64_t(M) << 32) | uint32_t(N));
    GT_SET(gt_slot, 1, (uint64_t(K) << 32) | (blockIdx.z << 16) | uint32_t(nt));
    GT_SET(gt_slot, 2, gtimer());
    GT_SET(gt_slot, 7, smid | (uint64_t(mt) << 32));
  }
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC > 1 ? MC : 1);  // released by the MMAs of all MC CTAs sharing the stage
    }
    mbar_init(&accum_full, 1);
    mbar_init(&res_full, 1);
    mbar_init(&recv_full, 1);
    fence_barrier_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (has_res) prefetch_tmap(&tmR);
    if (!SPLIT && tma_out) prefetch_tmap(&tmD);
    // the other splits' blocks of this CTA's slice, in bytes
    if (SPLIT) mbar_expect_tx(&recv_full, uint32_t((S - 1) * nvalid * CW * 4));
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_pair<TMEM_COLS>(&tmem_base);
    else tmem_alloc<TMEM_COLS>(&tmem_base);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();  // the next layer's CTAs may start their prologue now
  // every split's receive barrier is initialised before anyone pushes into it
  // (off the critical path: this runs under the previous layer's tail)
  if (SPLIT || MC > 1 || PAIR) {
    cluster_arrive_relaxed();
    cluster_wait();
  }
  const uint32_t tmem = tmem_base;

  // multicast group of this CTA (same split z): cluster ranks z*MC .. z*MC+MC-1
  const uint16_t mc_mask = uint16_t(((1u << MC) - 1u) << (uint32_t(MC) * uint32_t(z)));
  // B stage of k-block kb: whole (MC = 1), or this CTA's BN/MC rows to the group
  // pair: every load completes on the LEADER's barrier (its MMA consumes both CTAs' stages)
  auto pair_bar = [&](uint64_t* bar) { return map_shared_rank(smem_u32(bar), crank(0, uint32_t(z))); };
  auto load_b = [&](uint8_t* sa, int kb, uint64_t* bar) {
    if constexpr (PAIR) {
      tma_load_2d_pair(sa + L::A_BYTES, &tmB, kb * BK, n0 + int(cx) * (BN / 2), pair_bar(bar));
    } else if constexpr (MC == 1) {
      tma_load_2d(sa + L::A_BYTES, &tmB, kb * BK, n0, bar);
    } else {
      constexpr int SR = BN / MC;  // rows per slice (>= 16: 1 KiB-aligned swizzle atoms)
      tma_load_2d_mc(sa + L::A_BYTES + cx * SR * 128, &tmB, kb * BK, n0 + int(cx) * SR, bar, mc_mask);
    }
  };
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      // Weights (B) do not depend on the previous kernel: the first stages'
      // B tiles are requested before waiting on it, the activations after.
      const int pre = min(STAGES, kb1 - kb0);
      // pair: the leader's barrier counts both CTAs' bytes; the peer only loads
      auto expect = [&](uint64_t* bar) {
        if constexpr (PAIR) {
          if (cx == 0) mbar_expect_tx(bar, 2 * L::STAGE_BYTES);
        } else {
          mbar_expect_tx(bar, L::STAGE_BYTES);
        }
      };
      for (int i = 0; i < pre; ++i) {
        uint8_t* sa = smem + i * L::STAGE_BYTES;
        expect(&full[i]);
        load_b(sa, kb0 + i, &full[i]);
      }
      pdl_wait();
#ifdef TRIMS_GEMM_TRACE
      GT_SET(gt_slot, 3, gtimer());
#endif
      for (int i = 0; i < pre; ++i) load_a(smem + i * L::STAGE_BYTES, kb0 + i, &full[i]);
      if (has_res) {  // the residual tile rides the same engine, behind the first A tiles
        mbar_expect_tx(&res_full, uint32_t(rboxes * BM * 128));
        for (int b = 0; b < rboxes; ++b) {
          uint8_t* dst = smem + L::RES + b * BM * 128;
          const int c = n0 + (rbox0 + b) * 64;
          if (cg.impl) tma_load_4d(dst, &tmR, c, tw * wbox, th * cg.hbox, ti, &res_full);
          else tma_load_2d(dst, &tmR, c, m0, &res_full);
        }
      }
      for (int kb = kb0 + pre, i = pre; kb < kb1; ++kb, ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        uint8_t* sa = smem + s * L::STAGE_BYTES;
        expect(&full[s]);
        load_a(sa, kb, &full[s]);
        load_b(sa, kb, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && (!PAIR || cx == 0)) {  // ---- MMA issuer (a pair's leader only)
      constexpr uint32_t idesc = idesc_bf16_f32(PAIR ? 2 * BM : BM, BN);
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (i / STAGES) & 1);
#ifdef TRIMS_GEMM_TRACE
        if (i == 0) GT_SET(gt_slot, 4, gtimer());
#endif
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES), sb = sa + L::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          if constexpr (PAIR)
            mma_bf16_pair(tmem, smem_desc_sw128(sa + k * 32), smem_desc_sw128(sb + k * 32), idesc, (i | k) != 0);
          else
            mma_bf16(tmem, smem_desc_sw128(sa + k * 32), smem_desc_sw128(sb + k * 32), idesc, (i | k) != 0);
        }
        // the stage is free once these MMAs have read it; with multicast every
        // CTA of the group refills it, so each needs this CTA's release --
        // except for the last STAGES k-blocks, whose stages are never refilled
        // (no release arrives at a peer that may already have exited)
        if constexpr (PAIR) {
          if (i + STAGES < kb1 - kb0) mma_commit_pair(&empty[s], uint16_t(3));  // both CTAs' stage s
        } else if constexpr (MC == 1) {
          mma_commit(&empty[s]);
        } else if (i + STAGES < kb1 - kb0) {
          mma_commit_mc(&empty[s], mc_mask);
        }
      }
      if constexpr (PAIR) mma_commit_pair(&accum_full, uint16_t(3));  // each CTA's 128 rows of D
      else mma_commit(&accum_full);
    }
  } else if (warp < 4) {  // ---- folded-BN scale / bias -> smem (bind-time constants)
    const int t = threadIdx.x - 64;  // 64 threads
#pragma unroll
    for (int j = t; j < BN; j += 64) {
      const int n = n0 + j;
      s_scale[j] = (scale && n < N) ? __ldg(scale + n) : 1.f;
      s_bias[j] = (bias && n < N) ? __ldg(bias + n) : 0.f;
    }
#ifdef TRIMS_GEMM_TRACE
    if (t == 0) GT_SET(gt_slot, 8, gtimer());
#endif
    asm volatile("bar.arrive 1, 320;" ::: "memory");  // operands ready for warps 4-11
  } else {  // ---- epilogue: TMEM -> registers -> bf16 global
    pdl_wait();
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;  // which half of the columns
    const int rl = q * 32 + lane;
    const uint32_t tq = tmem + (uint32_t(q * 32) << 16);
    mbar_wait(&accum_full, 0);
#ifdef TRIMS_GEMM_TRACE
    if (threadIdx.x == 128) GT_SET(gt_slot, 5, gtimer());
#endif
    tc_fence_after();
    if constexpr (!SPLIT) {
      asm volatile("bar.sync 1, 320;" ::: "memory");  // scale / bias in smem
      s_scale = after_here(s_scale);  // the clobber-free scale / bias loads stay below the barrier
      s_bias = after_here(s_bias);
      if (has_res) mbar_wait(&res_full, 0);
#ifdef TRIMS_GEMM_TRACE
      if (threadIdx.x == 128) GT_SET(gt_slot, 9, gtimer());
#endif
#ifdef TRIMS_EPI_COMPACT
      // A/B: one 8-column group per TMEM round trip (tcgen05.ld ~25 cycles),
      // one copy of the epilogue code (the epilogue runs once per CTA, so
      // its instructions are fetched cold; a compact loop fetches them once)
#pragma unroll 1
      for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 8) {
        uint32_t r[8], o[4];
        tmem_ld8_nw(tq + uint32_t(c), r);
        tmem_wait_ld();
        epi8(rl, c, reinterpret_cast<const float*>(r), o);
        *reinterpret_cast<uint4*>(stage_at(rl, c)) = make_uint4(o[0], o[1], o[2], o[3]);
      }
      asm volatile("bar.sync 2, 256;" ::: "memory");  // the whole tile is staged
      {
        constexpr int lg = BN == 64 ? 3 : BN == 128 ? 4 : 5;  // 16-byte chunks per row
#pragma unroll 1
        for (int k = threadIdx.x - 128; k < (BM << lg); k += 256) {
          const int rr = k >> lg, c = (k & ((1 << lg) - 1)) * 8;
          const int row = row_of(rr), n = n0 + c;
          if (row < 0 || n >= N) continue;
          const uint4 v = *reinterpret_cast<const uint4*>(stage_at(rr, c));
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
          store8(row, n, w);
        }
      }
#else
      // this warp's BN/2 columns, 32 per TMEM round trip
#pragma unroll 1
      for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += 32) {
#ifdef TRIMS_GEMM_TRACE
        const long long q0 = clock64();
#endif
        uint32_t r[32];
        tmem_ld16_nw(tq + uint32_t(c0), r);
        tmem_ld16_nw(tq + uint32_t(c0 + 16), r + 16);
        tmem_wait_ld();
#ifdef TRIMS_GEMM_TRACE
        {  // diagnostic: consume the loaded registers (data actually arrived)
          uint32_t x = 0;
#pragma unroll
          for (int u = 0; u < 32; ++u) x ^= r[u];
          asm volatile("" ::"r"(x));
        }
        const long long q1 = clock64();
#endif
        {
          auto both = [&](auto hr, auto rlu) {
            finish_t(rl, c0, std::integral_constant<int, 32>{}, reinterpret_cast<const float*>(r), hr, rlu);
          };
          using T = std::true_type;
          using F = std::false_type;
          if (has_res) {
            if (relu) both(T{}, T{});
            else both(T{}, F{});
          } else {
            if (relu) both(F{}, T{});
            else both(F{}, F{});
          }
        }
#ifdef TRIMS_GEMM_TRACE
        if (threadIdx.x == 128 && c0 == 0) {  // cycles: TMEM loads until consumed, then the two finishes
          GT_SET(gt_slot, 12, uint64_t(q1 - q0));
          GT_SET(gt_slot, 13, uint64_t(clock64() - q1));
        }
#endif
      }
#ifdef TRIMS_GEMM_TRACE
      if (threadIdx.x == 128) GT_SET(gt_slot, 14, gtimer());
#endif
      if (tma_out) fence_proxy_async_smem();  // staged tile -> async proxy (the TMA store reads it)
      asm volatile("bar.sync 2, 256;" ::: "memory");  // the whole tile is staged
#ifdef TRIMS_GEMM_TRACE
      if (threadIdx.x == 128) GT_SET(gt_slot, 15, gtimer());
#endif
      if (cg.pool) {  // fused 2x2 max pool: the pooled tile replaces rows [0, 32)
        pool_staged_tile<BN>(s_out, threadIdx.x - 128, cg.wbox_log2);
        fence_proxy_async_smem();
        asm volatile("bar.sync 2, 256;" ::: "memory");
      }
      if (tma_out) {
        // one TMA store per 64-channel box; the engine clips rows / channels
        // outside the output. The CTA stays until the boxes are read out.
        if (threadIdx.x == 128) {
          const int pl = cg.pool;  // pooled: box coordinates halve
#pragma unroll
          for (int b = 0; b < BN / 64; ++b) {
            const uint16_t* src = s_out + b * BM * 64;
            if (cg.impl) tma_store_4d(&tmD, src, n0 + b * 64, (tw * wbox) >> pl, (th * cg.hbox) >> pl, ti);
            else tma_store_2d(&tmD, src, n0 + b * 64, m0);
          }
          bulk_commit();
          bulk_wait_read();
        }
      } else {
        copy_out(threadIdx.x - 128, 0, BN);
      }
#endif
#ifdef TRIMS_GEMM_TRACE
      if (threadIdx.x == 128) GT_SET(gt_slot, 10, gtimer());
#endif
    } else {
      // This warp's half of the accumulator row in one TMEM round trip. A
      // split can own no k-blocks (ceil(kblocks / S) * (S - 1) >= kblocks):
      // no MMA wrote its accumulator, so its partial is zero.
      constexpr int HC = BN / 2;
      uint32_t r[HC];
      if (kb0 >= kb1) {
#pragma unroll
        for (int u = 0; u < HC; ++u) r[u] = 0u;
      } else {
#pragma unroll
        for (int c = 0; c < HC; c += 16) tmem_ld16_nw(tq + uint32_t(half * HC + c), r + c);
        tmem_wait_ld();
      }
      // park: column group c (4 floats) of owner j -> block j, chunk (c % CW) / 4,
      // compact row; my own slice goes straight into my receive block z
      const uint32_t blk = uint32_t(nvalid) * CW * 4;
      const int ci = cidx(rl);
      if (ci >= 0) {
#pragma unroll
        for (int c = 0; c < HC; c += 4) {
          const int col = half * HC + c, j = col / CW, kk = (col % CW) / 4;
          uint8_t* base = j == z ? smem + L::RECV + uint32_t(z) * blk : smem + uint32_t(j) * blk;
          *reinterpret_cast<float4*>(base + (uint32_t(kk) * nvalid + ci) * 16) =
              make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]), __uint_as_float(r[c + 2]),
                          __uint_as_float(r[c + 3]));
        }
      }
#ifdef TRIMS_GEMM_TRACE
      if (threadIdx.x == 128) GT_SET(gt_slot, 14, gtimer());
#endif
      fence_proxy_async_smem();
      asm volatile("bar.sync 2, 256;" ::: "memory");  // all outgoing blocks written
#ifdef TRIMS_GEMM_TRACE
      if (threadIdx.x == 128) GT_SET(gt_slot, 15, gtimer());
#endif
      // warp 4 + i ships block (z + 1 + i) % S: S - 1 bulk copies issued in parallel
      if (lane == 0 && warp - 4 < S - 1) {
        const uint32_t j = uint32_t(z + 1 + warp - 4) % S;
        if (blk)  // (a padding tile of a multicast group has no rows)
          bulk_copy_to_cluster(map_shared_rank(smem_u32(smem + L::RECV) + uint32_t(z) * blk, crank(cx, j)),
                               smem_u32(smem) + j * blk, blk, map_shared_rank(smem_u32(&recv_full), crank(cx, j)));
      }
#ifdef TRIMS_GEMM_TRACE
      if (threadIdx.x == 128) GT_SET(gt_slot, 11, gtimer());
#endif
      // every other split's block of my slice has landed (bulk-copied data is
      // visible to the observers of its mbarrier's phase completion, like a
      // TMA load's); from here on nobody reads my outgoing blocks but me...
      mbar_wait(&recv_full, 0);
      // ...and my peers' blocks are read: they may leave once all owners say so
      cluster_arrive_relaxed();
#ifdef TRIMS_GEMM_TRACE
      if (threadIdx.x == 128) GT_SET(gt_slot, 12, gtimer());
#endif
      asm volatile("bar.sync 1, 320;" ::: "memory");  // scale / bias in smem; own partials written
      s_scale = after_here(s_scale);  // the clobber-free scale / bias loads stay below the barrier
      s_bias = after_here(s_bias);
      if (has_res) mbar_wait(&res_full, 0);
      // reduce: thread t takes tile row t % 128 and 8-column groups t / 128,
      // + 2, ... of the slice; v = p0 + p1 + ... in split order (deterministic)
      const int t = threadIdx.x - 128, rr = t & (BM - 1), cr = cidx(rr), row = row_of(rr);
      const uint8_t* recv = smem + L::RECV;
      if (cr >= 0) {
#pragma unroll
        for (int g = t >> 7; g < CW / 8; g += 2) {
          float v[8];
#pragma unroll
          for (int zz = 0; zz < S; ++zz) {
            const float4 a = *reinterpret_cast<const float4*>(recv + zz * blk + (uint32_t(2 * g) * nvalid + cr) * 16);
            const float4 b =
                *reinterpret_cast<const float4*>(recv + zz * blk + (uint32_t(2 * g + 1) * nvalid + cr) * 16);
            const float pv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = zz ? v[u] + pv[u] : pv[u];
          }
          const int c = z * CW + 8 * g;
          if (n0 + c < N) {
            uint32_t o[4];
            epi8(rr, c, v, o);
            if (cg.pool == 3) {  // global average pool: bf16 outputs as fp32 [pixel][CW] in the idle ring
              float* st = reinterpret_cast<float*>(smem + uint32_t(S) * uint32_t(nvalid) * CW * 4) + cr * CW + 8 * g;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                st[2 * u] = bf16_lo(o[u]);
                st[2 * u + 1] = bf16_hi(o[u]);
              }
            } else if (cg.pool)  // staged (the residual box is free: no residual with a fused pool)
              *reinterpret_cast<uint4*>(smem + L::RES + (uint32_t(rr) * (CW / 8) + g) * 16) =
                  make_uint4(o[0], o[1], o[2], o[3]);
            else
              store8(row, n0 + c, o);
          }
        }
      }
      if (cg.pool == 3) {
        // fused global average pool: the tile holds whole images (host-checked:
        // an implicit conv's tile = one image ti; a 1x1 conv's single M-tile =
        // all M / HW images), its compact rows are the pixels in order. Thread
        // q averages column q % CW of image q / CW in nn::avgpool_kernel's exact
        // summation order (32 pixel slices j = k, k + 32, ..., then the slices
        // in order, / HW): bit-identical to pooling the stored map. The staging
        // sits past my outgoing blocks in the ring (host-checked:
        // (S + 1) * rows <= 128 * S).
        asm volatile("bar.sync 2, 256;" ::: "memory");  // every pixel of the slice staged
        const float* st = reinterpret_cast<const float*>(smem + uint32_t(S) * uint32_t(nvalid) * CW * 4);
        const int HW = cg.P * cg.Q, imgs = nvalid / HW;
        // slice sums (image, k, column) into the receive blocks (every partial
        // was read before the barrier above), 256 in parallel...
        float* slc = reinterpret_cast<float*>(smem + L::RECV);
        for (int q = t; q < 32 * CW * imgs; q += 256) {
          const int col = q % CW, k = (q / CW) % 32, im = q / (32 * CW);
          const float* sp = st + im * HW * CW + col;
          float sl = 0.f;
          for (int j = k; j < HW; j += 32) sl += sp[j * CW];
          slc[q] = sl;
        }
        asm volatile("bar.sync 2, 256;" ::: "memory");
        // ...then each (image, column) adds its 32 slices in order (independent
        // loads first, one dependent add chain)
        for (int q = t; q < CW * imgs; q += 256) {
          const int col = q % CW, im = q / CW;
          float v[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = slc[(im * 32 + k) * CW + col];
          float tot = 0.f;
#pragma unroll
          for (int k = 0; k < 32; ++k) tot += v[k];
          if (n0 + z * CW + col < N)
            D[size_t(cg.impl ? ti : im) * ldd + n0 + z * CW + col] =
                uint16_t(pack_bf16x2(tot / float(HW), 0.f) & 0xffffu);
        }
      } else if (cg.pool) {  // fused 2x2 max pool of my slice: 32 pooled rows x CW / 8 chunks
        asm volatile("bar.sync 2, 256;" ::: "memory");  // every row of the slice staged
        constexpr int CH = CW / 8;
        if (t < 32 * CH) {
          const int pr = t / CH, gch = t % CH, wl = cg.wbox_log2;
          const int ph = pr >> (wl - 1), pw = pr & ((1 << (wl - 1)) - 1), r = ((2 * ph) << wl) + 2 * pw;
          const int P2 = cg.P / 2, Q2 = cg.Q / 2, py = th * (cg.hbox / 2) + ph, px = tw * (wbox / 2) + pw;
          const int c = z * CW + 8 * gch;
          if (py < P2 && px < Q2 && n0 + c < N) {  // a valid pooled pixel's window rows are all valid
            auto at = [&](int rw) {
              return *reinterpret_cast<const uint4*>(smem + L::RES + (uint32_t(rw) * CH + gch) * 16);
            };
            const uint4 m = max4_bf16x8(at(r), at(r + 1), at(r + wbox), at(r + wbox + 1));
            const uint32_t o[4] = {m.x, m.y, m.z, m.w};
            if (cg.pool == 2) {  // NCHW (torch's flatten order for the FC layer that follows)
              uint16_t* dp = D + (size_t(ti) * ldd + n0 + c) * P2 * Q2 + size_t(py) * Q2 + px;
              for (int j = 0; j < 8 && n0 + c + j < N; ++j) dp[size_t(j) * P2 * Q2] = uint16_t(o[j >> 1] >> (16 * (j & 1)));
            } else {
              store8((ti * P2 + py) * Q2 + px, n0 + c, o);
            }
          }
        }
      }
#ifdef TRIMS_GEMM_TRACE
      if (threadIdx.x == 128) GT_SET(gt_slot, 13, gtimer());
#endif
    }
  }
  // split-K: no CTA leaves while a bulk copy may still be reading its
  // outgoing blocks (every owner arrived after receiving all its bytes)
  if constexpr (SPLIT) {
    if (warp < 4) cluster_arrive_relaxed();
    cluster_wait();
  } else if constexpr (MC > 1 || PAIR) {
    // no CTA leaves while a group peer's multicast loads / releases may still
    // target it (every peer arrives once its own MMAs are complete); a pair
    // also frees its TMEM together
    cluster_arrive_relaxed();
    cluster_wait();
  }
  tc_fence_before();
  __syncthreads();
#ifdef TRIMS_GEMM_TRACE
  if (threadIdx.x == 0) GT_SET(gt_slot, 6, gtimer());
#endif
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_free_pair<TMEM_COLS>(tmem);
    else tmem_free<TMEM_COLS>(tmem);
  }
}

// Persistent variant for multi-wave layers (batch > 1; VGG's first layers at
// batch 1): one CTA per SM walks the output tiles t = blockIdx.x,
// + gridDim.x, ... (M-tile fastest, so co-running CTAs share the weight
// tile). The TMA ring runs on across tiles, and TWO TMEM accumulators let
// tile i's epilogue (TMEM -> bf16 staging -> TMA store) overlap tile i+1's
// k-loop: the one-tile-per-CTA kernel leaves the tensor pipe idle for each
// tile's prologue and epilogue, which dominates short k-loops (K = 64..576).
// Unsplit, one GEMM per launch, TMA-store epilogue, same arithmetic as
// gemm_tc_kernel (bit-identical outputs).
template <int BN, int STAGES>
struct PSmem {
  static constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t RING = STAGES * STAGE_BYTES;
  static constexpr uint32_t OUT = RING, OUT_BYTES = BM * BN * 2;  // staging tile (residual in, bf16 out)
  static constexpr uint32_t SCALE = OUT + OUT_BYTES, BIAS = SCALE + BN * 4;
  static constexpr uint32_t TOTAL = BIAS + BN * 4 + 1024;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1) gemm_persist_kernel(const __grid_constant__ Job J) {
  using L = PSmem<BN, STAGES>;
  constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulators
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], acc_full[2], acc_empty[2], res_full;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* s_scale = reinterpret_cast<float*>(smem + L::SCALE);
  float* s_bias = reinterpret_cast<float*>(smem + L::BIAS);
  uint16_t* s_out = reinterpret_cast<uint16_t*>(smem + L::OUT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = J.M, N = J.N, K = J.K, has_res = J.has_res, relu = J.relu;
  const ConvGeom cg = J.cg;
  const int kblocks = (K + BK - 1) / BK;
  const int tiles_m = J.tiles_m, tiles = tiles_m * ((N + BN - 1) / BN);
  const int wbox = 1 << cg.wbox_log2;
  (void)M;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);  // one arrive per epilogue warp
    }
    mbar_init(&res_full, 1);
    fence_barrier_init();
    prefetch_tmap(&J.ta);
    prefetch_tmap(&J.tb);
    if (has_res) prefetch_tmap(&J.tr);
    prefetch_tmap(&J.td);
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem = tmem_base;

  // tile -> (m-tile, n-tile) and, for an implicit conv, (image, row box, col box)
  struct T {
    int m0, n0, ti, th, tw;
  };
  auto tile_of = [&](int t) {
    T r;
    const int mt = t % tiles_m, nt = t / tiles_m;
    r.m0 = mt * BM;
    r.n0 = nt * BN;
    r.ti = r.th = r.tw = 0;
    if (cg.impl) {
      r.tw = mt % cg.tiles_w;
      r.th = (mt / cg.tiles_w) % cg.tiles_h;
      r.ti = mt / (cg.tiles_w * cg.tiles_h);
    }
    return r;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: the ring continues across tiles
      pdl_wait();
      uint32_t it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const T tl = tile_of(t);
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const uint32_t s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          uint8_t* sa = smem + s * L::STAGE_BYTES;
          mbar_expect_tx(&full[s], L::STAGE_BYTES);
          if (cg.impl) {
            const int rs = kb / cg.cblocks, cb = kb - rs * cg.cblocks, r = rs / cg.S, ss = rs - r * cg.S;
            tma_load_4d(sa, &J.ta, cg.c_off + cb * BK, tl.tw * wbox * cg.stride - cg.pad + ss,
                        tl.th * cg.hbox * cg.stride - cg.pad + r, tl.ti, &full[s]);
          } else {
            tma_load_2d(sa, &J.ta, kb * BK, tl.m0, &full[s]);
          }
          tma_load_2d(sa + L::A_BYTES, &J.tb, kb * BK, tl.n0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: accumulator lt & 1 for local tile lt
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      uint32_t it = 0, lt = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
        const uint32_t b = lt & 1;
        if (lt >= 2) mbar_wait(&acc_empty[b], ((lt >> 1) - 1) & 1);  // its previous tile's epilogue drained it
        tc_fence_after();
        const uint32_t acc = tmem + b * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const uint32_t s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES), sb = sa + L::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16(acc, smem_desc_sw128(sa + k * 32), smem_desc_sw128(sb + k * 32), idesc, (kb | k) != 0);
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[b]);
      }
    }
  } else if (warp >= 4) {  // ---- epilogue: 8 warps, two per TMEM lane quarter
    const int q = warp & 3, half = (warp - 4) >> 2, rl = q * 32 + lane, et = threadIdx.x - 128;
    const uint32_t tq = tmem + (uint32_t(q * 32) << 16);
    pdl_wait();  // the residual may be the previous kernel's output
    uint32_t lt = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
      const T tl = tile_of(t);
      const uint32_t b = lt & 1;
      // the staging tile is free once the previous tile's TMA store has read it
      if (et == 0) {
        bulk_wait_read();
        if (has_res) {
          mbar_expect_tx(&res_full, uint32_t((BN / 64) * BM * 128));
#pragma unroll
          for (int bx = 0; bx < BN / 64; ++bx) {
            uint8_t* dst = smem + L::OUT + bx * BM * 128;
            if (cg.impl) tma_load_4d(dst, &J.tr, tl.n0 + bx * 64, tl.tw * wbox, tl.th * cg.hbox, tl.ti, &res_full);
            else tma_load_2d(dst, &J.tr, tl.n0 + bx * 64, tl.m0, &res_full);
          }
        }
      }
      if (et < BN) {
        const int n = tl.n0 + et;
        s_scale[et] = (J.scale && n < N) ? __ldg(J.scale + n) : 1.f;
        s_bias[et] = (J.bias && n < N) ? __ldg(J.bias + n) : 0.f;
      }
      asm volatile("bar.sync 2, 256;" ::: "memory");  // scale / bias staged; staging tile free
      // scale / bias are rewritten every tile: their clobber-free loads must
      // stay below this barrier (not be hoisted out of the tile loop)
      const float* tsc = after_here(s_scale);
      const float* tbi = after_here(s_bias);
      mbar_wait(&acc_full[b], (lt >> 1) & 1);
      tc_fence_after();
      if (has_res) mbar_wait(&res_full, lt & 1);
      auto fin = [&](auto hr_tag, auto rl_tag) {
        constexpr bool HR = decltype(hr_tag)::value, RL = decltype(rl_tag)::value;
#pragma unroll 1
        for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += 32) {
          uint32_t r[32];
          tmem_ld16_nw(tq + b * BN + uint32_t(c0), r);
          tmem_ld16_nw(tq + b * BN + uint32_t(c0 + 16), r + 16);
          tmem_wait_ld();
          const float* v = reinterpret_cast<const float*>(r);
          uint16_t* srow = s_out + (c0 / 64) * BM * 64 + rl * 64;
          const int chunk0 = (c0 & 63) >> 3, sw = rl & 7;
          uint4 res[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            res[u] = HR ? *reinterpret_cast<const uint4*>(srow + (((chunk0 + u) ^ sw) << 3)) : make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + 8 * u;
            const uint32_t rw[4] = {res[u].x, res[u].y, res[u].z, res[u].w};
            const float4 sc0 = lds_f4(tsc + c), sc1 = lds_f4(tsc + c + 4);
            const float4 bi0 = lds_f4(tbi + c), bi1 = lds_f4(tbi + c + 4);
            const float sc[8] = {sc0.x, sc0.y, sc0.z, sc0.w, sc1.x, sc1.y, sc1.z, sc1.w};
            const float bi[8] = {bi0.x, bi0.y, bi0.z, bi0.w, bi1.x, bi1.y, bi1.z, bi1.w};
            uint32_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float2 ab = fma2(make_float2(v[8 * u + 2 * j], v[8 * u + 2 * j + 1]), make_float2(sc[2 * j], sc[2 * j + 1]),
                               make_float2(bi[2 * j], bi[2 * j + 1]));
              if constexpr (HR) ab = add2(ab, make_float2(bf16_lo(rw[j]), bf16_hi(rw[j])));
              if constexpr (RL) {
                ab.x = fmaxf(ab.x, 0.f);
                ab.y = fmaxf(ab.y, 0.f);
              }
              o[j] = pack_bf16x2(ab.x, ab.y);
            }
            *reinterpret_cast<uint4*>(srow + (((chunk0 + u) ^ sw) << 3)) = make_uint4(o[0], o[1], o[2], o[3]);
          }
        }
      };
      using Tt = std::true_type;
      using Ff = std::false_type;
      if (has_res) {
        if (relu) fin(Tt{}, Tt{});
        else fin(Tt{}, Ff{});
      } else {
        if (relu) fin(Ff{}, Tt{});
        else fin(Ff{}, Ff{});
      }
      // accumulator b is drained: the MMA warp may start tile lt + 2 in it
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
      fence_proxy_async_smem();                       // staged tile -> async proxy
      asm volatile("bar.sync 2, 256;" ::: "memory");  // the whole tile is staged
      if (cg.pool) {  // fused 2x2 max pool: the pooled tile replaces rows [0, 32)
        pool_staged_tile<BN>(s_out, et, cg.wbox_log2);
        fence_proxy_async_smem();
        asm volatile("bar.sync 2, 256;" ::: "memory");
      }
      if (et == 0) {
        const int pl = cg.pool;  // pooled: box coordinates halve
#pragma unroll
        for (int bx = 0; bx < BN / 64; ++bx) {
          const uint16_t* src = s_out + bx * BM * 64;
          if (cg.impl)
            tma_store_4d(&J.td, src, tl.n0 + bx * 64, (tl.tw * wbox) >> pl, (tl.th * cg.hbox) >> pl, tl.ti);
          else tma_store_2d(&J.td, src, tl.n0 + bx * 64, tl.m0);
        }
        bulk_commit();
      }
    }
    if (et == 0) bulk_wait_read();
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

void fill_job(Job& j, const Prepared& p, int S) {
  const Epilogue& e = p.e;
  j.ta = p.ta;
  j.tb = p.tb;
  j.tr = p.tr;
  j.td = p.td;
  j.D = e.out;
  j.scale = e.scale;
  j.bias = e.bias;
  j.M = int(p.M);
  j.N = int(p.N);
  j.K = int(p.K);
  j.ldd = int(e.ldo);
  j.has_res = e.residual ? 1 : 0;
  j.relu = e.relu ? 1 : 0;
  const int kblocks = int((p.K + BK - 1) / BK);
  j.kper = (kblocks + S - 1) / S;
  j.tma_out = p.tma_out;
  const int mc = p.pair ? 2 : std::max(1, p.mc);
  j.tiles_m = (int(tile_rows(p) / BM) + mc - 1) / mc * mc;  // whole groups / pairs (padding tiles have no rows)
  j.cg = p.g;
}

template <int BN, int STAGES, int S, int MC = 1>
void run_bn(const Prepared& p, const Prepared* q, cudaStream_t stream) {
  constexpr int CX = MC < 0 ? -MC : MC;
  constexpr size_t smem = Smem<BN, STAGES, S, (MC < 0)>::TOTAL;
  static_assert(smem <= 227 * 1024, "GEMM shared memory");
  static_assert(S * CX <= 8, "portable cluster size");
  static bool smem_set = false;
  if (!smem_set) {
    TRIMS_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES, S, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem)));
    smem_set = true;
  }
  if (CX > 1 && q) raise(Errc::InvalidArgument, "multicast / paired GEMMs run alone");
  Jobs jobs{};
  fill_job(jobs.j[0], p, S);
  jobs.t0 = jobs.j[0].tiles_m * int((p.N + BN - 1) / BN);
  int tiles = jobs.t0;
  if (q) {
    fill_job(jobs.j[1], *q, S);
    tiles += jobs.j[1].tiles_m * int((q->N + BN - 1) / BN);
  }
  dim3 grid(unsigned(tiles), 1, unsigned(S));
  // PDL always; split-K / multicast launch (MC, 1, S) clusters: the MC
  // consecutive M-tiles of one N-tile x the S splits of each
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = unsigned(CX);
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = unsigned(S);
  if (!pdl_enabled()) attr[0] = attr[1];  // keep only the cluster shape
  cfg.attrs = attr;
  cfg.numAttrs = (S > 1 || CX > 1 ? 2 : 1) - (pdl_enabled() ? 0 : 1);
  TRIMS_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, STAGES, S, MC>, jobs));
}

// Residual tile maps: bf16 [rows][ldr] (or NHWC [n][P][Q][ldr] for an
// implicit conv), N channels wide, SWIZZLE_128B boxes of 64 channels x the
// tile's 128 rows. Out-of-range rows / channels are zero-filled.
CUtensorMap tile_map_2d(const uint16_t* ptr, uint64_t ld, uint64_t M, uint64_t N) {
  CUtensorMap m;
  cuuint64_t dims[2] = {N, M};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, uint32_t(BM)};
  cuuint32_t estr[2] = {1, 1};
  cu_check(encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(ptr), dims, strides, box,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
           "cuTensorMapEncodeTiled (tile)");
  return m;
}

CUtensorMap tile_map_conv(const uint16_t* ptr, uint64_t ld, const ConvGeom& g, uint64_t N) {
  CUtensorMap m;
  cuuint64_t dims[4] = {N, cuuint64_t(g.Q), cuuint64_t(g.P), cuuint64_t(g.N)};
  cuuint64_t strides[3] = {ld * 2, cuuint64_t(g.Q) * ld * 2, cuuint64_t(g.P) * g.Q * ld * 2};
  cuuint32_t box[4] = {64, uint32_t(1 << g.wbox_log2), uint32_t(g.hbox), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  cu_check(encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(ptr), dims, strides, box,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
           "cuTensorMapEncodeTiled (conv tile)");
  return m;
}

// Pooled output map of a conv with a fused 2x2 / 2 max pool: NHWC
// [n][P/2][Q/2][ld], boxes of 64 channels x (Wbox/2 x Hbox/2) pooled pixels.
CUtensorMap tile_map_pool(const uint16_t* ptr, uint64_t ld, const ConvGeom& g, uint64_t N) {
  CUtensorMap m;
  cuuint64_t dims[4] = {N, cuuint64_t(g.Q / 2), cuuint64_t(g.P / 2), cuuint64_t(g.N)};
  cuuint64_t strides[3] = {ld * 2, cuuint64_t(g.Q / 2) * ld * 2, cuuint64_t(g.P / 2) * (g.Q / 2) * ld * 2};
  cuuint32_t box[4] = {64, uint32_t(1 << (g.wbox_log2 - 1)), uint32_t(g.hbox / 2), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  cu_check(encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(ptr), dims, strides, box,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
           "cuTensorMapEncodeTiled (pool tile)");
  return m;
}

// TRIMS_TMA_OUT=0: the staged output tile leaves by thread stores (A/B switch).
bool tma_out_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("TRIMS_TMA_OUT");
    return !(v && std::string(v) == "0");
  }();
  return on;
}

// TMA stores need 16-byte aligned rows and base.
bool tma_out_ok(const Epilogue& e) {
  return tma_out_enabled() && e.ldo % 8 == 0 && reinterpret_cast<uintptr_t>(e.out) % 16 == 0;
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
  static const int forced = [] {  // A/B switch: TRIMS_GEMM_BN=64|128|256
    const char* e = std::getenv("TRIMS_GEMM_BN");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 64 || forced == 128 || (forced == 256 && N % 256 == 0)) return forced;
  // Enough CTAs to cover the SMs first, then the widest tile.
  const uint64_t mt = (M + BM - 1) / BM;
  if (N <= 64) return 64;
  if (mt * ((N + 255) / 256) >= uint64_t(sms) && N % 256 == 0) return 256;
  // 64-wide tiles whenever they still fit one wave: there latency (batch-1
  // layers) wins with more, narrower CTAs (ResNet-50 b1 forward 0.294 vs
  // 0.307 ms, AlexNet 0.100 vs 0.107, same box); multi-wave layers keep the
  // wider tile (VGG-16). TRIMS_GEMM_PICK=old keeps the previous rule.
  static const bool old_rule = [] {
    const char* e = std::getenv("TRIMS_GEMM_PICK");
    return e && std::string(e) == "old";
  }();
  if (old_rule) return (mt * ((N + 127) / 128) >= uint64_t(sms) / 2 || N <= 128) ? 128 : 64;
  if (mt * ((N + 63) / 64) <= uint64_t(sms)) return 64;  // 64-wide tiles still fit one wave
  return (mt * ((N + 127) / 128) >= uint64_t(sms) / 2 || N <= 128) ? 128 : 64;
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
  if (e.residual) p.tr = tile_map_2d(e.residual, e.ldr, p.M, p.N);
  p.tma_out = tma_out_ok(e) ? 1 : 0;
  if (p.tma_out) p.td = tile_map_2d(e.out, e.ldo, p.M, p.N);
  return p;
}

namespace {
template <int BN, int STAGES>
void run_persist(const Prepared& p, cudaStream_t stream) {
  constexpr size_t smem = PSmem<BN, STAGES>::TOTAL;
  static_assert(smem <= 227 * 1024, "persistent GEMM shared memory");
  static bool smem_set = false;
  if (!smem_set) {
    TRIMS_CUDA(cudaFuncSetAttribute(gemm_persist_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem)));
    smem_set = true;
  }
  Job j{};
  fill_job(j, p, 1);
  const int tiles = j.tiles_m * int((p.N + BN - 1) / BN);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(std::min(tiles, sms)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  TRIMS_CUDA(cudaLaunchKernelEx(&cfg, gemm_persist_kernel<BN, STAGES>, j));
}
}  // namespace

// TMA ring depths (stages in flight per CTA: at batch 1 a CTA's k-loop is
// bound by bytes in flight / L2 latency, so deeper is faster while it fits).
#ifndef TRIMS_ST64
#define TRIMS_ST64 6
#endif
#ifndef TRIMS_ST64S
#define TRIMS_ST64S 6
#endif
#ifndef TRIMS_ST128
#define TRIMS_ST128 5
#endif
constexpr int kSt64 = TRIMS_ST64, kSt64S = TRIMS_ST64S, kSt128 = TRIMS_ST128;

void run(const Prepared& p, cudaStream_t stream) { run_pair(p, nullptr, stream); }

void run_pair(const Prepared& p, const Prepared* q, cudaStream_t stream) {
  if (p.splits < 1 || p.splits > kMaxSplits || (p.splits & (p.splits - 1)) || (p.bn / p.splits) % 8 ||
      (p.bn == 256 && p.splits > 1))
    raise(Errc::InvalidArgument, "GEMM split count");
  if ((p.g.pool || (q && q->g.pool)) &&
      (p.pair || p.mc > 1 || (p.splits == 1 && (!p.tma_out || p.g.pool == 2 || (q && q->g.pool == 2)))))
    raise(Errc::InvalidArgument, "a fused pool needs a single-CTA (split or TMA-stored) GEMM");
  for (const Prepared* x : {&p, q})
    if (x && x->g.pool == 3) {
      const uint64_t hw = uint64_t(x->g.P) * x->g.Q, rows = x->g.impl ? hw : x->M;  // rows of the one tile
      if (x->splits < 2 || uint64_t(x->splits + 1) * rows > uint64_t(128) * x->splits ||
          (!x->g.impl && (hw == 0 || x->M > 128 || x->M % hw)))
        raise(Errc::InvalidArgument,
              "a fused global average pool needs a split-K launch over whole images with (S + 1) * rows <= 128 * S");
    }
  if (q && (q->bn != p.bn || q->splits != p.splits || q->lean != p.lean))
    raise(Errc::InvalidArgument, "grouped GEMMs need the same tile width, split count and variant");
  if (p.persist) {  // persistent, double-buffered accumulators: unsplit, single GEMM, TMA-store output
    if (q || p.splits != 1 || p.pair || p.mc > 1 || !p.tma_out) raise(Errc::InvalidArgument, "persistent GEMM variant");
    if (p.bn == 64) run_persist<64, 6>(p, stream);
    else if (p.bn == 128) run_persist<128, 5>(p, stream);
    else run_persist<256, 3>(p, stream);
    return;
  }
  if (p.pair) {  // 2-SM pairs (cta_group::2): unsplit, BN 128 / 256
    if (p.splits != 1 || p.mc > 1 || p.lean || p.bn < 128) raise(Errc::InvalidArgument, "2-SM pair variant");
    if (p.bn == 128) run_bn<128, 6, 1, -2>(p, q, stream);
    else run_bn<256, 4, 1, -2>(p, q, stream);
    return;
  }
  if (p.mc > 1) {  // weight-multicast groups (single GEMM launches, latency mode)
    switch (p.bn * 1000 + p.splits * 10 + p.mc) {
      case 64 * 1000 + 14: run_bn<64, kSt64, 1, 4>(p, q, stream); return;
      case 64 * 1000 + 18: run_bn<64, kSt64, 1, 8>(p, q, stream); return;
      case 64 * 1000 + 24: run_bn<64, kSt64S, 2, 4>(p, q, stream); return;
      case 64 * 1000 + 42: run_bn<64, kSt64S, 4, 2>(p, q, stream); return;
      case 128 * 1000 + 14: run_bn<128, kSt128, 1, 4>(p, q, stream); return;
      case 128 * 1000 + 18: run_bn<128, kSt128, 1, 8>(p, q, stream); return;
      case 128 * 1000 + 24: run_bn<128, 4, 2, 4>(p, q, stream); return;
      case 128 * 1000 + 42: run_bn<128, 4, 4, 2>(p, q, stream); return;
      default: raise(Errc::InvalidArgument, "no multicast variant for this tile width / split count");
    }
  }
  if (p.lean && p.splits == 1 && p.bn != 256) {  // <= ~110 KB: two CTAs per SM
    if (p.bn == 64) run_bn<64, 3, 1>(p, q, stream);
    else run_bn<128, 2, 1>(p, q, stream);
    return;
  }
  switch (p.bn * 16 + p.splits) {
    case 64 * 16 + 1: run_bn<64, kSt64, 1>(p, q, stream); break;
    case 64 * 16 + 2: run_bn<64, kSt64S, 2>(p, q, stream); break;
    case 64 * 16 + 4: run_bn<64, kSt64S, 4>(p, q, stream); break;
    case 64 * 16 + 8: run_bn<64, kSt64S, 8>(p, q, stream); break;
    case 128 * 16 + 1: run_bn<128, kSt128, 1>(p, q, stream); break;
    case 128 * 16 + 2: run_bn<128, 4, 2>(p, q, stream); break;
    case 128 * 16 + 4: run_bn<128, 4, 4>(p, q, stream); break;
    case 128 * 16 + 8: run_bn<128, 4, 8>(p, q, stream); break;
    default: run_bn<256, 3, 1>(p, q, stream); break;
  }
}


uint32_t b_box_rows(const Prepared& p) { return uint32_t(p.bn / (p.pair ? 2 : std::max(1, p.mc))); }

namespace {
// Co-resident (MC, 1, S) clusters of one GEMM variant on this device.
template <int BN, int STAGES, int S, int MC>
int max_clusters() {
  static const int n = [] {
    constexpr size_t smem = Smem<BN, STAGES, S, (MC < 0)>::TOTAL;
    cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES, S, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(MC * 64), 1, unsigned(S));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a{};
    a.id = cudaLaunchAttributeClusterDimension;
    a.val.clusterDim.x = unsigned(MC);
    a.val.clusterDim.y = 1;
    a.val.clusterDim.z = unsigned(S);
    cfg.attrs = &a;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, gemm_tc_kernel<BN, STAGES, S, MC>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    return c;
  }();
  return n;
}

int mc_capacity(int bn, int splits, int mc) {
  switch (bn * 1000 + splits * 10 + mc) {
    case 64 * 1000 + 14: return max_clusters<64, kSt64, 1, 4>();
    case 64 * 1000 + 18: return max_clusters<64, kSt64, 1, 8>();
    case 64 * 1000 + 24: return max_clusters<64, kSt64S, 2, 4>();
    case 64 * 1000 + 42: return max_clusters<64, kSt64S, 4, 2>();
    case 128 * 1000 + 14: return max_clusters<128, kSt128, 1, 4>();
    case 128 * 1000 + 18: return max_clusters<128, kSt128, 1, 8>();
    case 128 * 1000 + 24: return max_clusters<128, 4, 2, 4>();
    case 128 * 1000 + 42: return max_clusters<128, 4, 4, 2>();
    default: return 0;
  }
}
}  // namespace

int pick_mc(const Prepared& p, int sms) {
  // Off by default: measured slower at batch 1 (VGG-16 0.2147 -> 0.2198 ms
  // with groups of 4, 0.2204 with 8; ResNet-50 0.2141 -> 0.2150; AlexNet flat;
  // profiles/r3/weight_multicast_ab.log): the k-loops are bound by each SM's
  // own ingress, not by L2 egress, and a shared stage refills only when the
  // slowest CTA of the group released it. TRIMS_MC=N enables groups <= N.
  static const int forced = [] {
    const char* e = std::getenv("TRIMS_MC");
    return e ? std::atoi(e) : 1;
  }();
  if (forced <= 1 || p.lean || p.pair || p.bn == 256 || p.splits > 4) return 1;
  const uint64_t tm = tile_rows(p) / BM, tn = (p.N + p.bn - 1) / p.bn, kb = (p.K + BK - 1) / BK;
  if (kb / uint64_t(p.splits) < 4) return 1;  // a short k-loop gains nothing from sharing its few stages
  const uint64_t ctas = tm * tn * uint64_t(p.splits);
  for (int mc : {8, 4, 2}) {
    if (mc > forced || p.splits * mc > 8 || tm < uint64_t(mc)) continue;
    const uint64_t pad = (tm + mc - 1) / mc * mc;
    if ((pad - tm) * 8 > pad) continue;  // <= 1/8 of the tiles padding
    const int cap = mc_capacity(p.bn, p.splits, mc);
    if (cap <= 0) continue;
    const uint64_t clusters = pad * tn / uint64_t(mc);
    // one wave stays one wave (a multi-wave launch keeps its wave count)
    const uint64_t waves_before = (ctas + uint64_t(sms) - 1) / uint64_t(sms);
    const uint64_t waves_after = (clusters + uint64_t(cap) - 1) / uint64_t(cap);
    if (waves_after > waves_before) continue;
    return mc;
  }
  return 1;
}

int pick_splits(uint64_t M, uint64_t N, uint64_t K, int bn, int sms) {
  // Split K only while the output tiles leave most SMs idle, each split keeps
  // >= 2 k-blocks (4 before the cheaper reduction; 2 measured best, AlexNet
  // b1 0.0883 -> 0.0862 ms, others flat, profiles/r3/split_minkb_ab.log) and
  // every split's column slice of the tile is >= 8 wide.
  const uint64_t tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn), kb = (K + BK - 1) / BK;
  int s = 1;
  if (bn == 256) return 1;  // no split variant of the widest tile (shared memory)
  // 8 splits only for the tiniest tile counts (<= 8 tiles, e.g. ResNet-50
  // layer3/4 3x3 convs at batch 1); measured slower for 16 tiles (VGG-16
  // conv5), profiles/r03d_split.log.
  const int max_s = tiles <= 8 ? kMaxSplits : 4;
  static const uint64_t min_kb = [] {  // k-blocks each split keeps at least (A/B: TRIMS_SPLIT_MINKB)
    const char* e = std::getenv("TRIMS_SPLIT_MINKB");
    return e ? uint64_t(std::max(1, std::atoi(e))) : uint64_t(2);
  }();
  while (s < max_s && bn / (s * 2) >= 8 && tiles * uint64_t(s * 2) <= uint64_t(sms) && kb / uint64_t(s * 2) >= min_kb)
    s *= 2;
  return s;
}

void choose_tiles(uint64_t rows, uint64_t N, uint64_t K, int sms, int* bn_out, int* splits_out, bool* pair_out) {
  // Cost model of one batch-1 layer (per-CTA phases measured by
  // scripts/gemm_trace.py): each CTA streams ceil(kblocks / S) stages of
  // (16 KiB A + BN x 128 B of B) from L2 at ~95 KB/us per SM, plus ~2 us of
  // fixed cost per wave (dependent-launch release, first tile, epilogue) and
  // ~0.8 us more for a split-K reduction. Candidates: BN 64/128/256 (256 only
  // unsplit, N % 256 == 0), S 1/2/4/8 with slices >= 8 columns, >= 2 k-blocks
  // per split and split launches within one wave.
  const double bw = 95.0, c_wave = 2.0, c_split = 0.8;
  const uint64_t mt = (rows + BM - 1) / BM, kb = (K + BK - 1) / BK;
  double best = 1e30;
  int bb = 64, bs = 1;
  for (int bn : {64, 128, 256}) {
    if (bn == 256 && N % 256) continue;
    for (int sp : {1, 2, 4, 8}) {
      if ((bn == 256 && sp > 1) || bn / sp < 8 || (sp > 1 && kb / uint64_t(sp) < 2)) continue;
      const uint64_t ctas = mt * ((N + bn - 1) / bn) * uint64_t(sp);
      if (sp > 1 && ctas > uint64_t(sms)) continue;
      const double waves = double((ctas + uint64_t(sms) - 1) / uint64_t(sms));
      const double per_kb = (16.0 + bn * 128.0 / 1024.0);  // KB per stage
      const double c = waves * (c_wave + double((kb + sp - 1) / sp) * per_kb / bw) + (sp > 1 ? c_split : 0.0);
      if (c < best - 1e-9) {
        best = c;
        bb = bn;
        bs = sp;
      }
    }
  }
  // 2-SM pairs (unsplit, BN 128 / 256): each SM streams 16 KiB of A and only
  // half of B per stage; M-tiles padded to whole pairs
  bool bp = false;
  // Default: 256-wide pairs only (VGG-16 b32 2.249 -> 2.162 ms, b8 0.848 ->
  // 0.824; ResNet-50 b32 +0.7 %; batch 1 flat; 128-wide pairs lost on
  // ResNet-50: profiles/r3/pair_sm_ab.log). TRIMS_PAIR_SM=0 off, =1 all widths.
  static const int pairs_on = [] {
    const char* e = std::getenv("TRIMS_PAIR_SM");
    return e ? std::atoi(e) : 256;
  }();
  if (pair_out && pairs_on && mt >= 2) {
    for (int bn : {128, 256}) {
      if (pairs_on == 256 && bn != 256) continue;
      if (bn == 256 && N % 256) continue;
      const uint64_t ctas = (mt + 1) / 2 * 2 * ((N + bn - 1) / bn);
      const double waves = double((ctas + uint64_t(sms) - 1) / uint64_t(sms));
      const double per_kb = 16.0 + bn * 64.0 / 1024.0;
      const double c = waves * (c_wave + double(kb) * per_kb / bw);
      if (c < best - 1e-9) {
        best = c;
        bb = bn;
        bs = 1;
        bp = true;
      }
    }
  }
  if (pair_out) *pair_out = bp;
  *bn_out = bb;
  *splits_out = bs;
}

uint64_t tile_rows(const Prepared& p) {
  if (p.g.impl) return uint64_t(p.g.N) * p.g.tiles_h * p.g.tiles_w * BM;
  return (p.M + BM - 1) / BM * BM;
}

ConvGeom conv_geom(int N, int H, int W, int C, int R, int S, int stride, int pad, int P, int Q, int cgroup,
                   int c_off, int pool_box) {
  ConvGeom g;
  g.impl = 1;
  g.N = N, g.H = H, g.W = W, g.C = C, g.R = R, g.S = S, g.stride = stride, g.pad = pad, g.P = P, g.Q = Q;
  int wl = 0;
  while ((1 << wl) < Q && wl < 7) ++wl;   // Wbox = next power of two >= Q, at most 128
  if (pool_box) {
    // even box sides: Wbox <= 64 (Hbox >= 2); pool_box 1: the box whose
    // tiles cover the fewest pixels outside the P x Q map, 2: the fewest
    // columns outside it (taller boxes); the widest on a tie
    int best = -1;
    uint64_t waste_best = ~0ull;
    for (int w = std::min(wl, 6); w >= 1; --w) {
      if ((BM >> w) * stride > 256 || (1 << w) * stride > 256) continue;
      const uint64_t hb = uint64_t(BM >> w);
      static const int forced = [] {  // A/B: TRIMS_POOL_BOX=area|col
        const char* e = std::getenv("TRIMS_POOL_BOX");
        return !e ? 0 : std::string(e) == "col" ? 2 : std::string(e) == "area" ? 1 : 0;
      }();
      const bool col_rule = (forced ? forced : pool_box) == 2;
      const uint64_t waste = col_rule ? uint64_t(((Q + (1 << w) - 1) >> w) << w) - uint64_t(Q)
                                      : uint64_t(((Q + (1 << w) - 1) >> w) << w) * ((uint64_t(P) + hb - 1) / hb * hb) -
                                            uint64_t(P) * uint64_t(Q);
      if (waste < waste_best) {
        waste_best = waste;
        best = w;
      }
    }
    if (best < 0) raise(Errc::InvalidArgument, "no pooling tile box for this conv");
    wl = best;
  }
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
  if (e.residual) p.tr = tile_map_conv(e.residual, e.ldr, g, p.N);
  if (g.pool == 3) {  // global average pool in the split-K owners' epilogue: one tile = one whole image
    if (!g.impl || g.tiles_w != 1 || g.tiles_h != 1)
      raise(Errc::InvalidArgument, "fused global average pool: one tile per image");
  } else if (g.pool) {
    if (!p.tma_out || g.P % 2 || g.Q % 2 || g.wbox_log2 < 1 || g.hbox % 2 || e.residual)
      raise(Errc::InvalidArgument, "fused pool: even output / tile sides, a TMA-stored output, no residual");
    p.td = tile_map_pool(e.out, e.ldo, g, p.N);
  } else if (p.tma_out) {
    p.td = tile_map_conv(e.out, e.ldo, g, p.N);
  }
  return p;
}

void launch(const Operand& A, const Operand& B, const Epilogue& e, cudaStream_t stream, int bn, int splits, int mc) {
  Prepared p = prepare(A, B, e, bn);
  if (mc == -3) {
    p.persist = true;
    splits = 1;
  } else if (mc > 1 || mc == -2) {
    if (mc == -2) p.pair = true;
    else p.mc = mc;
    p.tb = make_tmap(B.ptr, B.rows, B.k, B.ld, b_box_rows(p));
  }
  if (splits == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    splits = pick_splits(tile_rows(p), p.N, p.K, p.bn, sms);
  }
  p.splits = splits;
  run(p, stream);
}

}  // namespace trims::gemm

#ifdef TRIMS_GEMM_TRACE
// Copies out up to `cap` records (16 u64 each) and returns how many CTAs
// recorded since the last reset; reset != 0 zeroes the counter afterwards.
extern "C" int trims_debug_gemm_trace(unsigned long long* out, int cap, int reset) {
  unsigned int n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, trims::gemm::g_gtrace_n, sizeof(n));
  const int take = int(std::min<unsigned>(n, unsigned(std::min(cap, trims::gemm::kGTCap))));
  if (out && take) cudaMemcpyFromSymbol(out, trims::gemm::g_gtrace, sizeof(unsigned long long) * trims::gemm::kGTW * size_t(take));
  if (reset) {
    unsigned int z = 0;
    cudaMemcpyToSymbol(trims::gemm::g_gtrace_n, &z, sizeof(z));
  }
  return int(n);
}
#endif
