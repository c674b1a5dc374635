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
struct Prepared;
// Rows of the B (weight) TMA box of a prepared GEMM: BN, or BN / mc.
uint32_t b_box_rows(const Prepared& p);
// Weight-multicast group size for a prepared GEMM (its tile width and split
// count set): 1 when it does not pay or does not fit one wave of clusters.
int pick_mc(const Prepared& p, int sms);

// Implicit-GEMM convolution geometry: A is read straight from the NHWC bf16
// activation [N][H][W][C] by 4-D TMA boxes of 64 channels x Wbox x Hbox output
// pixels (tap-shifted, stride via TMA element strides, padding = OOB zero
// fill); an M tile is a Hbox x Wbox block of one image's output (Wbox*Hbox =
// 128). K order = (r, s, c), the resident KRSC weight order. Needs C % 64 == 0.
struct ConvGeom {
  int impl{0};
  int N, H, W, C, R, S, stride, pad, P, Q;
  int wbox_log2, hbox, tiles_w, tiles_h, cblocks;
  int c_off{0};  // grouped conv: first channel of this group (the group has cblocks * 64 channels)
  // 1: a 2x2 / stride-2 max pool is fused into the epilogue (the output is
  // the pooled P/2 x Q/2 map, NHWC); 2: the same written NCHW (a flatten
  // follows; split-K launches only); 3: a global average pool (output
  // [N][Cout]; split-K launches whose tile is one whole image)
  int pool{0};
};
// C = the activation's channels; cg / c_off = this group's channel count and
// first channel (cg = C, c_off = 0 for an ungrouped conv; cg % 64 == 0).
// pool_box != 0: a tile box with an even number of rows and columns (>= 2
// each), so every 2x2 pooling window lies inside one tile: 1 = the least
// padded tile area, 2 = the fewest padded columns (taller boxes; measured
// faster for single-wave layers, 1 for multi-wave ones).
ConvGeom conv_geom(int N, int H, int W, int C, int R, int S, int stride, int pad, int P, int Q, int cg = 0,
                   int c_off = 0, int pool_box = 0);
int pick_bn(uint64_t M, uint64_t N, int sms);

// A GEMM with its tensor maps encoded once (the executor builds these at
// bind time so a forward pass costs only kernel launches).
struct Prepared {
  CUtensorMap ta, tb;
  // Residual tile loader (e.residual != nullptr): SWIZZLE_128B boxes of 64
  // channels x the tile's 128 output rows (2-D rows, or the implicit conv's
  // Wbox x Hbox pixel block), staged by TMA during the mainloop.
  CUtensorMap tr;
  // Output tile store map (same box shape as the residual map) when the
  // output rows are 16-byte aligned: the staged bf16 tile leaves by TMA.
  CUtensorMap td;
  int tma_out{0};
  uint64_t M{0}, N{0}, K{0};
  int bn{128};
  Epilogue e;
  // Split-K (grid.z = splits, one (1,1,splits) cluster per output tile):
  // the splits reduce their fp32 partials through distributed shared memory.
  int splits{1};
  // Lean variants (splits == 1, BN 64/128): a shallower TMA ring so two CTAs
  // fit one SM's shared memory (throughput mode: many clients' kernels).
  bool lean{false};
  // Weight multicast: MC consecutive M-tiles (one cluster dimension) share
  // each B stage by TMA multicast, BN/MC rows loaded by each (the B tensor
  // map's box is then BN/MC rows: b_box_rows()). 1 = off.
  int mc{1};
  // 2-SM pair (tcgen05 cta_group::2, M = 256 over two CTAs; each loads half
  // of B: b_box_rows() = BN / 2). Unsplit, BN 128 / 256.
  bool pair{false};
  // Persistent (one CTA per SM over all output tiles, two TMEM accumulators:
  // a tile's epilogue overlaps the next tile's k-loop). Unsplit, single GEMM,
  // TMA-store output; for multi-wave layers.
  bool persist{false};
  ConvGeom g{};  // g.impl: A is the implicit im2col of an NHWC activation
};
Prepared prepare(const Operand& A, const Operand& B, const Epilogue& e, int bn = 0);
// Implicit-GEMM conv: `act` = NHWC input, B = [Cout][R*S*C] KRSC weights.
Prepared prepare_conv(const void* act, const ConvGeom& g, const Operand& B, const Epilogue& e, int bn = 0);
// Output-tile rows of a prepared GEMM (M rounded up to whole tiles).
uint64_t tile_rows(const Prepared& p);
void run(const Prepared& p, cudaStream_t stream);
// Two independent GEMMs (same bn, splits and variant) in one launch.
void run_pair(const Prepared& p, const Prepared* q, cudaStream_t stream);
// Tile width and split count from a per-CTA cost model (L2 -> SMEM stage
// bytes, per-wave fixed cost, split-K reduction cost); `rows` = tile rows.
void choose_tiles(uint64_t rows, uint64_t N, uint64_t K, int sms, int* bn, int* splits, bool* pair = nullptr);
// Split count for a GEMM shape on `sms` SMs.
int pick_splits(uint64_t M, uint64_t N, uint64_t K, int bn, int sms);
// D = epi(A . B^T); bn = 0 picks the tile width; splits = split-K count
// (1, 2, 4, 8; 0 picks it as the executor does).
// mc: weight-multicast group size (1 = off; 2 / 4 / 8 with splits * mc <= 8);
// mc = -2: a 2-SM pair (cta_group::2; splits 1, bn 128 / 256).
void launch(const Operand& A, const Operand& B, const Epilogue& e, cudaStream_t stream, int bn = 0, int splits = 1,
            int mc = 1);

}  // namespace trims::gemm
