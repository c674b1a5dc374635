// nn_kernels.cu — K8: the bandwidth-bound layers of the forward pass on the
// shared weights (NHWC bf16 activations): input layout/precision prep,
// im2col feeding the tcgen05 GEMM, max/avg pooling, NHWC->NCHW flatten for
// torchvision-ordered FC weights, the small-batch FC GEMV, batch-norm
// folding into per-channel fp32 scale/shift, and softmax.
#include <cuda_bf16.h>

#include <cstdlib>

#include "cuda_util.hpp"
#include "nn.hpp"

namespace trims::nn {

namespace {

__device__ __forceinline__ float bf(uint16_t v) { return __uint_as_float(uint32_t(v) << 16); }
__device__ __forceinline__ uint16_t to_bf(float x) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(0.f), "f"(x));
  return uint16_t(r & 0xffffu);
}

inline unsigned blocks(uint64_t n, unsigned t = 256) { return unsigned(std::min<uint64_t>((n + t - 1) / t, 1u << 20)); }

__global__ void input_prep_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int N, int C, int H, int W) {
  pdl_wait();  // reads the previous layer's output / writes shared scratch
  pdl_trigger();
  const uint64_t total = uint64_t(N) * H * W * C;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const int c = int(i % C);
    uint64_t r = i / C;
    const int w = int(r % W);
    r /= W;
    const int h = int(r % H);
    const int n = int(r / H);
    out[i] = to_bf(in[((uint64_t(n) * C + c) * H + h) * W + w]);
  }
}

// A[m, (r*S + s)*Cg + c] = in[n, p*stride - pad + r, q*stride - pad + s, c_off + c]; zero outside / in padding cols.
__global__ void im2col_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ A, int N, int H, int W, int Ctot,
                              int c_off, int Cg, int R, int S, int stride, int pad, int P, int Q, int Kp) {
  pdl_wait();  // reads the previous layer's output / writes shared scratch
  pdl_trigger();
  const int RSC = R * S * Cg;
  const bool vec = (Cg % 8 == 0) && (Ctot % 8 == 0) && (c_off % 8 == 0) && (Kp % 8 == 0);
  const uint64_t M = uint64_t(N) * P * Q;
  // grid.y = channel groups written side by side: group g's columns go to A + g * M * Kp
  c_off += int(blockIdx.y) * Cg;
  A += uint64_t(blockIdx.y) * M * Kp;
  if (vec) {
    const int cols8 = Kp / 8;
    const uint64_t total = M * cols8;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
      const int col = int(i % cols8) * 8;
      const uint64_t m = i / cols8;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (col < RSC) {
        const int c = col % Cg, rs = col / Cg, s = rs % S, r = rs / S;
        const int q = int(m % Q), p = int((m / Q) % P), n = int(m / (uint64_t(P) * Q));
        const int y = p * stride - pad + r, x = q * stride - pad + s;
        if (y >= 0 && y < H && x >= 0 && x < W)
          v = *reinterpret_cast<const uint4*>(in + ((uint64_t(n) * H + y) * W + x) * Ctot + c_off + c);
      }
      *reinterpret_cast<uint4*>(A + m * Kp + col) = v;
    }
  } else {
    // Narrow channel groups (conv1: Cg = 3): one thread per (row m, filter
    // row r) copies the S*Cg contiguous NHWC elements of that tap row (zero
    // outside the image); the r = R-1 thread also zeroes the K padding.
    const uint32_t rows = uint32_t(M) * R, SC = S * Cg;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
      const uint32_t m = i / R, r = i - m * R;
      const uint32_t q = m % Q, pn = m / Q, p = pn % P, n = pn / P;
      const int y = int(p) * stride - pad + int(r), x0 = int(q) * stride - pad;
      uint16_t* dst = A + uint64_t(m) * Kp + r * SC;
      const bool yok = y >= 0 && y < H;
      const uint16_t* srow = in + (uint64_t(n) * H + (yok ? y : 0)) * W * Ctot + c_off;
      for (int s = 0; s < S; ++s) {
        const int x = x0 + s;
        const bool ok = yok && x >= 0 && x < W;
        for (int c = 0; c < Cg; ++c) dst[s * Cg + c] = ok ? srow[uint64_t(x) * Ctot + c] : uint16_t(0);
      }
      if (r == uint32_t(R - 1))
        for (int c = RSC; c < Kp; ++c) A[uint64_t(m) * Kp + c] = 0;
    }
  }
}

// Max pool, 8 channels per thread, 32-bit index math; KS = the window size
// when it is a compile-time 2 or 3 (all KS*KS loads issued before the max),
// 0 = generic runtime window.
// nchw != 0: write the output in NCHW order (torch's flatten order for a
// following FC layer), so no separate flatten pass is needed.
template <int KS>
__global__ void __launch_bounds__(256) maxpool_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                                                      int N, int H, int W, int C, int k, int stride, int pad, int P,
                                                      int Q, int nchw) {
  pdl_wait();  // reads the previous layer's output / writes shared scratch
  pdl_trigger();
  const uint32_t C8 = uint32_t(C) / 8, total = uint32_t(N) * P * Q * C8;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t pix = i / C8, c = (i - pix * C8) * 8, q = pix % Q, pn = pix / Q, p = pn % P, n = pn / P;
    const int y0 = int(p) * stride - pad, x0 = int(q) * stride - pad;
    const uint16_t* img = in + uint64_t(n) * H * W * C + c;
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = -INFINITY;
    auto fold = [&](const uint4 v) {
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        m[2 * j] = fmaxf(m[2 * j], bf(uint16_t(w[j] & 0xffff)));
        m[2 * j + 1] = fmaxf(m[2 * j + 1], bf(uint16_t(w[j] >> 16)));
      }
    };
    if constexpr (KS > 0) {
      uint4 v[KS * KS];
      bool ok[KS * KS];
#pragma unroll
      for (int t = 0; t < KS * KS; ++t) {
        const int y = y0 + t / KS, x = x0 + t % KS;
        ok[t] = y >= 0 && y < H && x >= 0 && x < W;
        if (ok[t]) v[t] = *reinterpret_cast<const uint4*>(img + (uint64_t(y) * W + x) * C);
      }
#pragma unroll
      for (int t = 0; t < KS * KS; ++t)
        if (ok[t]) fold(v[t]);
    } else {
      for (int dy = 0; dy < k; ++dy) {
        const int y = y0 + dy;
        if (y < 0 || y >= H) continue;
        for (int dx = 0; dx < k; ++dx) {
          const int x = x0 + dx;
          if (x >= 0 && x < W) fold(*reinterpret_cast<const uint4*>(img + (uint64_t(y) * W + x) * C));
        }
      }
    }
    if (nchw) {  // 8 channels of one pixel -> 8 planes
      uint16_t* o = out + (uint64_t(n) * C + c) * P * Q + uint64_t(p) * Q + q;
#pragma unroll
      for (int j = 0; j < 8; ++j) o[uint64_t(j) * P * Q] = to_bf(m[j]);
      continue;
    }
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = uint32_t(to_bf(m[2 * j])) | (uint32_t(to_bf(m[2 * j + 1])) << 16);
    *reinterpret_cast<uint4*>(out + uint64_t(i) * 8) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Global average pool: one block per (image, 64 channels); 8 threads of
// 8 channels x 32 pixel slices, 128-bit loads, shared-memory reduction.
__global__ void __launch_bounds__(256) avgpool_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                                                      int N, int HW, int C) {
  pdl_wait();  // reads the previous layer's output
  pdl_trigger();
  __shared__ float red[32][65];
  const int groups = (C + 63) / 64, n = blockIdx.x / groups, c0 = (blockIdx.x - n * groups) * 64;
  const int cg = threadIdx.x & 7, sl = threadIdx.x >> 3, c = c0 + cg * 8;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c + 8 <= C && C % 8 == 0) {
    for (int j = sl; j < HW; j += 32) {
      const uint4 v = *reinterpret_cast<const uint4*>(in + (uint64_t(n) * HW + j) * C + c);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        s[2 * q] += bf(uint16_t(w[q] & 0xffff));
        s[2 * q + 1] += bf(uint16_t(w[q] >> 16));
      }
    }
  } else {
    for (int j = sl; j < HW; j += 32)
      for (int q = 0; q < 8 && c + q < C; ++q) s[q] += bf(in[(uint64_t(n) * HW + j) * C + c + q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) red[sl][cg * 8 + q] = s[q];
  __syncthreads();
  if (threadIdx.x < 64 && c0 + int(threadIdx.x) < C) {
    float t = 0.f;
    for (int k = 0; k < 32; ++k) t += red[k][threadIdx.x];
    out[uint64_t(n) * C + c0 + threadIdx.x] = to_bf(t / float(HW));
  }
}

// A[m, (r*S + s)*C + c] = bf16(in[n, c, y, x]) for the first conv. Thread i
// fills 16-byte chunk i of A (row i / G, columns 8 (i % G) .., G = Kp / 8):
// consecutive lanes write consecutive chunks, so a warp's stores are one
// contiguous run of A (a thread per row put every chunk of a warp store in
// a different row: 1.8x the DRAM writes, ResNet-50 b32 142 us). Each
// column's tap (plane offset, dy, dx) is decoded once per block into shared
// memory; the scattered input loads hit L1 (a pixel feeds up to R*S/stride^2
// rows of the block).
constexpr int kIm2colMaxK = 512;
__global__ void __launch_bounds__(256) im2col_input_kernel(const float* __restrict__ in, uint16_t* __restrict__ A,
                                                           int N, int C, int H, int W, int R, int S, int stride,
                                                           int pad, int P, int Q, int Kp) {
  __shared__ int s_plane[kIm2colMaxK];
  __shared__ short s_dy[kIm2colMaxK], s_dx[kIm2colMaxK];
  const int RSC = R * S * C;
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    const int rs = k / C, c = k - rs * C;
    s_dy[k] = short(k < RSC ? rs / S : -16384);  // out of every image: a zero column
    s_dx[k] = short(rs - (rs / S) * S);
    s_plane[k] = c * H * W;
  }
  pdl_wait();  // the input H2D / previous forward's readers of A
  pdl_trigger();
  __syncthreads();
  const uint32_t G = uint32_t(Kp) / 8;
  const uint64_t chunks = uint64_t(N) * P * Q * G;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < chunks; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t m = uint32_t(i / G), col = uint32_t(i - uint64_t(m) * G) * 8;
    const uint32_t q = m % Q, pn = m / Q, p = pn % P, n = pn / P;
    const int y0 = int(p) * stride - pad, x0 = int(q) * stride - pad;
    const float* img = in + uint64_t(n) * C * H * W;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int y = y0 + s_dy[col + e], x = x0 + s_dx[col + e];
      v[e] = (y >= 0 && y < H && x >= 0 && x < W) ? __ldg(img + s_plane[col + e] + y * W + x) : 0.f;
    }
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = uint32_t(to_bf(v[2 * j])) | (uint32_t(to_bf(v[2 * j + 1])) << 16);
    *reinterpret_cast<uint4*>(A + i * 8) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void flatten_nchw_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out, int N, int HW, int C) {
  pdl_wait();  // reads the previous layer's output / writes shared scratch
  pdl_trigger();
  const uint64_t total = uint64_t(N) * HW * C;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const int hw = int(i % HW);
    uint64_t r = i / HW;
    const int c = int(r % C);
    const int n = int(r / C);
    out[i] = in[(uint64_t(n) * HW + hw) * C + c];
  }
}

// Small-batch FC: out[m, n] = relu?(sum_k x[m,k] W[n,k] + bias[n]), HBM-bound
// on the weights, which are streamed exactly once. A block owns R consecutive
// rows, i.e. one contiguous R*K region of W, and its 8 warps sweep that region
// linearly in 512-byte pieces (warp w takes pieces w, w+8, ...), 16 pieces in
// flight per lane: each block is one sequential DRAM stream, not R*8
// interleaved row streams (measured: the per-row mapping capped at ~3.3 TB/s).
// A piece never straddles rows (K % 256 == 0); a warp flushes its running sum
// when its row changes, into a per-(row, warp) slot summed in a fixed order.
// The head of the block's region is prefetched into L2 before waiting on the
// previous layer.
constexpr int kGemvRows = 8;
template <int MB, int kGemvUnroll>
__global__ void __launch_bounds__(256) gemv_kernel(const uint16_t* __restrict__ x, int M, int K,
                                                   const uint16_t* __restrict__ Wt, int N, const float* __restrict__ bias,
                                                   int relu, uint16_t* __restrict__ out_bf, float* __restrict__ out_f32,
                                                   int ldo, int R) {
  __shared__ float red[kGemvRows][8][MB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // R > 0: R rows per block. R == 0: rows spread evenly over the grid (a
  // multiple of the SM count: every SM streams the same share of W)
  const int n0 = R ? int(blockIdx.x) * R : int(uint64_t(blockIdx.x) * N / gridDim.x);
  const int rows = R ? min(R, N - n0) : int(uint64_t(blockIdx.x + 1) * N / gridDim.x) - n0;
  const int ppr = K / 256, pieces = rows * ppr;  // 256-element pieces per row / in the block
  const uint16_t* base = Wt + uint64_t(n0) * K;
  for (int i = threadIdx.x; i < kGemvRows * 8 * MB; i += blockDim.x) reinterpret_cast<float*>(red)[i] = 0.f;
  if (threadIdx.x == 0) {
    const uint32_t bytes = uint32_t(min(pieces, 128)) * 512;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base), "r"(bytes) : "memory");
  }
  pdl_wait();  // x is the previous layer's output
  pdl_trigger();
  __syncthreads();
  float acc[MB];
#pragma unroll
  for (int m = 0; m < MB; ++m) acc[m] = 0.f;
  int cur = 0;  // block-local row of the running sums
  auto flush = [&](int next) {
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      float v = acc[m];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[cur][warp][m] += v;
      acc[m] = 0.f;
    }
    cur = next;
  };
  auto fma8 = [&](const uint4 wv, int col) {
    const uint32_t w[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      if (m >= M) break;
      const uint4 xv = __ldg(reinterpret_cast<const uint4*>(x + uint64_t(m) * K + col));
      const uint32_t xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[m] = fmaf(bf(uint16_t(w[j] & 0xffff)), bf(uint16_t(xx[j] & 0xffff)), acc[m]);
        acc[m] = fmaf(bf(uint16_t(w[j] >> 16)), bf(uint16_t(xx[j] >> 16)), acc[m]);
      }
    }
  };
  for (int p0 = warp; p0 < pieces; p0 += 8 * kGemvUnroll) {  // kGemvUnroll pieces of this warp per step
    uint4 wv[kGemvUnroll];
#pragma unroll
    for (int u = 0; u < kGemvUnroll; ++u) {
      const int p = p0 + 8 * u;
      if (p < pieces)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(wv[u].x), "=r"(wv[u].y), "=r"(wv[u].z), "=r"(wv[u].w)
                     : "l"(base + uint64_t(p) * 256 + lane * 8));
    }
#pragma unroll
    for (int u = 0; u < kGemvUnroll; ++u) {
      const int p = p0 + 8 * u;
      if (p >= pieces) break;
      const int row = p / ppr;  // warp-uniform
      if (row != cur) flush(row);
      fma8(wv[u], (p - row * ppr) * 256 + lane * 8);
    }
  }
  flush(0);
  __syncthreads();
  if (threadIdx.x >= rows) return;
  const int r = threadIdx.x, n = n0 + r;
  for (int m = 0; m < M && m < MB; ++m) {
    float v = 0.f;
    for (int w = 0; w < 8; ++w) v += red[r][w][m];  // fixed order: deterministic
    if (bias) v += bias[n];
    if (relu) v = fmaxf(v, 0.f);
    if (out_f32) out_f32[uint64_t(m) * ldo + n] = v;
    else out_bf[uint64_t(m) * ldo + n] = to_bf(v);
  }
}

__global__ void bn_fold_batched_kernel(const FoldJob* __restrict__ jobs, float eps) {
  const FoldJob j = jobs[blockIdx.y];
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= j.C) return;
  const float s = bf(j.gamma[c]) / sqrtf(bf(j.var[c]) + eps);
  j.scale[c] = s;
  j.shift[c] = bf(j.beta[c]) - bf(j.mean[c]) * s;
}

__global__ void bn_fold_kernel(const uint16_t* gamma, const uint16_t* beta, const uint16_t* mean, const uint16_t* var,
                               float eps, int C, float* scale, float* shift) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const float s = bf(gamma[c]) / sqrtf(bf(var[c]) + eps);
  scale[c] = s;
  shift[c] = bf(beta[c]) - bf(mean[c]) * s;
}

__global__ void bf16_to_f32_kernel(const uint16_t* in, float* out, int n) {
  pdl_wait();  // reads the previous layer's output / writes shared scratch
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = bf(in[i]);
}

__global__ void pad_rows_kernel(const uint16_t* in, int rows, int k, uint16_t* out, int kp) {
  const uint64_t total = uint64_t(rows) * kp;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const int col = int(i % kp);
    const uint64_t r = i / kp;
    out[i] = col < k ? in[r * k + col] : uint16_t(0);
  }
}

__global__ void softmax_kernel(const float* in, float* out, int M, int N) {
  pdl_wait();  // reads the previous layer's output / writes shared scratch
  pdl_trigger();
  const int m = blockIdx.x;
  if (m >= M) return;
  __shared__ float red[32];
  const float* x = in + uint64_t(m) * N;
  float mx = -INFINITY;
  for (int i = threadIdx.x; i < N; i += blockDim.x) mx = fmaxf(mx, x[i]);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float s = 0.f;
  for (int i = threadIdx.x; i < N; i += blockDim.x) s += __expf(x[i] - mx);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  s = 0.f;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
  for (int i = threadIdx.x; i < N; i += blockDim.x) out[uint64_t(m) * N + i] = __expf(x[i] - mx) / s;
}

}  // namespace

void input_prep(const float* in, uint16_t* out, int N, int C, int H, int W, cudaStream_t s) {
  launch_pdl(input_prep_kernel, dim3(blocks(uint64_t(N) * C * H * W)), dim3(256), 0, s, in, out, N, C, H, W);
  TRIMS_CUDA(cudaGetLastError());
}

void im2col(const uint16_t* in, uint16_t* A, int N, int H, int W, int Ctot, int c_off, int Cg, int R, int S, int stride,
            int pad, int P, int Q, int Kp, cudaStream_t s, int groups) {
  const uint64_t work = uint64_t(N) * P * Q * ((Cg % 8 == 0 && Ctot % 8 == 0 && c_off % 8 == 0 && Kp % 8 == 0) ? Kp / 8 : R);
  launch_pdl(im2col_kernel, dim3(blocks(work), unsigned(groups)), dim3(256), 0, s, in, A, N, H, W, Ctot, c_off, Cg, R, S,
             stride, pad, P, Q, Kp);
  TRIMS_CUDA(cudaGetLastError());
}

void im2col_input(const float* in, uint16_t* A, int N, int C, int H, int W, int R, int S, int stride, int pad, int P,
                  int Q, int Kp, cudaStream_t s) {
  if (Kp % 8 || Kp > kIm2colMaxK) raise(Errc::InvalidArgument, "im2col_input needs Kp % 8 == 0, Kp <= 512");
  const uint64_t chunks = uint64_t(N) * P * Q * (Kp / 8);
  launch_pdl(im2col_input_kernel, dim3(unsigned(std::min<uint64_t>((chunks + 255) / 256, 148 * 16))), dim3(256), 0, s,
             in, A, N, C, H, W, R, S, stride, pad, P, Q, Kp);
}

void maxpool(const uint16_t* in, uint16_t* out, int N, int H, int W, int C, int k, int stride, int pad, int P, int Q,
             cudaStream_t s, bool nchw) {
  if (C % 8) raise(Errc::InvalidArgument, "maxpool needs C % 8 == 0");
  const dim3 g(blocks(uint64_t(N) * P * Q * C / 8));
  const int o = nchw ? 1 : 0;
  if (k == 3) launch_pdl(maxpool_kernel<3>, g, dim3(256), 0, s, in, out, N, H, W, C, k, stride, pad, P, Q, o);
  else if (k == 2) launch_pdl(maxpool_kernel<2>, g, dim3(256), 0, s, in, out, N, H, W, C, k, stride, pad, P, Q, o);
  else launch_pdl(maxpool_kernel<0>, g, dim3(256), 0, s, in, out, N, H, W, C, k, stride, pad, P, Q, o);
  TRIMS_CUDA(cudaGetLastError());
}

void avgpool_global(const uint16_t* in, uint16_t* out, int N, int HW, int C, cudaStream_t s) {
  launch_pdl(avgpool_kernel, dim3(unsigned(N * ((C + 63) / 64))), dim3(256), 0, s, in, out, N, HW, C);
  TRIMS_CUDA(cudaGetLastError());
}

void flatten_nchw(const uint16_t* in, uint16_t* out, int N, int HW, int C, cudaStream_t s) {
  launch_pdl(flatten_nchw_kernel, dim3(blocks(uint64_t(N) * HW * C)), dim3(256), 0, s, in, out, N, HW, C);
  TRIMS_CUDA(cudaGetLastError());
}

void gemv(const uint16_t* x, int M, int K, const uint16_t* W, int N, const float* bias, bool relu, uint16_t* out_bf,
          float* out_f32, int ldo, int sms, cudaStream_t s) {
  if (K % 256) raise(Errc::InvalidArgument, "gemv needs K % 256 == 0");
  // rows per block: 8, or fewer when that leaves fewer than 2 blocks per SM
  // (TRIMS_GEMV_R / TRIMS_GEMV_U override rows per block / loads in flight)
  static const int r_env = std::getenv("TRIMS_GEMV_R") ? std::atoi(std::getenv("TRIMS_GEMV_R")) : 0;
  static const int u_env = std::getenv("TRIMS_GEMV_U") ? std::atoi(std::getenv("TRIMS_GEMV_U")) : 8;
  // Balanced (default): b blocks per SM, b = the fewest that keep a block
  // <= kGemvRows rows (>= 2), rows spread evenly: every SM streams the same
  // share of W (fixed R rows per block left up to a third of the SMs with
  // one block more than the rest). TRIMS_GEMV_R=n: n rows per block (A/B).
  int R = 0;
  unsigned grid = 0;
  if (r_env >= 1 && r_env <= kGemvRows) {
    R = r_env;
    grid = unsigned((N + R - 1) / R);
  } else {
    const int per_sm = std::max(2, (N + sms * kGemvRows - 1) / (sms * kGemvRows));
    grid = unsigned(std::min(N, sms * per_sm));
  }
  auto go = [&](auto k) { launch_pdl(k, dim3(grid), dim3(256), 0, s, x, M, K, W, N, bias, relu, out_bf, out_f32, ldo, R); };
  if (M > 8) raise(Errc::InvalidArgument, "gemv is for M <= 8");
  if (u_env == 4) {
    if (M <= 1) go(gemv_kernel<1, 4>);
    else if (M <= 4) go(gemv_kernel<4, 4>);
    else go(gemv_kernel<8, 4>);
  } else if (u_env == 16) {
    if (M <= 1) go(gemv_kernel<1, 16>);
    else if (M <= 4) go(gemv_kernel<4, 16>);
    else go(gemv_kernel<8, 16>);
  } else {
    if (M <= 1) go(gemv_kernel<1, 8>);
    else if (M <= 4) go(gemv_kernel<4, 8>);
    else go(gemv_kernel<8, 8>);
  }
  TRIMS_CUDA(cudaGetLastError());
}

void bn_fold_batched(const FoldJob* d_jobs, int njobs, int max_c, float eps, cudaStream_t s) {
  if (!njobs) return;
  bn_fold_batched_kernel<<<dim3((max_c + 255) / 256, njobs), 256, 0, s>>>(d_jobs, eps);  // bind time: no PDL
  TRIMS_CUDA(cudaGetLastError());
}

void bn_fold(const uint16_t* gamma, const uint16_t* beta, const uint16_t* mean, const uint16_t* var, float eps, int C,
             float* scale, float* shift, cudaStream_t s) {
  bn_fold_kernel<<<(C + 255) / 256, 256, 0, s>>>(gamma, beta, mean, var, eps, C, scale, shift);  // bind time: no PDL
  TRIMS_CUDA(cudaGetLastError());
}

void bf16_to_f32(const uint16_t* in, float* out, int n, cudaStream_t s) {
  launch_pdl(bf16_to_f32_kernel, dim3((n + 255) / 256), dim3(256), 0, s, in, out, n);
  TRIMS_CUDA(cudaGetLastError());
}

void pad_rows(const uint16_t* in, int rows, int k, uint16_t* out, int kp, cudaStream_t s) {
  pad_rows_kernel<<<blocks(uint64_t(rows) * kp), 256, 0, s>>>(in, rows, k, out, kp);  // bind time: no PDL
  TRIMS_CUDA(cudaGetLastError());
}

void softmax(const float* in, float* out, int M, int N, cudaStream_t s) {
  launch_pdl(softmax_kernel, dim3(M), dim3(256), 0, s, in, out, M, N);
  TRIMS_CUDA(cudaGetLastError());
}

}  // namespace trims::nn
