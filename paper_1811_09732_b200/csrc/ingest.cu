// ingest.cu — K2 (dtype convert) + K3 (KCRS->KRSC permute) + K4 (block
// checksum) fused in one persistent tile kernel, plus K5 synthetic fills.
//
// HBM-bound byte work: 128-bit coalesced loads of the staged raw blob, one
// 64-bit store per resident word, the checksum of every stored word folded in
// registers and reduced once per tile (warp shuffle + one u64 atomic). The
// conversions are integer-defined so they are bit-identical to the CPU oracle
// (oracle/trims_oracle.c) — no reliance on hardware NaN canonicalisation.
#include <algorithm>
#include <queue>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "cuda_util.hpp"
#include "ingest.hpp"

namespace trims::ingest {

namespace {

constexpr uint64_t kGold = 0x9e3779b97f4a7c15ull;
constexpr int kThreads = 256;
constexpr uint32_t kHashTile = 64u << 10;     // bytes per OP_HASH tile
constexpr uint32_t kPermSmem = 24u << 10;     // smem of the direct (non-TMA) permute path
constexpr int kUnroll = 4;                    // 128-bit loads in flight per thread (direct paths)
constexpr int kMaxStages = 16;                // TMA ring depth limit (runtime depth <= this)

// TMA ring geometry (host side): stage bytes = raw source bytes per tile,
// depth, CTAs per SM. Defaults tuned on B200; TRIMS_TMA_{STAGE_KB,STAGES,CTAS}
// override them for sweeps (scripts/prof_transform.py).
struct RingCfg {
  uint32_t stage_bytes, stages, ctas_per_sm;
  uint32_t stage_alloc() const { return stage_bytes + 128; }  // + 16-byte realignment slack, 128-aligned
};
const RingCfg& ring_cfg() {
  static const RingCfg c = [] {
    auto env = [](const char* k, uint32_t d) {
      const char* v = std::getenv(k);
      return v ? uint32_t(std::strtoul(v, nullptr, 10)) : d;
    };
    // 64 KiB x 3 stages x 1 CTA/SM won the sweep (scripts/sweep_ring.sh): the
    // per-tile fixed cost dominates below 32 KiB stages.
    RingCfg r{env("TRIMS_TMA_STAGE_KB", 64) << 10, env("TRIMS_TMA_STAGES", 3), env("TRIMS_TMA_CTAS", 1)};
    r.stages = std::max(2u, std::min<uint32_t>(r.stages, kMaxStages));
    // the ring + the static descriptor batch (18 KiB) + barriers must fit the
    // 227 KiB a CTA can opt into: an A/B setting that does not is refused here
    // with a clear message rather than by cudaFuncSetAttribute
    constexpr uint64_t kSmemCap = 227u << 10, kStatic = 20u << 10;
    if (r.stage_bytes < (4u << 10) || uint64_t(r.stages) * r.stage_alloc() + kStatic > kSmemCap)
      raise(Errc::InvalidArgument, "TRIMS_TMA_STAGES x TRIMS_TMA_STAGE_KB = " + std::to_string(r.stages) + " x " +
                                       std::to_string(r.stage_bytes >> 10) + " KiB does not fit shared memory");
    return r;
  }();
  return c;
}
#ifndef TRIMS_CONSUMER_WARPS
#define TRIMS_CONSUMER_WARPS 16
#endif
constexpr int kConsumerWarps = TRIMS_CONSUMER_WARPS;  // TMA kernel: 1 producer warp + consumer warps
constexpr int kTmaThreads = 32 * (kConsumerWarps + 1);

#ifdef TRIMS_TRACE
// Diagnostic build only (make EXTRA=-DTRIMS_TRACE ...; scripts/transform_trace.py):
// one record per CTA launch, appended in start order (so back-to-back
// launches are all kept): [start, first stage ready, last push issued, end,
// staged bytes, tiles, static bin issued, dynamic tiles taken, launch ticket
// base (distinct per launch), blockIdx.x] (times in %globaltimer ns).
constexpr int kTraceW = 10, kTraceCap = 16384;
__device__ unsigned long long g_ttrace[kTraceCap * kTraceW];
__device__ unsigned int g_tslot_n;
__shared__ unsigned int g_tslot;  // this CTA's record
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE_SET(i, v) (g_tslot < kTraceCap ? (void)(g_ttrace[g_tslot * kTraceW + (i)] = (v)) : (void)0)
#define TRACE_MAX(i, v) (g_tslot < kTraceCap ? (void)atomicMax(&g_ttrace[g_tslot * kTraceW + (i)], (v)) : (void)0)
#define TRACE_ADD(i, v) (g_tslot < kTraceCap ? (void)(g_ttrace[g_tslot * kTraceW + (i)] += (v)) : (void)0)
#else
#define TRACE_SET(i, v) ((void)0)
#define TRACE_MAX(i, v) ((void)0)
#define TRACE_ADD(i, v) ((void)0)
#endif
constexpr uint32_t kDescCap = 384;  // static-schedule descriptors staged in smem per batch (18 KiB)
// dynamic share of a TMA group's tile cost: 20 % measured best back to back
// (ResNet-50 28.3 vs 28.8 us at 15 %, VGG-16 125.7 vs 126.3 us; profiles/r01f/transform_tail_ab.log)
constexpr int kDefaultTailPct = 20;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t word_hash(uint64_t w, uint64_t gw) { return checksum_term(w, gw); }

// dtype codes are fmt::DType: F64=0 F32=1 F16=2 I8=3 BF16=4
template <int DT> struct Bits;
template <> struct Bits<0> { using T = uint64_t; };
template <> struct Bits<1> { using T = uint32_t; };
template <> struct Bits<2> { using T = uint16_t; };
template <> struct Bits<3> { using T = uint8_t; };
template <> struct Bits<4> { using T = uint16_t; };
template <int DT> constexpr int esize() { return int(sizeof(typename Bits<DT>::T)); }

// bf16 NaN encoding is the canonical 0x7fff: what the B200 cvt.rn.bf16x2.f32
// instruction produces (probed: scripts/probe_cvt.cu, 4M values, no other
// difference from integer RNE), so the hardware pair-convert below and these
// scalar integer paths agree bit for bit.
__device__ __forceinline__ uint16_t f32_to_bf16(uint32_t u) {
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t(0x7fffu);
  return uint16_t((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

// Two fp32 -> packed bf16x2 (x0 in the low half) in one instruction.
__device__ __forceinline__ uint32_t f32x2_to_bf16x2(uint32_t x0, uint32_t x1) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(x1)), "f"(__uint_as_float(x0)));
  return r;
}

__device__ __forceinline__ uint16_t f64_to_bf16(uint64_t u) {
  uint16_t sign = uint16_t((u >> 48) & 0x8000u);
  uint64_t e = (u >> 52) & 0x7ff, m = u & ((1ull << 52) - 1);
  if (e == 0x7ff) return m ? uint16_t(0x7fffu) : uint16_t(sign | 0x7f80u);
  if (e == 0) return sign;
  int64_t eb = int64_t(e) - 1023 + 127;
  if (eb >= 255) return uint16_t(sign | 0x7f80u);
  uint64_t sig = (1ull << 52) | m, q, r, half;
  if (eb >= 1) {
    q = (uint64_t(eb) << 7) | ((sig >> 45) & 0x7f);
    r = sig & ((1ull << 45) - 1);
    half = 1ull << 44;
  } else {
    uint64_t shift = 45 + uint64_t(1 - eb);
    if (shift > 54) return sign;
    q = sig >> shift;
    r = sig & ((1ull << shift) - 1);
    half = 1ull << (shift - 1);
  }
  if (r > half || (r == half && (q & 1))) q += 1;
  return uint16_t(sign | q);
}

__device__ __forceinline__ uint32_t f64_to_f32(uint64_t u) {
  if ((u & 0x7fffffffffffffffull) > 0x7ff0000000000000ull) return uint32_t((u >> 32) & 0x80000000u) | 0x7fc00000u;
  return __float_as_uint(__double2float_rn(__longlong_as_double((long long)u)));
}

// f16 -> f32 is exact; the hardware widening convert handles normals and
// subnormals in one instruction (the software normalisation loop it replaces
// made the f16 transform variants spill). Inf/NaN keep their payload bits
// verbatim, as the oracle does (the hardware would quiet a signalling NaN).
__device__ __forceinline__ uint32_t f16_to_f32(uint16_t hbits) {
  if ((hbits & 0x7c00u) == 0x7c00u)
    return (uint32_t(hbits & 0x8000u) << 16) | 0x7f800000u | (uint32_t(hbits & 0x3ffu) << 13);
  float f;
  asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(hbits));
  return __float_as_uint(f);
}

template <int S, int D>
__device__ __forceinline__ typename Bits<D>::T cvt(typename Bits<S>::T x) {
  if constexpr (S == D) return x;
  else if constexpr (S == 1 && D == 4) return f32_to_bf16(x);
  else if constexpr (S == 0 && D == 1) return f64_to_f32(x);
  else if constexpr (S == 0 && D == 4) return f64_to_bf16(x);
  else if constexpr (S == 2 && D == 1) return f16_to_f32(x);
  else if constexpr (S == 2 && D == 4) return f32_to_bf16(f16_to_f32(x));
  else if constexpr (S == 4 && D == 1) return uint32_t(x) << 16;
  else return 0;  // unreachable: build_tiles rejects other pairs
}

// One resident word from EPW source elements (the pair-convert instruction
// for fp32 -> bf16).
template <int S, int D, int N>
__device__ __forceinline__ uint64_t pack_word(const typename Bits<S>::T (&v)[N]) {
  if constexpr (S == 1 && D == 4 && N == 4) {
    return uint64_t(f32x2_to_bf16x2(v[0], v[1])) | (uint64_t(f32x2_to_bf16x2(v[2], v[3])) << 32);
  } else {
    uint64_t word = 0;
#pragma unroll
    for (int q = 0; q < N; ++q) word |= uint64_t(cvt<S, D>(v[q])) << (8 * esize<D>() * q);
    return word;
  }
}

// One element S -> D; fp32 -> bf16 through the (probed) hardware convert.
template <int S, int D>
__device__ __forceinline__ typename Bits<D>::T cvt1(typename Bits<S>::T x) {
  if constexpr (S == 1 && D == 4) return uint16_t(f32x2_to_bf16x2(x, 0u));
  else return cvt<S, D>(x);
}

// Load N elements of type T starting at p (p aligned to N*sizeof(T)) with
// the widest vector loads available (16 B), read-only path.
template <typename T, int N>
__device__ __forceinline__ void load_vec(const uint8_t* p, T (&v)[N]) {
  constexpr int B = N * int(sizeof(T));
  if constexpr (B >= 16) {
#pragma unroll
    for (int i = 0; i < B / 16; ++i) {
      uint4 q = __ldg(reinterpret_cast<const uint4*>(p) + i);
      memcpy(reinterpret_cast<uint8_t*>(v) + 16 * i, &q, 16);
    }
  } else if constexpr (B == 8) {
    uint2 q = __ldg(reinterpret_cast<const uint2*>(p));
    memcpy(v, &q, 8);
  } else if constexpr (B == 4) {
    uint32_t q = __ldg(reinterpret_cast<const unsigned int*>(p));
    memcpy(v, &q, 4);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = reinterpret_cast<const T*>(p)[i];
  }
}

// Per-warp checksum accumulator that flushes (warp reduce + one atomic) only
// when the bucket changes: a CTA's consecutive tiles mostly belong to the same
// large tensor, so the atomics on a hot bucket stay few.
struct WarpSum {
  uint32_t bucket{~0u};
  uint64_t acc{0};
  __device__ __forceinline__ void flush(unsigned long long* sums) {
    if (bucket == ~0u) return;
    uint64_t v = acc;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sums[bucket], (unsigned long long)v);
    acc = 0;
  }
  __device__ __forceinline__ void add(uint32_t b, uint64_t v, unsigned long long* sums) {
    if (b != bucket) {  // warp-uniform
      flush(sums);
      bucket = b;
    }
    acc += v;
  }
};

__device__ __forceinline__ uint64_t block_sum(uint64_t v, unsigned long long* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  uint64_t s = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  __syncthreads();
  return s;
}

// OP_HASH: resident bytes already in place (identity ingest); hash them.
__device__ uint64_t tile_hash(const Tile& t, const uint8_t* dst) {
  const uint8_t* base = dst + t.dst_off;
  const uint64_t gw0 = t.dst_off >> 3;
  const uint32_t words = t.dst_bytes >> 3;
  uint64_t acc = 0;
  uint32_t pairs = words >> 1;
  if ((t.dst_off & 15) == 0) {
    for (uint32_t i = threadIdx.x; i < pairs; i += kThreads) {
      uint4 q = __ldg(reinterpret_cast<const uint4*>(base) + i);
      uint64_t a = (uint64_t(q.y) << 32) | q.x, b = (uint64_t(q.w) << 32) | q.z;
      acc += word_hash(a, gw0 + 2 * i) + word_hash(b, gw0 + 2 * i + 1);
    }
    if ((words & 1) && threadIdx.x == 0) {
      uint64_t a = __ldg(reinterpret_cast<const unsigned long long*>(base) + words - 1);
      acc += word_hash(a, gw0 + words - 1);
    }
  } else {
    for (uint32_t i = threadIdx.x; i < words; i += kThreads)
      acc += word_hash(__ldg(reinterpret_cast<const unsigned long long*>(base) + i), gw0 + i);
  }
  return acc;
}

// OP_HASH tile of a peer pull: copy the resident bytes from `src` (a peer
// GPU's sealed segment, mapped into this device over NVLink) to `dst` and hash
// them in the same pass. Four 16-byte loads in flight per thread to cover the
// NVLink round trip.
__device__ uint64_t tile_pull(const Tile& t, const uint8_t* src, uint8_t* dst) {
  const uint8_t* s = src + t.dst_off;
  uint8_t* d = dst + t.dst_off;
  const uint64_t gw0 = t.dst_off >> 3;
  const uint32_t words = t.dst_bytes >> 3;
  uint64_t acc = 0;
  if ((t.dst_off & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    const uint32_t pairs = words >> 1;
    uint32_t i = threadIdx.x;
    for (; i + 3 * kThreads < pairs; i += 4 * kThreads) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = __ldcs(s4 + i + u * kThreads);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t j = i + u * kThreads;
        d4[j] = q[u];
        acc += word_hash((uint64_t(q[u].y) << 32) | q[u].x, gw0 + 2 * j) +
               word_hash((uint64_t(q[u].w) << 32) | q[u].z, gw0 + 2 * j + 1);
      }
    }
    for (; i < pairs; i += kThreads) {
      const uint4 q = __ldcs(s4 + i);
      d4[i] = q;
      acc += word_hash((uint64_t(q.y) << 32) | q.x, gw0 + 2 * i) + word_hash((uint64_t(q.w) << 32) | q.z, gw0 + 2 * i + 1);
    }
    if ((words & 1) && threadIdx.x == 0) {
      const unsigned long long a = reinterpret_cast<const unsigned long long*>(s)[words - 1];
      reinterpret_cast<unsigned long long*>(d)[words - 1] = a;
      acc += word_hash(a, gw0 + words - 1);
    }
  } else {
    for (uint32_t i = threadIdx.x; i < words; i += kThreads) {
      const unsigned long long a = reinterpret_cast<const unsigned long long*>(s)[i];
      reinterpret_cast<unsigned long long*>(d)[i] = a;
      acc += word_hash(a, gw0 + i);
    }
  }
  return acc;
}

// OP_CVT: elementwise convert S -> D; one resident word per thread step,
// kCvtUnroll independent 128-bit loads in flight per thread.
constexpr int kCvtUnroll = 8;
template <int S, int D>
__device__ uint64_t tile_cvt(const Tile& t, const uint8_t* src, uint8_t* dst) {
  // f64 sources: a word is 32 source bytes, so half the groups keep the same
  // bytes in flight without spilling
  constexpr int kUnroll = S == 0 ? kCvtUnroll / 2 : kCvtUnroll;
  using ST = typename Bits<S>::T;
  using DT = typename Bits<D>::T;
  constexpr int DS = esize<D>(), SS = esize<S>(), EPW = 8 / DS;
  const uint8_t* s = src + t.src_off;
  uint64_t* d = reinterpret_cast<uint64_t*>(dst + t.dst_off);
  const uint64_t gw0 = t.dst_off >> 3;
  const uint32_t words = t.dst_bytes >> 3, n = t.n_elem;
  uint64_t acc = 0;
  // kUnroll independent 128-bit loads in flight per thread before any use.
  for (uint32_t base = threadIdx.x; base < words; base += kThreads * kUnroll) {
    ST v[kUnroll][EPW];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t e0 = (base + u * kThreads) * EPW;
      if (e0 + EPW <= n) load_vec<ST, EPW>(s + uint64_t(e0) * SS, v[u]);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t w = base + u * kThreads;
      if (w >= words) break;
      const uint32_t e0 = w * EPW;
      uint64_t word = 0;
      if (e0 + EPW <= n) {
        word = pack_word<S, D>(v[u]);
      } else if (e0 < n) {
        for (int q = 0; q < EPW && e0 + q < n; ++q) {
          ST x;
          memcpy(&x, s + uint64_t(e0 + q) * SS, SS);
          word |= uint64_t(cvt<S, D>(x)) << (8 * DS * q);
        }
      }
      d[w] = word;
      acc += word_hash(word, gw0 + w);
    }
  }
  return acc;
}

// OP_PERM: g k-slices [C][RS] -> [RS][C], converted, via shared memory.
template <int S, int D>
__device__ uint64_t tile_perm(const Tile& t, const uint8_t* src, uint8_t* dst, uint8_t* smem) {
  using ST = typename Bits<S>::T;
  using DT = typename Bits<D>::T;
  constexpr int DS = esize<D>(), SS = esize<S>(), EPW = 8 / DS;
  const uint8_t* s = src + t.src_off;
  DT* sm = reinterpret_cast<DT*>(smem);
  const uint32_t n = t.n_elem, C = t.C, RS = t.RS, CRS = C * RS;
  // slice group too large for this path's smem: read the source directly
  const bool gather = t.pad_ != 0 || uint64_t(n) * DS > kPermSmem;
  // phase 1: coalesced vector loads in source order -> converted in smem
  const uint32_t groups = gather ? 0 : n / EPW;
  for (uint32_t base = threadIdx.x; base < groups; base += kThreads * kUnroll) {
    ST v[kUnroll][EPW];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t g = base + u * kThreads;
      if (g < groups) load_vec<ST, EPW>(s + uint64_t(g) * EPW * SS, v[u]);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t g = base + u * kThreads;
      if (g < groups) {  // one packed 8-byte shared store per group
        uint64_t word = 0;
#pragma unroll
        for (int q = 0; q < EPW; ++q) word |= uint64_t(cvt<S, D>(v[u][q])) << (8 * DS * q);
        reinterpret_cast<uint64_t*>(sm)[g] = word;
      }
    }
  }
  for (uint32_t e = groups * EPW + threadIdx.x; !gather && e < n; e += kThreads) {
    ST x;
    memcpy(&x, s + uint64_t(e) * SS, SS);
    sm[e] = cvt<S, D>(x);
  }
  __syncthreads();
  auto elem = [&](uint32_t i) -> DT {
    if (!gather) return sm[i];
    ST x;
    memcpy(&x, s + uint64_t(i) * SS, SS);
    return cvt<S, D>(x);
  };
  // phase 2: resident order o = (k*RS + rs)*C + c
  uint64_t* d = reinterpret_cast<uint64_t*>(dst + t.dst_off);
  const uint64_t gw0 = t.dst_off >> 3;
  const uint32_t words = t.dst_bytes >> 3;
  uint64_t acc = 0;
  if (!gather && (C * DS) % 8 == 0) {
    // Row path: one warp per output row (k, rs) of C contiguous elements, so
    // the only division is per row; lanes write consecutive words.
    const uint32_t wpr = C / EPW, rows = (n / CRS) * RS;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t row = warp; row < rows; row += kThreads / 32) {
      const uint32_t k = row / RS, rs = row - k * RS;
      const DT* col = sm + k * CRS + rs;
      uint64_t* drow = d + uint64_t(row) * wpr;
      const uint64_t gwr = gw0 + uint64_t(row) * wpr;
      for (uint32_t wi = lane; wi < wpr; wi += 32) {
        const DT* e = col + wi * EPW * RS;
        uint64_t word = 0;
#pragma unroll
        for (int q = 0; q < EPW; ++q) word |= uint64_t(e[q * RS]) << (8 * DS * q);
        drow[wi] = word;
        acc += word_hash(word, gwr + wi);
      }
    }
    for (uint32_t w = n * DS / 8 + threadIdx.x; w < words; w += kThreads) {  // trailing pad
      d[w] = 0;
      acc += word_hash(0, gw0 + w);
    }
    __syncthreads();  // smem reuse by the next tile
    return acc;
  }
  for (uint32_t w = threadIdx.x; w < words; w += kThreads) {
    uint32_t o = w * EPW;
    uint64_t word = 0;
    if (o < n) {
      uint32_t k = o / CRS, rem = o - k * CRS, rs = rem / C, c = rem - rs * C;
#pragma unroll
      for (int q = 0; q < EPW; ++q) {
        if (o + q < n) word |= uint64_t(elem(k * CRS + c * RS + rs)) << (8 * DS * q);
        if (++c == C) {
          c = 0;
          if (++rs == RS) {
            rs = 0;
            ++k;
          }
        }
      }
    }
    d[w] = word;
    acc += word_hash(word, gw0 + w);
  }
  __syncthreads();  // smem reuse by the next tile
  return acc;
}

// One specialisation per (source dtype, resident dtype) pair keeps register
// pressure at what that pair needs; tiles of other pairs in the same range are
// skipped (the host launches one kernel per pair present, usually exactly one).
template <int S, int D>
__global__ void __launch_bounds__(kThreads, 2) transform_kernel(const Tile* __restrict__ tiles, uint32_t ntiles,
                                                             const uint8_t* __restrict__ src,
                                                             uint8_t* __restrict__ dst,
                                                             unsigned long long* __restrict__ sums) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long red[kThreads / 32];
  Tile next = blockIdx.x < ntiles ? tiles[blockIdx.x] : Tile{};
  WarpSum ws;
  for (uint32_t i = blockIdx.x; i < ntiles; i += gridDim.x) {
    const Tile t = next;
    if (i + gridDim.x < ntiles) next = tiles[i + gridDim.x];  // descriptor prefetch
    if (t.op == OP_HASH || t.sdt != S || t.ddt != D) continue;  // block-uniform
    if (t.op == OP_PERM) {
      const uint64_t acc = block_sum(tile_perm<S, D>(t, src, dst, smem), red);
      if (threadIdx.x == 0) atomicAdd(&sums[t.tensor], (unsigned long long)acc);
    } else {  // no CTA barrier: warps run ahead into the next tile
      ws.add(t.tensor, tile_cvt<S, D>(t, src, dst), sums);
    }
  }
  ws.flush(sums);
}

__global__ void __launch_bounds__(kThreads) hash_tiles_kernel(const Tile* __restrict__ tiles, uint32_t ntiles,
                                                              const uint8_t* __restrict__ dst,
                                                              unsigned long long* __restrict__ sums) {
  __shared__ unsigned long long red[kThreads / 32];
  for (uint32_t i = blockIdx.x; i < ntiles; i += gridDim.x) {
    const Tile t = tiles[i];
    if (t.op != OP_HASH) continue;
    uint64_t acc = block_sum(tile_hash(t, dst), red);
    if (threadIdx.x == 0) atomicAdd(&sums[t.tensor], (unsigned long long)acc);
  }
}

__global__ void __launch_bounds__(kThreads) pull_tiles_kernel(const Tile* __restrict__ tiles, uint32_t ntiles,
                                                              const uint8_t* __restrict__ src,
                                                              uint8_t* __restrict__ dst,
                                                              unsigned long long* __restrict__ sums) {
  __shared__ unsigned long long red[kThreads / 32];
  for (uint32_t i = blockIdx.x; i < ntiles; i += gridDim.x) {
    const Tile t = tiles[i];
    if (t.op != OP_HASH) continue;
    uint64_t acc = block_sum(tile_pull(t, src, dst), red);
    if (threadIdx.x == 0) atomicAdd(&sums[t.tensor], (unsigned long long)acc);
  }
}

// ---------------------------------------------------------------------------
// TMA-staged variant (the production path): each persistent CTA streams its
// tiles' raw source bytes into a multi-stage shared-memory ring with 1-D bulk
// async copies (cp.async.bulk, mbarrier complete_tx), and converts / permutes
// straight out of shared memory while the next tiles are in flight.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TRIMS_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TRIMS_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// 64-bit warp sum from three 32-bit redux.sync adds (16 + 16 + 32 bits): the
// low pieces cannot overflow 32 lanes, the high piece only matters mod 2^32.
__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
  const uint32_t l = __reduce_add_sync(0xffffffffu, uint32_t(v) & 0xffffu);
  const uint32_t m = __reduce_add_sync(0xffffffffu, uint32_t(v) >> 16);
  const uint32_t h = __reduce_add_sync(0xffffffffu, uint32_t(v >> 32));
  return uint64_t(l) + (uint64_t(m) << 16) + (uint64_t(h) << 32);
}

// EPW source elements at stride `stride` (shared memory) -> one resident word;
// fp32 -> bf16 through the pair-convert instruction.
template <int S, int D, int EPW>
__device__ __forceinline__ uint64_t gather_word(const typename Bits<S>::T* e, uint32_t stride) {
  typename Bits<S>::T v[EPW];
#pragma unroll
  for (int q = 0; q < EPW; ++q) v[q] = e[q * stride];
  return pack_word<S, D, EPW>(v);
}

// Consumer warps of transform_tma_kernel: wait for a staged tile, convert /
// permute it out of shared memory, store + hash the resident words, hand the
// stage back.
template <int S, int D>
__device__ __forceinline__ void consume_tiles(const uint8_t* ring, uint64_t* full, uint64_t* empty, const Tile* staged,
                                              uint8_t* __restrict__ dst, unsigned long long* __restrict__ sums,
                                              uint32_t stages, uint32_t stage_alloc) {
  using ST = typename Bits<S>::T;
  constexpr int DS = esize<D>(), SS = esize<S>(), EPW = 8 / DS;
  constexpr uint32_t kC = kConsumerWarps * 32;  // consumer threads
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ct = threadIdx.x - 32, cw = warp - 1;
  uint32_t bucket = ~0u;  // per-warp checksum accumulator, flushed when the tensor changes
  uint64_t wacc = 0;
  uint32_t s = 0, phase = 0;
  pdl_wait();  // no write (dst, sums) before the previous grid completes
#ifdef TRIMS_TRACE
  bool first = true;
#endif
  for (;;) {
    mbar_wait(&full[s], phase);
#ifdef TRIMS_TRACE
    if (first && cw == 0 && lane == 0) TRACE_SET(1, gtimer());
    first = false;
#endif
    const Tile t = staged[s];
    if (t.op == OP_END) break;
    const ST* el = reinterpret_cast<const ST*>(ring + s * stage_alloc + (t.src_off & 15));
    uint64_t* d = reinterpret_cast<uint64_t*>(dst + t.dst_off);
    const uint64_t gw0 = t.dst_off >> 3;
    const uint32_t words = t.dst_bytes >> 3, n = t.n_elem;
    uint64_t acc = 0;
    if (t.op == OP_CVT) {
      const bool vec = ((t.src_off & 15) % (EPW * SS)) == 0;
      const uint32_t full_words = vec ? n / EPW : 0;
#pragma unroll 4
      for (uint32_t w = ct; w < full_words; w += kC) {
        ST v[EPW];
        if constexpr (EPW * SS >= 16) {
#pragma unroll
          for (int i = 0; i < EPW * SS / 16; ++i) reinterpret_cast<uint4*>(v)[i] = reinterpret_cast<const uint4*>(el + w * EPW)[i];
        } else if constexpr (EPW * SS == 8) {
          *reinterpret_cast<uint2*>(v) = *reinterpret_cast<const uint2*>(el + w * EPW);
        } else {
#pragma unroll
          for (int q = 0; q < EPW; ++q) v[q] = el[w * EPW + q];
        }
        const uint64_t word = pack_word<S, D, EPW>(v);
        d[w] = word;
        acc += word_hash(word, gw0 + w);
      }
      for (uint32_t w = full_words + ct; w < words; w += kC) {  // partial word, trailing pad
        const uint32_t e0 = w * EPW;
        uint64_t word = 0;
        for (int q = 0; q < EPW && e0 + q < n; ++q) word |= uint64_t(cvt<S, D>(el[e0 + q])) << (8 * DS * q);
        d[w] = word;
        acc += word_hash(word, gw0 + w);
      }
    } else {  // OP_PERM: source [g][C][RS] in smem -> resident [g][RS][C]
      const uint32_t C = t.C, RS = t.RS, CRS = C * RS;
      const uint32_t wpr = (C * DS) / 8, rows = t.rows;
      const uint32_t rs_magic = t.rs_magic;  // k = row / RS = umulhi(row, ceil(2^32/RS))
      uint32_t body = 0;  // words written by the fast paths below
      if ((C * DS) % 8 == 0 && RS > 1 && (wpr & 7) == 0) {
        // Units of 4 rows x 8 words: lane (lane>>3, lane&7) takes row 4u'+lane>>3,
        // word 8o+lane&7. For odd RS the 32 lanes of one shared load then hit 32
        // distinct banks (row offsets 0..3 + multiples of 4), with no rotation,
        // so the EPW loads pack straight into pair converts.
        const uint32_t oct = wpr >> 3, units = ((rows + 3) >> 2) * oct;
        const bool pow2 = (oct & (oct - 1)) == 0;
        const uint32_t sh = __ffs(oct) - 1, oct_magic = pow2 ? 0u : 0xffffffffu / oct + 1;
        const uint32_t g = lane >> 3, o = lane & 7;
        body = rows * wpr;
#pragma unroll 2
        for (uint32_t u = cw; u < units; u += kConsumerWarps) {
          const uint32_t q4 = pow2 ? u >> sh : __umulhi(u, oct_magic);
          const uint32_t row = 4 * q4 + g, wi = 8 * (u - q4 * oct) + o;
          if (row < rows) {
            const uint32_t k = __umulhi(row, rs_magic), r = row - k * RS;
            const uint64_t word = gather_word<S, D, EPW>(el + k * CRS + r + wi * EPW * RS, RS);
            const uint32_t it = row * wpr + wi;
            d[it] = word;
            acc += word_hash(word, gw0 + it);
          }
        }
      } else if ((C * DS) % 8 == 0 && RS > 1) {
        // Flattened (row, word) items, 32 consecutive words per warp step.
        const uint32_t items = rows * wpr;
        body = items;
        for (uint32_t it = ct; it < items; it += kC) {
          const uint32_t row = it / wpr, wi = it - row * wpr;
          const uint32_t k = __umulhi(row, rs_magic), r = row - k * RS;
          const uint64_t word = gather_word<S, D, EPW>(el + k * CRS + r + wi * EPW * RS, RS);
          d[it] = word;
          acc += word_hash(word, gw0 + it);
        }
      }
      for (uint32_t w = body + ct; w < words; w += kC) {  // generic path, partial word, pad
        const uint32_t o = w * EPW;
        uint64_t word = 0;
        if (o < n) {
          uint32_t k = o / CRS, rem = o - k * CRS, r = rem / C, c = rem - r * C;
          for (int q = 0; q < EPW && o + q < n; ++q) {
            word |= uint64_t(cvt<S, D>(el[k * CRS + c * RS + r])) << (8 * DS * q);
            if (++c == C) {
              c = 0;
              if (++r == RS) {
                r = 0;
                ++k;
              }
            }
          }
        }
        d[w] = word;
        acc += word_hash(word, gw0 + w);
      }
    }
    if (t.tensor != bucket) {  // warp-uniform
      if (bucket != ~0u) {
        const uint64_t v = warp_sum64(wacc);
        if (lane == 0 && v) atomicAdd(&sums[bucket], (unsigned long long)v);
      }
      bucket = t.tensor;
      wacc = 0;
    }
    wacc += acc;
    __syncwarp();  // every lane's shared-memory reads of stage s are done
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    if (++s == stages) {
      s = 0;
      phase ^= 1;
    }
  }
  if (bucket != ~0u) {
    const uint64_t v = warp_sum64(wacc);
    if (lane == 0 && v) atomicAdd(&sums[bucket], (unsigned long long)v);
  }
#ifdef TRIMS_TRACE
  if (lane == 0) TRACE_MAX(3, gtimer());
#endif
}

// Warp-specialised: warp 0 is the producer (one elected lane issues the bulk
// copies and recycles ring stages through `empty` mbarriers); kConsumerWarps
// warps convert / permute / hash straight out of shared memory. No CTA-wide
// barrier on the steady path: every consumer warp reduces its checksum with
// shuffles and adds it with one atomic per tile.
template <int S, int D>
__global__ void __launch_bounds__(kTmaThreads) transform_tma_kernel(const Tile* __restrict__ tiles, uint32_t ntiles,
                                                                    const uint8_t* __restrict__ src,
                                                                    uint8_t* __restrict__ dst,
                                                                    unsigned long long* __restrict__ sums,
                                                                    uint32_t stages, uint32_t stage_alloc,
                                                                    unsigned int* __restrict__ sched,
                                                                    uint32_t ticket_base, uint32_t stride,
                                                                    uint32_t tail0, uint32_t early) {
  using ST = typename Bits<S>::T;
  constexpr int DS = esize<D>(), SS = esize<S>(), EPW = 8 / DS;
  constexpr uint32_t kC = kConsumerWarps * 32;  // consumer threads
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ Tile staged[kMaxStages];
  __shared__ __align__(16) Tile descs[kDescCap];  // static schedule: this CTA's descriptors

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // PDL: let the next launch in the stream start its prologue on SMs as ours
  // free up. Everything here that touches memory a previous kernel may have
  // written (src, dst, sums, the ticket counters) happens after the
  // producer's griddepcontrol.wait below: consumers only act on staged data.
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#ifdef TRIMS_TRACE
    g_tslot = atomicAdd(&g_tslot_n, 1u);
    TRACE_SET(0, gtimer());
    TRACE_SET(8, ticket_base);
    TRACE_SET(9, blockIdx.x);
    TRACE_SET(3, 0);
    TRACE_SET(4, 0);
    TRACE_SET(5, 0);
    TRACE_SET(7, 0);
#endif
  }
  __syncthreads();

  if (warp == 0) {  // ---------------- producer
    // early != 0: the host guarantees no kernel that triggers its dependents
    // early (a transform, a forward-pass kernel) writes this launch's source
    // (sources are filled by DMA copies or by non-PDL fill kernels), so the
    // first ring fill is requested BEFORE griddepcontrol.wait, while the
    // previous launch drains: consecutive ingests keep HBM busy across the
    // launch boundary. Everything that writes (consumers: dst, sums) and the
    // ticket draws still wait for the previous grid.
    if (!early) pdl_wait();
    bool gated = !early;
    auto gate = [&] {
      if (!gated) {
        pdl_wait();
        gated = true;
      }
    };
    uint32_t s = 0, round = 0;  // ring slot, and how many times the ring has wrapped
    auto push = [&](const Tile& t) {  // lane 0: stage t's raw bytes into slot s
      if (round) mbar_wait(&empty[s], (round - 1) & 1);
      staged[s] = t;
      const uint64_t b = t.src_off & ~15ull, e = (t.src_off + uint64_t(t.n_elem) * SS + 15) & ~15ull;
      mbar_expect_tx(&full[s], uint32_t(e - b));
      bulk_g2s(ring + s * stage_alloc, src + b, uint32_t(e - b), &full[s]);
      TRACE_ADD(4, e - b);
      TRACE_ADD(5, 1);
      if (++s == stages) {
        s = 0;
        ++round;
      }
    };
    if (stride) {
      // Static part: this CTA's bin (balanced on the host) sits at
      // blockIdx.x * stride, padded with OP_END. Its descriptors are copied
      // into shared memory by the whole warp in one round trip per kDescCap
      // entries, so issuing a tile never waits on a global load.
      const Tile* mine = tiles + size_t(blockIdx.x) * stride;
      bool more = true;
      for (uint32_t base = 0; more && base < stride; base += kDescCap) {
        const uint32_t cnt = min(kDescCap, stride - base);
        const uint4* g4 = reinterpret_cast<const uint4*>(mine + base);
        uint4* s4 = reinterpret_cast<uint4*>(descs);
        constexpr uint32_t kW = sizeof(Tile) / 16;
        for (uint32_t i = lane; i < cnt * kW; i += 32) s4[i] = g4[i];
        __syncwarp();
        if (lane == 0) {
          uint32_t j = 0;
          for (; j < cnt && descs[j].op != OP_END; ++j) push(descs[j]);
          more = j == cnt;
        }
        more = __shfl_sync(0xffffffffu, more, 0);
        __syncwarp();
      }
    }
    if (lane == 0) {
      TRACE_SET(6, gtimer());
      gate();
      if (sched && tail0 < ntiles) {
        // Dynamic part: tiles [tail0, ntiles) handed out by a ticket counter,
        // so CTAs that ran slow take fewer of them. The next ticket and its
        // descriptor are fetched while the ring waits.
        uint32_t ti = tail0 + (atomicAdd(sched, 1u) - ticket_base);
        Tile next = ti < ntiles ? tiles[ti] : Tile{};
        while (ti < ntiles) {
          const Tile t = next;
          ti = tail0 + (atomicAdd(sched, 1u) - ticket_base);
          if (ti < ntiles) next = tiles[ti];
          push(t);
          TRACE_ADD(7, 1);
        }
      } else if (!stride) {  // no schedule at all: static round robin
        for (uint32_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) push(tiles[ti]);
      }
      // end marker: consumers leave
      TRACE_SET(2, gtimer());
      if (round) mbar_wait(&empty[s], (round - 1) & 1);
      staged[s].op = OP_END;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    }
  } else {
    consume_tiles<S, D>(ring, full, empty, staged, dst, sums, stages, stage_alloc);
  }
}

using TransformFn = void (*)(const Tile*, uint32_t, const uint8_t*, uint8_t*, unsigned long long*);
using TmaFn = void (*)(const Tile*, uint32_t, const uint8_t*, uint8_t*, unsigned long long*, uint32_t, uint32_t,
                       unsigned int*, uint32_t, uint32_t, uint32_t, uint32_t);

TmaFn pair_tma_kernel(int s, int d) {
  switch (s * 8 + d) {
    case 0 * 8 + 0: return transform_tma_kernel<0, 0>;
    case 1 * 8 + 1: return transform_tma_kernel<1, 1>;
    case 2 * 8 + 2: return transform_tma_kernel<2, 2>;
    case 3 * 8 + 3: return transform_tma_kernel<3, 3>;
    case 4 * 8 + 4: return transform_tma_kernel<4, 4>;
    case 1 * 8 + 4: return transform_tma_kernel<1, 4>;
    case 0 * 8 + 1: return transform_tma_kernel<0, 1>;
    case 0 * 8 + 4: return transform_tma_kernel<0, 4>;
    case 2 * 8 + 1: return transform_tma_kernel<2, 1>;
    case 2 * 8 + 4: return transform_tma_kernel<2, 4>;
    case 4 * 8 + 1: return transform_tma_kernel<4, 1>;
    default: return nullptr;
  }
}

TransformFn pair_kernel(int s, int d) {
  switch (s * 8 + d) {
    case 0 * 8 + 0: return transform_kernel<0, 0>;
    case 1 * 8 + 1: return transform_kernel<1, 1>;
    case 2 * 8 + 2: return transform_kernel<2, 2>;
    case 3 * 8 + 3: return transform_kernel<3, 3>;
    case 4 * 8 + 4: return transform_kernel<4, 4>;
    case 1 * 8 + 4: return transform_kernel<1, 4>;
    case 0 * 8 + 1: return transform_kernel<0, 1>;
    case 0 * 8 + 4: return transform_kernel<0, 4>;
    case 2 * 8 + 1: return transform_kernel<2, 1>;
    case 2 * 8 + 4: return transform_kernel<2, 4>;
    case 4 * 8 + 1: return transform_kernel<4, 1>;
    default: return nullptr;
  }
}

__global__ void __launch_bounds__(kThreads) checksum_kernel(const uint8_t* __restrict__ p, uint64_t nbytes,
                                                            uint64_t word0, unsigned long long* out) {
  __shared__ unsigned long long red[kThreads / 32];
  const uint64_t words = nbytes >> 3;
  uint64_t acc = 0;
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  const bool vec = (reinterpret_cast<uintptr_t>(p) & 15) == 0;
  if (vec) {
    for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < words / 2; i += stride) {
      uint4 q = __ldg(reinterpret_cast<const uint4*>(p) + i);
      acc += word_hash((uint64_t(q.y) << 32) | q.x, word0 + 2 * i) +
             word_hash((uint64_t(q.w) << 32) | q.z, word0 + 2 * i + 1);
    }
  }
  const uint64_t done = vec ? (words / 2) * 2 : 0;
  for (uint64_t i = done + uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < words; i += stride)
    acc += word_hash(__ldg(reinterpret_cast<const unsigned long long*>(p) + i), word0 + i);
  if ((nbytes & 7) && blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t w = 0;
    for (uint64_t b = 0; b < (nbytes & 7); ++b) w |= uint64_t(p[words * 8 + b]) << (8 * b);
    acc += word_hash(w, word0 + words);
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)acc);
}

__global__ void fill_splitmix_kernel(uint64_t* dst, uint64_t n, uint64_t stream, uint64_t k0) {
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += uint64_t(gridDim.x) * blockDim.x)
    dst[j] = mix64(stream + (k0 + j + 1) * kGold);
}

__global__ void fill_uniform_kernel(float* dst, uint64_t n, uint64_t stream, uint64_t j0, float lo, float hi) {
  const float span = __fsub_rn(hi, lo);
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += uint64_t(gridDim.x) * blockDim.x) {
    float u = __fmul_rn(float(mix64(stream + (j0 + j + 1) * kGold) >> 40), 0x1p-24f);
    dst[j] = __fmaf_rn(span, u, lo);
  }
}

bool floating(fmt::DType t) { return t != fmt::DType::I8; }

bool supported_pair(fmt::DType s, fmt::DType d) {
  using fmt::DType;
  if (s == d) return true;
  return (s == DType::F32 && d == DType::BF16) || (s == DType::F64 && d == DType::F32) ||
         (s == DType::F64 && d == DType::BF16) || (s == DType::F16 && d == DType::F32) ||
         (s == DType::F16 && d == DType::BF16) || (s == DType::BF16 && d == DType::F32);
}

// One group's tiles -> nb bins (LPT: largest cost first onto the least loaded
// bin) plus a dynamic tail of the smallest tiles, written back in the group's
// range as [bin 0 | bin 1 | ... | tail]; bin sizes go to `bin_sizes`. Tiles
// keep source order inside a bin, the tail is largest first.
void schedule_bins(std::vector<Tile>& table, Group& g, uint32_t grid, std::vector<uint32_t>& bin_sizes) {
  constexpr uint64_t kFixed = 8u << 10;  // per-tile charge in byte-equivalents
  const uint32_t n = g.end - g.begin, nb = std::min(n, grid);
  std::vector<uint32_t> order(n);
  std::vector<uint64_t> cost(n);
  // TRIMS_PERM_WEIGHT (percent, A/B): extra weight of gathered (RS > 1)
  // permute tiles over streaming ones
  static const uint64_t perm_w = [] {
    const char* e = std::getenv("TRIMS_PERM_WEIGHT");
    return e ? uint64_t(std::clamp(std::atoi(e), 50, 400)) : uint64_t(100);
  }();
  for (uint32_t i = 0; i < n; ++i) {
    const Tile& t = table[g.begin + i];
    order[i] = i;
    cost[i] = kFixed + t.dst_bytes + uint64_t(t.n_elem) * fmt::element_size(fmt::DType(t.sdt));
    if (t.op == OP_PERM && t.RS > 1) cost[i] = cost[i] * perm_w / 100;
  }
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cost[a] > cost[b]; });
  // The smallest tiles worth `tail_pct` % of the cost form the dynamic tail
  // (TRIMS_TILE_TAIL, percent), handed out by tickets after the static bins.
  static const uint64_t tail_pct = [] {
    const char* e = std::getenv("TRIMS_TILE_TAIL");
    return e ? uint64_t(std::clamp(std::atoi(e), 0, 100)) : uint64_t(kDefaultTailPct);
  }();
  uint64_t total = 0;
  for (uint64_t c : cost) total += c;
  uint32_t head = n;
  for (uint64_t acc = 0; head > 0 && (acc + cost[order[head - 1]]) * 100 <= total * tail_pct; --head)
    acc += cost[order[head - 1]];
  using Load = std::pair<uint64_t, uint32_t>;
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (uint32_t b = 0; b < nb; ++b) heap.push({0, b});
  std::vector<uint32_t> bin_of(n, nb);  // nb = the dynamic tail
  for (uint32_t k = 0; k < head; ++k) {
    const uint32_t i = order[k];
    Load l = heap.top();
    heap.pop();
    bin_of[i] = l.second;
    heap.push({l.first + cost[i], l.second});
  }
  std::vector<uint32_t> start(nb + 2, 0);
  for (uint32_t i = 0; i < n; ++i) ++start[bin_of[i] + 1];
  for (uint32_t b = 0; b <= nb; ++b) start[b + 1] += start[b];
  std::vector<Tile> out(n);
  std::vector<uint32_t> fill(start.begin(), start.end() - 1);
  for (uint32_t i = 0; i < n; ++i) out[fill[bin_of[i]]++] = table[g.begin + i];
  for (uint32_t k = head; k < n; ++k) out[start[nb] + (k - head)] = table[g.begin + order[k]];
  std::copy(out.begin(), out.end(), table.begin() + g.begin);
  g.nbins = nb;
  g.tail = n - start[nb];
  g.bin_first = uint32_t(bin_sizes.size());
  for (uint32_t b = 0; b < nb; ++b) bin_sizes.push_back(start[b + 1] - start[b]);
}

// Device image of a tile table: every group's range in order; a scheduled
// group's bins are padded with OP_END entries to a common stride, so CTA b
// finds its bin at b * stride without a lookup (one global round trip to
// fetch its descriptors), followed by the tail.
std::vector<Tile> device_image(const std::vector<Tile>& table, std::vector<Group*> groups,
                               const std::vector<uint32_t>& bin_sizes) {
  std::vector<Tile> dev;
  Tile pad{};
  pad.op = OP_END;
  for (Group* g : groups) {
    g->dev_begin = uint32_t(dev.size());
    if (!g->nbins) {
      dev.insert(dev.end(), table.begin() + g->begin, table.begin() + g->end);
      g->dev_count = g->end - g->begin;
      continue;
    }
    uint32_t stride = 1;
    for (uint32_t b = 0; b < g->nbins; ++b) stride = std::max(stride, bin_sizes[g->bin_first + b] + 1);
    g->stride = stride;
    uint32_t at = g->begin;
    for (uint32_t b = 0; b < g->nbins; ++b) {
      const uint32_t sz = bin_sizes[g->bin_first + b];
      dev.insert(dev.end(), table.begin() + at, table.begin() + at + sz);
      dev.insert(dev.end(), stride - sz, pad);
      at += sz;
    }
    dev.insert(dev.end(), table.begin() + at, table.begin() + g->end);  // tail
    g->dev_count = uint32_t(dev.size()) - g->dev_begin;
  }
  return dev;
}

}  // namespace

TilePlan build_tiles(const fmt::Manifest& src, const fmt::Manifest& dst, bool identity, uint64_t chunk_bytes,
                     int sm_count) {
  // kernel key: hash | (TMA ring or direct) x dtype pair. TRIMS_CVT_PATH /
  // TRIMS_PERM_PATH = "direct" | "tma" select the kernel per op (A/B switch).
  static const bool cvt_direct = [] {  // default: elementwise tiles ride the TMA ring too (one launch)
    const char* e = std::getenv("TRIMS_CVT_PATH");
    return e && std::string(e) == "direct";
  }();
  static const bool perm_direct = [] {
    const char* e = std::getenv("TRIMS_PERM_PATH");
    return e && std::string(e) == "direct";
  }();
  // Elementwise tiles on the direct path: enough tiles for ~4 waves of the
  // direct grid (148 SMs x 4 CTAs) so the last wave is not half empty, but
  // 16..64 KiB of source each so the per-tile reduction stays noise (A/B in
  // profiles/r01_transform_ab.log). TRIMS_CVT_TILE_KB (source KiB) overrides.
  static const uint64_t cvt_tile_env = [] {
    const char* e = std::getenv("TRIMS_CVT_TILE_KB");
    return e ? uint64_t(std::max(1, std::atoi(e))) << 10 : 0;
  }();
  uint64_t cvt_src_bytes = 0;
  for (size_t i = 0; i < src.tensors.size() && i < dst.tensors.size(); ++i) {
    const auto& s = src.tensors[i];
    const auto& d = dst.tensors[i];
    const bool perm = d.layout == fmt::Layout::KRSC && s.layout == fmt::Layout::Native && s.dims.size() == 4 &&
                      s.dims[2] * s.dims[3] > 1;
    if (!perm) cvt_src_bytes += s.nbytes;
  }
  uint64_t cvt_tile = cvt_tile_env;
  if (!cvt_tile) {
    cvt_tile = 16u << 10;
    while (cvt_tile < (64u << 10) && cvt_src_bytes / cvt_tile > 148ull * 4 * 4) cvt_tile *= 2;
  }
  TilePlan p;
  p.identity = identity;
  p.src_bytes = src.blob_bytes;
  p.dst_bytes = dst.blob_bytes;
  const size_t nt = dst.tensors.size();
  p.buckets = uint32_t(nt + 1);
  if (src.tensors.size() != nt) raise(Errc::InvalidArgument, "plan tensor count mismatch");
  auto extent_end = [&](size_t i) { return i + 1 < nt ? dst.tensors[i + 1].offset : dst.blob_bytes; };
  std::vector<Tile> tiles;

  if (identity) {
    auto hash_range = [&](uint64_t b, uint64_t e, uint32_t bucket) {
      for (uint64_t off = b; off < e; off += kHashTile) {
        Tile t{};
        t.src_off = t.dst_off = off;
        t.dst_bytes = uint32_t(std::min<uint64_t>(kHashTile, e - off));
        t.tensor = bucket;
        t.op = OP_HASH;
        tiles.push_back(t);
      }
    };
    if (nt && dst.tensors[0].offset > 0) hash_range(0, dst.tensors[0].offset, uint32_t(nt));
    for (size_t i = 0; i < nt; ++i) hash_range(dst.tensors[i].offset, extent_end(i), uint32_t(i));
    p.algo_read_bytes = dst.blob_bytes;
  } else {
    for (size_t i = 0; i < nt; ++i) {
      const auto& s = src.tensors[i];
      const auto& d = dst.tensors[i];
      if (!supported_pair(s.dtype, d.dtype))
        raise(Errc::InvalidArgument, std::string("no ingest conversion ") + fmt::dtype_name(s.dtype) + "->" +
                                         fmt::dtype_name(d.dtype));
      if (!floating(s.dtype) && s.dtype != d.dtype) raise(Errc::InvalidArgument, "integer tensors are copied verbatim");
      const uint64_t ss = fmt::element_size(s.dtype), ds = fmt::element_size(d.dtype);
      const uint64_t n = s.nbytes / ss, end = extent_end(i);
      p.algo_read_bytes += s.nbytes;
      // 1x1 kernels: KCRS and KRSC are the same byte order -> elementwise tile.
      const bool perm = d.layout == fmt::Layout::KRSC && s.layout == fmt::Layout::Native &&
                        s.dims[2] * s.dims[3] > 1;
      if (perm) {
        const uint64_t K = s.dims[0], C = s.dims[1], RS = s.dims[2] * s.dims[3], CRS = C * RS;
        uint64_t g = 1;
        while ((g * CRS * ds) % 8) ++g;
        // a slice group whose raw bytes exceed a ring stage is gathered straight from HBM
        const uint64_t stage = ring_cfg().stage_bytes;
        const bool gather = g * CRS * ss > stage;
        // as many whole aligned slice groups as fill one ring stage
        if (!gather) g = std::max<uint64_t>(g, std::min<uint64_t>(K, stage / (g * CRS * ss) * g));
        p.has_perm = true;
        for (uint64_t k0 = 0; k0 < K; k0 += g) {
          const uint64_t kn = std::min(g, K - k0);
          Tile t{};
          t.op = OP_PERM;
          t.src_off = s.offset + k0 * CRS * ss;
          t.dst_off = d.offset + k0 * CRS * ds;
          t.n_elem = uint32_t(kn * CRS);
          t.dst_bytes = uint32_t(k0 + kn == K ? end - t.dst_off : kn * CRS * ds);
          t.tensor = uint32_t(i);
          t.sdt = uint8_t(s.dtype);
          t.ddt = uint8_t(d.dtype);
          t.C = uint32_t(C);
          t.RS = uint32_t(RS);
          t.rows = uint32_t(kn * RS);
          t.rs_magic = uint32_t(0xffffffffu / RS + 1);
          t.pad_ = gather ? 1 : 0;
          tiles.push_back(t);
        }
      } else {
        const uint64_t per = (cvt_direct ? cvt_tile : ring_cfg().stage_bytes) / ss;
        for (uint64_t e0 = 0; e0 < n; e0 += per) {
          const uint64_t cnt = std::min<uint64_t>(per, n - e0);
          Tile t{};
          t.op = OP_CVT;
          t.src_off = s.offset + e0 * ss;
          t.dst_off = d.offset + e0 * ds;
          t.n_elem = uint32_t(cnt);
          t.dst_bytes = uint32_t(e0 + cnt == n ? end - t.dst_off : cnt * ds);
          t.tensor = uint32_t(i);
          t.sdt = uint8_t(s.dtype);
          t.ddt = uint8_t(d.dtype);
          tiles.push_back(t);
        }
      }
    }
    p.algo_write_bytes = dst.blob_bytes;
  }

  auto src_end = [](const Tile& t) -> uint64_t {
    if (t.op == OP_HASH) return t.src_off + t.dst_bytes;
    return t.src_off + uint64_t(t.n_elem) * fmt::element_size(fmt::DType(t.sdt));
  };
  auto kind_of = [](const Tile& t) -> uint8_t {
    if (t.op == OP_HASH) return 0;
    if (t.pad_) return 2;
    return (t.op == OP_CVT ? cvt_direct : perm_direct) ? 2 : 1;
  };
  auto key_of = [&](const Tile& t) { return uint32_t(kind_of(t)) << 16 | uint32_t(t.sdt) << 8 | t.ddt; };
  auto group_range = [&](std::vector<Tile>& v, uint32_t b, uint32_t e, std::vector<Group>& out) {
    std::stable_sort(v.begin() + b, v.begin() + e, [&](const Tile& x, const Tile& y) { return key_of(x) < key_of(y); });
    for (uint32_t i = b; i < e;) {
      uint32_t j = i + 1;
      while (j < e && key_of(v[j]) == key_of(v[i])) ++j;
      uint8_t smem = 0;
      for (uint32_t k = i; k < j; ++k) smem |= v[k].op == OP_PERM && !v[k].pad_;
      out.push_back({i, j, kind_of(v[i]), v[i].sdt, v[i].ddt, smem});
      i = j;
    }
  };
  // Chunks: consecutive (source-ordered) tiles until their span reaches chunk_bytes.
  uint32_t b = 0;
  while (b < tiles.size()) {
    uint64_t s0 = tiles[b].src_off, s1 = src_end(tiles[b]);
    uint32_t e = b + 1;
    while (e < tiles.size() && s1 - s0 < chunk_bytes) {
      s1 = std::max(s1, src_end(tiles[e]));
      ++e;
    }
    p.chunks.push_back({b, e, s0, s1, {}});
    b = e;
  }
  p.tiles = tiles;
  for (auto& ch : p.chunks) group_range(p.tiles, ch.tile_begin, ch.tile_end, ch.groups);
  p.tiles_by_kernel = tiles;
  group_range(p.tiles_by_kernel, 0, uint32_t(tiles.size()), p.groups);
  // TRIMS_TILE_LPT=1: largest tiles first (A/B: source order measured faster,
  // profiles/r01_transform_ab_sched.log)
  static const bool lpt = std::getenv("TRIMS_TILE_LPT") && std::atoi(std::getenv("TRIMS_TILE_LPT"));
  for (const Group& g : p.groups)
    if (lpt) std::stable_sort(p.tiles_by_kernel.begin() + g.begin, p.tiles_by_kernel.begin() + g.end,
                     [](const Tile& x, const Tile& y) { return x.dst_bytes > y.dst_bytes; });
  // Static schedule of the TMA groups (default; TRIMS_TILE_SCHED=dynamic uses
  // the ticket counter): greedy largest-cost-first bin packing onto one bin
  // per CTA, cost = bytes moved + a fixed per-tile charge.
  static const bool dyn = [] {
    const char* e = std::getenv("TRIMS_TILE_SCHED");
    return e && std::string(e) == "dynamic";
  }();
  const uint32_t grid = uint32_t(std::max(1, sm_count)) * ring_cfg().ctas_per_sm;
  std::vector<uint32_t> sizes, sizes_k;
  std::vector<Group*> gp, gp_k;
  for (auto& ch : p.chunks)
    for (Group& g : ch.groups) {
      if (!dyn && g.kind == 1 && g.end > g.begin) schedule_bins(p.tiles, g, grid, sizes);
      gp.push_back(&g);
    }
  for (Group& g : p.groups) {
    if (!dyn && g.kind == 1 && g.end > g.begin) schedule_bins(p.tiles_by_kernel, g, grid, sizes_k);
    gp_k.push_back(&g);
  }
  p.dev_tiles = device_image(p.tiles, gp, sizes);
  p.dev_tiles_k = device_image(p.tiles_by_kernel, gp_k, sizes_k);
  return p;
}

uint32_t launch_groups(const Tile* d_tiles, const std::vector<Group>& groups, const uint8_t* src, uint8_t* dst,
                       unsigned long long* d_sums, cudaStream_t stream, int sm_count, SideStream* side) {
  // With a side stream, the direct-path groups run concurrently with the TMA
  // ring groups: the ring kernel holds one CTA and ~200 KB of shared memory
  // per SM, the smem-free direct CTAs fill the remaining warps and registers.
  bool has_tma = false, has_direct = false;
  for (const Group& g : groups) {
    has_tma |= g.kind == 1 && g.end > g.begin;
    has_direct |= g.kind == 2 && g.end > g.begin;
  }
  static const bool serial = std::getenv("TRIMS_TRANSFORM_SERIAL") != nullptr;  // A/B switch
  const bool fork = !serial && side && side->stream && has_tma && has_direct;
  if (fork) {
    TRIMS_CUDA(cudaEventRecord(side->fork, stream));
    TRIMS_CUDA(cudaStreamWaitEvent(side->stream, side->fork, 0));
  }
  uint32_t launches = 0;
  for (const Group& g : groups) {
    const uint32_t n = g.dev_count;
    if (!n) continue;
    const Tile* t = d_tiles + g.dev_begin;
    cudaStream_t st = fork && g.kind == 2 ? side->stream : stream;
    if (g.kind == 0) {
      hash_tiles_kernel<<<std::min<uint32_t>(n, sm_count * 8), kThreads, 0, st>>>(t, n, dst, d_sums);
    } else if (g.kind == 1) {
      TmaFn fn = pair_tma_kernel(g.sdt, g.ddt);
      if (!fn) raise(Errc::InvalidArgument, "unsupported dtype pair in plan");
      const RingCfg& rc = ring_cfg();
      const int smem = int(rc.stages * rc.stage_alloc());
      TRIMS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      if (!side || !side->sched) raise(Errc::Internal, "TMA transform launch without a scheduler slot");
      static const bool dynamic = [] {  // A/B switch: TRIMS_TILE_SCHED=static
        const char* e = std::getenv("TRIMS_TILE_SCHED");
        return !(e && std::string(e) == "static");
      }();
      // Ticket counters are never reset: a launch draws exactly (dynamic
      // tiles + CTAs) tickets (every CTA ends on one failing draw), so the
      // host advances the slot's base by that and passes it in -- only once
      // the launch is accepted (commit_slot): a launch that never ran drew
      // nothing, and the slot's base must stay equal to its device counter.
      int pending_k = -1;
      uint32_t pending_adv = 0;
      auto take_slot = [&](uint32_t dyn_tiles, uint32_t ctas, unsigned int** slot, uint32_t* base) {
        const uint32_t k = side->sched_next % kSchedSlots;
        *slot = side->sched + 2 * k;
        *base = side->sched_base[k];
        pending_k = int(k);
        pending_adv = dyn_tiles + ctas;
      };
      auto commit_slot = [&] {
        if (pending_k < 0) return;
        side->sched_base[pending_k] += pending_adv;
        ++side->sched_next;
        pending_k = -1;
      };
      unsigned int* slot = nullptr;
      uint32_t base = 0;
      static const bool pdl = [] {  // A/B switch: TRIMS_TRANSFORM_PDL=0
        const char* e = std::getenv("TRIMS_TRANSFORM_PDL");
        return !(e && std::string(e) == "0");
      }();
      // Early ring fill (see transform_tma_kernel): transform sources are only
      // ever written by DMA copies or non-PDL kernels. A/B: TRIMS_TRANSFORM_EARLY=0.
      static const uint32_t early = [] {
        const char* e = std::getenv("TRIMS_TRANSFORM_EARLY");
        return (e && std::string(e) == "0") ? 0u : 1u;
      }();
      auto go = [&](uint32_t ctas, const unsigned int* sl, uint32_t b, uint32_t stride, uint32_t tail0) {
        if (pdl)
          launch_pdl(fn, dim3(ctas), dim3(kTmaThreads), size_t(smem), st, t, n, src, dst, d_sums, rc.stages,
                     rc.stage_alloc(), const_cast<unsigned int*>(sl), b, stride, tail0, early);
        else
          fn<<<ctas, kTmaThreads, smem, st>>>(t, n, src, dst, d_sums, rc.stages, rc.stage_alloc(),
                                              const_cast<unsigned int*>(sl), b, stride, tail0, 0u);
      };
      if (g.nbins) {  // static schedule: one CTA per bin (+ dynamic tail)
        if (g.tail) take_slot(g.tail, g.nbins, &slot, &base);
        go(g.nbins, slot, base, g.stride, g.nbins * g.stride);
      } else {
        const uint32_t ctas = std::min<uint32_t>(n, sm_count * rc.ctas_per_sm);
        if (dynamic) take_slot(n, ctas, &slot, &base);
        go(ctas, slot, base, 0u, 0u);
      }
      TRIMS_CUDA(cudaGetLastError());
      commit_slot();
    } else {
      TransformFn fn = pair_kernel(g.sdt, g.ddt);
      if (!fn) raise(Errc::InvalidArgument, "unsupported dtype pair in plan");
      const uint32_t smem = g.smem ? uint32_t(kPermSmem) : 0;
      TRIMS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPermSmem)));
      int per_sm = 0;  // persistent grid = exactly the resident CTAs
      TRIMS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem));
      fn<<<std::min<uint32_t>(n, sm_count * std::max(1, per_sm)), kThreads, smem, st>>>(t, n, src, dst, d_sums);
    }
    TRIMS_CUDA(cudaGetLastError());
    ++launches;
  }
  if (fork) {
    TRIMS_CUDA(cudaEventRecord(side->join, side->stream));
    TRIMS_CUDA(cudaStreamWaitEvent(stream, side->join, 0));
  }
  return launches;
}

uint32_t launch_pull(const Tile* d_tiles, const std::vector<Group>& groups, const uint8_t* src, uint8_t* dst,
                     unsigned long long* d_sums, cudaStream_t stream, int sm_count) {
  uint32_t launches = 0;
  for (const Group& g : groups) {
    const uint32_t n = g.end - g.begin;
    if (!n) continue;
    if (g.kind != 0) raise(Errc::InvalidArgument, "peer pull needs an identity (hash-only) plan");
    pull_tiles_kernel<<<std::min<uint32_t>(n, sm_count * 8), kThreads, 0, stream>>>(d_tiles + g.dev_begin, n, src,
                                                                                    dst, d_sums);
    TRIMS_CUDA(cudaGetLastError());
    ++launches;
  }
  return launches;
}

void launch_checksum(const uint8_t* p, uint64_t nbytes, uint64_t word0, unsigned long long* d_out,
                     cudaStream_t stream, int sm_count) {
  if (!nbytes) return;
  uint64_t words = (nbytes + 7) / 8;
  uint32_t grid = uint32_t(std::min<uint64_t>((words / 2 + kThreads - 1) / kThreads + 1, uint64_t(sm_count) * 8));
  checksum_kernel<<<grid, kThreads, 0, stream>>>(p, nbytes, word0, d_out);
  TRIMS_CUDA(cudaGetLastError());
}

void launch_fill_splitmix(uint64_t* dst, uint64_t n, uint64_t stream_seed, uint64_t k0, cudaStream_t s) {
  if (!n) return;
  uint32_t grid = uint32_t(std::min<uint64_t>((n + 255) / 256, 148ull * 16));
  fill_splitmix_kernel<<<grid, 256, 0, s>>>(dst, n, stream_seed, k0);
  TRIMS_CUDA(cudaGetLastError());
}

void launch_fill_uniform(float* dst, uint64_t n, uint64_t stream_seed, uint64_t j0, float lo, float hi,
                         cudaStream_t s) {
  if (!n) return;
  uint32_t grid = uint32_t(std::min<uint64_t>((n + 255) / 256, 148ull * 16));
  fill_uniform_kernel<<<grid, 256, 0, s>>>(dst, n, stream_seed, j0, lo, hi);
  TRIMS_CUDA(cudaGetLastError());
}

}  // namespace trims::ingest

#ifdef TRIMS_TRACE
// Copies out up to n words (kTraceW = 10 per CTA record) and resets the
// record counter; returns the number of records since the last reset, or -1.
extern "C" int trims_debug_transform_trace(unsigned long long* out, int n) {
  unsigned int recs = 0, zero = 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  cudaMemcpyFromSymbol(&recs, trims::ingest::g_tslot_n, sizeof(recs));
  const size_t words = std::min<size_t>(size_t(n), size_t(recs) * trims::ingest::kTraceW);
  if (words && cudaMemcpyFromSymbol(out, trims::ingest::g_ttrace, sizeof(unsigned long long) * words) != cudaSuccess)
    return -1;
  cudaMemcpyToSymbol(trims::ingest::g_tslot_n, &zero, sizeof(zero));
  return int(recs);
}

__global__ void trims_debug_empty_kernel() {}

// An empty launch with the transform's shared-memory footprint on every SM:
// separates the SM carve-out reconfiguration from the transform itself.
extern "C" int trims_debug_carveout(int smem, int ctas, void* stream) {
  cudaFuncSetAttribute(trims_debug_empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  trims_debug_empty_kernel<<<ctas, 544, smem, static_cast<cudaStream_t>(stream)>>>();
  return int(cudaGetLastError());
}
#endif
