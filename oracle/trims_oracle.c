/* trims_oracle.c — CPU restatement (TEST INFRASTRUCTURE ONLY; see the header).
 * Every function cites the reference file:line it follows, or says that it is
 * our own definition of a transform the reference does not have. */
#include "trims_oracle.h"

#include <math.h>
#include <string.h>

/* ---------------- SHA-256 (proj/src/sha256.cpp:24-123) ---------------- */

static const uint32_t K256[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u,
    0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu,
    0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu,
    0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau, 0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u,
    0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu,
    0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
    0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u, 0x19a4c116u,
    0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u,
    0xc67178f2u};

static uint32_t ror32(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

static void sha_block(uint32_t st[8], const uint8_t* b) {
  uint32_t w[64];
  for (int i = 0; i < 16; ++i)
    w[i] = ((uint32_t)b[4 * i] << 24) | ((uint32_t)b[4 * i + 1] << 16) |
           ((uint32_t)b[4 * i + 2] << 8) | (uint32_t)b[4 * i + 3];
  for (int i = 16; i < 64; ++i) {
    uint32_t x = w[i - 15], y = w[i - 2];
    w[i] = w[i - 16] + (ror32(x, 7) ^ ror32(x, 18) ^ (x >> 3)) + w[i - 7] +
           (ror32(y, 17) ^ ror32(y, 19) ^ (y >> 10));
  }
  uint32_t a = st[0], bb = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
  for (int i = 0; i < 64; ++i) {
    uint32_t t1 = h + (ror32(e, 6) ^ ror32(e, 11) ^ ror32(e, 25)) + ((e & f) ^ (~e & g)) + K256[i] + w[i];
    uint32_t t2 = (ror32(a, 2) ^ ror32(a, 13) ^ ror32(a, 22)) + ((a & bb) ^ (a & c) ^ (bb & c));
    h = g; g = f; f = e; e = d + t1; d = c; c = bb; bb = a; a = t1 + t2;
  }
  st[0] += a; st[1] += bb; st[2] += c; st[3] += d; st[4] += e; st[5] += f; st[6] += g; st[7] += h;
}

void tro_sha256(const void* data, uint64_t n, uint8_t out[32]) {
  uint32_t st[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                    0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  const uint8_t* p = (const uint8_t*)data;
  uint64_t full = n / 64;
  for (uint64_t i = 0; i < full; ++i) sha_block(st, p + 64 * i);
  uint8_t tail[128];
  uint64_t rem = n - full * 64;
  memset(tail, 0, sizeof tail);
  if (rem) memcpy(tail, p + full * 64, rem);
  tail[rem] = 0x80;
  uint64_t tl = (rem + 1 + 8 <= 64) ? 64 : 128;
  uint64_t bits = n * 8;
  for (int i = 0; i < 8; ++i) tail[tl - 1 - i] = (uint8_t)(bits >> (8 * i));
  sha_block(st, tail);
  if (tl == 128) sha_block(st, tail + 64);
  for (int i = 0; i < 8; ++i) {
    out[4 * i] = (uint8_t)(st[i] >> 24);
    out[4 * i + 1] = (uint8_t)(st[i] >> 16);
    out[4 * i + 2] = (uint8_t)(st[i] >> 8);
    out[4 * i + 3] = (uint8_t)st[i];
  }
}

/* ------------- catalog RNG (catalog.hpp:59-71, catalog.cpp:79-86,142) ------------- */

#define GOLDEN 0x9e3779b97f4a7c15ull

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t tro_fnv1a_str(const char* s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= (uint8_t)*s;
    h *= 0x100000001b3ull;
  }
  return h;
}

uint64_t tro_splitmix_at(uint64_t stream_seed, uint64_t k) {
  return mix64(stream_seed + (k + 1) * GOLDEN);
}

void tro_splitmix_fill(uint64_t stream_seed, uint64_t k0, uint64_t n, uint64_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = tro_splitmix_at(stream_seed, k0 + i);
}

uint64_t tro_catalog_stream(uint64_t seed, const char* model_name) {
  return seed ^ tro_fnv1a_str(model_name);
}

/* ---------------- Client::touch (client.cpp:338-359) ---------------- */

uint64_t tro_touch(const uint8_t* blob, const uint64_t* offsets, const uint64_t* nbytes,
                   uint64_t ntensors) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t t = 0; t < ntensors; ++t) {
    const uint8_t* p = blob + offsets[t];
    uint64_t n = nbytes[t], words = n / 8;
    for (uint64_t i = 0; i < words; ++i) {
      uint64_t w;
      memcpy(&w, p + 8 * i, 8);
      h ^= w;
      h *= 0x100000001b3ull;
    }
    for (uint64_t i = words * 8; i < n; ++i) {
      h ^= p[i];
      h *= 0x100000001b3ull;
    }
  }
  return h;
}

double tro_share_benefit(double bytes, double n_objects, double q, double o, double s) {
  return bytes / q - n_objects * (o + s);
}

/* ---------------- conversions (our definition; parity unpinned) ---------------- */

uint16_t tro_f32_to_bf16_1(uint32_t u) {
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)0x7fffu; /* canonical NaN */
  uint32_t lsb = (u >> 16) & 1u;
  return (uint16_t)((u + 0x7fffu + lsb) >> 16);
}

void tro_f32_to_bf16(const uint32_t* src, uint64_t n, uint16_t* dst) {
  for (uint64_t i = 0; i < n; ++i) dst[i] = tro_f32_to_bf16_1(src[i]);
}

void tro_f64_to_f32(const double* src, uint64_t n, float* dst) {
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t u;
    memcpy(&u, &src[i], 8);
    if ((u & 0x7fffffffffffffffull) > 0x7ff0000000000000ull) { /* NaN: canonical quiet, sign kept */
      uint32_t q = (uint32_t)((u >> 32) & 0x80000000u) | 0x7fc00000u;
      memcpy(&dst[i], &q, 4);
    } else {
      dst[i] = (float)src[i];
    }
  }
}

static uint16_t f64_to_bf16_1(uint64_t u) {
  uint16_t sign = (uint16_t)((u >> 48) & 0x8000u);
  uint64_t e = (u >> 52) & 0x7ff, m = u & ((1ull << 52) - 1);
  if (e == 0x7ff) return m ? (uint16_t)0x7fffu : (uint16_t)(sign | 0x7f80u);
  if (e == 0) return sign; /* f64 subnormals are far below bf16's range */
  int64_t eb = (int64_t)e - 1023 + 127;
  if (eb >= 255) return (uint16_t)(sign | 0x7f80u);
  uint64_t sig = (1ull << 52) | m;
  if (eb >= 1) {
    uint64_t q = ((uint64_t)eb << 7) | ((sig >> 45) & 0x7f);
    uint64_t r = sig & ((1ull << 45) - 1), half = 1ull << 44;
    if (r > half || (r == half && (q & 1))) q += 1; /* may carry into Inf: RNE overflow */
    return (uint16_t)(sign | q);
  }
  uint64_t shift = 45 + (uint64_t)(1 - eb);
  if (shift > 54) return sign;
  uint64_t q = sig >> shift, r = sig & ((1ull << shift) - 1), half = 1ull << (shift - 1);
  if (r > half || (r == half && (q & 1))) q += 1;
  return (uint16_t)(sign | q);
}

void tro_f64_to_bf16(const double* src, uint64_t n, uint16_t* dst) {
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t u;
    memcpy(&u, &src[i], 8);
    dst[i] = f64_to_bf16_1(u);
  }
}

void tro_f16_to_f32(const uint16_t* src, uint64_t n, float* dst) {
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t h = src[i], sign = (h & 0x8000u) << 16, e = (h >> 10) & 0x1f, m = h & 0x3ff, out;
    if (e == 0x1f) {
      out = sign | 0x7f800000u | (m << 13);
    } else if (e == 0) {
      if (m == 0) {
        out = sign;
      } else { /* normalise the subnormal */
        int ex = -1;
        do { m <<= 1; ++ex; } while (!(m & 0x400));
        out = sign | ((uint32_t)(127 - 15 - ex) << 23) | ((m & 0x3ff) << 13);
      }
    } else {
      out = sign | ((e + 112) << 23) | (m << 13);
    }
    memcpy(&dst[i], &out, 4);
  }
}

void tro_permute_kcrs_krsc(const void* src, uint64_t K, uint64_t C, uint64_t R, uint64_t S,
                           uint64_t esize, void* dst) {
  const uint8_t* s = (const uint8_t*)src;
  uint8_t* d = (uint8_t*)dst;
  for (uint64_t k = 0; k < K; ++k)
    for (uint64_t c = 0; c < C; ++c)
      for (uint64_t r = 0; r < R; ++r)
        for (uint64_t q = 0; q < S; ++q) {
          uint64_t si = ((k * C + c) * R + r) * S + q;
          uint64_t di = ((k * R + r) * S + q) * C + c;
          memcpy(d + di * esize, s + si * esize, esize);
        }
}

/* per-position odd key of the block checksum (trims_oracle.h) */
static uint64_t tro_checksum_key(uint64_t g) {
  uint32_t t = (uint32_t)g * 0x9e3779b1u;
  uint32_t klo = (t ^ (t >> 16)) | 1u, khi = t * 0xc2b2ae3du;
  return ((uint64_t)khi << 32) | klo;
}

uint64_t tro_block_checksum(const uint8_t* p, uint64_t nbytes, uint64_t word0) {
  uint64_t sum = 0, words = (nbytes + 7) / 8;
  for (uint64_t i = 0; i < words; ++i) {
    uint64_t w = 0;
    uint64_t take = (nbytes - 8 * i) < 8 ? (nbytes - 8 * i) : 8;
    memcpy(&w, p + 8 * i, take);
    sum += w * tro_checksum_key(word0 + i);
  }
  return sum;
}

void tro_uniform_fill_f32(uint64_t stream, uint64_t j0, uint64_t n, float lo, float hi,
                          float* dst) {
  float span = hi - lo;
  for (uint64_t j = 0; j < n; ++j) {
    float u = (float)(tro_splitmix_at(stream, j0 + j) >> 40) * 0x1p-24f;
    dst[j] = fmaf(span, u, lo);
  }
}
