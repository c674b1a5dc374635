// sha256.cpp — SHA-256 (FIPS 180-4) with an x86 SHA-NI fast path.
#include "sha256.hpp"

#include <cpuid.h>
#include <immintrin.h>

#include <algorithm>
#include <cstring>

namespace trims {

namespace {

alignas(64) const uint32_t K[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void blocks_scalar(uint32_t st[8], const uint8_t* p, size_t n) {
  for (; n; --n, p += 64) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = uint32_t(p[4 * i]) << 24 | uint32_t(p[4 * i + 1]) << 16 | uint32_t(p[4 * i + 2]) << 8 |
             uint32_t(p[4 * i + 3]);
    for (int i = 16; i < 64; ++i)
      w[i] = w[i - 16] + (rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3)) + w[i - 7] +
             (rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10));
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
    for (int i = 0; i < 64; ++i) {
      uint32_t t1 = h + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K[i] + w[i];
      uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    st[0] += a; st[1] += b; st[2] += c; st[3] += d; st[4] += e; st[5] += f; st[6] += g; st[7] += h;
  }
}

// SHA-NI: sha256rnds2 does two rounds; per 4-round quad q the message
// schedule for quad q+1 is finished with msg2 and quad q-1 seeded with msg1.
__attribute__((target("sha,sse4.1"))) void blocks_shani(uint32_t st[8], const uint8_t* p, size_t n) {
  const __m128i MASK = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
  __m128i tmp = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&st[0]));
  __m128i s1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&st[4]));
  tmp = _mm_shuffle_epi32(tmp, 0xB1);              // CDAB
  s1 = _mm_shuffle_epi32(s1, 0x1B);                // EFGH
  __m128i s0 = _mm_alignr_epi8(tmp, s1, 8);        // ABEF
  s1 = _mm_blend_epi16(s1, tmp, 0xF0);             // CDGH
  for (; n; --n, p += 64) {
    __m128i abef = s0, cdgh = s1;
    __m128i m[4];
    for (int i = 0; i < 4; ++i)
      m[i] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16 * i)), MASK);
    for (int q = 0; q < 16; ++q) {
      __m128i msg = _mm_add_epi32(m[q & 3], _mm_load_si128(reinterpret_cast<const __m128i*>(&K[4 * q])));
      s1 = _mm_sha256rnds2_epu32(s1, s0, msg);
      if (q >= 3 && q <= 14) {
        __m128i t = _mm_alignr_epi8(m[q & 3], m[(q - 1) & 3], 4);
        m[(q + 1) & 3] = _mm_sha256msg2_epu32(_mm_add_epi32(m[(q + 1) & 3], t), m[q & 3]);
      }
      msg = _mm_shuffle_epi32(msg, 0x0E);
      s0 = _mm_sha256rnds2_epu32(s0, s1, msg);
      if (q >= 1 && q <= 12) m[(q - 1) & 3] = _mm_sha256msg1_epu32(m[(q - 1) & 3], m[q & 3]);
    }
    s0 = _mm_add_epi32(s0, abef);
    s1 = _mm_add_epi32(s1, cdgh);
  }
  tmp = _mm_shuffle_epi32(s0, 0x1B);   // FEBA
  s1 = _mm_shuffle_epi32(s1, 0xB1);    // DCHG
  s0 = _mm_blend_epi16(tmp, s1, 0xF0); // DCBA
  s1 = _mm_alignr_epi8(s1, tmp, 8);    // ABEF -> HGFE
  _mm_storeu_si128(reinterpret_cast<__m128i*>(&st[0]), s0);
  _mm_storeu_si128(reinterpret_cast<__m128i*>(&st[4]), s1);
}

bool detect_shani() {
  unsigned a, b, c, d;
  if (!__get_cpuid_count(7, 0, &a, &b, &c, &d)) return false;
  bool sha = (b >> 29) & 1;
  if (!__get_cpuid(1, &a, &b, &c, &d)) return false;
  bool sse41 = (c >> 19) & 1, ssse3 = (c >> 9) & 1;
  return sha && sse41 && ssse3;
}

const bool g_shani = detect_shani();

}  // namespace

bool Sha256::hw_accelerated() { return g_shani; }

void Sha256::reset() {
  static const uint32_t iv[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  std::memcpy(st_, iv, sizeof iv);
  total_ = 0;
  buf_len_ = 0;
}

void Sha256::blocks(const uint8_t* p, size_t n) {
  if (g_shani) blocks_shani(st_, p, n);
  else blocks_scalar(st_, p, n);
}

void Sha256::update(const void* data, size_t len) {
  const uint8_t* p = static_cast<const uint8_t*>(data);
  total_ += len;
  if (buf_len_) {
    size_t take = std::min(len, 64 - buf_len_);
    std::memcpy(buf_ + buf_len_, p, take);
    buf_len_ += take;
    p += take;
    len -= take;
    if (buf_len_ == 64) {
      blocks(buf_, 1);
      buf_len_ = 0;
    }
  }
  if (len >= 64) {
    blocks(p, len / 64);
    p += len / 64 * 64;
    len %= 64;
  }
  if (len) {
    std::memcpy(buf_, p, len);
    buf_len_ = len;
  }
}

std::array<uint8_t, 32> Sha256::finish() {
  uint64_t bits = total_ * 8;
  uint8_t pad[128] = {0x80};
  size_t padlen = (buf_len_ < 56) ? (56 - buf_len_) : (120 - buf_len_);
  uint8_t lenb[8];
  for (int i = 0; i < 8; ++i) lenb[i] = uint8_t(bits >> (56 - 8 * i));
  update(pad, padlen);
  update(lenb, 8);
  std::array<uint8_t, 32> out;
  for (int i = 0; i < 8; ++i) {
    out[4 * i] = uint8_t(st_[i] >> 24);
    out[4 * i + 1] = uint8_t(st_[i] >> 16);
    out[4 * i + 2] = uint8_t(st_[i] >> 8);
    out[4 * i + 3] = uint8_t(st_[i]);
  }
  reset();
  return out;
}

std::string hex(const uint8_t* p, size_t n) {
  static const char* h = "0123456789abcdef";
  std::string s;
  for (size_t i = 0; i < n; ++i) {
    s.push_back(h[p[i] >> 4]);
    s.push_back(h[p[i] & 15]);
  }
  return s;
}

}  // namespace trims
