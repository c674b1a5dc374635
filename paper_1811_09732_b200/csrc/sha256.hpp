// sha256.hpp — host SHA-256 for the artifact trailer and the manifest digest
// (the reference's proj/src/sha256.cpp role). Uses the x86 SHA-NI extension
// when the CPU has it (~1.2+ GB/s/core vs 0.145 GB/s for the reference's
// scalar loop), scalar FIPS 180-4 otherwise; both produce identical digests.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <string>

namespace trims {

class Sha256 {
 public:
  Sha256() { reset(); }
  void reset();
  void update(const void* data, size_t len);
  std::array<uint8_t, 32> finish();
  static std::array<uint8_t, 32> of(const void* data, size_t len) {
    Sha256 h;
    h.update(data, len);
    return h.finish();
  }
  static bool hw_accelerated();

 private:
  void blocks(const uint8_t* p, size_t nblocks);
  uint32_t st_[8];
  uint64_t total_{0};
  uint8_t buf_[64];
  size_t buf_len_{0};
};

std::string hex(const uint8_t* p, size_t n);

}  // namespace trims
