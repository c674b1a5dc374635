// ingest.hpp — the weight-ingest transform: staged raw artifact blob ->
// resident blob (dtype convert, KCRS->KRSC permute, zero padding) with the
// TRIMS block checksum of every resident word fused in (K2+K3+K4 of
// SURVEY.md §2). Work is cut into tiles on the host; one persistent kernel
// launch processes a tile range.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "format.hpp"

namespace trims::ingest {

enum Op : uint8_t { OP_HASH = 0, OP_CVT = 1, OP_PERM = 2 };

// 40 bytes. dst_off/dst_bytes are multiples of 8 so every tile owns whole
// checksum words; the last tile of a tensor extends over its trailing pad.
struct Tile {
  uint64_t src_off;    // byte offset in the staged raw blob
  uint64_t dst_off;    // byte offset in the resident blob
  uint32_t dst_bytes;  // resident bytes written (and hashed) by this tile
  uint32_t n_elem;     // source elements consumed (OP_CVT / OP_PERM)
  uint32_t tensor;     // checksum bucket (resident tensor index; ntensors = leading pad)
  uint8_t op, sdt, ddt, pad_;
  uint32_t C, RS;      // OP_PERM geometry: n_elem / (C*RS) k-slices
};
static_assert(sizeof(Tile) == 40, "tile layout");

struct TilePlan {
  std::vector<Tile> tiles;
  // Pipeline chunks: [tile_begin, tile_end) with the source byte span the
  // chunk's tiles read, so the H2D of chunk c can overlap tiles of chunk c-1.
  struct Chunk {
    uint32_t tile_begin, tile_end;
    uint64_t src_begin, src_end;
    uint64_t pairs;  // dtype pairs present (bit s*8+d), kHashPairBit for OP_HASH
  };
  std::vector<Chunk> chunks;
  uint64_t pairs{0};
  uint32_t buckets{0};     // checksum buckets (ntensors + 1)
  bool identity{false};    // resident == source bytes: tiles only hash
  bool has_perm{false};
  uint64_t src_bytes{0}, dst_bytes{0};
  uint64_t algo_read_bytes{0}, algo_write_bytes{0};  // roofline accounting
};

// src: the artifact manifest; dst: resident_manifest(src, plan).
TilePlan build_tiles(const fmt::Manifest& src, const fmt::Manifest& dst, bool identity,
                     uint64_t chunk_bytes = 16ull << 20);

inline constexpr uint64_t kHashPairBit = 1ull << 63;

// Persistent tile kernels over tiles [0, ntiles) of `d_tiles` (device copy):
// one launch per dtype pair in `pairs` (+ one hash launch). Per-bucket
// checksums are atomically accumulated into d_sums (mod 2^64). Returns the
// number of kernel launches issued.
uint32_t launch_transform(const Tile* d_tiles, uint32_t ntiles, uint64_t pairs, bool has_perm, const uint8_t* src,
                          uint8_t* dst, unsigned long long* d_sums, cudaStream_t stream, int sm_count);

// Checksum of an arbitrary device range (word0 = global index of its first word).
void launch_checksum(const uint8_t* p, uint64_t nbytes, uint64_t word0, unsigned long long* d_out,
                     cudaStream_t stream, int sm_count);

// K5 synthetic weights on the device: catalog words (splitmix at k0+j) and
// uniform fp32 values (fmaf(hi-lo, u24*2^-24, lo)); both bit-identical to the
// host generators and the oracle.
void launch_fill_splitmix(uint64_t* dst, uint64_t n, uint64_t stream_seed, uint64_t k0, cudaStream_t s);
void launch_fill_uniform(float* dst, uint64_t n, uint64_t stream_seed, uint64_t j0, float lo, float hi,
                         cudaStream_t s);

}  // namespace trims::ingest
