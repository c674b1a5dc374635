// ingest.hpp — the weight-ingest transform: staged raw artifact blob ->
// resident blob (dtype convert, KCRS->KRSC permute, zero padding) with the
// TRIMS block checksum of every resident word fused in (K2+K3+K4 of
// SURVEY.md §2). Work is cut into tiles on the host; persistent kernels
// stream tile ranges through a TMA-fed shared-memory ring.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "format.hpp"

namespace trims::ingest {

// TRIMS block checksum term of resident word w at global word index g
// (oracle/trims_oracle.h: tro_block_checksum): w * K(g) mod 2^64 with an odd
// per-position key, so every single-word change moves the sum. Four 32-bit
// IMADs + three key ops per word on the GPU; the region checksum is the sum of
// its words' terms (additive over disjoint ranges).
__host__ __device__ __forceinline__ uint64_t checksum_term(uint64_t w, uint64_t g) {
  const uint32_t t = uint32_t(g) * 0x9e3779b1u;
  const uint32_t klo = (t ^ (t >> 16)) | 1u, khi = t * 0xc2b2ae3du;
  const uint32_t lo = uint32_t(w), hi = uint32_t(w >> 32);
  return uint64_t(lo) * klo + (uint64_t(lo * khi + hi * klo) << 32);
}

enum Op : uint8_t { OP_HASH = 0, OP_CVT = 1, OP_PERM = 2, OP_END = 0xff };

// 48 bytes. dst_off/dst_bytes are multiples of 8 so every tile owns whole
// checksum words; the last tile of a tensor extends over its trailing pad.
struct Tile {
  uint64_t src_off;    // byte offset in the staged raw blob
  uint64_t dst_off;    // byte offset in the resident blob
  uint32_t dst_bytes;  // resident bytes written (and hashed) by this tile
  uint32_t n_elem;     // source elements consumed (OP_CVT / OP_PERM)
  uint32_t tensor;     // checksum bucket (resident tensor index; ntensors = leading pad)
  uint8_t op, sdt, ddt, pad_;  // pad_ = 1: slice too large for the TMA ring (direct-gather kernel)
  uint32_t C, RS;      // OP_PERM geometry: n_elem / (C*RS) k-slices
  uint32_t rows;       // OP_PERM: resident rows (k, rs) in the tile = n_elem / C
  uint32_t rs_magic;   // OP_PERM: ceil(2^32 / RS), so row / RS = umulhi(row, rs_magic)
};
static_assert(sizeof(Tile) == 48, "tile layout");

// A contiguous tile range handled by one kernel: kind 0 hash, 1 TMA ring, 2 gather.
struct Group {
  uint32_t begin, end;
  uint8_t kind, sdt, ddt;
  uint8_t smem;  // a direct-path group holding smem-staged OP_PERM tiles
  // TMA groups: static schedule. The group's tiles are stored bin-major (one
  // bin per CTA, balanced on the host; nbins = 0: none), then the `tail`
  // smallest tiles, handed out dynamically by a ticket counter once a CTA's
  // bin is done. bin_first indexes the plan's bin sizes.
  uint32_t nbins{0}, tail{0}, bin_first{0};
  // Where the group lives in the device image of its table (bins padded to
  // `stride` entries each, see device_image in ingest.cu).
  uint32_t dev_begin{0}, dev_count{0}, stride{0};
};

struct TilePlan {
  // Chunk-major tile table (tiles grouped by kernel within each chunk).
  std::vector<Tile> tiles;
  // Pipeline chunks: the source byte span their tiles read, so the H2D of
  // chunk c+1 overlaps the kernels of chunk c.
  struct Chunk {
    uint32_t tile_begin, tile_end;
    uint64_t src_begin, src_end;
    std::vector<Group> groups;  // ranges inside `tiles`
  };
  std::vector<Chunk> chunks;
  // Whole-plan table sorted by kernel (one launch per group) for the
  // HBM-resident transform.
  std::vector<Tile> tiles_by_kernel;
  std::vector<Group> groups;
  // Device images of the two tables (what d_tiles / d_tiles_k hold).
  std::vector<Tile> dev_tiles, dev_tiles_k;
  uint32_t buckets{0};     // checksum buckets (ntensors + 1)
  bool identity{false};    // resident == source bytes: tiles only hash
  bool has_perm{false};
  uint64_t src_bytes{0}, dst_bytes{0};
  uint64_t algo_read_bytes{0}, algo_write_bytes{0};  // roofline accounting
};

// src: the artifact manifest; dst: resident_manifest(src, plan).
// sm_count sizes the static schedule of the TMA groups (one bin per CTA).
TilePlan build_tiles(const fmt::Manifest& src, const fmt::Manifest& dst, bool identity,
                     uint64_t chunk_bytes = 16ull << 20, int sm_count = 148);

// Launches one persistent kernel per group over `d_tiles` (device copy of the
// table the groups index). Per-bucket checksums accumulate atomically into
// d_sums (mod 2^64). Returns the number of kernel launches.
// Launch context of an Ingestor: an optional second stream for concurrent
// groups (fork/join through the events), and a ring of tile-scheduler
// counters in device memory for the TMA kernel's dynamic (work-stealing) tile
// order. Each launch takes the next slot. The counters are never reset: a
// launch draws exactly (dynamic tiles + CTAs) tickets, so the host keeps each
// slot's base (the counter value the next launch on it starts from) and
// advances it only after the launch is accepted; stream-ordered reuse is safe
// (slots >> launches in flight).
struct SideStream {
  cudaStream_t stream{nullptr};
  cudaEvent_t fork{nullptr}, join{nullptr};
  unsigned int* sched{nullptr};  // kSchedSlots x {ticket counter, unused}
  uint32_t sched_next{0};
  uint32_t sched_base[256]{};    // per slot: the counter value the next launch starts from
};
inline constexpr uint32_t kSchedSlots = 256;
uint32_t launch_groups(const Tile* d_tiles, const std::vector<Group>& groups, const uint8_t* src, uint8_t* dst,
                       unsigned long long* d_sums, cudaStream_t stream, int sm_count, SideStream* side);

// Peer pull over an identity plan's hash groups: copies src -> dst (src is a
// peer GPU's resident segment) and hashes the copied bytes in the same pass.
uint32_t launch_pull(const Tile* d_tiles, const std::vector<Group>& groups, const uint8_t* src, uint8_t* dst,
                     unsigned long long* d_sums, cudaStream_t stream, int sm_count);

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
