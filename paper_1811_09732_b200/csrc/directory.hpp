// directory.hpp — node-local fast-tier residency directory for the multi-GPU
// store (builder-defined: the reference runs one daemon per
// node and has no peer tier).
//
// One POSIX shared-memory table per node job: a header, then one row per rank
// (= per GPU process). Each rank is the single writer of its own row and
// every rank reads all rows, so there is no cross-process lock: each slot is a
// seqlock (odd sequence while the writer edits it). A row records where the
// rank's sealed fast-tier segments live (owner pid + fd of the exportable
// allocation, offset, generation, checksum); a peer maps that allocation and
// pulls the segment over NVLink (CudaTierBackend::publish_from_peer), and the
// segment's own sealed tail — not the directory — is the authority that the
// bytes are current. The directory is a hint that may lag by one eviction.
#pragma once

#include <atomic>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "cache_core.hpp"
#include "format.hpp"

namespace trims {

struct DirCoords {
  int32_t rank{-1}, device{-1}, pid{0}, fd{-1};
  uint32_t arena{0};     // the allocation outlives the segment (map once, reuse)
  uint32_t reserved{0};  // arena: its number in the owner process (token trims.<pid>.arena<device>.<n>)
  uint64_t alloc_bytes{0}, offset{0};
  uint64_t payload_bytes{0}, resident_blob_bytes{0}, generation{0}, checksum{0};
};

// Rendezvous weight of (key, rank): among several holders a requester pulls
// from the highest, which spreads the pulls of a hot model over its holders.
// Restated by oracle/simulator.py:peer_score.
uint64_t peer_score(const std::string& key, int rank);
uint64_t fnv1a64(const std::string& s);

class Directory {
 public:
  static constexpr uint32_t kKeyMax = 200;
  // Create or attach `name` (a /dev/shm name without the slash) sized for
  // world x slots; this rank's row is cleared (a restarted rank starts empty).
  static std::unique_ptr<Directory> open(const std::string& name, int world, int rank, uint32_t slots);
  static void unlink(const std::string& name);
  ~Directory();

  int rank() const { return rank_; }
  int world() const { return world_; }

  // Writer side (own row only).
  void publish(const fmt::ModelKey& key, const DirCoords& c);  // replaces an existing slot of `key`
  void retract(const fmt::ModelKey& key);
  void clear();

  // Reader side: the other ranks' live copies of `key`, best peer first.
  std::vector<DirCoords> holders(const fmt::ModelKey& key) const;
  // Every live slot of `rank` (tests / diagnostics).
  std::vector<std::pair<std::string, DirCoords>> row(int rank) const;

 private:
  struct Slot;
  struct Header;
  Directory() = default;
  Slot* slot(int rank, uint32_t i) const;
  bool read_slot(const Slot& s, std::string* key, DirCoords* c) const;

  int fd_{-1};
  void* map_{nullptr};
  uint64_t bytes_{0};
  int world_{0}, rank_{0};
  uint32_t slots_{0};
};

// The multi-GPU open (builder-defined; restated by oracle/simulator.py
// simulate_cluster): a model already fast-resident here is a plain hit; else
// each peer holding it, best first, is tried as a PeerSource; a peer whose
// copy went stale or cannot be mapped is skipped (counted as a fallback); with
// no usable peer this is exactly the reference's open. Admission failures of
// the peer open (TooLargeForFast, NoEvictableSpace) are decisions, not
// fallbacks, and propagate.
struct PeerCounters {
  std::atomic<uint64_t> attempts{0}, fallbacks{0};
};
using ManifestFn = std::function<std::shared_ptr<const fmt::Manifest>(const fmt::ModelKey&)>;
// Returns the source for one holder; may park a keep-alive (a temporary
// mapping) in *hold for the duration of the open.
using SourceFn = std::function<PeerSource(const DirCoords&, std::shared_ptr<void>* hold)>;
PlacementResult open_with_peers(CacheCore& core, const Directory* dir, const fmt::ModelKey& key, const Granularity& g,
                                uint64_t now, const ManifestFn& manifest_for, const SourceFn& source_for,
                                PeerCounters* ctr, int* peer_rank);
bool peer_retryable(Errc e);

}  // namespace trims
