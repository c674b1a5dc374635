// cache_core.hpp — the placement manager of the store: tiered residency
// (fast = HBM, host = pinned DRAM, disk cache, remote), refcounts, LRU/LCU
// eviction, per-key single-flight. Decision-for-decision identical to the
// reference's proj/src/cache_core.cpp (pinned against the reference live core
// and simulator by tests/test_decisions.py); the physical work goes through
// the same TierBackend plugin boundary (proj/include/mrm/cache_core.hpp:76-98).
#pragma once

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "errc.hpp"
#include "format.hpp"

namespace trims {

enum class Tier : uint8_t { Fast = 0, Host = 1, Disk = 2, Remote = 3 };
inline constexpr int kTiers = 4;
enum class Policy : uint8_t { LRU = 0, LCU = 1 };
// PeerHit is the multi-GPU extension (served by an NVLink peer copy).
enum class Outcome : uint8_t { FastHit = 0, HostHit = 1, DiskLoad = 2, RemoteFetch = 3, PeerHit = 4 };

enum class GranKind : uint8_t { Model = 0, Layer = 1, Block = 2 };
struct Granularity {
  GranKind kind{GranKind::Model};
  uint64_t block_bytes{2ull << 20};
};
bool valid_granularity(const Granularity& g);

struct ObjectSpan {
  std::string name;
  uint32_t segment_index{0};
  uint64_t offset{0}, length{0};
};
// shm::layout_for (proj/src/shared_segment.cpp:63-95).
std::vector<ObjectSpan> layout_for(const fmt::Manifest& m, const Granularity& g);

struct PhaseTimings {
  uint64_t fetch_ns{0}, disk_read_ns{0}, host_to_fast_copy_ns{0}, handle_export_ns{0};
};

// What the fast tier exports for one model: the device segment and how a
// client reaches it. `token` names it; for the CUDA backend the handle is an
// exportable cuMem allocation (fd) plus a legacy cudaIpc handle.
struct ExportedSegment {
  std::string token;
  uint64_t generation{0};
  uint64_t length{0};         // payload bytes: resident blob + JSON + tail
  int device{0};
  void* dev_ptr{nullptr};     // owner-process address
  int fd{-1};                 // owner-process POSIX fd of the allocation (-1: none)
  uint64_t alloc_bytes{0};    // physical allocation (granularity-rounded)
  uint64_t offset{0};         // segment offset inside that allocation (arena ranges)
  uint8_t ipc_handle[64]{};   // cudaIpcMemHandle_t bytes (legacy import path)
  uint64_t resident_blob_bytes{0};
  uint64_t ingest_checksum{0};  // TRIMS block checksum of the resident blob
};

struct FastPublication {
  std::vector<ExportedSegment> segments;
  fmt::Digest manifest_digest{};
};

struct Located {
  enum class Kind { DiskCache, Remote, Absent };
  Kind kind{Kind::Absent};
  std::string path;
  uint64_t file_bytes{0};
};
struct FetchResult {
  std::string path;
  uint64_t file_bytes{0};
};

// Multi-GPU extension: a sealed fast-tier copy of the model on
// a peer GPU, mapped into this process and readable from this device. The
// open becomes a PeerHit: the manifest comes with the source, no disk or host
// tier is touched, and the backend pulls the resident segment over NVLink.
struct PeerSource {
  std::shared_ptr<const fmt::Manifest> manifest;  // artifact manifest of the model
  int rank{-1}, device{-1};
  const uint8_t* payload{nullptr};  // peer segment base (resident blob | JSON | jlen | SegTail)
  uint64_t payload_bytes{0}, resident_blob_bytes{0}, generation{0}, checksum{0};
};

// The plugin boundary, same eight operations and threading contract as the
// reference: everything but evict_* is called outside the core lock; evict_*
// runs under it and must not block long.
class TierBackend {
 public:
  virtual ~TierBackend() = default;
  virtual Located locate(const fmt::ModelKey& key) = 0;
  virtual FetchResult fetch_remote(const fmt::ModelKey& key) = 0;
  virtual fmt::Manifest read_manifest(const fmt::ModelKey& key, const std::string& path) = 0;
  virtual void stage_host(uint64_t model_id, const fmt::Manifest& m, const std::string& path) = 0;
  virtual FastPublication publish_fast(uint64_t model_id, const fmt::Manifest& m, bool from_host,
                                       const std::string& path) = 0;
  virtual void evict_fast(uint64_t model_id) = 0;
  virtual void evict_host(uint64_t model_id) = 0;
  virtual void evict_disk(const fmt::ModelKey& key, const std::string& path) = 0;
  // Extension, not part of the reference's eight: fill the fast tier from a
  // peer's sealed segment. The default refuses.
  virtual FastPublication publish_from_peer(uint64_t model_id, const fmt::Manifest& m, const PeerSource& src);
  // Extension: the open of `key` that called read_manifest has settled
  // (published or failed). Called under the core mutex; must not block. Lets a
  // backend drop per-load state, e.g. a blob it read while verifying.
  virtual void load_settled(const fmt::ModelKey&) {}
};

struct PlacementResult {
  Outcome outcome{Outcome::FastHit};
  uint64_t model_id{0};
  std::shared_ptr<const fmt::Manifest> manifest;  // artifact manifest (shared, immutable)
  uint64_t weights_bytes{0}, workspace_bytes{0};
  std::vector<ExportedSegment> segments;
  std::vector<ObjectSpan> layout;
  fmt::Digest manifest_digest{};
  PhaseTimings timings;
};

struct TierStats {
  uint64_t hits{0}, misses{0}, evictions{0}, used_bytes{0}, capacity_bytes{0};
};
struct ModelStats {
  fmt::ModelKey key;
  uint32_t refcount{0};
  uint64_t use_count{0}, last_access{0};
  uint8_t residency{0};
};
struct StatsSnapshot {
  TierStats tiers[kTiers];
  std::vector<ModelStats> models;
  uint64_t open_requests{0}, open_errors{0}, disk_reads{0}, remote_fetches{0};
  uint64_t peer_hits{0};  // multi-GPU extension
  PhaseTimings cumulative;
};

struct CoreConfig {
  uint64_t fast_capacity_bytes{0}, host_capacity_bytes{0}, disk_capacity_bytes{0};
  Policy policy{Policy::LRU};
  bool eager_reclaim{false};
};

struct Candidate {
  fmt::ModelKey key;
  uint32_t refcount{0};
  uint64_t last_access{0}, use_count{0}, seq{0};
};
// cache_core.cpp:56-65: refcount==0 entries ordered by the policy metric, then seq.
std::vector<Candidate> evict_candidates(Policy p, std::vector<Candidate> c);

class CacheCore {
 public:
  // A peer attempt that failed for good (open_with_peers rethrows it): one user-level open error.
  void note_open_error() {
    std::lock_guard lk(mu_);
    ++open_errors_;
  }
  CacheCore(CoreConfig cfg, TierBackend& backend);
  // `peer` (multi-GPU extension): a peer copy to serve a fast-tier miss from;
  // nullptr is exactly the reference's open.
  PlacementResult open_model(const fmt::ModelKey& key, const Granularity& g, uint64_t now,
                             const PeerSource* peer = nullptr);
  uint64_t close_model(const fmt::ModelKey& key);
  std::vector<fmt::ModelKey> reclaim(Tier t, uint64_t bytes_needed, Policy p);
  StatsSnapshot stats() const;
  void register_disk_file(const fmt::ModelKey& key, const std::string& path, uint64_t bytes);
  uint64_t used_bytes(Tier t) const;
  uint64_t capacity_bytes(Tier t) const;
  uint32_t refcount(const fmt::ModelKey& key) const;
  bool drained() const;
  void drop_all();
  // Multi-GPU extension: is the model fast-resident here (no state change)?
  bool fast_resident(const fmt::ModelKey& key) const;

 private:
  struct Entry {
    fmt::ModelKey key;
    uint64_t model_id{0}, seq{0};
    std::shared_ptr<const fmt::Manifest> manifest;
    uint32_t refcount{0};
    uint64_t last_access{0}, use_count{0};
    bool in_fast{false}, in_host{false}, on_disk{false}, loading{false};
    std::vector<ExportedSegment> segments;
    fmt::Digest digest{};
    std::string disk_path;
    uint64_t disk_bytes{0}, weights{0};
  };
  struct Flight {
    bool done{false};
  };

  Entry* find(const fmt::ModelKey& k);
  const Entry* find(const fmt::ModelKey& k) const;
  Entry& entry_for(const fmt::ModelKey& k);
  uint64_t capacity(Tier t) const;
  bool resident(const Entry& e, Tier t) const;
  uint64_t charge(const Entry& e, Tier t) const;
  void drop_residency(Entry& e, Tier t);  // backend evict + accounting, no stats
  void evict(Entry& e, Tier t);           // drop_residency + eviction counter
  std::vector<fmt::ModelKey> reclaim_held(Tier t, uint64_t need, Policy p);
  PlacementResult result_held(Entry& e, Outcome o, const Granularity& g, PhaseTimings tm);

  CoreConfig cfg_;
  TierBackend& be_;
  mutable std::mutex mu_;
  std::condition_variable flight_cv_;
  std::map<fmt::ModelKey, Entry> entries_;
  std::map<fmt::ModelKey, std::shared_ptr<Flight>> flights_;
  uint64_t next_seq_{1}, next_id_{1};
  uint64_t used_[kTiers]{};
  uint64_t hits_[kTiers]{}, misses_[kTiers]{}, evictions_[kTiers]{};
  uint64_t opens_{0}, open_errors_{0}, disk_reads_{0}, remote_fetches_{0}, peer_hits_{0};
  PhaseTimings cumulative_;
};

}  // namespace trims
