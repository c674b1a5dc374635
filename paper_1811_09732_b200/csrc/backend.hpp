// backend.hpp — CudaTierBackend: the B200 implementation of the reference's
// TierBackend plugin (proj/include/mrm/cache_core.hpp:76-98, implemented there
// by ShmTierBackend, proj/src/daemon.cpp:120-224), and the Ingestor that
// runs the disk -> pinned host -> HBM pipeline behind publish_fast.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "cache_core.hpp"
#include "device_mem.hpp"
#include "directory.hpp"
#include "format.hpp"
#include "ingest.hpp"

namespace trims {

struct IngestStats {
  double h2d_ms{0};        // copy-engine time of the blob (first chunk start -> last chunk end)
  double total_ms{0};      // ingest call wall time on the device (first copy -> last tile)
  double read_ms{0};       // host file reads (from_file only)
  uint64_t h2d_bytes{0};
  uint32_t launches{0};    // transform kernel launches
  double alloc_ms{0};      // publish_fast: cuMem create/map/export of the segment
  double seal_ms{0};       // publish_fast: tail (JSON + SegTail) write + digest
};

// A compiled ingest plan: tiles + chunks on the host, the tile table in HBM.
// Built once per (artifact manifest, plan) and reused by every ingest of it.
struct IngestPlan {
  fmt::Manifest src, dst;
  bool identity{false};
  ingest::TilePlan plan;
  ingest::Tile* d_tiles{nullptr};    // chunk-major table (pipelined H2D ingest)
  ingest::Tile* d_tiles_k{nullptr};  // kernel-grouped table (HBM-resident transform)
  int device{0};
  std::string dst_json;
  ~IngestPlan();
};

// One per device. Serialises its own ingests (PCIe is the shared resource).
class Ingestor {
 public:
  explicit Ingestor(int device);
  ~Ingestor();
  int device() const { return device_; }
  int sm_count() const { return sms_; }

  std::shared_ptr<IngestPlan> compile(const fmt::Manifest& src, const fmt::Plan& plan);

  // Raw artifact blob in host memory (pinned for full PCIe rate) -> resident
  // blob at d_dst. Returns the resident checksum; per-bucket sums optional.
  uint64_t from_host(const IngestPlan& p, const uint8_t* host_blob, uint8_t* d_dst, std::vector<uint64_t>* buckets,
                     IngestStats* st);
  // Streams the blob from an artifact file through a pinned bounce ring
  // (publish_fast without host staging, daemon.cpp:184-193).
  uint64_t from_file(const IngestPlan& p, int fd, uint64_t blob_file_off, uint8_t* d_dst,
                     std::vector<uint64_t>* buckets, IngestStats* st);
  // Raw blob already in HBM -> resident blob (the HBM-resident transform),
  // asynchronous on `stream`; bucket sums accumulate into d_sums.
  uint32_t from_device(const IngestPlan& p, const uint8_t* d_src, uint8_t* d_dst, unsigned long long* d_sums,
                       cudaStream_t stream);
  // Raw blob already uploaded to d_raw (ready once `ready` fires) -> resident
  // blob at d_dst: the transform (or, for an identity plan, the fused copy +
  // hash), then the checksums. Used by a publish whose stage_host streamed
  // the blob to the device while reading it.
  uint64_t from_staged(const IngestPlan& p, const uint8_t* d_raw, cudaEvent_t ready, uint8_t* d_dst,
                       std::vector<uint64_t>* buckets, IngestStats* st);
  // Peer pull: an identity plan's resident bytes from `d_src` (a peer GPU's
  // segment mapped here) to d_dst, copied and hashed by one fused kernel.
  uint64_t pull(const IngestPlan& p, const uint8_t* d_src, uint8_t* d_dst, std::vector<uint64_t>* buckets,
                IngestStats* st);
  // Waits for everything queued on the ingest streams (error paths: before
  // buffers a failed ingest may still be touching are freed). Never throws.
  void drain();

 private:
  uint8_t* staging(uint64_t bytes);
  unsigned long long* sums(uint32_t n);
  uint64_t finish(const ingest::TilePlan& p, std::vector<uint64_t>* buckets);

  int device_{0}, sms_{148};
  cudaStream_t copy_{}, compute_{};
  ingest::SideStream side_;  // concurrent direct-path groups (fork/join off compute_ or the caller's stream)
  std::vector<cudaEvent_t> events_;
  cudaEvent_t t0_{}, t1_{}, c0_{}, c1_{};
  uint8_t* staging_{nullptr};
  uint64_t staging_cap_{0};
  unsigned long long* d_sums_{nullptr};
  unsigned long long* h_sums_{nullptr};
  uint32_t sums_cap_{0};
  uint8_t* bounce_[2]{};
  uint64_t bounce_cap_{0};
  cudaEvent_t bounce_ev_[2]{};
  std::mutex mu_;
};

struct BackendConfig {
  int device{0};
  std::string disk_cache_dir;
  std::string remote_url;  // daemon.hpp:26 (http://... or dir:<path>; empty = no remote tier)
  bool full_verify{false};
  fmt::Plan plan;
  uint64_t pinned_pool_bytes{0};
  unsigned read_threads{8};
  // Cold-load reads into the pinned host tier: 0 buffered, 1 O_DIRECT, 2 auto
  // (O_DIRECT when most of the blob is not in the page cache).
  int direct_io{0};
  uint64_t arena_bytes{0};  // HBM arena for the fast tier (0 = one cuMem allocation per model)
  std::shared_ptr<Directory> directory;  // multi-GPU: publish sealed segments for peers (null = single GPU)
  // Keep the host tier in the RESIDENT form: after a converting publish, the
  // host copy is replaced (async D2H) by the converted blob, so a later warm
  // reload moves the bf16 bytes over PCIe (half of fp32) and only hashes them.
  // Off when the host copy is dropped on close anyway (eager reclaim).
  bool resident_host_tier{true};
};

// Fast-tier record of one published model: a range of the arena, or a
// dedicated segment when the arena has no fitting extent.
struct FastRecord {
  DeviceSegment seg;             // dedicated allocation (arena == nullptr)
  std::shared_ptr<DeviceArena> arena;  // arena range [offset, offset + reserved); kept alive by pinned records
  uint64_t offset{0}, reserved{0};
  uint8_t* base() const { return arena ? arena->base() + offset : seg.ptr(); }
  ~FastRecord() {
    if (arena) arena->free(offset);
  }
  fmt::ModelKey key;
  fmt::Manifest resident;
  std::string json;
  uint64_t generation{0};
  uint64_t checksum{0};
  std::vector<uint64_t> bucket_sums;
  IngestStats stats;
};

// Startup calibration of the share-benefit cost model (daemon.hpp:42-46,
// Daemon::run_startup_calibration daemon.cpp:342-390), measured on the B200
// path: q = artifact read rate, o = per-object export (place + seal a
// segment), s = per-object attach (read back + validate its sealed tail).
struct Calibration {
  double q{0};  // disk bytes/second
  double o{0};  // per-object export seconds
  double s{0};  // per-object attach seconds
};

class CudaTierBackend : public TierBackend {
 public:
  explicit CudaTierBackend(BackendConfig cfg);
  ~CudaTierBackend() override;

  Located locate(const fmt::ModelKey& key) override;
  FetchResult fetch_remote(const fmt::ModelKey& key) override;
  fmt::Manifest read_manifest(const fmt::ModelKey& key, const std::string& path) override;
  void stage_host(uint64_t model_id, const fmt::Manifest& m, const std::string& path) override;
  FastPublication publish_fast(uint64_t model_id, const fmt::Manifest& m, bool from_host,
                               const std::string& path) override;
  void evict_fast(uint64_t model_id) override;
  void evict_host(uint64_t model_id) override;
  void evict_disk(const fmt::ModelKey& key, const std::string& path) override;
  void load_settled(const fmt::ModelKey& key) override;
  FastPublication publish_from_peer(uint64_t model_id, const fmt::Manifest& m, const PeerSource& src) override;

  std::shared_ptr<FastRecord> fast_record(uint64_t model_id);
  // nullopt when the disk cache holds no artifact of >= 1 MiB to time (as the reference)
  std::optional<Calibration> calibrate();
  const uint8_t* host_buffer(uint64_t model_id, uint64_t* bytes);
  Ingestor& ingestor() { return ing_; }
  const BackendConfig& config() const { return cfg_; }
  uint64_t direct_loads() const { return direct_loads_.load(); }

 private:
  struct HostBuf {
    uint8_t* p{nullptr};           // the blob
    uint8_t* base{nullptr};        // the allocation (p - head: direct reads keep p congruent to the file offset)
    uint64_t bytes{0};
    bool pooled{false};
    bool resident{false};          // holds the resident (converted) blob, valid once `ready` fires
    cudaEvent_t ready{nullptr};    // the D2H that wrote it (null: raw artifact bytes)
  };
  void to_resident_form(uint64_t model_id, const FastRecord& rec, const IngestPlan& plan);
  void free_host(HostBuf& h);
  // head: bytes before the blob in the allocation (< 4096); a head or direct
  // read also reserves 4 KiB after it (the last aligned block)
  HostBuf alloc_host(uint64_t bytes, uint64_t head = 0, bool direct = false);
  int direct_fd_for(const std::string& path, int fd, uint64_t off, uint64_t len);
  std::atomic<uint64_t> direct_loads_{0};  // disk reads done with O_DIRECT
  uint32_t arena_seq_{0};                   // this arena's number in the process (its token's suffix)
  bool take_verified(const fmt::ModelKey& key, uint64_t bytes, HostBuf* out);

  std::shared_ptr<IngestPlan> plan_for(uint64_t model_id, const fmt::Manifest& m);
  std::shared_ptr<IngestPlan> pull_plan_for(uint64_t model_id, const fmt::Manifest& resident);
  void place(FastRecord& rec, uint64_t payload);  // arena range or dedicated segment + generation
  FastPublication seal(uint64_t model_id, std::shared_ptr<FastRecord> rec, const fmt::Manifest& m);

  BackendConfig cfg_;
  Ingestor ing_;
  std::unique_ptr<PinnedPool> pool_;
  std::shared_ptr<DeviceArena> arena_;  // shared with every record placed in it (a pin may outlive the backend)
  std::mutex mu_;
  std::map<uint64_t, HostBuf> host_;
  // full_verify: read_manifest reads the blob into pinned memory while hashing
  // it (one pass, pread.hpp) and keeps the verified bytes here until the same
  // open stages / publishes them, so they are neither read nor hashed twice
  // (the reference reads + hashes in read_manifest, then again in read_model).
  std::map<std::string, HostBuf> verified_;
  std::map<uint64_t, std::shared_ptr<FastRecord>> fast_;
  std::map<uint64_t, std::shared_ptr<IngestPlan>> plans_;  // model_id -> compiled plan (manifests are immutable)
  std::map<uint64_t, std::shared_ptr<IngestPlan>> pull_plans_;  // model_id -> identity plan of the resident blob
  std::atomic<uint64_t> next_gen_{1};

  // Cold-path overlap: stage_host reads the artifact in chunks into the
  // pinned host tier and uploads each chunk to `pre_raw_` while reading the
  // next, so the publish_fast that follows (same open, same thread) only
  // transforms. One model at a time owns the buffer (pre_owner_); a
  // concurrent cold open takes the plain path.
  static constexpr uint64_t kNoOwner = ~0ull;
  static constexpr uint64_t kPrestageKeep = 256ull << 20;  // pool memory parked between cold opens
  std::atomic<uint64_t> pre_owner_{kNoOwner};
  uint8_t* pre_raw_{nullptr};      // from pre_pool_, owned by pre_owner_ until its publish (converting plans)
  std::shared_ptr<FastRecord> pre_rec_;  // identity plans: the placed segment the file streams into
  uint8_t* claim_prestage(uint64_t model_id, const fmt::Manifest& m, uint64_t bytes);
  cudaMemPool_t pre_pool_{nullptr};
  cudaStream_t pre_stream_{nullptr};
  cudaStream_t d2h_stream_{nullptr};  // host tier -> resident form
  cudaEvent_t pre_t0_{nullptr}, pre_done_{nullptr}, pre_used_{nullptr};
  double pre_read_ms_{0};
  void release_prestage(uint64_t model_id);
};

// Multi-threaded pread of [off, off+len) into dst (page cache -> pinned).
// (parallel_pread_upload, the same with the in-order upload + hash, is local to backend.cu)
void parallel_pread(int fd, uint8_t* dst, uint64_t len, uint64_t off, unsigned threads);

}  // namespace trims
