// backend.cu — Ingestor (pinned host / file -> HBM, copy-engine chunks
// overlapped with the fused transform kernel) and CudaTierBackend.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <filesystem>
#include <mutex>
#include <thread>

#include "backend.hpp"
#include "cuda_util.hpp"
#include "pread.hpp"
#include "remote.hpp"
#include "sha256.hpp"

namespace trims {

namespace fs = std::filesystem;

void parallel_pread(int fd, uint8_t* dst, uint64_t len, uint64_t off, unsigned threads) {
  // 2 MiB pieces handed out by a counter (measured faster from the page cache
  // than one large piece per thread)
  pipelined_read(fd, off, len, dst, threads, nullptr);
}

// Reads [off, off+len) into the pinned host buffer in 2 MiB pieces handed out
// to `threads` readers, while the calling thread uploads the pieces to `dev`
// as they land (async on `stream`): the PCIe copy of the blob runs
// under the file read instead of after it, and one thread owns the stream
// (readers issuing their own copies contended in the driver). Pieces upload
// in the order they land, not in file order. With `hash`, a further thread
// hashes the pieces in file order under both.
void parallel_pread_upload(int fd, uint8_t* host, uint8_t* dev, uint64_t len, uint64_t off, unsigned threads,
                           int device, cudaStream_t stream, Sha256* hash, int direct_fd) {
  DeviceGuard g(device);
  static const bool any_order = [] {  // A/B switch: TRIMS_UPLOAD_IN_ORDER=1
    const char* e = std::getenv("TRIMS_UPLOAD_IN_ORDER");
    return !(e && std::string(e) == "1");
  }();
  pipelined_read(
      fd, off, len, host, threads, hash,
      [&](const uint8_t* p, uint64_t b, uint64_t n) {
        TRIMS_CUDA(cudaMemcpyAsync(dev + b, p, n, cudaMemcpyHostToDevice, stream));
      },
      any_order, direct_fd);
}

// ---------------------------------------------------------------------------
// Ingestor

Ingestor::Ingestor(int device) : device_(device) {
  DeviceGuard g(device);
  TRIMS_CUDA(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device));
  TRIMS_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
  TRIMS_CUDA(cudaStreamCreateWithFlags(&compute_, cudaStreamNonBlocking));
  TRIMS_CUDA(cudaStreamCreateWithFlags(&side_.stream, cudaStreamNonBlocking));
  TRIMS_CUDA(cudaEventCreateWithFlags(&side_.fork, cudaEventDisableTiming));
  TRIMS_CUDA(cudaEventCreateWithFlags(&side_.join, cudaEventDisableTiming));
  TRIMS_CUDA(cudaMalloc(&side_.sched, 2 * ingest::kSchedSlots * sizeof(unsigned int)));
  // ordered before every launch of this Ingestor: compute_ is a non-blocking
  // stream, so a legacy-stream memset would not be
  TRIMS_CUDA(cudaMemsetAsync(side_.sched, 0, 2 * ingest::kSchedSlots * sizeof(unsigned int), compute_));
  TRIMS_CUDA(cudaStreamSynchronize(compute_));
  events_.resize(512);
  for (auto& e : events_) TRIMS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto* e : {&t0_, &t1_, &c0_, &c1_}) TRIMS_CUDA(cudaEventCreate(e));
  for (auto& e : bounce_ev_) TRIMS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

Ingestor::~Ingestor() {
  DeviceGuard g(device_, /*nothrow=*/true);
  for (auto e : events_) cudaEventDestroy(e);
  for (auto e : {t0_, t1_, c0_, c1_}) cudaEventDestroy(e);
  for (auto e : bounce_ev_) cudaEventDestroy(e);
  if (staging_) cudaFree(staging_);
  if (d_sums_) cudaFree(d_sums_);
  if (h_sums_) cudaFreeHost(h_sums_);
  for (auto* b : bounce_)
    if (b) cudaFreeHost(b);
  cudaStreamDestroy(copy_);
  cudaStreamDestroy(compute_);
  cudaStreamDestroy(side_.stream);
  cudaEventDestroy(side_.fork);
  cudaEventDestroy(side_.join);
  cudaFree(side_.sched);
}

uint8_t* Ingestor::staging(uint64_t bytes) {
  if (bytes > staging_cap_) {
    if (staging_) TRIMS_CUDA(cudaFree(staging_));
    staging_ = nullptr;
    staging_cap_ = 0;
    uint64_t cap = std::max<uint64_t>(bytes, 64ull << 20);
    TRIMS_CUDA(cudaMalloc(&staging_, cap));
    staging_cap_ = cap;
  }
  return staging_;
}

unsigned long long* Ingestor::sums(uint32_t n) {
  if (n > sums_cap_) {
    if (d_sums_) TRIMS_CUDA(cudaFree(d_sums_));
    if (h_sums_) TRIMS_CUDA(cudaFreeHost(h_sums_));
    uint32_t cap = std::max<uint32_t>(n, 1024);
    TRIMS_CUDA(cudaMalloc(&d_sums_, cap * sizeof(unsigned long long)));
    TRIMS_CUDA(cudaHostAlloc(&h_sums_, cap * sizeof(unsigned long long), cudaHostAllocDefault));
    sums_cap_ = cap;
  }
  return d_sums_;
}

IngestPlan::~IngestPlan() {
  if (d_tiles || d_tiles_k) {
    DeviceGuard g(device, /*nothrow=*/true);
    if (d_tiles) cudaFree(d_tiles);
    if (d_tiles_k) cudaFree(d_tiles_k);
  }
}

std::shared_ptr<IngestPlan> Ingestor::compile(const fmt::Manifest& src, const fmt::Plan& plan) {
  DeviceGuard g(device_);
  auto p = std::make_shared<IngestPlan>();
  p->device = device_;
  p->src = src;
  p->dst = fmt::resident_manifest(src, plan);
  p->dst_json = fmt::manifest_to_json(p->dst);
  p->identity = plan.identity();
  const uint64_t chunk = std::max<uint64_t>(16ull << 20, src.blob_bytes / (events_.size() - 8) + 1);
  p->plan = ingest::build_tiles(p->src, p->dst, p->identity, chunk, sms_);
  if (!p->plan.tiles.empty()) {
    // the device images: scheduled groups' bins padded to a common stride
    auto upload = [](ingest::Tile** d, const std::vector<ingest::Tile>& t) {
      const size_t tb = std::max<size_t>(1, t.size()) * sizeof(ingest::Tile);
      TRIMS_CUDA(cudaMalloc(d, tb));
      if (!t.empty()) TRIMS_CUDA(cudaMemcpy(*d, t.data(), t.size() * sizeof(ingest::Tile), cudaMemcpyHostToDevice));
    };
    upload(&p->d_tiles, p->plan.dev_tiles);
    upload(&p->d_tiles_k, p->plan.dev_tiles_k);
    // A pageable-memory cudaMemcpy may return before its DMA lands, and the
    // ingest kernels run on non-blocking streams that do not order after the
    // legacy stream: wait for the tables here (a cold open once raced this).
    TRIMS_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
  }
  return p;
}

uint64_t Ingestor::finish(const ingest::TilePlan& p, std::vector<uint64_t>* buckets) {
  TRIMS_CUDA(cudaMemcpyAsync(h_sums_, d_sums_, p.buckets * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             compute_));
  TRIMS_CUDA(cudaStreamSynchronize(compute_));
  uint64_t total = 0;
  if (buckets) buckets->assign(h_sums_, h_sums_ + p.buckets);
  for (uint32_t i = 0; i < p.buckets; ++i) total += h_sums_[i];
  return total;
}

uint64_t Ingestor::from_host(const IngestPlan& ip, const uint8_t* host_blob, uint8_t* d_dst,
                             std::vector<uint64_t>* buckets, IngestStats* st) {
  std::lock_guard lk(mu_);
  DeviceGuard g(device_);
  const ingest::TilePlan& p = ip.plan;
  unsigned long long* ds = sums(p.buckets);
  TRIMS_CUDA(cudaMemsetAsync(ds, 0, p.buckets * sizeof(unsigned long long), compute_));
  uint8_t* raw = ip.identity ? d_dst : staging(ip.src.blob_bytes);
  TRIMS_CUDA(cudaEventRecord(t0_, copy_));
  uint32_t launches = 0;
  for (size_t c = 0; c < p.chunks.size(); ++c) {
    const auto& ch = p.chunks[c];
    cudaEvent_t ev = events_[c % events_.size()];
    TRIMS_CUDA(cudaMemcpyAsync(raw + ch.src_begin, host_blob + ch.src_begin, ch.src_end - ch.src_begin,
                               cudaMemcpyHostToDevice, copy_));
    TRIMS_CUDA(cudaEventRecord(ev, copy_));
    TRIMS_CUDA(cudaStreamWaitEvent(compute_, ev, 0));
    launches += ingest::launch_groups(ip.d_tiles, ch.groups, raw, d_dst, ds, compute_, sms_, &side_);
  }
  TRIMS_CUDA(cudaEventRecord(t1_, copy_));
  TRIMS_CUDA(cudaEventRecord(c1_, compute_));
  uint64_t total = finish(p, buckets);
  if (st) {
    float ms = 0;
    // t1_ sits on the copy stream after the last chunk's event; the compute
    // stream waited for that event, not for t1_ itself
    TRIMS_CUDA(cudaEventSynchronize(t1_));
    TRIMS_CUDA(cudaEventElapsedTime(&ms, t0_, t1_));
    st->h2d_ms = ms;
    TRIMS_CUDA(cudaEventElapsedTime(&ms, t0_, c1_));
    st->total_ms = ms;
    st->h2d_bytes = p.chunks.empty() ? 0 : p.chunks.back().src_end - p.chunks.front().src_begin;
    st->launches = launches;
  }
  return total;
}

uint64_t Ingestor::from_file(const IngestPlan& ip, int fd, uint64_t blob_file_off, uint8_t* d_dst,
                             std::vector<uint64_t>* buckets, IngestStats* st) {
  std::lock_guard lk(mu_);
  DeviceGuard g(device_);
  const ingest::TilePlan& p = ip.plan;
  uint64_t need = 0;
  for (const auto& ch : p.chunks) need = std::max(need, ch.src_end - ch.src_begin);
  if (need > bounce_cap_) {
    for (auto*& b : bounce_) {
      if (b) TRIMS_CUDA(cudaFreeHost(b));
      b = nullptr;
    }
    bounce_cap_ = 0;
    for (auto*& b : bounce_) TRIMS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b), need, cudaHostAllocDefault));
    bounce_cap_ = need;
  }
  unsigned long long* ds = sums(p.buckets);
  TRIMS_CUDA(cudaMemsetAsync(ds, 0, p.buckets * sizeof(unsigned long long), compute_));
  uint8_t* raw = ip.identity ? d_dst : staging(ip.src.blob_bytes);
  TRIMS_CUDA(cudaEventRecord(t0_, copy_));
  double read_ms = 0;
  uint32_t launches = 0;
  for (size_t c = 0; c < p.chunks.size(); ++c) {
    const auto& ch = p.chunks[c];
    const int slot = int(c & 1);
    TRIMS_CUDA(cudaEventSynchronize(bounce_ev_[slot]));  // previous H2D out of this slot done
    auto r0 = std::chrono::steady_clock::now();
    parallel_pread(fd, bounce_[slot], ch.src_end - ch.src_begin, blob_file_off + ch.src_begin, 8);
    read_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - r0).count();
    cudaEvent_t ev = events_[c % events_.size()];
    TRIMS_CUDA(cudaMemcpyAsync(raw + ch.src_begin, bounce_[slot], ch.src_end - ch.src_begin,
                               cudaMemcpyHostToDevice, copy_));
    TRIMS_CUDA(cudaEventRecord(ev, copy_));
    TRIMS_CUDA(cudaEventRecord(bounce_ev_[slot], copy_));
    TRIMS_CUDA(cudaStreamWaitEvent(compute_, ev, 0));
    launches += ingest::launch_groups(ip.d_tiles, ch.groups, raw, d_dst, ds, compute_, sms_, &side_);
  }
  TRIMS_CUDA(cudaEventRecord(t1_, copy_));
  TRIMS_CUDA(cudaEventRecord(c1_, compute_));
  uint64_t total = finish(p, buckets);
  if (st) {
    float ms = 0;
    // t1_ sits on the copy stream after the last chunk's event; the compute
    // stream waited for that event, not for t1_ itself
    TRIMS_CUDA(cudaEventSynchronize(t1_));
    TRIMS_CUDA(cudaEventElapsedTime(&ms, t0_, t1_));
    st->h2d_ms = ms;
    TRIMS_CUDA(cudaEventElapsedTime(&ms, t0_, c1_));
    st->total_ms = ms;
    st->read_ms = read_ms;
    st->h2d_bytes = p.chunks.empty() ? 0 : p.chunks.back().src_end - p.chunks.front().src_begin;
    st->launches = launches;
  }
  return total;
}

uint32_t Ingestor::from_device(const IngestPlan& ip, const uint8_t* d_src, uint8_t* d_dst,
                               unsigned long long* d_sums, cudaStream_t stream) {
  std::lock_guard lk(mu_);  // side_ is shared
  DeviceGuard g(device_);
  return ingest::launch_groups(ip.d_tiles_k, ip.plan.groups, d_src, d_dst, d_sums, stream, sms_, &side_);
}

uint64_t Ingestor::from_staged(const IngestPlan& ip, const uint8_t* d_raw, cudaEvent_t ready, uint8_t* d_dst,
                               std::vector<uint64_t>* buckets, IngestStats* st) {
  std::lock_guard lk(mu_);
  DeviceGuard g(device_);
  const ingest::TilePlan& p = ip.plan;
  unsigned long long* ds = sums(p.buckets);
  TRIMS_CUDA(cudaMemsetAsync(ds, 0, p.buckets * sizeof(unsigned long long), compute_));
  TRIMS_CUDA(cudaStreamWaitEvent(compute_, ready, 0));
  TRIMS_CUDA(cudaEventRecord(c0_, compute_));
  const uint32_t launches = ip.identity ? ingest::launch_pull(ip.d_tiles_k, p.groups, d_raw, d_dst, ds, compute_, sms_)
                                        : ingest::launch_groups(ip.d_tiles_k, p.groups, d_raw, d_dst, ds, compute_,
                                                                sms_, &side_);
  TRIMS_CUDA(cudaEventRecord(c1_, compute_));
  const uint64_t total = finish(p, buckets);
  if (st) {
    float ms = 0;
    TRIMS_CUDA(cudaEventElapsedTime(&ms, c0_, c1_));
    st->total_ms = ms;
    st->launches = launches;
  }
  return total;
}

void Ingestor::drain() {
  DeviceGuard g(device_, /*nothrow=*/true);
  if (copy_) cudaStreamSynchronize(copy_);
  if (compute_) cudaStreamSynchronize(compute_);
  if (side_.stream) cudaStreamSynchronize(side_.stream);
  cudaGetLastError();
}

uint64_t Ingestor::pull(const IngestPlan& ip, const uint8_t* d_src, uint8_t* d_dst, std::vector<uint64_t>* buckets,
                        IngestStats* st) {
  if (!ip.identity) raise(Errc::Internal, "peer pull needs an identity plan");
  std::lock_guard lk(mu_);
  DeviceGuard g(device_);
  const ingest::TilePlan& p = ip.plan;
  unsigned long long* ds = sums(p.buckets);
  TRIMS_CUDA(cudaMemsetAsync(ds, 0, p.buckets * sizeof(unsigned long long), compute_));
  TRIMS_CUDA(cudaEventRecord(c0_, compute_));
  const uint32_t launches = ingest::launch_pull(ip.d_tiles_k, p.groups, d_src, d_dst, ds, compute_, sms_);
  TRIMS_CUDA(cudaEventRecord(c1_, compute_));
  const uint64_t total = finish(p, buckets);
  if (st) {
    float ms = 0;
    TRIMS_CUDA(cudaEventElapsedTime(&ms, c0_, c1_));
    st->total_ms = ms;
    st->h2d_ms = 0;
    st->h2d_bytes = 0;
    st->launches = launches;
  }
  return total;
}

// ---------------------------------------------------------------------------
// CudaTierBackend

namespace {
// TRIMS_PRESTAGE=0: stage_host reads the whole blob first, publish uploads (A/B).
bool prestage_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_PRESTAGE");
    return !(e && std::string(e) == "0");
  }();
  return on;
}
}  // namespace

CudaTierBackend::CudaTierBackend(BackendConfig cfg) : cfg_(std::move(cfg)), ing_(cfg_.device) {
  DeviceGuard g(cfg_.device);
  if (cfg_.pinned_pool_bytes) pool_ = std::make_unique<PinnedPool>(cfg_.pinned_pool_bytes);
  if (cfg_.arena_bytes) {
    // one name per arena, also with several stores in one process (their
    // lease tables must not collide): trims.<pid>.arena<device>.<n>
    static std::atomic<uint32_t> arenas{0};
    arena_seq_ = arenas.fetch_add(1);
    arena_ = std::make_shared<DeviceArena>(cfg_.device, cfg_.arena_bytes,
                                           "trims." + std::to_string(::getpid()) + ".arena" +
                                               std::to_string(cfg_.device) + "." + std::to_string(arena_seq_));
  }
  TRIMS_CUDA(cudaStreamCreateWithFlags(&pre_stream_, cudaStreamNonBlocking));
  TRIMS_CUDA(cudaStreamCreateWithFlags(&d2h_stream_, cudaStreamNonBlocking));
  cudaMemPoolProps pp{};
  pp.allocType = cudaMemAllocationTypePinned;
  pp.location.type = cudaMemLocationTypeDevice;
  pp.location.id = cfg_.device;
  TRIMS_CUDA(cudaMemPoolCreate(&pre_pool_, &pp));
  uint64_t keep = kPrestageKeep;  // parked between cold opens; the rest is released at the next sync point
  TRIMS_CUDA(cudaMemPoolSetAttribute(pre_pool_, cudaMemPoolAttrReleaseThreshold, &keep));
  TRIMS_CUDA(cudaEventCreate(&pre_t0_));
  TRIMS_CUDA(cudaEventCreate(&pre_done_));
  TRIMS_CUDA(cudaEventCreateWithFlags(&pre_used_, cudaEventDisableTiming));
  TRIMS_CUDA(cudaEventRecord(pre_used_, pre_stream_));
}

CudaTierBackend::~CudaTierBackend() {
  std::lock_guard lk(mu_);
  fast_.clear();
  for (auto& [id, h] : host_) free_host(h);
  host_.clear();
  for (auto& [k, h] : verified_) free_host(h);
  verified_.clear();
  DeviceGuard g(cfg_.device, /*nothrow=*/true);
  if (pre_stream_) cudaStreamSynchronize(pre_stream_);
  if (pre_raw_) cudaFreeAsync(pre_raw_, pre_stream_);
  if (pre_stream_) cudaStreamSynchronize(pre_stream_);
  if (pre_pool_) cudaMemPoolDestroy(pre_pool_);
  if (pre_stream_) cudaStreamDestroy(pre_stream_);
  if (d2h_stream_) cudaStreamDestroy(d2h_stream_);
  if (pre_t0_) cudaEventDestroy(pre_t0_);
  if (pre_done_) cudaEventDestroy(pre_done_);
  if (pre_used_) cudaEventDestroy(pre_used_);
}

void CudaTierBackend::release_prestage(uint64_t model_id) {
  if (pre_owner_.load() != model_id) return;
  if (pre_raw_) {  // back to the pool once the transform that read it is done (stream-ordered)
    DeviceGuard g(cfg_.device, /*nothrow=*/true);
    cudaStreamWaitEvent(pre_stream_, pre_used_, 0);
    cudaFreeAsync(pre_raw_, pre_stream_);
    pre_raw_ = nullptr;
  }
  pre_rec_.reset();  // a segment placed for an identity stream that was never published
  uint64_t want = model_id;
  pre_owner_.compare_exchange_strong(want, kNoOwner);
}

uint8_t* CudaTierBackend::claim_prestage(uint64_t model_id, const fmt::Manifest& m, uint64_t bytes) {
  uint64_t none = kNoOwner;
  if (!prestage_enabled() || !bytes || !pre_owner_.compare_exchange_strong(none, model_id)) return nullptr;
  try {
    DeviceGuard g(cfg_.device);
    std::shared_ptr<IngestPlan> plan = plan_for(model_id, m);
    if (plan->identity) {
      // The resident blob IS the raw blob: stream it straight into the
      // fast-tier segment (placed now, sealed by publish_fast) -- no second
      // copy of the weights in HBM, no device-to-device pass.
      auto rec = std::make_shared<FastRecord>();
      rec->resident = plan->dst;
      rec->json = plan->dst_json;
      place(*rec, rec->resident.blob_bytes + rec->json.size() + 8);
      pre_rec_ = std::move(rec);
      return pre_rec_->base();
    }
    // A converting plan reads the raw blob from a transient buffer. Its pool
    // parks at most kPrestageKeep bytes between cold opens; larger buffers go
    // back to the driver after the publish (release_prestage).
    const cudaError_t e =
        cudaMallocFromPoolAsync(reinterpret_cast<void**>(&pre_raw_), bytes, pre_pool_, pre_stream_);
    if (e != cudaSuccess) {
      cudaGetLastError();  // out of memory for the overlap buffer: the plain path needs none
      pre_raw_ = nullptr;
      release_prestage(model_id);
      return nullptr;
    }
    return pre_raw_;
  } catch (...) {
    release_prestage(model_id);
    throw;
  }
}

// daemon.cpp:128-136
Located CudaTierBackend::locate(const fmt::ModelKey& key) {
  fs::path p = fs::path(cfg_.disk_cache_dir) / fmt::canonical_filename(key);
  std::error_code ec;
  if (fs::exists(p, ec)) return {Located::Kind::DiskCache, p.string(), uint64_t(fs::file_size(p, ec))};
  if (!cfg_.remote_url.empty()) return {Located::Kind::Remote, "", 0};
  return {Located::Kind::Absent, "", 0};
}

// daemon.cpp:138-142: download into the disk cache (remote.cpp)
FetchResult CudaTierBackend::fetch_remote(const fmt::ModelKey& key) {
  if (cfg_.remote_url.empty()) raise(Errc::RemoteNotFound, fmt::to_string(key));
  std::string p = remote::fetch(remote::make_ref(cfg_.remote_url, key), cfg_.disk_cache_dir);
  std::error_code ec;
  return {p, uint64_t(fs::file_size(p, ec))};
}

// daemon.cpp:144-151. With full_verify the blob is read into pinned memory
// by parallel readers while one thread hashes it in order; the verified bytes
// are kept for this open's stage_host / publish_fast (take_verified).
fmt::Manifest CudaTierBackend::read_manifest(const fmt::ModelKey& key, const std::string& path) {
  fmt::ArtifactInfo a = fmt::read_artifact_info(path, false);
  if (a.manifest.key != key)
    raise(Errc::Corrupt, "artifact at " + path + " holds " + fmt::to_string(a.manifest.key) + ", expected " +
                             fmt::to_string(key));
  if (!cfg_.full_verify) return a.manifest;
  int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) raise(Errc::NotFound, path);
  HostBuf hb;
  const int dfd = direct_fd_for(path, fd, a.blob_offset, a.manifest.blob_bytes);
  if (dfd >= 0) direct_loads_.fetch_add(1);
  try {
    hb = alloc_host(a.manifest.blob_bytes, dfd >= 0 ? a.blob_offset % 4096 : 0, dfd >= 0);
    Sha256 h;
    pipelined_read(fd, a.blob_offset, a.manifest.blob_bytes, hb.p, cfg_.read_threads, &h, {}, false, dfd);
    if (h.finish() != a.manifest.checksum) raise(Errc::ChecksumMismatch, path);
  } catch (...) {
    ::close(fd);
    if (dfd >= 0) ::close(dfd);
    free_host(hb);
    throw;
  }
  ::close(fd);
  if (dfd >= 0) ::close(dfd);
  std::lock_guard lk(mu_);
  auto& slot = verified_[fmt::to_string(key)];
  free_host(slot);  // a stale one from an open that never settled
  slot = hb;
  return a.manifest;
}

CudaTierBackend::HostBuf CudaTierBackend::alloc_host(uint64_t bytes, uint64_t head, bool direct) {
  HostBuf hb;
  hb.bytes = bytes;
  const uint64_t total = std::max<uint64_t>(bytes + head + (head || direct ? 4096 : 0), 1);
  if (pool_) hb.base = pool_->alloc(total);
  hb.pooled = hb.base != nullptr;
  if (!hb.base) {
    DeviceGuard g(cfg_.device);
    TRIMS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hb.base), total, cudaHostAllocPortable));
  }
  hb.p = hb.base + head;
  return hb;
}

// Cold-load read mode for one artifact (cfg_.direct_io): an O_DIRECT fd of
// the same file, or -1 for buffered reads.
int CudaTierBackend::direct_fd_for(const std::string& path, int fd, uint64_t off, uint64_t len) {
  if (cfg_.direct_io == 0) return -1;
  if (cfg_.direct_io == 2 && page_cache_fraction(fd, off, len) > 0.5) return -1;  // mostly cached: buffered
  return ::open(path.c_str(), O_RDONLY | O_CLOEXEC | O_DIRECT);  // -1 where unsupported: buffered
}

bool CudaTierBackend::take_verified(const fmt::ModelKey& key, uint64_t bytes, HostBuf* out) {
  std::lock_guard lk(mu_);
  auto it = verified_.find(fmt::to_string(key));
  if (it == verified_.end()) return false;
  HostBuf hb = it->second;
  verified_.erase(it);
  if (hb.bytes != bytes) {
    free_host(hb);
    return false;
  }
  *out = hb;
  return true;
}

void CudaTierBackend::load_settled(const fmt::ModelKey& key) {
  std::lock_guard lk(mu_);
  auto it = verified_.find(fmt::to_string(key));
  if (it == verified_.end()) return;
  free_host(it->second);
  verified_.erase(it);
}

void CudaTierBackend::free_host(HostBuf& h) {
  if (h.ready) {  // a resident-form D2H may still be writing it
    cudaEventSynchronize(h.ready);
    cudaEventDestroy(h.ready);
    h.ready = nullptr;
  }
  if (!h.base) return;
  if (h.pooled) pool_->free(h.base);
  else cudaFreeHost(h.base);
  h.p = h.base = nullptr;
}

// daemon.cpp:153-158: disk -> host tier, here straight into pinned memory.
void CudaTierBackend::stage_host(uint64_t model_id, const fmt::Manifest& m, const std::string& path) {
  HostBuf hb;
  if (take_verified(m.key, m.blob_bytes, &hb)) {
    // read_manifest already read + verified these bytes: only the upload is left
    uint8_t* target = nullptr;
    try {
      target = claim_prestage(model_id, m, hb.bytes);
    } catch (...) {
      free_host(hb);
      throw;
    }
    if (target) {
      try {
        DeviceGuard g(cfg_.device);
        TRIMS_CUDA(cudaEventRecord(pre_t0_, pre_stream_));
        TRIMS_CUDA(cudaMemcpyAsync(target, hb.p, hb.bytes, cudaMemcpyHostToDevice, pre_stream_));
        TRIMS_CUDA(cudaEventRecord(pre_done_, pre_stream_));
        pre_read_ms_ = 0;
      } catch (...) {
        release_prestage(model_id);
        free_host(hb);
        throw;
      }
    }
  } else {
    int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
    if (fd < 0) raise(Errc::NotFound, path);
    int dfd = -1;
    try {
      uint8_t hdr[16];
      if (::pread(fd, hdr, 16, 0) != 16) raise(Errc::Corrupt, "short read on " + path);
      uint64_t mlen = 0;
      for (int i = 0; i < 8; ++i) mlen |= uint64_t(hdr[8 + i]) << (8 * i);
      const uint64_t off = fmt::blob_file_offset(mlen);
      struct stat st {};
      ::fstat(fd, &st);
      if (uint64_t(st.st_size) < off + m.blob_bytes) raise(Errc::Corrupt, "blob truncated in " + path);
      dfd = direct_fd_for(path, fd, off, m.blob_bytes);
      hb = alloc_host(m.blob_bytes, dfd >= 0 ? off % 4096 : 0, dfd >= 0);
      if (dfd >= 0) direct_loads_.fetch_add(1);
      // verify (daemon.cpp:155 read_model(path, full_verify)) in order under the read + upload
      Sha256 h;
      Sha256* hp = cfg_.full_verify ? &h : nullptr;
      if (uint8_t* target = claim_prestage(model_id, m, hb.bytes)) {
        // Read chunk c into the host tier while chunk c-1 uploads to the
        // device (into the segment itself for an identity plan).
        try {
          DeviceGuard g(cfg_.device);
          auto r0 = std::chrono::steady_clock::now();
          TRIMS_CUDA(cudaEventRecord(pre_t0_, pre_stream_));
          parallel_pread_upload(fd, hb.p, target, hb.bytes, off, cfg_.read_threads, cfg_.device, pre_stream_, hp,
                                dfd);
          TRIMS_CUDA(cudaEventRecord(pre_done_, pre_stream_));
          pre_read_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - r0).count();
        } catch (...) {
          release_prestage(model_id);
          throw;
        }
      } else {
        pipelined_read(fd, off, hb.bytes, hb.p, cfg_.read_threads, hp, {}, false, dfd);
      }
      if (hp && h.finish() != m.checksum) raise(Errc::ChecksumMismatch, path);
    } catch (...) {
      release_prestage(model_id);
      ::close(fd);
      if (dfd >= 0) ::close(dfd);
      free_host(hb);
      throw;
    }
    ::close(fd);
    if (dfd >= 0) ::close(dfd);
  }
  std::lock_guard lk(mu_);
  auto it = host_.find(model_id);
  if (it != host_.end()) free_host(it->second);
  host_[model_id] = hb;
}

const uint8_t* CudaTierBackend::host_buffer(uint64_t model_id, uint64_t* bytes) {
  std::lock_guard lk(mu_);
  auto it = host_.find(model_id);
  if (it == host_.end()) return nullptr;
  if (bytes) *bytes = it->second.bytes;
  return it->second.p;
}

std::shared_ptr<IngestPlan> CudaTierBackend::plan_for(uint64_t model_id, const fmt::Manifest& m) {
  {
    std::lock_guard lk(mu_);
    auto it = plans_.find(model_id);
    if (it != plans_.end()) return it->second;
  }
  auto p = ing_.compile(m, cfg_.plan);
  std::lock_guard lk(mu_);
  return plans_.emplace(model_id, std::move(p)).first->second;
}

std::optional<Calibration> CudaTierBackend::calibrate() {
  using clock = std::chrono::steady_clock;
  auto secs = [](clock::time_point a) { return std::chrono::duration<double>(clock::now() - a).count(); };
  Calibration cal;
  // q: one full sequential read (1 MiB reads) of the largest artifact in the
  // disk cache (daemon.cpp:343-364); nothing >= 1 MiB -> no calibration.
  std::filesystem::path biggest;
  uintmax_t biggest_size = 0;
  std::error_code ec;
  for (const auto& e : std::filesystem::directory_iterator(cfg_.disk_cache_dir, ec)) {
    if (!e.is_regular_file(ec)) continue;
    const uintmax_t sz = e.file_size(ec);
    if (!ec && sz > biggest_size) {
      biggest_size = sz;
      biggest = e.path();
    }
  }
  if (biggest_size < (1u << 20)) return std::nullopt;
  {
    const int fd = ::open(biggest.c_str(), O_RDONLY | O_CLOEXEC);
    if (fd < 0) return std::nullopt;
    std::vector<char> buf(1 << 20);
    const auto t0 = clock::now();
    uint64_t total = 0;
    for (;;) {
      const ssize_t n = ::read(fd, buf.data(), buf.size());
      if (n <= 0) break;
      total += uint64_t(n);
    }
    const double dt = secs(t0);
    ::close(fd);
    if (dt <= 0 || total == 0) return std::nullopt;
    cal.q = double(total) / dt;
  }
  // o and s: medians over 32 export / attach reps of a 64 KiB segment
  // (daemon.cpp:366-385): export = place it in the fast tier and seal its
  // tail; attach = read the sealed tail back and validate it, which is what
  // an importer does per object (trims_import_attach).
  DeviceGuard g(cfg_.device);
  std::vector<double> exports, attaches;
  for (int i = 0; i < 32; ++i) {
    auto rec = std::make_shared<FastRecord>();
    const uint64_t payload = 64 * 1024;
    auto e0 = clock::now();
    place(*rec, payload);
    SegTail t{};
    t.magic = kSegMagic;
    t.generation = rec->generation;
    t.length = payload;
    t.sealed = 1;
    t.device = uint32_t(cfg_.device);
    TRIMS_CUDA(cudaMemcpy(rec->base() + payload, &t, sizeof t, cudaMemcpyHostToDevice));
    exports.push_back(secs(e0));
    auto a0 = clock::now();
    SegTail back{};
    TRIMS_CUDA(cudaMemcpy(&back, rec->base() + payload, sizeof back, cudaMemcpyDeviceToHost));
    if (back.magic != kSegMagic || back.generation != t.generation || !back.sealed)
      raise(Errc::Internal, "calibration segment tail did not read back");
    attaches.push_back(secs(a0));
  }
  auto median = [](std::vector<double>& v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  cal.o = median(exports);
  cal.s = median(attaches);
  return cal;
}

void CudaTierBackend::place(FastRecord& rec, uint64_t payload) {
  auto a0 = std::chrono::steady_clock::now();
  uint64_t off = 0, reserved = 0;
  if (arena_ && arena_->alloc(payload + sizeof(SegTail), &off, &reserved)) {
    rec.arena = arena_;
    rec.offset = off;
    rec.reserved = reserved;
  } else {
    rec.seg = DeviceSegment::create(cfg_.device, payload + sizeof(SegTail));
  }
  rec.stats.alloc_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a0).count();
  rec.generation = next_gen_.fetch_add(1);
}

// Tail: JSON, its length, the sealed SegTail; then the export record.
FastPublication CudaTierBackend::seal(uint64_t model_id, std::shared_ptr<FastRecord> rec, const fmt::Manifest& m) {
  auto s0 = std::chrono::steady_clock::now();
  uint8_t* const base = rec->base();
  const uint64_t rb = rec->resident.blob_bytes;
  const uint64_t payload = rb + rec->json.size() + 8;
  std::vector<uint8_t> tail(rec->json.size() + 8 + sizeof(SegTail));
  std::memcpy(tail.data(), rec->json.data(), rec->json.size());
  uint64_t jlen = rec->json.size();
  for (int i = 0; i < 8; ++i) tail[rec->json.size() + i] = uint8_t(jlen >> (8 * i));
  SegTail t{};
  t.magic = kSegMagic;
  t.generation = rec->generation;
  t.length = payload;
  t.sealed = 1;
  t.device = uint32_t(cfg_.device);
  t.blob_bytes = rb;
  t.checksum = rec->checksum;
  std::memcpy(tail.data() + rec->json.size() + 8, &t, sizeof t);
  {
    DeviceGuard g(cfg_.device);
    TRIMS_CUDA(cudaMemcpy(base + rb, tail.data(), tail.size(), cudaMemcpyHostToDevice));
    TRIMS_CUDA(cudaStreamSynchronize(cudaStreamLegacy));  // sealed before anyone can see the segment
  }

  FastPublication pub;
  ExportedSegment es;
  es.token = "trims." + std::to_string(::getpid()) + "." + std::to_string(rec->generation) + "." + m.key.name;
  es.generation = rec->generation;
  es.length = payload;
  es.device = cfg_.device;
  es.dev_ptr = base;
  es.fd = rec->arena ? rec->arena->fd() : rec->seg.fd();
  es.alloc_bytes = rec->arena ? rec->arena->size() : rec->seg.size();
  es.offset = rec->offset;
  if (rec->arena) es.token = rec->arena->token();
  es.resident_blob_bytes = rb;
  es.ingest_checksum = rec->checksum;
  pub.segments.push_back(es);
  pub.manifest_digest = Sha256::of(rec->json.data(), rec->json.size());
  rec->key = m.key;
  rec->stats.seal_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - s0).count();
  if (cfg_.directory) {
    DirCoords c;
    c.device = cfg_.device;
    c.pid = int32_t(::getpid());
    c.fd = es.fd;
    c.arena = rec->arena ? 1 : 0;
    c.reserved = arena_seq_;  // names the arena (and its lease table) with pid and device
    c.alloc_bytes = es.alloc_bytes;
    c.offset = es.offset;
    c.payload_bytes = payload;
    c.resident_blob_bytes = rb;
    c.generation = rec->generation;
    c.checksum = rec->checksum;
    cfg_.directory->publish(m.key, c);  // only after the tail is sealed
  }
  std::lock_guard lk(mu_);
  fast_[model_id] = std::move(rec);
  return pub;
}

// daemon.cpp:160-209: the fast-tier (HBM) segment holds the RESIDENT blob
// (converted / permuted per the plan), then its JSON manifest and the
// 64-byte SegTail.
FastPublication CudaTierBackend::publish_fast(uint64_t model_id, const fmt::Manifest& m, bool from_host,
                                              const std::string& path) {
  std::shared_ptr<IngestPlan> plan = plan_for(model_id, m);
  const bool staged = from_host && pre_owner_.load() == model_id;
  std::shared_ptr<FastRecord> rec;
  if (staged && pre_rec_) {
    rec = std::move(pre_rec_);  // the identity stream already filled this segment
  } else {
    rec = std::make_shared<FastRecord>();
    rec->resident = plan->dst;
    rec->json = plan->dst_json;
    place(*rec, rec->resident.blob_bytes + rec->json.size() + 8);
  }
  uint8_t* const base = rec->base();
  const double alloc_ms = rec->stats.alloc_ms;

  // Any failure below: wait for queued ingest work before `rec` (and with it
  // the arena range) is released by the unwinding.
  try {
    if (staged) {
      // stage_host already streamed the raw blob to the device: transform only
      // (an identity plan: hash the segment in place -- the fused copy+hash
      // kernel with source == destination rewrites every word with itself)
      const uint8_t* raw = pre_raw_ ? pre_raw_ : base;
      try {
        rec->checksum = ing_.from_staged(*plan, raw, pre_done_, base, &rec->bucket_sums, &rec->stats);
        TRIMS_CUDA(cudaEventRecord(pre_used_, pre_stream_));  // from_staged returned: the reads are done
        float ms = 0;
        TRIMS_CUDA(cudaEventElapsedTime(&ms, pre_t0_, pre_done_));
        rec->stats.h2d_ms = ms;  // overlapped with the file read
        rec->stats.read_ms = pre_read_ms_;
        rec->stats.h2d_bytes = m.blob_bytes;
      } catch (...) {
        ing_.drain();  // no queued kernel may still touch the buffers freed below
        release_prestage(model_id);
        throw;
      }
      release_prestage(model_id);
    } else if (from_host) {
      const uint8_t* src = nullptr;
      bool resident = false;
      cudaEvent_t ready = nullptr;
      {
        std::lock_guard lk(mu_);
        auto it = host_.find(model_id);
        if (it == host_.end()) raise(Errc::Internal, "host buffer missing for publish");
        if (it->second.bytes != m.blob_bytes) raise(Errc::Internal, "host buffer size mismatch");
        src = it->second.p;  // single-flight pins the entry while loading
        resident = it->second.resident;
        ready = it->second.ready;
      }
      if (resident) {
        // The host tier already holds the resident blob: copy it straight into
        // the segment and hash it (the identity plan of the resident manifest).
        if (ready) TRIMS_CUDA(cudaEventSynchronize(ready));
        std::shared_ptr<IngestPlan> ident = pull_plan_for(model_id, rec->resident);
        rec->checksum = ing_.from_host(*ident, src, base, &rec->bucket_sums, &rec->stats);
      } else {
        rec->checksum = ing_.from_host(*plan, src, base, &rec->bucket_sums, &rec->stats);
      }
    } else if (HostBuf vb; take_verified(m.key, m.blob_bytes, &vb)) {
      // host tier skipped under pressure, but read_manifest holds the verified
      // bytes: publish from them instead of reading the file again
      try {
        rec->checksum = ing_.from_host(*plan, vb.p, base, &rec->bucket_sums, &rec->stats);
      } catch (...) {
        free_host(vb);
        throw;
      }
      free_host(vb);
    } else {
      int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
      if (fd < 0) raise(Errc::NotFound, path);
      try {
        uint8_t hdr[16];
        if (::pread(fd, hdr, 16, 0) != 16) raise(Errc::Corrupt, "short read on " + path);
        uint64_t mlen = 0;
        for (int i = 0; i < 8; ++i) mlen |= uint64_t(hdr[8 + i]) << (8 * i);
        rec->checksum = ing_.from_file(*plan, fd, fmt::blob_file_offset(mlen), base, &rec->bucket_sums,
                                       &rec->stats);
      } catch (...) {
        ::close(fd);
        throw;
      }
      ::close(fd);
    }
  } catch (...) {
    ing_.drain();
    throw;
  }
  rec->stats.alloc_ms = alloc_ms;
  if (cfg_.resident_host_tier && !plan->identity) to_resident_form(model_id, *rec, *plan);
  return seal(model_id, std::move(rec), m);
}

// Replace a staged raw host copy with the resident blob just published
// (async D2H on its own stream; evictions of either tier wait for it).
void CudaTierBackend::to_resident_form(uint64_t model_id, const FastRecord& rec, const IngestPlan& plan) {
  std::lock_guard lk(mu_);
  auto it = host_.find(model_id);
  if (it == host_.end() || it->second.resident || rec.resident.blob_bytes > it->second.bytes) return;
  HostBuf& hb = it->second;
  DeviceGuard g(cfg_.device);
  if (!hb.ready) TRIMS_CUDA(cudaEventCreateWithFlags(&hb.ready, cudaEventDisableTiming));
  TRIMS_CUDA(cudaMemcpyAsync(hb.p, rec.base(), rec.resident.blob_bytes, cudaMemcpyDeviceToHost, d2h_stream_));
  TRIMS_CUDA(cudaEventRecord(hb.ready, d2h_stream_));
  hb.resident = true;
  (void)plan;
}

// Multi-GPU extension: fill this GPU's fast tier from a peer's
// sealed segment. One fused kernel pulls the resident blob over NVLink and
// hashes it; the peer's tail must show the same sealed generation before and
// after the pull (a seqlock: an eviction scrubs the tail before the range can
// be reused), and the pulled checksum must equal the one the peer sealed.
FastPublication CudaTierBackend::publish_from_peer(uint64_t model_id, const fmt::Manifest& m, const PeerSource& src) {
  auto rec = std::make_shared<FastRecord>();
  std::shared_ptr<IngestPlan> plan = plan_for(model_id, m);
  rec->resident = plan->dst;
  rec->json = plan->dst_json;
  const uint64_t rb = rec->resident.blob_bytes;
  const uint64_t payload = rb + rec->json.size() + 8;
  if (!src.payload || src.resident_blob_bytes != rb || src.payload_bytes != payload)
    raise(Errc::InvalidArgument, "peer segment of " + fmt::to_string(m.key) + " has a different resident layout " +
                                     "(stores must share the ingest plan)");
  DeviceGuard g(cfg_.device);
  auto read_tail = [&](std::string* json) {
    SegTail t{};
    TRIMS_CUDA(cudaMemcpy(&t, src.payload + payload, sizeof t, cudaMemcpyDefault));
    if (t.magic != kSegMagic || !t.sealed || t.generation != src.generation || t.length != payload ||
        t.blob_bytes != rb)
      raise(Errc::StaleGeneration, "peer segment of " + fmt::to_string(m.key) + " changed (generation " +
                                       std::to_string(src.generation) + ")");
    if (json) {
      json->resize(rec->json.size());
      TRIMS_CUDA(cudaMemcpy(json->data(), src.payload + rb, json->size(), cudaMemcpyDefault));
    }
  };
  std::string peer_json;
  read_tail(&peer_json);
  if (peer_json != rec->json) raise(Errc::InvalidArgument, "peer resident manifest differs (plan mismatch)");
  place(*rec, payload);
  std::shared_ptr<IngestPlan> ident = pull_plan_for(model_id, rec->resident);
  try {
    rec->checksum = ing_.pull(*ident, src.payload, rec->base(), &rec->bucket_sums, &rec->stats);
  } catch (...) {
    ing_.drain();  // the pull may still be writing the range `rec` releases
    throw;
  }
  read_tail(nullptr);
  if (rec->checksum != src.checksum)
    raise(Errc::ChecksumMismatch, "peer pull of " + fmt::to_string(m.key) + ": checksum " +
                                      std::to_string(rec->checksum) + " != sealed " + std::to_string(src.checksum));
  return seal(model_id, std::move(rec), m);
}

std::shared_ptr<IngestPlan> CudaTierBackend::pull_plan_for(uint64_t model_id, const fmt::Manifest& resident) {
  {
    std::lock_guard lk(mu_);
    auto it = pull_plans_.find(model_id);
    if (it != pull_plans_.end()) return it->second;
  }
  std::shared_ptr<IngestPlan> p = ing_.compile(resident, fmt::Plan{});
  std::lock_guard lk(mu_);
  return pull_plans_.emplace(model_id, std::move(p)).first->second;
}

void CudaTierBackend::evict_fast(uint64_t model_id) {
  std::shared_ptr<FastRecord> victim;
  {
    std::lock_guard lk(mu_);
    auto it = fast_.find(model_id);
    if (it == fast_.end()) return;
    victim = std::move(it->second);
    fast_.erase(it);
  }
  {
    std::lock_guard lk(mu_);  // a resident-form D2H may still be reading the segment
    auto h = host_.find(model_id);
    if (h != host_.end() && h->second.ready) cudaEventSynchronize(h->second.ready);
  }
  if (cfg_.directory) cfg_.directory->retract(victim->key);  // before the scrub: peers stop choosing it
  if (victim->arena) {
    // The range returns to the arena: scrub the sealed tail so an importer
    // holding the old (offset, generation) can never validate it again, even
    // when the next occupant is shorter and leaves these bytes untouched.
    DeviceGuard g(cfg_.device, /*nothrow=*/true);
    const uint64_t payload = victim->resident.blob_bytes + victim->json.size() + 8;
    cudaMemset(victim->base() + payload, 0, sizeof(SegTail));
    cudaStreamSynchronize(cudaStreamLegacy);  // scrubbed before the range can be reallocated
  }
  // A dedicated segment's physical memory lives on in importers' mappings.
}

void CudaTierBackend::evict_host(uint64_t model_id) {
  release_prestage(model_id);
  std::lock_guard lk(mu_);
  auto it = host_.find(model_id);
  if (it == host_.end()) return;
  free_host(it->second);
  host_.erase(it);
}

void CudaTierBackend::evict_disk(const fmt::ModelKey&, const std::string& path) {
  std::error_code ec;
  fs::remove(path, ec);
}

std::shared_ptr<FastRecord> CudaTierBackend::fast_record(uint64_t model_id) {
  std::lock_guard lk(mu_);
  auto it = fast_.find(model_id);
  return it == fast_.end() ? nullptr : it->second;
}

}  // namespace trims
