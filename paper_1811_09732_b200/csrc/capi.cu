// capi.cu — the extern "C" boundary (include/trims.h). Every entry point
// converts exceptions to reference Errc codes; nothing C++ crosses the ABI.
#include <dirent.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <filesystem>
#include <map>
#include <memory>
#include <sstream>
#include <thread>

#include "../../include/trims.h"
#include "backend.hpp"
#include "cache_core.hpp"
#include "cuda_util.hpp"
#include "directory.hpp"
#include "format.hpp"
#include "gemm.hpp"
#include "nn.hpp"
#include "remote.hpp"
#include "sha256.hpp"
#include "store_api.hpp"

using namespace trims;

namespace {

thread_local std::string g_last_error;

std::string f64(double v) {  // round-trippable JSON number
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

template <class F>
int guard(F&& f) {
  try {
    g_last_error.clear();
    return f();
  } catch (const Error& e) {
    g_last_error = e.what();
    return int(e.code());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return int(Errc::Internal);
  } catch (...) {
    g_last_error = "unknown exception";
    return int(Errc::Internal);
  }
}

int put(const std::string& s, char* out, uint64_t cap) {
  if (!out || s.size() + 1 > cap) {
    g_last_error = "output buffer too small (need " + std::to_string(s.size() + 1) + ")";
    return int(Errc::InvalidArgument);
  }
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = '\0';
  return 0;
}

std::vector<fmt::TensorDecl> parse_decls(const char* text) {
  std::vector<fmt::TensorDecl> out;
  std::istringstream is(text ? text : "");
  std::string line;
  while (std::getline(is, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string name, dt, dims;
    ls >> name >> dt >> dims;
    auto t = fmt::dtype_from_name(dt);
    if (!t) raise(Errc::InvalidArgument, "dtype " + dt);
    fmt::TensorDecl d{name, {}, *t};
    size_t pos = 0;
    while (pos < dims.size()) {
      size_t c = dims.find(',', pos);
      if (c == std::string::npos) c = dims.size();
      d.dims.push_back(std::stoull(dims.substr(pos, c - pos)));
      pos = c + 1;
    }
    out.push_back(std::move(d));
  }
  return out;
}

fmt::Plan make_plan(uint32_t flags, uint32_t out_dtype) {
  fmt::Plan p;
  p.convert = flags & TRIMS_PLAN_CONVERT;
  p.permute_4d = flags & TRIMS_PLAN_PERMUTE_4D;
  if (out_dtype > 4) raise(Errc::InvalidArgument, "out_dtype");
  p.out_dtype = fmt::DType(out_dtype);
  return p;
}

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <class F>
void parallel_for(uint64_t n, F&& f) {
  unsigned t = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < (1u << 20)) t = 1;
  std::vector<std::thread> ts;
  uint64_t piece = (n + t - 1) / t;
  for (unsigned i = 1; i < t; ++i) {
    uint64_t b = std::min(n, i * piece), e = std::min(n, (i + 1) * piece);
    ts.emplace_back([&, b, e] { f(b, e); });
  }
  f(0, std::min(n, piece));
  for (auto& x : ts) x.join();
}

}  // namespace

// Serving in place across GPUs (StoreOptions.peer_serve = "map"): an open
// of a model held by a peer rank borrows the peer's sealed segment -- mapped
// read-only for this store's device, its range leased in the holder's lease
// table (a freed range stays retired until the lease goes) -- instead of
// copying it into this store's fast tier. No local admission: the aggregate
// fast-tier capacity of N stores holds N x capacity distinct bytes.
namespace trims {
struct PeerMapHold {
  fmt::ModelKey key;
  std::shared_ptr<Import> map;
  std::shared_ptr<LeaseTable> table;
  int row{-1};
  uint64_t offset{0}, generation{0};
  std::string json;
  ~PeerMapHold() {
    if (table && row >= 0) table->release(row, offset, generation);
  }
};
constexpr uint64_t kPeerMapIdBit = 1ull << 62;  // model ids of peer-mapped opens
}  // namespace trims

struct trims_store {
  std::unique_ptr<CudaTierBackend> be;
  std::unique_ptr<CacheCore> core;
  std::atomic<uint64_t> clock{0};
  // multi-GPU
  std::shared_ptr<Directory> dir;
  // DaemonConfig::workspace_headroom_fraction (daemon.hpp:29) and the startup
  // calibration published in StatsResponse (daemon.cpp:535-539)
  double workspace_headroom{0.25};
  std::optional<Calibration> calibration;
  PeerCounters peers;
  bool peer_map{false};
  std::mutex pm_mu;
  std::map<uint64_t, std::shared_ptr<PeerMapHold>> peer_maps;  // open peer-mapped views by id
  uint64_t next_pm{1};
  std::atomic<uint64_t> peer_maps_total{0};
  std::mutex peer_mu;
  std::map<std::tuple<int, int, uint64_t>, std::shared_ptr<Import>> peer_arenas;  // (pid, fd, bytes) -> mapping
  std::map<fmt::ModelKey, std::shared_ptr<const fmt::Manifest>> manifests;

  // The peer path needs the artifact's manifest from this store's own disk
  // cache (same rule as oracle/simulator.py simulate_cluster); parsed once.
  std::shared_ptr<const fmt::Manifest> manifest_for(const fmt::ModelKey& key) {
    Located l = be->locate(key);
    if (l.kind != Located::Kind::DiskCache) return nullptr;
    {
      std::lock_guard lk(peer_mu);
      auto it = manifests.find(key);
      if (it != manifests.end()) return it->second;
    }
    // The manifest only (no full_verify pass over the blob): a PeerHit never
    // reads the local artifact's bytes, and the pulled copy is checked
    // against the holder's sealed checksum instead.
    fmt::ArtifactInfo a = fmt::read_artifact_info(l.path, false);
    if (a.manifest.key != key) raise(Errc::Corrupt, "artifact at " + l.path + " holds " + fmt::to_string(a.manifest.key));
    auto m = std::make_shared<const fmt::Manifest>(std::move(a.manifest));
    std::lock_guard lk(peer_mu);
    return manifests.emplace(key, std::move(m)).first->second;
  }

  // Map a peer's exportable allocation into this process with read access for
  // this store's device: the fd is taken from the owner with pidfd_getfd.
  std::shared_ptr<Import> map_peer(const DirCoords& c) {
    const auto k = std::make_tuple(c.pid, c.fd, c.alloc_bytes);
    if (c.arena) {
      std::lock_guard lk(peer_mu);
      auto it = peer_arenas.find(k);
      if (it != peer_arenas.end()) return it->second;
    }
    const int pidfd = int(::syscall(SYS_pidfd_open, c.pid, 0));
    if (pidfd < 0) raise(Errc::NoSuchSegment, "peer rank " + std::to_string(c.rank) + " (pid " + std::to_string(c.pid) + ") is gone");
    const int fd = int(::syscall(SYS_pidfd_getfd, pidfd, c.fd, 0));
    const int err = errno;
    ::close(pidfd);
    if (fd < 0) raise(Errc::NoSuchSegment, "pidfd_getfd from rank " + std::to_string(c.rank) + ": " + std::strerror(err));
    std::shared_ptr<Import> imp;
    try {
      imp.reset(Import::open(be->config().device, fd, c.alloc_bytes, /*read_only=*/true));
    } catch (...) {
      ::close(fd);
      throw;
    }
    ::close(fd);
    if (c.arena) {
      std::lock_guard lk(peer_mu);
      peer_arenas.emplace(k, imp);
    }
    return imp;
  }

  PlacementResult open(const fmt::ModelKey& key, const Granularity& g, uint64_t now, int* peer_rank) {
    return open_with_peers(
        *core, dir.get(), key, g, now, [this](const fmt::ModelKey& k) { return manifest_for(k); },
        [this](const DirCoords& c, std::shared_ptr<void>* hold) {
          std::shared_ptr<Import> imp = map_peer(c);
          *hold = imp;
          PeerSource src;
          src.rank = c.rank;
          src.device = c.device;
          src.payload = imp->ptr() + c.offset;
          src.payload_bytes = c.payload_bytes;
          src.resident_blob_bytes = c.resident_blob_bytes;
          src.generation = c.generation;
          src.checksum = c.checksum;
          if (c.offset + c.payload_bytes + sizeof(SegTail) > imp->size())
            raise(Errc::NoSuchSegment, "peer segment outside its allocation");
          return src;
        },
        &peers, peer_rank);
  }
};

struct trims_dir {
  std::unique_ptr<Directory> d;
};

struct trims_import {
  std::unique_ptr<Import> map;
  int device{0};
};

// In-process view lifetime: holds the published record, so its arena range
// is neither freed nor reused while the view may be read.
struct trims_pin {
  std::shared_ptr<FastRecord> rec;
  std::shared_ptr<PeerMapHold> peer;  // a peer-mapped view: its lease
};

// Cross-process view lifetime: one row of the owner's lease table.
struct trims_lease {
  std::shared_ptr<LeaseTable> table;
  int row{-1};
  uint64_t offset{0}, generation{0};
};

extern "C" {

const char* trims_errc_name(int code) { return errc_name(Errc(code)); }
int trims_wire_code(int code) { return int(wire_code(Errc(code))); }
const char* trims_last_error(void) { return g_last_error.c_str(); }

int trims_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int trims_device_init(int device) {
  return guard([&] {
    if (device < 0 || device >= trims_device_count()) raise(Errc::NoDevice, "no CUDA device " + std::to_string(device));
    TRIMS_CUDA(cudaSetDevice(device));
    TRIMS_CUDA(cudaFree(nullptr));  // creates the primary context now, not inside the first open
    return 0;
  });
}

int trims_sha_hw(void) { return Sha256::hw_accelerated() ? 1 : 0; }

int trims_sha256(const void* data, uint64_t n, uint8_t out[32]) {
  return guard([&] {
    auto d = Sha256::of(data, n);
    std::memcpy(out, d.data(), 32);
    return 0;
  });
}

int trims_read_manifest(const char* path, int full_verify, char* json_out, uint64_t cap, uint8_t checksum_out[32],
                        uint64_t* blob_bytes, uint64_t* blob_file_offset) {
  return guard([&] {
    fmt::ArtifactInfo a = fmt::read_artifact_info(path, full_verify != 0);
    if (checksum_out) std::memcpy(checksum_out, a.manifest.checksum.data(), 32);
    if (blob_bytes) *blob_bytes = a.manifest.blob_bytes;
    if (blob_file_offset) *blob_file_offset = a.blob_offset;
    return json_out ? put(fmt::manifest_to_json(a.manifest), json_out, cap) : 0;
  });
}

int trims_manifest_canonical(const char* json_in, char* json_out, uint64_t cap) {
  return guard([&] { return put(fmt::manifest_to_json(fmt::manifest_from_json(json_in)), json_out, cap); });
}

int trims_make_manifest(const char* ns, const char* name, const char* version, const char* decls,
                        uint64_t workspace_bytes, char* json_out, uint64_t cap) {
  return guard([&] {
    fmt::Manifest m = fmt::make_manifest({ns, name, version}, parse_decls(decls), workspace_bytes);
    return put(fmt::manifest_to_json(m), json_out, cap);
  });
}

int trims_write_model(const char* path, const char* manifest_json, const void* blob) {
  return guard([&] {
    fmt::Manifest m = fmt::manifest_from_json(manifest_json);
    static const uint8_t empty = 0;
    fmt::write_artifact(path, m, blob ? static_cast<const uint8_t*>(blob) : &empty);
    return 0;
  });
}

int trims_layout_for(const char* manifest_json, uint32_t kind, uint64_t block_bytes, char* out, uint64_t cap) {
  return guard([&] {
    if (kind > 2) raise(Errc::InvalidArgument, "granularity kind");
    fmt::Manifest m = fmt::manifest_from_json(manifest_json);
    std::ostringstream os;
    for (const auto& o : layout_for(m, {GranKind(kind), block_bytes}))
      os << o.name << ' ' << o.segment_index << ' ' << o.offset << ' ' << o.length << '\n';
    return put(os.str(), out, cap);
  });
}

int trims_resident_manifest(const char* src_json, uint32_t plan_flags, uint32_t out_dtype, char* json_out,
                            uint64_t cap) {
  return guard([&] {
    fmt::Manifest m = fmt::manifest_from_json(src_json);
    return put(fmt::manifest_to_json(fmt::resident_manifest(m, make_plan(plan_flags, out_dtype))), json_out, cap);
  });
}

int trims_fill_splitmix_host(uint64_t* dst, uint64_t n, uint64_t stream_seed, uint64_t k0) {
  return guard([&] {
    parallel_for(n, [&](uint64_t b, uint64_t e) {
      for (uint64_t j = b; j < e; ++j) dst[j] = mix64(stream_seed + (k0 + j + 1) * 0x9e3779b97f4a7c15ull);
    });
    return 0;
  });
}

int trims_fill_uniform_host(float* dst, uint64_t n, uint64_t stream_seed, uint64_t j0, float lo, float hi) {
  return guard([&] {
    const float span = hi - lo;
    parallel_for(n, [&](uint64_t b, uint64_t e) {
      for (uint64_t j = b; j < e; ++j) {
        float u = float(mix64(stream_seed + (j0 + j + 1) * 0x9e3779b97f4a7c15ull) >> 40) * 0x1p-24f;
        dst[j] = std::fma(span, u, lo);
      }
    });
    return 0;
  });
}

uint64_t trims_fnv1a(const char* s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= uint8_t(*s);
    h *= 0x100000001b3ull;
  }
  return h;
}

int trims_touch_host(const void* blob, const char* manifest_json, uint64_t* out) {
  return guard([&] {
    fmt::Manifest m = fmt::manifest_from_json(manifest_json);
    const uint8_t* base = static_cast<const uint8_t*>(blob);
    uint64_t h = 0xcbf29ce484222325ull;
    for (const auto& t : m.tensors) {
      const uint8_t* p = base + t.offset;
      uint64_t words = t.nbytes / 8;
      for (uint64_t i = 0; i < words; ++i) {
        uint64_t w;
        std::memcpy(&w, p + 8 * i, 8);
        h = (h ^ w) * 0x100000001b3ull;
      }
      for (uint64_t i = words * 8; i < t.nbytes; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
    }
    *out = h;
    return 0;
  });
}

int trims_checksum_host(const void* p, uint64_t n, uint64_t word0, uint64_t* out) {
  return guard([&] {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    const uint64_t words = (n + 7) / 8;
    std::atomic<uint64_t> total{0};
    parallel_for(words, [&](uint64_t s, uint64_t e) {
      uint64_t acc = 0;
      for (uint64_t i = s; i < e; ++i) {
        uint64_t w = 0;
        std::memcpy(&w, b + 8 * i, std::min<uint64_t>(8, n - 8 * i));
        acc += ingest::checksum_term(w, word0 + i);
      }
      total.fetch_add(acc);
    });
    *out = total.load();
    return 0;
  });
}

// ---------------------------------------------------------------- store

namespace {
// DaemonConfig validation (daemon.cpp:26-36) + the B200 backend settings.
BackendConfig backend_config(const trims_store_config* cfg) {
  if (!cfg) raise(Errc::InvalidArgument, "null argument");
  if (!cfg->fast_capacity_bytes || !cfg->host_capacity_bytes || !cfg->disk_capacity_bytes)
    raise(Errc::InvalidArgument, "capacities must be > 0");
  if (!cfg->disk_cache_dir || !*cfg->disk_cache_dir) raise(Errc::InvalidArgument, "disk_cache_dir must be set");
  if (trims_device_count() <= cfg->device) raise(Errc::NoDevice, "no CUDA device " + std::to_string(cfg->device));
  std::filesystem::create_directories(cfg->disk_cache_dir);
  BackendConfig bc;
  bc.device = cfg->device;
  bc.disk_cache_dir = cfg->disk_cache_dir;
  bc.full_verify = cfg->full_verify != 0;
  if (cfg->remote_url) bc.remote_url = cfg->remote_url;
  bc.plan = make_plan(cfg->plan_flags, cfg->out_dtype);
  bc.pinned_pool_bytes = cfg->pinned_pool_bytes ? cfg->pinned_pool_bytes : cfg->host_capacity_bytes;
  bc.read_threads = cfg->read_threads ? cfg->read_threads : 8;
  bc.direct_io = int(cfg->direct_io);
  if (const char* e = std::getenv("TRIMS_DIRECT_IO")) bc.direct_io = std::atoi(e);  // A/B override
  // arena: 0 = auto (capacity + 1/16 + 64 MiB for per-segment rounding and tails), 1 = off
  bc.arena_bytes = cfg->arena_bytes == 1 ? 0
                   : cfg->arena_bytes ? cfg->arena_bytes
                                      : cfg->fast_capacity_bytes + cfg->fast_capacity_bytes / 16 + (64ull << 20);
  bc.resident_host_tier = cfg->eager_reclaim == 0;
  return bc;
}

void fill_export(const ExportedSegment& es, trims_export* out) {
  out->device = es.device;
  out->generation = es.generation;
  out->payload_bytes = es.length;
  out->resident_blob_bytes = es.resident_blob_bytes;
  out->alloc_bytes = es.alloc_bytes;
  out->ingest_checksum = es.ingest_checksum;
  out->dev_ptr = es.dev_ptr;
  out->fd = es.fd;
  out->segment_offset = es.offset;
  std::snprintf(out->token, sizeof out->token, "%s", es.token.c_str());
}
}  // namespace

struct trims_backend {
  std::unique_ptr<CudaTierBackend> be;
};

int trims_backend_create(const trims_store_config* cfg, trims_backend** out) {
  return guard([&] {
    auto b = std::make_unique<trims_backend>();
    b->be = std::make_unique<CudaTierBackend>(backend_config(cfg));
    *out = b.release();
    return 0;
  });
}

void trims_backend_destroy(trims_backend* b) {
  try {
    delete b;
  } catch (...) {
  }
}

int trims_backend_locate(trims_backend* b, const char* ns, const char* name, const char* version, char* path_out,
                         uint64_t cap, uint64_t* file_bytes) {
  return guard([&] {
    Located l = b->be->locate({ns, name, version});
    if (l.kind == Located::Kind::Absent) raise(Errc::NotFound, std::string(ns) + "/" + name + "@" + version);
    if (file_bytes) *file_bytes = l.file_bytes;
    return put(l.path, path_out, cap);
  });
}

int trims_backend_fetch_remote(trims_backend* b, const char* ns, const char* name, const char* version,
                               char* path_out, uint64_t cap, uint64_t* file_bytes) {
  return guard([&] {
    FetchResult f = b->be->fetch_remote({ns, name, version});
    if (file_bytes) *file_bytes = f.file_bytes;
    return put(f.path, path_out, cap);
  });
}

int trims_backend_load_settled(trims_backend* b, const char* ns, const char* name, const char* version) {
  return guard([&] {
    b->be->load_settled({ns, name, version});
    return 0;
  });
}

int trims_remote_fetch(const char* url, const char* ns, const char* name, const char* version, const char* dest_dir,
                       char* path_out, uint64_t cap, uint64_t* file_bytes) {
  return guard([&] {
    if (!url || !dest_dir) raise(Errc::InvalidArgument, "null argument");
    std::string p = remote::fetch(remote::make_ref(url, {ns, name, version}), dest_dir);
    std::error_code ec;
    if (file_bytes) *file_bytes = uint64_t(std::filesystem::file_size(p, ec));
    return put(p, path_out, cap);
  });
}

int trims_backend_read_manifest(trims_backend* b, const char* ns, const char* name, const char* version,
                                const char* path, char* json_out, uint64_t cap, uint8_t checksum_out[32]) {
  return guard([&] {
    fmt::Manifest m = b->be->read_manifest({ns, name, version}, path);
    if (checksum_out) std::memcpy(checksum_out, m.checksum.data(), 32);
    return put(fmt::manifest_to_json(m), json_out, cap);
  });
}

int trims_backend_stage_host(trims_backend* b, uint64_t model_id, const char* manifest_json,
                             const uint8_t checksum[32], const char* path) {
  return guard([&] {
    fmt::Manifest m = fmt::manifest_from_json(manifest_json);
    if (checksum) std::memcpy(m.checksum.data(), checksum, 32);
    b->be->stage_host(model_id, m, path);
    return 0;
  });
}

int trims_backend_publish_fast(trims_backend* b, uint64_t model_id, const char* manifest_json, int from_host,
                               const char* path, trims_export* out) {
  return guard([&] {
    FastPublication pub = b->be->publish_fast(model_id, fmt::manifest_from_json(manifest_json), from_host != 0,
                                              path ? path : "");
    std::memset(out, 0, sizeof *out);
    out->model_id = model_id;
    out->outcome = TRIMS_DISK_LOAD;
    std::memcpy(out->manifest_digest, pub.manifest_digest.data(), 32);
    fill_export(pub.segments.at(0), out);
    out->n_objects = 1;
    return 0;
  });
}

int trims_backend_evict_fast(trims_backend* b, uint64_t model_id) {
  return guard([&] {
    b->be->evict_fast(model_id);
    return 0;
  });
}

int trims_backend_evict_host(trims_backend* b, uint64_t model_id) {
  return guard([&] {
    b->be->evict_host(model_id);
    return 0;
  });
}

int trims_backend_evict_disk(trims_backend* b, const char* path) {
  return guard([&] {
    b->be->evict_disk({}, path);
    return 0;
  });
}

int trims_store_create(const trims_store_config* cfg, trims_store** out) {
  return guard([&] {
    if (!out) raise(Errc::InvalidArgument, "null argument");
    auto s = std::make_unique<trims_store>();
    BackendConfig bc = backend_config(cfg);
    if (cfg->directory && *cfg->directory) {
      s->dir = Directory::open(cfg->directory, cfg->world, cfg->rank,
                               cfg->directory_slots ? cfg->directory_slots : 1024);
      bc.directory = s->dir;
    }
    // validate_config (daemon.cpp): the headroom is a fraction
    if (!(cfg->workspace_headroom_fraction >= 0.0 && cfg->workspace_headroom_fraction <= 1.0))
      raise(Errc::InvalidArgument, "workspace_headroom_fraction must be in [0, 1]");
    s->workspace_headroom = cfg->workspace_headroom_fraction;
    s->be = std::make_unique<CudaTierBackend>(std::move(bc));
    CoreConfig cc{cfg->fast_capacity_bytes, cfg->host_capacity_bytes, cfg->disk_capacity_bytes,
                  Policy(cfg->policy ? 1 : 0), cfg->eager_reclaim != 0};
    s->core = std::make_unique<CacheCore>(cc, *s->be);
    if (cfg->scan_disk) {  // daemon.cpp:314-325: name-sorted for deterministic seq numbers
      std::vector<std::filesystem::path> files;
      for (const auto& e : std::filesystem::directory_iterator(cfg->disk_cache_dir))
        if (e.is_regular_file()) files.push_back(e.path());
      std::sort(files.begin(), files.end());
      for (const auto& p : files) {
        auto key = fmt::key_from_filename(p.filename().string());
        if (key) s->core->register_disk_file(*key, p.string(), std::filesystem::file_size(p));
      }
    }
    if (cfg->startup_calibration) s->calibration = s->be->calibrate();  // daemon.cpp:334
    s->peer_map = cfg->peer_map != 0 && s->dir != nullptr;
    *out = s.release();
    return 0;
  });
}

void trims_store_destroy(trims_store* s) {
  if (!s) return;
  try {
    s->core->drop_all();
  } catch (...) {
  }
  delete s;
}

}  // extern "C"

namespace {
SegTail read_tail_of(const Import& map, int device, uint64_t offset, uint64_t generation, uint64_t payload_bytes,
                     std::string* json) {
  if (payload_bytes < 8 || offset + payload_bytes + sizeof(SegTail) > map.size())
    raise(Errc::NoSuchSegment, "segment outside the mapped allocation");
  DeviceGuard g(device);
  uint8_t tail[8 + sizeof(SegTail)];
  TRIMS_CUDA(cudaMemcpy(tail, map.ptr() + offset + payload_bytes - 8, sizeof tail, cudaMemcpyDeviceToHost));
  uint64_t jlen = 0;
  for (int i = 0; i < 8; ++i) jlen |= uint64_t(tail[i]) << (8 * i);
  SegTail st;
  std::memcpy(&st, tail + 8, sizeof st);
  if (st.magic != kSegMagic) raise(Errc::NoSuchSegment, "bad segment tail");
  if (st.generation != generation)
    raise(Errc::StaleGeneration, "generation " + std::to_string(st.generation) + " != " + std::to_string(generation));
  if (!st.sealed) raise(Errc::NotSealed, "segment not sealed");
  if (st.length != payload_bytes || jlen + 8 > payload_bytes || st.blob_bytes + jlen + 8 != payload_bytes)
    raise(Errc::Corrupt, "segment length mismatch");
  if (json) {
    json->resize(jlen);
    TRIMS_CUDA(cudaMemcpy(json->data(), map.ptr() + offset + payload_bytes - 8 - jlen, jlen, cudaMemcpyDeviceToHost));
  }
  return st;
}


// Serve an open in place from a peer rank's sealed segment (peer_serve = map):
// best holder first; a holder whose copy is gone, stale or not an arena is
// skipped. Returns false when no peer serves it (the caller opens normally).
bool open_peer_mapped(trims_store* s, const fmt::ModelKey& key, uint32_t gran_kind, uint64_t block_bytes,
                      trims_export* out) {
  for (const DirCoords& c : s->dir->holders(key)) {
    if (!c.arena) continue;
    auto hold = std::make_shared<PeerMapHold>();
    try {
      hold->map = s->map_peer(c);
      const std::string token = "trims." + std::to_string(c.pid) + ".arena" + std::to_string(c.device) + "." +
                                std::to_string(c.reserved);
      hold->table = LeaseTable::open(token);
      if (!hold->table) continue;
      hold->row = hold->table->acquire(c.offset, c.generation);
      hold->offset = c.offset;
      hold->generation = c.generation;
      // leased first, then checked: a range the holder freed before the lease
      // shows a scrubbed or newer tail here and is skipped
      SegTail st = read_tail_of(*hold->map, s->be->config().device, c.offset, c.generation, c.payload_bytes,
                                &hold->json);
      fmt::Manifest m = fmt::manifest_from_json(hold->json);
      if (m.key != key) raise(Errc::NoSuchSegment, "peer segment holds another model");
      hold->key = key;
      std::memset(out, 0, sizeof *out);
      {
        std::lock_guard lk(s->pm_mu);
        out->model_id = kPeerMapIdBit | s->next_pm++;
        s->peer_maps[out->model_id] = hold;
      }
      s->peer_maps_total.fetch_add(1);
      out->outcome = TRIMS_PEER_MAP;
      out->device = s->be->config().device;
      out->generation = c.generation;
      out->payload_bytes = c.payload_bytes;
      out->resident_blob_bytes = st.blob_bytes;
      out->alloc_bytes = c.alloc_bytes;
      uint64_t w = 0;
      for (const auto& t : m.tensors) w += t.nbytes;
      out->weights_bytes = w;
      out->workspace_bytes = m.workspace_bytes;
      out->ingest_checksum = st.checksum;
      auto d = Sha256::of(hold->json.data(), hold->json.size());
      std::memcpy(out->manifest_digest, d.data(), 32);
      out->dev_ptr = hold->map->ptr() + c.offset;
      out->fd = -1;
      out->segment_offset = c.offset;
      std::snprintf(out->token, sizeof out->token, "%s", token.c_str());
      if (st.blob_bytes == 0 || gran_kind == 0) out->n_objects = 1;
      else if (gran_kind == 1) out->n_objects = uint32_t(m.tensors.size());
      else out->n_objects = uint32_t((st.blob_bytes + block_bytes - 1) / block_bytes);
      return true;
    } catch (const Error&) {
      s->peers.fallbacks.fetch_add(1);  // this holder's copy is gone / stale: try the next
    }
  }
  return false;
}
}  // namespace

extern "C" {

int trims_store_open(trims_store* s, const char* ns, const char* name, const char* version, uint32_t gran_kind,
                     uint64_t block_bytes, trims_export* out) {
  return guard([&] {
    if (gran_kind > 2) raise(Errc::InvalidArgument, "granularity kind");
    if (s->peer_map && s->dir && !s->core->fast_resident({ns, name, version}) &&
        open_peer_mapped(s, {ns, name, version}, gran_kind, block_bytes, out))
      return 0;
    uint64_t now = s->clock.fetch_add(1) + 1;  // daemon.cpp:457
    PlacementResult r = s->open({ns, name, version}, {GranKind(gran_kind), block_bytes}, now, nullptr);
    std::memset(out, 0, sizeof *out);
    out->model_id = r.model_id;
    out->outcome = uint32_t(r.outcome);
    out->weights_bytes = r.weights_bytes;
    out->workspace_bytes = r.workspace_bytes;
    out->timings_ns[0] = r.timings.fetch_ns;
    out->timings_ns[1] = r.timings.disk_read_ns;
    out->timings_ns[2] = r.timings.host_to_fast_copy_ns;
    out->timings_ns[3] = r.timings.handle_export_ns;
    std::memcpy(out->manifest_digest, r.manifest_digest.data(), 32);
    out->fd = -1;
    if (!r.segments.empty()) fill_export(r.segments[0], out);
    // objects of the resident blob at the requested granularity (count only)
    const uint64_t rbb = out->resident_blob_bytes;
    if (rbb == 0) out->n_objects = 1;
    else if (gran_kind == 0) out->n_objects = 1;
    else if (gran_kind == 1) out->n_objects = uint32_t(r.manifest->tensors.size());
    else out->n_objects = uint32_t((rbb + block_bytes - 1) / block_bytes);
    return 0;
  });
}

int trims_store_close(trims_store* s, const char* ns, const char* name, const char* version, uint64_t* rc) {
  return guard([&] {
    if (s->peer_map) {  // a peer-mapped open of this key first (its lease goes with the last view)
      const fmt::ModelKey key{ns, name, version};
      std::lock_guard lk(s->pm_mu);
      for (auto it = s->peer_maps.rbegin(); it != s->peer_maps.rend(); ++it) {
        if (it->second->key == key) {
          s->peer_maps.erase(std::next(it).base());
          if (rc) *rc = 0;
          return 0;
        }
      }
    }
    uint64_t v = s->core->close_model({ns, name, version});
    if (rc) *rc = v;
    return 0;
  });
}

int trims_store_reclaim(trims_store* s, uint32_t tier, uint64_t bytes, uint32_t policy, char* out, uint64_t cap) {
  return guard([&] {
    if (tier > 2) raise(Errc::InvalidArgument, "tier");
    auto ev = s->core->reclaim(Tier(tier), bytes, Policy(policy ? 1 : 0));
    std::string txt;
    for (const auto& k : ev) txt += fmt::to_string(k) + "\n";
    return out ? put(txt, out, cap) : 0;
  });
}

int trims_store_register_disk_file(trims_store* s, const char* ns, const char* name, const char* version,
                                   const char* path, uint64_t bytes) {
  return guard([&] {
    s->core->register_disk_file({ns, name, version}, path, bytes);
    return 0;
  });
}

int trims_store_drop_all(trims_store* s) {
  return guard([&] {
    s->core->drop_all();
    return 0;
  });
}

int trims_store_stats_json(trims_store* s, char* out, uint64_t cap) {
  return guard([&] {
    StatsSnapshot st = s->core->stats();
    std::ostringstream os;
    os << "{\"tiers\":[";
    for (int t = 0; t < kTiers; ++t) {
      const auto& x = st.tiers[t];
      os << (t ? "," : "") << "{\"hits\":" << x.hits << ",\"misses\":" << x.misses << ",\"evictions\":" << x.evictions
         << ",\"used_bytes\":" << x.used_bytes << ",\"capacity_bytes\":" << x.capacity_bytes << "}";
    }
    os << "],\"models\":[";
    for (size_t i = 0; i < st.models.size(); ++i) {
      const auto& m = st.models[i];
      os << (i ? "," : "") << "{\"key\":\"" << fmt::to_string(m.key) << "\",\"refcount\":" << m.refcount
         << ",\"use_count\":" << m.use_count << ",\"last_access\":" << m.last_access
         << ",\"residency\":" << int(m.residency) << "}";
    }
    os << "],\"open_requests\":" << st.open_requests << ",\"open_errors\":" << st.open_errors
       << ",\"disk_reads\":" << st.disk_reads << ",\"remote_fetches\":" << st.remote_fetches
       << ",\"fetch_ns\":" << st.cumulative.fetch_ns << ",\"disk_read_ns\":" << st.cumulative.disk_read_ns
       << ",\"copy_ns\":" << st.cumulative.host_to_fast_copy_ns << ",\"export_ns\":" << st.cumulative.handle_export_ns
       << ",\"peer_hits\":" << st.peer_hits << ",\"peer_attempts\":" << s->peers.attempts.load()
       << ",\"peer_fallbacks\":" << s->peers.fallbacks.load() << ",\"direct_reads\":" << s->be->direct_loads()
       << ",\"peer_maps\":" << s->peer_maps_total.load() << ",\"peer_maps_open\":" << [&] {
            std::lock_guard lk(s->pm_mu);
            return s->peer_maps.size();
          }()
       << ",\"rank\":" << (s->dir ? s->dir->rank() : 0)
       << ",\"world\":" << (s->dir ? s->dir->world() : 1) << ",\"workspace_headroom\":" << f64(s->workspace_headroom)
       << ",\"has_calibration\":" << (s->calibration ? "true" : "false");
    if (s->calibration)
      os << ",\"calib_q\":" << f64(s->calibration->q) << ",\"calib_o\":" << f64(s->calibration->o)
         << ",\"calib_s\":" << f64(s->calibration->s);
    os << "}";
    return put(os.str(), out, cap);
  });
}

int trims_store_pin(trims_store* s, uint64_t model_id, uint64_t generation, trims_pin** out) {
  return guard([&] {
    if (!s || !out) raise(Errc::InvalidArgument, "null argument");
    if (model_id & kPeerMapIdBit) {  // a peer-mapped view: holding its lease keeps the range
      std::lock_guard lk(s->pm_mu);
      auto it = s->peer_maps.find(model_id);
      if (it == s->peer_maps.end() || it->second->generation != generation)
        raise(Errc::NoSuchSegment, "peer-mapped view not open");
      *out = new trims_pin{nullptr, it->second};
      return 0;
    }
    auto rec = s->be->fast_record(model_id);
    if (!rec) raise(Errc::NoSuchSegment, "model " + std::to_string(model_id) + " is not fast-resident");
    if (rec->generation != generation) raise(Errc::StaleGeneration, "pin of a replaced generation");
    *out = new trims_pin{std::move(rec)};
    return 0;
  });
}

void trims_pin_release(trims_pin* p) { delete p; }

int trims_lease_acquire(const char* token, uint64_t offset, uint64_t generation, trims_lease** out) {
  return guard([&] {
    if (!token || !out) raise(Errc::InvalidArgument, "null argument");
    *out = nullptr;
    auto t = LeaseTable::open(token);
    if (!t) return 0;  // a dedicated segment (no arena): the mapping itself keeps the pages
    auto l = std::make_unique<trims_lease>();
    l->row = t->acquire(offset, generation);
    l->table = std::move(t);
    l->offset = offset;
    l->generation = generation;
    *out = l.release();
    return 0;
  });
}

void trims_lease_release(trims_lease* l) {
  if (!l) return;
  if (l->table) l->table->release(l->row, l->offset, l->generation);
  delete l;
}

int trims_store_resident_json(trims_store* s, uint64_t model_id, char* out, uint64_t cap) {
  return guard([&] {
    if (model_id & kPeerMapIdBit) {
      std::lock_guard lk(s->pm_mu);
      auto it = s->peer_maps.find(model_id);
      if (it == s->peer_maps.end()) raise(Errc::NotOpen, "peer-mapped view not open");
      return put(it->second->json, out, cap);
    }
    auto rec = s->be->fast_record(model_id);
    if (!rec) raise(Errc::NotOpen, "model not fast-resident");
    return put(rec->json, out, cap);
  });
}

int trims_store_ingest_stats(trims_store* s, uint64_t model_id, double out7[7]) {
  double* out5 = out7;
  return guard([&] {
    auto rec = s->be->fast_record(model_id);
    if (!rec) raise(Errc::NotOpen, "model not fast-resident");
    out5[0] = rec->stats.h2d_ms;
    out5[1] = rec->stats.total_ms;
    out5[2] = rec->stats.read_ms;
    out5[3] = double(rec->stats.h2d_bytes);
    out5[4] = rec->stats.launches;
    out7[5] = rec->stats.alloc_ms;
    out7[6] = rec->stats.seal_ms;
    return 0;
  });
}

int trims_store_checksums(trims_store* s, uint64_t model_id, uint64_t* out, uint64_t cap, uint64_t* n) {
  return guard([&] {
    auto rec = s->be->fast_record(model_id);
    if (!rec) raise(Errc::NotOpen, "model not fast-resident");
    *n = rec->bucket_sums.size();
    for (uint64_t i = 0; i < std::min<uint64_t>(cap, *n); ++i) out[i] = rec->bucket_sums[i];
    return 0;
  });
}

int trims_store_fast_resident(trims_store* s, const char* ns, const char* name, const char* version, int* out) {
  return guard([&] {
    if (!s || !out) raise(Errc::InvalidArgument, "null argument");
    *out = s->core->fast_resident({ns, name, version}) ? 1 : 0;
    return 0;
  });
}

// ------------------------------------------------------------- directory

static_assert(sizeof(trims_dir_coords) == sizeof(DirCoords), "trims_dir_coords mirrors DirCoords");

int trims_dir_open(const char* name, int world, int rank, uint32_t slots, trims_dir** out) {
  return guard([&] {
    if (!name || !out) raise(Errc::InvalidArgument, "null argument");
    auto d = std::make_unique<trims_dir>();
    d->d = Directory::open(name, world, rank, slots ? slots : 1024);
    *out = d.release();
    return 0;
  });
}

void trims_dir_close(trims_dir* d) {
  try {
    delete d;
  } catch (...) {
  }
}

int trims_dir_unlink(const char* name) {
  return guard([&] {
    if (!name) raise(Errc::InvalidArgument, "null argument");
    Directory::unlink(name);
    return 0;
  });
}

int trims_dir_publish(trims_dir* d, const char* ns, const char* name, const char* version, const trims_dir_coords* c) {
  return guard([&] {
    if (!d || !c) raise(Errc::InvalidArgument, "null argument");
    DirCoords dc;
    std::memcpy(&dc, c, sizeof dc);
    d->d->publish({ns, name, version}, dc);
    return 0;
  });
}

int trims_dir_retract(trims_dir* d, const char* ns, const char* name, const char* version) {
  return guard([&] {
    if (!d) raise(Errc::InvalidArgument, "null argument");
    d->d->retract({ns, name, version});
    return 0;
  });
}

int trims_dir_holders(trims_dir* d, const char* ns, const char* name, const char* version, trims_dir_coords* out,
                      uint64_t cap, uint64_t* n) {
  return guard([&] {
    if (!d || !n) raise(Errc::InvalidArgument, "null argument");
    std::vector<DirCoords> hs = d->d->holders({ns, name, version});
    *n = hs.size();
    for (uint64_t i = 0; i < std::min<uint64_t>(cap, hs.size()); ++i) std::memcpy(&out[i], &hs[i], sizeof hs[i]);
    return 0;
  });
}

uint64_t trims_peer_score(const char* key, int rank) { return peer_score(key ? key : "", rank); }

// ---------------------------------------------------------------- import

int trims_import_open(int device, int fd, uint64_t alloc_bytes, trims_import** out, void** base) {
  return guard([&] {
    auto im = std::make_unique<trims_import>();
    im->map.reset(Import::open(device, fd, alloc_bytes, /*read_only=*/true));
    im->device = device;
    if (base) *base = im->map->ptr();
    *out = im.release();
    return 0;
  });
}

namespace {
// Reads and validates the tail of the segment at `offset` (shared_segment.cpp:
// 233-237 checks: magic, generation, sealed, length) and returns it with the JSON.
SegTail read_tail(trims_import* im, uint64_t offset, uint64_t generation, uint64_t payload_bytes, std::string* json) {
  return read_tail_of(*im->map, im->device, offset, generation, payload_bytes, json);
}
}  // namespace

int trims_import_attach(trims_import* im, uint64_t offset, uint64_t generation, uint64_t payload_bytes,
                        const uint8_t digest[32], void** dev_ptr, char* json_out, uint64_t cap) {
  return guard([&] {
    std::string json;
    read_tail(im, offset, generation, payload_bytes, &json);
    if (digest) {
      auto d = Sha256::of(json.data(), json.size());
      if (std::memcmp(d.data(), digest, 32) != 0) raise(Errc::Corrupt, "manifest digest mismatch on attach");
    }
    if (dev_ptr) *dev_ptr = im->map->ptr() + offset;
    return json_out ? put(json, json_out, cap) : 0;
  });
}

int trims_import_read_only(trims_import* im) { return im && im->map && im->map->read_only() ? 1 : 0; }

int trims_import_verify(trims_import* im, uint64_t offset, uint64_t generation, uint64_t payload_bytes,
                        uint64_t* checksum_out) {
  return guard([&] {
    SegTail st = read_tail(im, offset, generation, payload_bytes, nullptr);
    DeviceGuard g(im->device);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, im->device);
    unsigned long long* d = nullptr;
    TRIMS_CUDA(cudaMalloc(&d, sizeof *d));
    unsigned long long h = 0;
    try {
      TRIMS_CUDA(cudaMemset(d, 0, sizeof *d));
      ingest::launch_checksum(im->map->ptr() + offset, st.blob_bytes, 0, d, nullptr, sms);
      TRIMS_CUDA(cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost));
    } catch (...) {
      cudaFree(d);
      throw;
    }
    cudaFree(d);
    if (checksum_out) *checksum_out = h;
    if (h != st.checksum) raise(Errc::Corrupt, "resident blob checksum mismatch on attach");
    return 0;
  });
}

void trims_import_close(trims_import* im) {
  try {
    delete im;
  } catch (...) {
  }
}

// ---------------------------------------------------------------- raw ingest

namespace {
// Raw-ingest engines live for the process: they are never destroyed at exit
// (static destructors would run after the CUDA driver has shut down).
std::mutex g_ing_mu;
std::map<int, Ingestor*>* g_ing = new std::map<int, Ingestor*>();
Ingestor& ingestor(int device) {
  std::lock_guard lk(g_ing_mu);
  Ingestor*& p = (*g_ing)[device];
  if (!p) p = new Ingestor(device);
  return *p;
}
}  // namespace

namespace {
// Plans compiled for the convenience (JSON-in) entry points, keyed by the
// exact request; callers on a hot path hold a trims_plan instead.
std::mutex g_plan_mu;
std::map<std::string, std::shared_ptr<IngestPlan>>* g_plans = new std::map<std::string, std::shared_ptr<IngestPlan>>();
std::shared_ptr<IngestPlan> cached_plan(int device, const char* src_json, uint32_t flags, uint32_t out_dtype) {
  std::string key = std::to_string(device) + ":" + std::to_string(flags) + ":" + std::to_string(out_dtype) + ":" + src_json;
  {
    std::lock_guard lk(g_plan_mu);
    auto it = g_plans->find(key);
    if (it != g_plans->end()) return it->second;
  }
  auto p = ingestor(device).compile(fmt::manifest_from_json(src_json), make_plan(flags, out_dtype));
  std::lock_guard lk(g_plan_mu);
  if (g_plans->size() > 32) g_plans->clear();
  return g_plans->emplace(std::move(key), std::move(p)).first->second;
}

void put_stats(const IngestStats& st, double* out5) {
  if (!out5) return;
  out5[0] = st.h2d_ms;
  out5[1] = st.total_ms;
  out5[2] = st.read_ms;
  out5[3] = double(st.h2d_bytes);
  out5[4] = st.launches;
}
}  // namespace

struct trims_plan {
  std::shared_ptr<IngestPlan> p;
};

int trims_plan_create(int device, const char* src_json, uint32_t plan_flags, uint32_t out_dtype, trims_plan** out) {
  return guard([&] {
    auto h = std::make_unique<trims_plan>();
    h->p = ingestor(device).compile(fmt::manifest_from_json(src_json), make_plan(plan_flags, out_dtype));
    *out = h.release();
    return 0;
  });
}

void trims_plan_destroy(trims_plan* p) { delete p; }

int trims_tile_plan_text(const char* src_json, uint32_t plan_flags, uint32_t out_dtype, int sm_count, char* out,
                         uint64_t cap) {
  return guard([&] {
    const fmt::Manifest src = fmt::manifest_from_json(src_json);
    const fmt::Plan plan = make_plan(plan_flags, out_dtype);
    const fmt::Manifest dst = fmt::resident_manifest(src, plan);
    const ingest::TilePlan t = ingest::build_tiles(src, dst, plan.identity(), 16ull << 20, sm_count);
    std::ostringstream os;
    auto tile = [&](const char* tag, const ingest::Tile& x) {
      os << tag << ' ' << int(x.op) << ' ' << x.src_off << ' ' << x.dst_off << ' ' << x.dst_bytes << ' ' << x.n_elem
         << ' ' << x.tensor << '\n';
    };
    for (const ingest::Tile& x : t.tiles_by_kernel) tile("tile", x);
    for (const ingest::Group& g : t.groups) {
      os << "group " << int(g.kind) << ' ' << (g.end - g.begin) << ' ' << g.nbins << ' ' << g.stride << ' ' << g.tail
         << ' ' << g.dev_begin << ' ' << g.dev_count << '\n';
      for (uint32_t i = 0; i < g.dev_count; ++i) tile("dev", t.dev_tiles_k[g.dev_begin + i]);
    }
    return put(os.str(), out, cap);
  });
}

int trims_plan_describe(trims_plan* p, uint64_t out8[8]) {
  return guard([&] {
    const auto& t = p->p->plan;
    out8[0] = t.tiles.size();
    out8[1] = t.buckets;
    out8[2] = t.algo_read_bytes;
    out8[3] = t.algo_write_bytes;
    out8[4] = p->p->src.blob_bytes;
    out8[5] = p->p->dst.blob_bytes;
    out8[6] = t.chunks.size();
    out8[7] = t.groups.size();  // kernel launches of one HBM-resident transform
    return 0;
  });
}

int trims_plan_resident_json(trims_plan* p, char* out, uint64_t cap) {
  return guard([&] { return put(p->p->dst_json, out, cap); });
}

int trims_plan_transform(trims_plan* p, const void* dev_src, void* dev_dst, unsigned long long* d_sums, void* stream,
                         uint32_t* launches) {
  return guard([&] {
    uint32_t n = ingestor(p->p->device).from_device(*p->p, static_cast<const uint8_t*>(dev_src),
                                                    static_cast<uint8_t*>(dev_dst), d_sums,
                                                    static_cast<cudaStream_t>(stream));
    if (launches) *launches = n;
    return 0;
  });
}

int trims_plan_ingest_host(trims_plan* p, const void* host_blob, void* dev_dst, uint64_t* checksum_out,
                           double stats_out5[5]) {
  return guard([&] {
    IngestStats st;
    uint64_t c = ingestor(p->p->device).from_host(*p->p, static_cast<const uint8_t*>(host_blob),
                                                  static_cast<uint8_t*>(dev_dst), nullptr, &st);
    if (checksum_out) *checksum_out = c;
    put_stats(st, stats_out5);
    return 0;
  });
}

int trims_ingest_host(int device, const void* host_blob, const char* src_json, uint32_t plan_flags,
                      uint32_t out_dtype, void* dev_dst, uint64_t* checksum_out, double stats_out5[5]) {
  return guard([&] {
    auto p = cached_plan(device, src_json, plan_flags, out_dtype);
    IngestStats st;
    uint64_t c = ingestor(device).from_host(*p, static_cast<const uint8_t*>(host_blob), static_cast<uint8_t*>(dev_dst),
                                            nullptr, &st);
    if (checksum_out) *checksum_out = c;
    put_stats(st, stats_out5);
    return 0;
  });
}

int trims_transform_device(int device, const void* dev_src, const char* src_json, uint32_t plan_flags,
                           uint32_t out_dtype, void* dev_dst, unsigned long long* d_sums, void* stream) {
  return guard([&] {
    auto p = cached_plan(device, src_json, plan_flags, out_dtype);
    ingestor(device).from_device(*p, static_cast<const uint8_t*>(dev_src), static_cast<uint8_t*>(dev_dst), d_sums,
                                 static_cast<cudaStream_t>(stream));
    return 0;
  });
}

int trims_plan_info(const char* src_json, uint32_t plan_flags, uint32_t out_dtype, uint64_t out4[4]) {
  return guard([&] {
    fmt::Manifest src = fmt::manifest_from_json(src_json);
    fmt::Plan plan = make_plan(plan_flags, out_dtype);
    fmt::Manifest dst = fmt::resident_manifest(src, plan);
    ingest::TilePlan p = ingest::build_tiles(src, dst, plan.identity());
    out4[0] = p.tiles.size();
    out4[1] = p.buckets;
    out4[2] = p.algo_read_bytes;
    out4[3] = p.algo_write_bytes;
    return 0;
  });
}

int trims_checksum_device(const void* dev, uint64_t nbytes, uint64_t word0, unsigned long long* d_out, void* stream) {
  return guard([&] {
    int dev_id = 0, sms = 148;
    cudaGetDevice(&dev_id);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev_id);
    ingest::launch_checksum(static_cast<const uint8_t*>(dev), nbytes, word0, d_out, static_cast<cudaStream_t>(stream),
                            sms);
    return 0;
  });
}

int trims_touch_device(int device, const void* dev, uint64_t nbytes, uint64_t* out) {
  return guard([&] {
    // per calling thread and device: a stream, a device accumulator, a pinned result word
    struct Scratch {
      int device{-1};
      cudaStream_t stream{nullptr};
      unsigned long long* d_sum{nullptr};
      unsigned long long* h_sum{nullptr};
      ~Scratch() {  // thread exit (errors ignored: the context may already be gone at process exit)
        if (device < 0) return;
        cudaSetDevice(device);
        cudaStreamDestroy(stream);
        cudaFree(d_sum);
        cudaFreeHost(h_sum);
        cudaGetLastError();
      }
    };
    thread_local std::map<int, Scratch> scratch;
    DeviceGuard g(device);
    Scratch& sc = scratch[device];
    if (sc.device < 0) {
      TRIMS_CUDA(cudaStreamCreateWithFlags(&sc.stream, cudaStreamNonBlocking));
      TRIMS_CUDA(cudaMalloc(&sc.d_sum, sizeof(unsigned long long)));
      TRIMS_CUDA(cudaMallocHost(&sc.h_sum, sizeof(unsigned long long)));
      sc.device = device;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    TRIMS_CUDA(cudaMemsetAsync(sc.d_sum, 0, sizeof(unsigned long long), sc.stream));
    ingest::launch_checksum(static_cast<const uint8_t*>(dev), nbytes, 0, sc.d_sum, sc.stream, sms);
    TRIMS_CUDA(cudaMemcpyAsync(sc.h_sum, sc.d_sum, sizeof(unsigned long long), cudaMemcpyDeviceToHost, sc.stream));
    TRIMS_CUDA(cudaStreamSynchronize(sc.stream));
    *out = *sc.h_sum;
    return 0;
  });
}

int trims_fill_splitmix_device(uint64_t* dev, uint64_t n, uint64_t stream_seed, uint64_t k0, void* stream) {
  return guard([&] {
    ingest::launch_fill_splitmix(dev, n, stream_seed, k0, static_cast<cudaStream_t>(stream));
    return 0;
  });
}

int trims_gemm_bf16(const void* A, uint64_t M, uint64_t K, uint64_t lda, const void* B, uint64_t N, uint64_t ldb,
                    void* D, uint64_t ldd, const float* scale, const float* bias, const void* residual, uint64_t ldr,
                    int relu, int bn, void* stream) {
  return guard([&] {
    gemm::Epilogue e{static_cast<uint16_t*>(D), ldd, scale, bias, static_cast<const uint16_t*>(residual), ldr,
                     relu != 0};
    gemm::launch({A, M, K, lda}, {B, N, K, ldb}, e, static_cast<cudaStream_t>(stream), bn);
    return 0;
  });
}

int trims_gemm_bf16_split(const void* A, uint64_t M, uint64_t K, uint64_t lda, const void* B, uint64_t N,
                          uint64_t ldb, void* D, uint64_t ldd, const float* scale, const float* bias,
                          const void* residual, uint64_t ldr, int relu, int bn, int splits, void* stream) {
  return guard([&] {
    gemm::Epilogue e{static_cast<uint16_t*>(D), ldd, scale, bias, static_cast<const uint16_t*>(residual), ldr,
                     relu != 0};
    gemm::launch({A, M, K, lda}, {B, N, K, ldb}, e, static_cast<cudaStream_t>(stream), bn, splits);
    return 0;
  });
}

int trims_gemm_bf16_ex(const void* A, uint64_t M, uint64_t K, uint64_t lda, const void* B, uint64_t N, uint64_t ldb,
                       void* D, uint64_t ldd, const float* scale, const float* bias, const void* residual,
                       uint64_t ldr, int relu, int bn, int splits, int mc, void* stream) {
  return guard([&] {
    if (mc != 1 && mc != 2 && mc != 4 && mc != 8 && mc != -2 && mc != -3)
      raise(Errc::InvalidArgument, "multicast group of 1, 2, 4 or 8, -2 (2-SM pair) or -3 (persistent)");
    gemm::Epilogue e{static_cast<uint16_t*>(D), ldd, scale, bias, static_cast<const uint16_t*>(residual), ldr,
                     relu != 0};
    gemm::launch({A, M, K, lda}, {B, N, K, ldb}, e, static_cast<cudaStream_t>(stream), bn, splits, mc);
    return 0;
  });
}

struct trims_net {
  std::unique_ptr<nn::Net> net;
};

int trims_net_create_ex(int device, const char* arch_text, const char* resident_json, const void* weights, int batch,
                        int flags, trims_net** out) {
  return guard([&] {
    if (batch < 1) raise(Errc::InvalidArgument, "batch must be >= 1");
    if (flags & ~(nn::kNetThroughput | nn::kNetLean)) raise(Errc::InvalidArgument, "unknown executor flags");
    auto h = std::make_unique<trims_net>();
    h->net = std::make_unique<nn::Net>(device, arch_text, fmt::manifest_from_json(resident_json),
                                       static_cast<const uint8_t*>(weights), batch, flags);
    *out = h.release();
    return 0;
  });
}

int trims_net_create(int device, const char* arch_text, const char* resident_json, const void* weights, int batch,
                     trims_net** out) {
  return trims_net_create_ex(device, arch_text, resident_json, weights, batch, 0, out);
}

void trims_net_destroy(trims_net* net) {
  try {
    delete net;
  } catch (...) {
  }
}

int trims_net_buffers(trims_net* net, void** input, void** logits, int* classes, int* input_hw) {
  return guard([&] {
    if (input) *input = net->net->input();
    if (logits) *logits = net->net->logits();
    if (classes) *classes = net->net->classes();
    if (input_hw) *input_hw = net->net->input_hw();
    return 0;
  });
}

int trims_net_rebind(trims_net* net, const void* weights) {
  return guard([&] {
    net->net->rebind(static_cast<const uint8_t*>(weights));
    return 0;
  });
}

int trims_net_run(trims_net* net, void* stream, int use_graph) {
  return guard([&] {
    net->net->run(static_cast<cudaStream_t>(stream), use_graph != 0);
    return 0;
  });
}

int trims_net_forward_host(trims_net* net, const float* host_input, float* host_logits, void* stream, int use_graph) {
  return guard([&] {
    if (!net || !host_input || !host_logits) raise(Errc::InvalidArgument, "null argument");
    DeviceGuard g(net->net->device());
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TRIMS_CUDA(cudaMemcpyAsync(net->net->input(), host_input, net->net->input_bytes(), cudaMemcpyHostToDevice, st));
    net->net->run(st, use_graph != 0);
    TRIMS_CUDA(cudaMemcpyAsync(host_logits, net->net->logits(), net->net->logits_bytes(), cudaMemcpyDeviceToHost, st));
    TRIMS_CUDA(cudaStreamSynchronize(st));
    return 0;
  });
}

int trims_host_alloc(uint64_t bytes, void** out) {
  return guard([&] {
    if (!out) raise(Errc::InvalidArgument, "null argument");
    *out = nullptr;
    TRIMS_CUDA(cudaHostAlloc(out, std::max<uint64_t>(bytes, 1), cudaHostAllocPortable));
    return 0;
  });
}

void trims_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int trims_net_info(trims_net* net, double out3[3]) {
  return guard([&] {
    out3[0] = net->net->flops();
    out3[1] = net->net->launches();
    out3[2] = double(net->net->workspace_bytes());
    return 0;
  });
}

int trims_net_tap(trims_net* net, int layer, const void** ptr, int dims4[4], int* dtype) {
  return guard([&] {
    if (!net) raise(Errc::InvalidArgument, "null net");
    if (layer < 0) return net->net->layers();
    const auto& t = net->net->tap(layer);
    if (ptr) *ptr = t.p;
    if (dims4) {
      dims4[0] = t.n;
      dims4[1] = t.h;
      dims4[2] = t.w;
      dims4[3] = t.c;
    }
    if (dtype) *dtype = t.dtype;
    return 0;
  });
}

int trims_softmax(const float* in, float* out, int M, int N, void* stream) {
  return guard([&] {
    nn::softmax(in, out, M, N, static_cast<cudaStream_t>(stream));
    return 0;
  });
}

int trims_fill_uniform_device(float* dev, uint64_t n, uint64_t stream_seed, uint64_t j0, float lo, float hi,
                              void* stream) {
  return guard([&] {
    ingest::launch_fill_uniform(dev, n, stream_seed, j0, lo, hi, static_cast<cudaStream_t>(stream));
    return 0;
  });
}

}  // extern "C"

// ------------------------------------------------------------ store_api
// (store_api.hpp: the surface the wire daemon drives)

namespace trims::store_api {

PlacementResult open(trims_store* s, const fmt::ModelKey& key, const Granularity& g) {
  const uint64_t now = s->clock.fetch_add(1) + 1;  // daemon.cpp:457
  return s->open(key, g, now, nullptr);
}

uint64_t close(trims_store* s, const fmt::ModelKey& key) { return s->core->close_model(key); }

StatsSnapshot stats(trims_store* s) { return s->core->stats(); }

std::shared_ptr<FastRecord> fast_record(trims_store* s, uint64_t model_id) { return s->be->fast_record(model_id); }

void set_last_error(const std::string& what) { g_last_error = what; }

double workspace_headroom(trims_store* s) { return s->workspace_headroom; }

std::optional<Calibration> calibration(trims_store* s) { return s->calibration; }

}  // namespace trims::store_api
