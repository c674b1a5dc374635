// mrm_cuda_backend.cpp — the reference-side binding of the B200 store.
//
// This is the adapter a maintainer of the reference (proj/, namespace mrm)
// adds to swap its shared-memory fast tier for the B200 HBM store: a
// mrm::cache::TierBackend (proj/include/mrm/cache_core.hpp:76-98) whose eight
// virtuals forward to libtrims's C ABI (include/trims.h, trims_backend_*).
// The reference's CacheCore, daemon and wire protocol stay unmodified; the
// exported segment token carries the CUDA arena coordinates instead of a shm
// name, so a client attaches with trims_import_open/attach.
//
// It is compiled against the reference headers by `make -C oracle
// integration` (oracle/_ref/libmrm_cuda.so, test infrastructure) and driven by
// tests/test_gpu_integration.py: the UNMODIFIED reference CacheCore runs on top
// of the CUDA backend.
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "../include/trims.h"
#include "mrm/bench/catalog.hpp"
#include "mrm/cache_core.hpp"
#include "mrm/model_format.hpp"

namespace mrm_b200 {

using namespace mrm;

namespace {
void check(int rc, const char* what) {
  if (rc == 0) return;
  // trims codes are the reference Errc values; the B200 additions (170+) are Internal here
  raise(rc >= 170 ? Errc::Internal : Errc(rc), std::string(what) + ": " + trims_last_error());
}
}  // namespace

class CudaTierBackend : public cache::TierBackend {
 public:
  explicit CudaTierBackend(const trims_store_config& cfg) { check(trims_backend_create(&cfg, &be_), "create"); }
  ~CudaTierBackend() override { trims_backend_destroy(be_); }

  cache::Located locate(const model::ModelKey& key) override {
    char path[4096];
    uint64_t bytes = 0;
    int rc = trims_backend_locate(be_, key.ns.c_str(), key.name.c_str(), key.version.c_str(), path, sizeof path,
                                  &bytes);
    if (rc == int(Errc::NotFound)) return {cache::Located::Kind::Absent, "", 0};
    check(rc, "locate");
    if (!path[0]) return {cache::Located::Kind::Remote, "", 0};  // not on disk, remote_url set
    return {cache::Located::Kind::DiskCache, path, bytes};
  }

  cache::FetchResult fetch_remote(const model::ModelKey& key) override {  // daemon.cpp:138-142
    char path[4096];
    uint64_t bytes = 0;
    check(trims_backend_fetch_remote(be_, key.ns.c_str(), key.name.c_str(), key.version.c_str(), path, sizeof path,
                                     &bytes),
          "fetch_remote");
    return {path, bytes};
  }

  model::ModelManifest read_manifest(const model::ModelKey& key, const std::string& path) override {
    std::vector<char> json(1 << 22);
    uint8_t cs[32];
    check(trims_backend_read_manifest(be_, key.ns.c_str(), key.name.c_str(), key.version.c_str(), path.c_str(),
                                      json.data(), json.size(), cs),
          "read_manifest");
    model::ModelManifest m = model::manifest_from_json(json.data());
    std::memcpy(m.checksum.data(), cs, 32);
    return m;
  }

  void stage_host(uint64_t model_id, const model::ModelManifest& m, const std::string& path) override {
    check(trims_backend_stage_host(be_, model_id, model::manifest_to_json(m).c_str(), m.checksum.data(),
                                   path.c_str()),
          "stage_host");
  }

  cache::FastPublication publish_fast(uint64_t model_id, const model::ModelManifest& m, bool from_host,
                                      const std::string& path) override {
    trims_export ex;
    check(trims_backend_publish_fast(be_, model_id, model::manifest_to_json(m).c_str(), from_host ? 1 : 0,
                                     path.c_str(), &ex),
          "publish_fast");
    // token: "<arena token>@<offset>:<payload>:<alloc>:<fd>" (fd valid in the owner process;
    // a daemon passes it to clients with SCM_RIGHTS)
    std::ostringstream tok;
    tok << ex.token << '@' << ex.segment_offset << ':' << ex.payload_bytes << ':' << ex.alloc_bytes << ':' << ex.fd;
    cache::FastPublication pub;
    pub.segments.push_back({tok.str(), ex.generation, ex.payload_bytes});
    std::memcpy(pub.manifest_digest.data(), ex.manifest_digest, 32);
    last_checksum_ = ex.ingest_checksum;
    return pub;
  }

  void evict_fast(uint64_t model_id) override { check(trims_backend_evict_fast(be_, model_id), "evict_fast"); }
  void evict_host(uint64_t model_id) override { check(trims_backend_evict_host(be_, model_id), "evict_host"); }
  void evict_disk(const model::ModelKey&, const std::string& path) override {
    check(trims_backend_evict_disk(be_, path.c_str()), "evict_disk");
  }

  uint64_t last_checksum() const { return last_checksum_; }

 private:
  trims_backend* be_{nullptr};
  uint64_t last_checksum_{0};
};

}  // namespace mrm_b200

// Test driver: the unmodified reference CacheCore over the CUDA backend.
// ops: "o <name>" / "c <name>" lines on catalog keys zoo/<name>@1.0.0 in `dir`.
// Output per op: "<outcome> <fast_used> <host_used> <refcount> <token>".
// remote (may be NULL): DaemonConfig::remote_url; full_verify as DaemonConfig.
extern "C" int refcuda_replay2(const char* dir, const char* remote, int full_verify, uint64_t fast_cap,
                               uint64_t host_cap, int eager, const char* ops, char* out, uint64_t cap) {
  using namespace mrm;
  try {
    trims_store_config cfg{};
    cfg.fast_capacity_bytes = fast_cap;
    cfg.host_capacity_bytes = host_cap;
    cfg.disk_capacity_bytes = 1ull << 40;
    cfg.disk_cache_dir = dir;
    cfg.remote_url = remote;
    cfg.full_verify = full_verify != 0;
    mrm_b200::CudaTierBackend be(cfg);
    cache::CoreConfig cc{fast_cap, host_cap, 1ull << 40, cache::Policy::LRU, eager != 0};
    cache::CacheCore core(cc, be);
    std::istringstream is(ops);
    std::ostringstream os;
    std::string op, name;
    uint64_t now = 0;
    while (is >> op >> name) {
      model::ModelKey key{"zoo", name, "1.0.0"};
      std::string token = "-";
      int outcome = 0;
      try {
        if (op == "o") {
          auto r = core.open_model(key, shm::ShareGranularity::model(), ++now);
          outcome = int(r.outcome);
          token = r.segments.at(0).token;
        } else {
          core.close_model(key);
        }
      } catch (const Error& e) {
        outcome = 100 + int(e.code());
      }
      os << outcome << ' ' << core.used_bytes(cache::Tier::Fast) << ' ' << core.used_bytes(cache::Tier::Host) << ' '
         << core.refcount(key) << ' ' << token << '\n';
    }
    core.drop_all();
    std::string s = os.str();
    if (s.size() + 1 > cap) return 160;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (const Error& e) {
    return int(e.code());
  } catch (...) {
    return 7;
  }
}

extern "C" int refcuda_replay(const char* dir, uint64_t fast_cap, uint64_t host_cap, int eager, const char* ops,
                              char* out, uint64_t cap) {
  return refcuda_replay2(dir, nullptr, 0, fast_cap, host_cap, eager, ops, out, cap);
}
