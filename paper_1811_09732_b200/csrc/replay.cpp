// replay.cpp — decision-trace replay through this library's CacheCore over an
// in-memory TierBackend with the reference FakeBackend contract
// (proj/src/bench/oracle.cpp:14-91): keys trace/m<i>@1, one F64 tensor of
// weights/8 elements, evictions recorded by model index. Output lines match
// oracle/ref_shim.cpp:ref_replay's "live" lines so tests diff them verbatim.
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/trims.h"
#include "cache_core.hpp"
#include "directory.hpp"

using namespace trims;

namespace {

struct Model {
  uint64_t weights{0}, file_bytes{0};
  bool on_disk{true}, on_remote{false};
};

class FakeBackend : public TierBackend {
 public:
  explicit FakeBackend(std::vector<Model> m) : models_(std::move(m)), present_(models_.size()), id_(models_.size()) {
    for (size_t i = 0; i < models_.size(); ++i) present_[i] = models_[i].on_disk;
  }
  static fmt::ModelKey key_of(uint32_t i) { return {"trace", "m" + std::to_string(i), "1"}; }
  static uint32_t index_of(const fmt::ModelKey& k) { return uint32_t(std::stoul(k.name.substr(1))); }

  Located locate(const fmt::ModelKey& k) override {
    uint32_t i = index_of(k);
    if (present_[i]) return {Located::Kind::DiskCache, "fake://" + std::to_string(i), models_[i].file_bytes};
    if (models_[i].on_remote) return {Located::Kind::Remote, "", 0};
    return {Located::Kind::Absent, "", 0};
  }
  FetchResult fetch_remote(const fmt::ModelKey& k) override {
    uint32_t i = index_of(k);
    if (!models_[i].on_remote) raise(Errc::RemoteNotFound, k.name);
    present_[i] = true;
    return {"fake://" + std::to_string(i), models_[i].file_bytes};
  }
  fmt::Manifest read_manifest(const fmt::ModelKey& k, const std::string&) override {
    return fmt::make_manifest(k, {{"t0", {models_[index_of(k)].weights / 8}, fmt::DType::F64}}, 0);
  }
  void stage_host(uint64_t id, const fmt::Manifest& m, const std::string&) override { id_[index_of(m.key)] = id; }
  FastPublication publish_fast(uint64_t id, const fmt::Manifest& m, bool, const std::string&) override {
    id_[index_of(m.key)] = id;
    FastPublication p;
    ExportedSegment s;
    s.token = "fake-seg-" + std::to_string(id);
    s.generation = ++gen_;
    s.length = m.blob_bytes;
    p.segments.push_back(s);
    if (dir) {
      DirCoords c;
      c.generation = s.generation;
      c.payload_bytes = s.length;
      dir->publish(m.key, c);
    }
    return p;
  }
  FastPublication publish_from_peer(uint64_t id, const fmt::Manifest& m, const PeerSource&) override {
    return publish_fast(id, m, false, "");
  }
  void evict_fast(uint64_t id) override {
    uint32_t i = record(id, ev_fast);
    if (dir && i != ~0u) dir->retract(key_of(i));
  }
  void evict_host(uint64_t id) override { record(id, ev_host); }
  void evict_disk(const fmt::ModelKey& k, const std::string&) override {
    uint32_t i = index_of(k);
    present_[i] = false;
    ev_disk.push_back(i);
  }
  std::shared_ptr<const fmt::Manifest> manifest_if_on_disk(uint32_t i) {
    if (!present_[i]) return nullptr;
    return std::make_shared<const fmt::Manifest>(read_manifest(key_of(i), ""));
  }
  std::vector<uint32_t> ev_fast, ev_host, ev_disk;
  Directory* dir{nullptr};

 private:
  uint32_t record(uint64_t id, std::vector<uint32_t>& v) {
    for (uint32_t i = 0; i < id_.size(); ++i)
      if (id_[i] == id) {
        v.push_back(i);
        return i;
      }
    return ~0u;
  }
  uint64_t gen_{0};
  std::vector<Model> models_;
  std::vector<bool> present_;
  std::vector<uint64_t> id_;
};

std::string list(std::vector<uint32_t>& v) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  v.clear();
  return s.empty() ? "-" : s;
}


void parse_spec(const char* spec, CoreConfig& cfg, std::vector<Model>& models,
                std::vector<std::pair<char, uint32_t>>& ops) {
    std::istringstream is(spec);
    std::string tag;
    while (is >> tag) {
      if (tag == "cfg") {
        int pol, eager;
        is >> cfg.fast_capacity_bytes >> cfg.host_capacity_bytes >> cfg.disk_capacity_bytes >> pol >> eager;
        cfg.policy = Policy(pol);
        cfg.eager_reclaim = eager != 0;
      } else if (tag == "model") {
        Model m;
        int d, r;
        is >> m.weights >> m.file_bytes >> d >> r;
        m.on_disk = d;
        m.on_remote = r;
        models.push_back(m);
      } else if (tag == "op") {
        std::string k;
        uint32_t i;
        is >> k >> i;
        ops.push_back({k[0], i});
      }
    }
}

int error_outcome(Errc c) {
  switch (c) {
    case Errc::NotFound:
    case Errc::RemoteNotFound: return 100;
    case Errc::TooLargeForFast: return 101;
    case Errc::NoEvictableSpace: return 102;
    case Errc::NotOpen:
    case Errc::UnknownModel: return 103;
    default: return 199;
  }
}

}  // namespace

// Op kinds: 'o' open, 'c' close, 'p' open with a peer copy available (the
// multi-GPU extension; oracle/simulator.py Core.step 'p').
extern "C" int trims_replay(const char* spec, char* out, uint64_t cap) {
  try {
    CoreConfig cfg;
    std::vector<Model> models;
    std::vector<std::pair<char, uint32_t>> ops;
    parse_spec(spec, cfg, models, ops);
    FakeBackend be(models);
    CacheCore core(cfg, be);
    for (uint32_t i = 0; i < models.size(); ++i)
      if (models[i].on_disk) core.register_disk_file(FakeBackend::key_of(i), "fake://" + std::to_string(i), models[i].file_bytes);
    std::ostringstream os;
    for (size_t s = 0; s < ops.size(); ++s) {
      auto key = FakeBackend::key_of(ops[s].second);
      int outcome = 0;
      try {
        if (ops[s].first == 'o') {
          outcome = int(core.open_model(key, {}, s + 1).outcome);
        } else if (ops[s].first == 'p') {
          PeerSource src;
          src.manifest = std::make_shared<const fmt::Manifest>(be.read_manifest(key, ""));
          outcome = int(core.open_model(key, {}, s + 1, &src).outcome);
        } else {
          core.close_model(key);
        }
      } catch (const Error& e) {
        outcome = error_outcome(e.code());
        if (ops[s].first == 'c') outcome = 103;
      }
      os << "live " << s << ' ' << outcome << ' ' << core.used_bytes(Tier::Fast) << ' ' << core.used_bytes(Tier::Host)
         << ' ' << core.refcount(key) << " f:" << list(be.ev_fast) << " h:" << list(be.ev_host)
         << " d:" << list(be.ev_disk) << '\n';
    }
    StatsSnapshot st = core.stats();
    os << "stats";
    for (int t = 0; t < kTiers; ++t)
      os << ' ' << st.tiers[t].hits << ' ' << st.tiers[t].misses << ' ' << st.tiers[t].evictions << ' '
         << st.tiers[t].used_bytes;
    os << ' ' << st.open_requests << ' ' << st.open_errors << ' ' << st.disk_reads << ' ' << st.remote_fetches << '\n';
    std::string txt = os.str();
    if (txt.size() + 1 > cap) return int(Errc::InvalidArgument);
    std::memcpy(out, txt.data(), txt.size() + 1);
    return 0;
  } catch (const Error& e) {
    return int(e.code());
  } catch (...) {
    return int(Errc::Internal);
  }
}

struct trims_simcore {
  CoreConfig cfg;
  std::vector<Model> models;
  std::unique_ptr<FakeBackend> be;
  std::unique_ptr<CacheCore> core;
  std::unique_ptr<Directory> dir;
  PeerCounters ctr;
};

extern "C" int trims_simcore_create(const char* spec, const char* directory, int world, int rank,
                                    trims_simcore** out) {
  try {
    if (!spec || !out) return int(Errc::InvalidArgument);
    auto c = std::make_unique<trims_simcore>();
    std::vector<std::pair<char, uint32_t>> ops;
    parse_spec(spec, c->cfg, c->models, ops);
    c->be = std::make_unique<FakeBackend>(c->models);
    if (directory && *directory) {
      c->dir = Directory::open(directory, world, rank, 1024);
      c->be->dir = c->dir.get();
    }
    c->core = std::make_unique<CacheCore>(c->cfg, *c->be);
    for (uint32_t i = 0; i < c->models.size(); ++i)
      if (c->models[i].on_disk)
        c->core->register_disk_file(FakeBackend::key_of(i), "fake://" + std::to_string(i), c->models[i].file_bytes);
    *out = c.release();
    return 0;
  } catch (const Error& e) {
    return int(e.code());
  } catch (...) {
    return int(Errc::Internal);
  }
}

extern "C" void trims_simcore_destroy(trims_simcore* c) {
  if (!c) return;
  c->core.reset();  // before the backend and the directory
  delete c;
}

extern "C" int trims_simcore_step(trims_simcore* c, char kind, uint32_t model, uint64_t now, char* out,
                                  uint64_t cap) {
  try {
    if (!c || model >= c->models.size()) return int(Errc::InvalidArgument);
    const auto key = FakeBackend::key_of(model);
    int outcome = 0, peer = -1;
    try {
      if (kind == 'o') {
        PlacementResult r = open_with_peers(
            *c->core, c->dir.get(), key, {}, now,
            [&](const fmt::ModelKey&) { return c->be->manifest_if_on_disk(model); },
            [&](const DirCoords& d, std::shared_ptr<void>*) {
              PeerSource s;
              s.rank = d.rank;
              s.generation = d.generation;
              return s;
            },
            &c->ctr, &peer);
        outcome = int(r.outcome);
      } else {
        c->core->close_model(key);
      }
    } catch (const Error& e) {
      outcome = kind == 'c' ? 103 : error_outcome(e.code());
    }
    c->be->ev_fast.clear();
    c->be->ev_host.clear();
    c->be->ev_disk.clear();
    std::string line = std::to_string(outcome) + ' ' + std::to_string(c->core->used_bytes(Tier::Fast)) + ' ' +
                       std::to_string(c->core->used_bytes(Tier::Host)) + ' ' +
                       std::to_string(c->core->refcount(key)) + ' ' + std::to_string(peer);
    if (line.size() + 1 > cap) return int(Errc::InvalidArgument);
    std::memcpy(out, line.c_str(), line.size() + 1);
    return 0;
  } catch (const Error& e) {
    return int(e.code());
  } catch (...) {
    return int(Errc::Internal);
  }
}
