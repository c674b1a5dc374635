// ref_shim.cpp — C-ABI driver over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. This file is ours; it is compiled together with
// the reference's own translation units, read in place from
// /root/reference/proj/src (see oracle/Makefile), into oracle/_ref/libmrm_ref.so.
// It replaces the CLI11 tools (proj/tools/*.cpp), which cannot build here, with
// a plain C ABI that tests/golden/make_golden.py and bench.py's reference arm
// call through ctypes. Nothing in the product package links or loads it.
//
// Each entry point names the reference API it drives.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <random>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "mrm/bench/catalog.hpp"
#include "mrm/bench/oracle.hpp"
#include "mrm/bench/simulator.hpp"
#include "mrm/bench/stats_math.hpp"
#include "mrm/cache_core.hpp"
#include "mrm/client.hpp"
#include "mrm/daemon.hpp"
#include "mrm/model_format.hpp"
#include "mrm/sha256.hpp"
#include "mrm/shared_segment.hpp"
#include "mrm/wire_protocol.hpp"

using namespace mrm;
namespace fs = std::filesystem;

namespace {

// Unique daemon socket per call (several reference daemons may run at once in
// one process: the bench's reference arm replays two traces concurrently).
std::string sock_path(const char* tag) {
  static std::atomic<uint64_t> seq{0};
  return "/tmp/mrm-refshim-" + std::string(tag) + "-" + std::to_string(::getpid()) + "-" +
         std::to_string(seq.fetch_add(1)) + ".sock";
}

int put_text(const std::string& s, char* out, uint64_t cap) {
  if (!out || cap == 0) return -1;
  if (s.size() + 1 > cap) return -2;
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = '\0';
  return 0;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    std::fprintf(stderr, "ref_shim: %s\n", e.what());
    return int(e.code());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_shim: %s\n", e.what());
    return 7;
  }
}

// "name dtype d0,d1,...\n" per tensor (manifest order).
std::vector<model::TensorDecl> parse_decls(const char* text) {
  std::vector<model::TensorDecl> decls;
  std::istringstream is(text ? text : "");
  std::string line;
  while (std::getline(is, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string name, dt, dims;
    ls >> name >> dt >> dims;
    model::TensorDecl d;
    d.name = name;
    auto t = model::dtype_from_name(dt);
    if (!t) raise(Errc::InvalidArgument, "dtype " + dt);
    d.dtype = *t;
    size_t pos = 0;
    while (pos < dims.size()) {
      size_t c = dims.find(',', pos);
      if (c == std::string::npos) c = dims.size();
      d.dims.push_back(std::stoull(dims.substr(pos, c - pos)));
      pos = c + 1;
    }
    decls.push_back(std::move(d));
  }
  return decls;
}

bench::CatalogSpec filtered(const char* catalog, const char* only_model) {
  bench::CatalogSpec spec = bench::catalog_by_name(catalog);
  if (only_model && *only_model) {
    std::vector<bench::CatalogModel> keep;
    for (auto& m : spec.models)
      if (m.name == only_model) keep.push_back(m);
    if (keep.empty()) raise(Errc::InvalidArgument, std::string("no model ") + only_model);
    spec.models = keep;
  }
  return spec;
}

double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- wire protocol text form (the same one-line form as our
// trims_wire_encode_text / trims_wire_decode_text, csrc/wire.cpp)
std::string wesc(const std::string& s) {
  std::string o;
  for (unsigned char c : s) {
    if (c <= ' ' || c == '%' || c >= 0x7f) {
      char h[4];
      std::snprintf(h, sizeof h, "%%%02X", c);
      o += h;
    } else {
      o += char(c);
    }
  }
  return o.empty() ? "%" : o;
}

std::string wunesc(const std::string& s) {
  if (s == "%") return "";
  std::string o;
  for (size_t i = 0; i < s.size(); ++i) {
    if (s[i] == '%' && i + 2 < s.size()) {
      o += char(std::stoi(s.substr(i + 1, 2), nullptr, 16));
      i += 2;
    } else {
      o += s[i];
    }
  }
  return o;
}

std::string wf64(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

wire::Message wire_from_text(const std::string& text) {
  std::istringstream is(text);
  std::string kind;
  is >> kind;
  auto s = [&] {
    std::string t;
    if (!(is >> t)) throw std::runtime_error("message text ends early");
    return wunesc(t);
  };
  auto u = [&] { return std::stoull(s()); };
  auto d = [&] { return std::stod(s()); };
  auto gran = [&](uint64_t kind_v, uint64_t block) {
    shm::ShareGranularity g;
    g.kind = shm::GranularityKind(kind_v);
    if (g.kind == shm::GranularityKind::Block) g.block_bytes = block;
    return g;
  };
  if (kind == "open") {
    wire::OpenRequest m;
    m.protocol_version = uint16_t(u());
    m.ns = s();
    m.name = s();
    m.version = s();
    const uint64_t k = u(), b = u();
    m.granularity = gran(k, b);
    m.client_id = u();
    return m;
  }
  if (kind == "openresp") {
    wire::OpenResponse m;
    m.model_id = u();
    m.handle_id = u();
    m.footprint.weights_bytes = u();
    m.footprint.workspace_bytes = u();
    m.footprint.total_bytes = u();
    const uint64_t c = u();
    for (uint64_t i = 0; i < c; ++i) {
      wire::ObjectRef o;
      o.name = s();
      o.segment_token = s();
      o.generation = u();
      o.offset = u();
      o.length = u();
      m.objects.push_back(o);
    }
    const std::string h = s();
    for (int i = 0; i < 32; ++i) m.manifest_digest[size_t(i)] = uint8_t(std::stoi(h.substr(size_t(2 * i), 2), nullptr, 16));
    return m;
  }
  if (kind == "close") {
    wire::CloseRequest m;
    m.protocol_version = uint16_t(u());
    m.model_id = u();
    m.handle_id = u();
    return m;
  }
  if (kind == "closeresp") {
    wire::CloseResponse m;
    m.model_id = u();
    m.refcount = u();
    return m;
  }
  if (kind == "stats") {
    wire::StatsRequest m;
    m.protocol_version = uint16_t(u());
    return m;
  }
  if (kind == "statsresp") {
    wire::StatsResponse m;
    for (auto& t : m.tiers) {
      t.hits = u();
      t.misses = u();
      t.evictions = u();
      t.used_bytes = u();
      t.capacity_bytes = u();
    }
    const uint64_t c = u();
    for (uint64_t i = 0; i < c; ++i) {
      wire::ModelStatsMsg r;
      r.ns = s();
      r.name = s();
      r.version = s();
      r.refcount = u();
      r.use_count = u();
      r.residency = uint8_t(u());
      m.models.push_back(r);
    }
    m.open_requests = u();
    m.open_errors = u();
    m.disk_reads = u();
    m.remote_fetches = u();
    m.fetch_ns = u();
    m.disk_read_ns = u();
    m.copy_ns = u();
    m.export_ns = u();
    m.workspace_headroom = d();
    m.has_calibration = u() != 0;
    if (m.has_calibration) {
      m.calib_q = d();
      m.calib_o = d();
      m.calib_s = d();
    }
    return m;
  }
  if (kind == "error") {
    wire::ErrorMsg m;
    m.code = uint16_t(u());
    m.detail = s();
    return m;
  }
  throw std::runtime_error("unknown message kind " + kind);
}

std::string wire_to_text(const wire::Message& msg) {
  std::ostringstream os;
  auto hex = [](const Digest& dg) {
    std::string h;
    char b[3];
    for (uint8_t x : dg) {
      std::snprintf(b, sizeof b, "%02x", x);
      h += b;
    }
    return h;
  };
  if (const auto* m = std::get_if<wire::OpenRequest>(&msg)) {
    const bool blk = m->granularity.kind == shm::GranularityKind::Block;
    os << "open " << m->protocol_version << ' ' << wesc(m->ns) << ' ' << wesc(m->name) << ' ' << wesc(m->version)
       << ' ' << int(m->granularity.kind) << ' ' << (blk ? m->granularity.block_bytes : 0) << ' ' << m->client_id;
  } else if (const auto* m = std::get_if<wire::OpenResponse>(&msg)) {
    os << "openresp " << m->model_id << ' ' << m->handle_id << ' ' << m->footprint.weights_bytes << ' '
       << m->footprint.workspace_bytes << ' ' << m->footprint.total_bytes << ' ' << m->objects.size();
    for (const auto& o : m->objects)
      os << ' ' << wesc(o.name) << ' ' << wesc(o.segment_token) << ' ' << o.generation << ' ' << o.offset << ' '
         << o.length;
    os << ' ' << hex(m->manifest_digest);
  } else if (const auto* m = std::get_if<wire::CloseRequest>(&msg)) {
    os << "close " << m->protocol_version << ' ' << m->model_id << ' ' << m->handle_id;
  } else if (const auto* m = std::get_if<wire::CloseResponse>(&msg)) {
    os << "closeresp " << m->model_id << ' ' << m->refcount;
  } else if (const auto* m = std::get_if<wire::StatsRequest>(&msg)) {
    os << "stats " << m->protocol_version;
  } else if (const auto* m = std::get_if<wire::StatsResponse>(&msg)) {
    os << "statsresp";
    for (const auto& t : m->tiers)
      os << ' ' << t.hits << ' ' << t.misses << ' ' << t.evictions << ' ' << t.used_bytes << ' ' << t.capacity_bytes;
    os << ' ' << m->models.size();
    for (const auto& r : m->models)
      os << ' ' << wesc(r.ns) << ' ' << wesc(r.name) << ' ' << wesc(r.version) << ' ' << r.refcount << ' '
         << r.use_count << ' ' << int(r.residency);
    os << ' ' << m->open_requests << ' ' << m->open_errors << ' ' << m->disk_reads << ' ' << m->remote_fetches << ' '
       << m->fetch_ns << ' ' << m->disk_read_ns << ' ' << m->copy_ns << ' ' << m->export_ns << ' '
       << wf64(m->workspace_headroom) << ' ' << (m->has_calibration ? 1 : 0);
    if (m->has_calibration) os << ' ' << wf64(m->calib_q) << ' ' << wf64(m->calib_o) << ' ' << wf64(m->calib_s);
  } else if (const auto* m = std::get_if<wire::ErrorMsg>(&msg)) {
    os << "error " << m->code << ' ' << wesc(m->detail);
  }
  return os.str();
}

}  // namespace

extern "C" {

// mrm::Sha256::of (proj/src/sha256.cpp)
int ref_sha256(const void* p, uint64_t n, uint8_t* out32) {
  Digest d = Sha256::of({static_cast<const uint8_t*>(p), size_t(n)});
  std::memcpy(out32, d.data(), 32);
  return 0;
}

// bench::gen_catalog (proj/src/bench/catalog.cpp:130-159)
int ref_gen_catalog(const char* catalog, const char* out_dir, uint64_t seed, const char* only) {
  return guarded([&] {
    bench::gen_catalog(filtered(catalog, only), out_dir, seed);
    return 0;
  });
}

// bench::catalog_manifest + model::manifest_to_json (catalog.cpp:111-128,
// model_format.cpp:179-197)
int ref_catalog_manifest_json(const char* catalog, const char* model, char* out, uint64_t cap) {
  return guarded([&] {
    bench::CatalogSpec spec = filtered(catalog, model);
    model::ModelManifest m = bench::catalog_manifest(spec.models[0], spec.scale_divisor);
    return put_text(model::manifest_to_json(m), out, cap);
  });
}

// model::make_manifest + manifest_to_json (model_format.cpp:158-197)
int ref_make_manifest_json(const char* ns, const char* name, const char* version,
                           const char* decls, uint64_t workspace, char* out, uint64_t cap) {
  return guarded([&] {
    model::ModelManifest m = model::make_manifest({ns, name, version}, parse_decls(decls), workspace);
    return put_text(model::manifest_to_json(m), out, cap);
  });
}

// model::write_model_file (model_format.cpp:293-305). `data` is the tensors'
// bytes concatenated in manifest order with no padding.
int ref_write_model(const char* path, const char* ns, const char* name, const char* version,
                    const char* decls, uint64_t workspace, const uint8_t* data) {
  return guarded([&] {
    model::ModelManifest m = model::make_manifest({ns, name, version}, parse_decls(decls), workspace);
    std::vector<std::vector<uint8_t>> blocks;
    uint64_t pos = 0;
    for (const auto& t : m.tensors) {
      blocks.emplace_back(data + pos, data + pos + t.nbytes);
      pos += t.nbytes;
    }
    model::write_model_file(path, m, blocks);
    return 0;
  });
}

// model::read_manifest(path, full_verify) (model_format.cpp:370-409)
int ref_read_manifest(const char* path, int full_verify, char* json_out, uint64_t cap,
                      uint8_t* checksum, uint64_t* blob_bytes) {
  return guarded([&] {
    model::ModelManifest m = model::read_manifest(fs::path(path), full_verify != 0);
    if (checksum) std::memcpy(checksum, m.checksum.data(), 32);
    if (blob_bytes) *blob_bytes = m.blob_bytes;
    return put_text(model::manifest_to_json(m), json_out, cap);
  });
}

// client::Client::open(force_private) + Client::touch (client.cpp:224-241, 338-359)
int ref_touch_file(const char* path, uint64_t* out) {
  return guarded([&] {
    model::ModelManifest m = model::read_manifest(fs::path(path), false);
    client::ClientConfig cc;
    cc.endpoint = "/nonexistent-mrm-oracle.sock";
    client::Client cli(cc);
    client::OpenOptions o;
    o.force_private = true;
    o.local_path = path;
    client::ModelView v = cli.open(m.key, o);
    *out = cli.touch(v);
    cli.close(v);
    return 0;
  });
}

// shm::layout_for (shared_segment.cpp:63-95) over an artifact's manifest.
// kind: 0 model, 1 layer, 2 block. Emits "name seg offset length\n".
int ref_layout_for(const char* path, int kind, uint64_t block_bytes, char* out, uint64_t cap) {
  return guarded([&] {
    model::ModelManifest m = model::read_manifest(fs::path(path), false);
    shm::ShareGranularity g{shm::GranularityKind(kind), block_bytes};
    shm::ObjectLayout l = shm::layout_for(m, g);
    std::ostringstream os;
    for (const auto& o : l.objects)
      os << o.name << ' ' << o.segment_index << ' ' << o.offset << ' ' << o.length << '\n';
    return put_text(os.str(), out, cap);
  });
}

// Replays one decision trace through BOTH the reference's live CacheCore over
// its FakeBackend (oracle.cpp:14-91) and the reference simulator
// (simulator.cpp:131-254), recording per-op outcome, eviction lists, used
// bytes and refcount. Spec text:
//   cfg <fast> <host> <disk> <policy 0|1> <eager 0|1>
//   model <weights> <file_bytes> <on_disk> <on_remote>     (one per model)
//   op <o|c> <model>                                        (one per op)
// Output, one line per op and per engine:
//   <live|sim> <step> <outcome> <fast_used> <host_used> <refcount> f:<..> h:<..> d:<..>
int ref_replay(const char* spec, char* out, uint64_t cap) {
  return guarded([&] {
    bench::sim::SimConfig cfg;
    std::vector<bench::sim::SimModel> models;
    std::vector<bench::sim::TraceOp> trace;
    std::istringstream is(spec);
    std::string tag;
    while (is >> tag) {
      if (tag == "cfg") {
        int pol, eager;
        is >> cfg.fast_capacity >> cfg.host_capacity >> cfg.disk_capacity >> pol >> eager;
        cfg.policy = cache::Policy(pol);
        cfg.eager_reclaim = eager != 0;
      } else if (tag == "model") {
        bench::sim::SimModel m;
        int d, r;
        is >> m.weights_bytes >> m.file_bytes >> d >> r;
        m.name = "m" + std::to_string(models.size());
        m.on_disk = d != 0;
        m.on_remote = r != 0;
        models.push_back(m);
      } else if (tag == "op") {
        std::string k;
        uint32_t mi;
        is >> k >> mi;
        trace.push_back({k == "o" ? bench::sim::TraceOp::Kind::Open : bench::sim::TraceOp::Kind::Close, mi});
      }
    }
    auto lst = [](const std::vector<uint32_t>& v) {
      std::string s;
      for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
      return s.empty() ? std::string("-") : s;
    };
    std::ostringstream os;
    auto sim_ev = bench::sim::simulate(cfg, models, trace);
    for (size_t s = 0; s < sim_ev.size(); ++s) {
      const auto& e = sim_ev[s];
      os << "sim " << s << ' ' << int(e.outcome) << ' ' << e.fast_used << ' ' << e.host_used << ' '
         << e.refcount << " f:" << lst(e.evicted_fast) << " h:" << lst(e.evicted_host)
         << " d:" << lst(e.evicted_disk) << '\n';
    }

    bench::FakeBackend backend(models);
    cache::CoreConfig cc{cfg.fast_capacity, cfg.host_capacity, cfg.disk_capacity, cfg.policy,
                         cfg.eager_reclaim};
    cache::CacheCore core(cc, backend);
    for (uint32_t i = 0; i < models.size(); ++i)
      if (models[i].on_disk)
        core.register_disk_file(bench::FakeBackend::key_of(i), "fake://" + std::to_string(i),
                                models[i].file_bytes);
    for (size_t s = 0; s < trace.size(); ++s) {
      const auto& op = trace[s];
      auto key = bench::FakeBackend::key_of(op.model);
      int outcome = 0;
      if (op.kind == bench::sim::TraceOp::Kind::Open) {
        try {
          auto r = core.open_model(key, shm::ShareGranularity::model(), s + 1);
          outcome = int(r.outcome);
        } catch (const Error& e) {
          switch (e.code()) {
            case Errc::NotFound: case Errc::RemoteNotFound: outcome = 100; break;
            case Errc::TooLargeForFast: outcome = 101; break;
            case Errc::NoEvictableSpace: outcome = 102; break;
            default: outcome = 199; break;
          }
        }
      } else {
        try {
          core.close_model(key);
        } catch (const Error& e) {
          outcome = 103;
        }
      }
      auto ev = backend.take_evictions();
      os << "live " << s << ' ' << outcome << ' ' << core.used_bytes(cache::Tier::Fast) << ' '
         << core.used_bytes(cache::Tier::Host) << ' ' << core.refcount(key) << " f:" << lst(ev.fast)
         << " h:" << lst(ev.host) << " d:" << lst(ev.disk) << '\n';
    }
    auto st = core.stats();
    os << "stats";
    for (size_t t = 0; t < cache::kTierCount; ++t)
      os << ' ' << st.tiers[t].hits << ' ' << st.tiers[t].misses << ' ' << st.tiers[t].evictions
         << ' ' << st.tiers[t].used_bytes;
    os << ' ' << st.open_requests << ' ' << st.open_errors << ' ' << st.disk_reads << ' '
       << st.remote_fetches << '\n';
    return put_text(os.str(), out, cap);
  });
}

// bench::run_oracle (oracle.cpp:200-323). out6 = traces, ops, divergences,
// pinned, budget, refcount violations.
int ref_run_oracle(uint32_t traces, uint64_t seed, uint32_t max_models, uint32_t max_ops,
                   uint64_t* out6) {
  return guarded([&] {
    bench::OracleParams p;
    p.traces = traces;
    p.seed = seed;
    p.max_models = max_models;
    p.max_ops = max_ops;
    bench::OracleReport r = bench::run_oracle(p);
    out6[0] = r.traces_run;
    out6[1] = r.ops_run;
    out6[2] = r.divergences;
    out6[3] = r.pinned_violations;
    out6[4] = r.budget_violations;
    out6[5] = r.refcount_violations;
    if (!r.first_divergence.empty()) std::fprintf(stderr, "%s\n", r.first_divergence.c_str());
    return 0;
  });
}

// The reference's ingest leg on one artifact: ShmTierBackend::stage_host
// (daemon.cpp:153-158) then publish_fast(from_host) (daemon.cpp:160-209),
// evicting in between reps. out[0] = median stage seconds, out[1] = median
// publish (host -> fast copy) seconds, out[2] = blob bytes.
int ref_ingest(const char* path, int reps, double* out) {
  return guarded([&] {
    model::ModelManifest m = model::read_manifest(fs::path(path), false);
    daemon::ShmTierBackend be(fs::path(path).parent_path().string(), std::nullopt, false);
    std::vector<double> st, pu;
    for (int r = 0; r < reps; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      be.stage_host(1, m, path);
      st.push_back(secs_since(t0));
      auto t1 = std::chrono::steady_clock::now();
      cache::FastPublication pub = be.publish_fast(1, m, true, path);
      pu.push_back(secs_since(t1));
      be.evict_fast(1);
      be.evict_host(1);
    }
    std::sort(st.begin(), st.end());
    std::sort(pu.begin(), pu.end());
    out[0] = st[st.size() / 2];
    out[1] = pu[pu.size() / 2];
    out[2] = double(m.blob_bytes);
    return 0;
  });
}

// The same publish path driven by `threads` concurrent callers, as the
// reference daemon's per-connection threads would (distinct model ids, one
// ShmTierBackend): aggregate bytes/second of publish_fast over `reps` rounds.
// out: [aggregate GB/s of the publishes, threads used]
int ref_ingest_parallel(const char* path, int threads, int reps, double* out) {
  return guarded([&] {
    model::ModelManifest m = model::read_manifest(fs::path(path), false);
    daemon::ShmTierBackend be(fs::path(path).parent_path().string(), std::nullopt, false);
    for (int t = 0; t < threads; ++t) be.stage_host(uint64_t(100 + t), m, path);
    double best = 0;
    for (int r = 0; r < reps; ++r) {
      std::vector<std::thread> ts;
      std::vector<int> ok(size_t(threads), 1);
      auto t0 = std::chrono::steady_clock::now();
      for (int t = 0; t < threads; ++t)
        ts.emplace_back([&, t] {
          try {
            be.publish_fast(uint64_t(100 + t), m, true, path);
          } catch (...) {
            ok[size_t(t)] = 0;
          }
        });
      for (auto& x : ts) x.join();
      const double dt = secs_since(t0);
      for (int t = 0; t < threads; ++t) be.evict_fast(uint64_t(100 + t));
      for (int v : ok)
        if (!v) throw std::runtime_error("a parallel publish failed");
      best = std::max(best, double(threads) * double(m.blob_bytes) / dt / 1e9);
    }
    for (int t = 0; t < threads; ++t) be.evict_host(uint64_t(100 + t));
    out[0] = best;
    out[1] = threads;
    return 0;
  });
}

// bench::run_latency's per-request loop (harness.cpp:99-188) restated over an
// arbitrary artifact (the reference's helper only accepts its catalogs), using
// the reference Daemon + Client unmodified. mode: "cold" (eager reclaim: disk
// load every open), "warm" (fast-tier hit), "host" (host-tier hit: the fast
// tier holds one model and a 64-byte filler evicts it between reps),
// "nodaemon" (private load). out: load_disk_s, init_copy_s, share_overhead_s,
// compute_s, end_to_end_s, open_s (medians by e2e), then touch value bits.
int ref_latency(const char* dir, const char* ns, const char* name, const char* version,
                const char* mode_c, int reps, double* out, uint64_t* touch_out) {
  return guarded([&] {
    std::string mode(mode_c);
    model::ModelKey key{ns, name, version};
    fs::path art = fs::path(dir) / model::canonical_filename(key);
    model::ModelManifest m = model::read_manifest(art, false);
    uint64_t weights = model::estimate_footprint(m).weights_bytes;
    model::ModelKey filler{ns, std::string(name) + "-filler", version};
    if (mode == "host") {
      fs::path fp = fs::path(dir) / model::canonical_filename(filler);
      if (!fs::exists(fp)) {
        model::ModelManifest fm = model::make_manifest(filler, {{"w", {8}, model::DType::F64}}, 0);
        model::write_model_file(fp, fm, {std::vector<uint8_t>(64, 1)});
      }
    }
    std::unique_ptr<daemon::Daemon> dmn;
    if (mode != "nodaemon") {
      daemon::DaemonConfig cfg;
      cfg.listen_path = sock_path("lat");
      cfg.disk_cache_dir = dir;
      cfg.startup_calibration = false;
      cfg.workspace_headroom_fraction = 1.0;
      cfg.fast_capacity_bytes = mode == "host" ? weights : std::max<uint64_t>(weights * 2, 1 << 20);
      cfg.host_capacity_bytes = std::max<uint64_t>(weights * 4, 1 << 20);
      cfg.disk_capacity_bytes = weights * 64 + (64ull << 20);
      cfg.eager_reclaim = mode == "cold";
      dmn = std::make_unique<daemon::Daemon>(cfg);
      dmn->start();
    }
    client::ClientConfig cc;
    cc.endpoint = dmn ? dmn->config().listen_path : "/nonexistent-mrm-oracle.sock";
    cc.model_dirs = {dir};
    client::Client cli(cc);
    client::OpenOptions opts;
    if (mode == "nodaemon") opts.force_private = true;
    else opts.force_shared = true;
    if (mode == "warm" || mode == "host") {
      client::ModelView v = cli.open(key, opts);
      cli.close(v);
    }
    struct Row { double disk, copy, share, compute, e2e, open; };
    std::vector<Row> rows;
    uint64_t touch = 0;
    for (int r = 0; r < reps; ++r) {
      if (mode == "host") {
        client::ModelView f = cli.open(filler, opts);  // evicts `key` from the fast tier
        cli.close(f);
      }
      cache::StatsSnapshot before{};
      if (dmn) before = dmn->stats();
      auto t0 = std::chrono::steady_clock::now();
      client::ModelView v = cli.open(key, opts);
      auto t_open = std::chrono::steady_clock::now();
      touch = cli.touch(v);
      auto t1 = std::chrono::steady_clock::now();
      Row row{};
      if (dmn) {
        cache::StatsSnapshot after = dmn->stats();
        row.disk = double(after.cumulative.disk_read_ns - before.cumulative.disk_read_ns +
                          after.cumulative.fetch_ns - before.cumulative.fetch_ns) / 1e9;
        row.copy = double(after.cumulative.host_to_fast_copy_ns -
                          before.cumulative.host_to_fast_copy_ns) / 1e9;
        row.share = std::max(0.0, v.timings().rpc_s - row.disk - row.copy) + v.timings().attach_s;
      } else {
        row.disk = v.timings().private_load_s;
      }
      cli.close(v);
      row.open = std::chrono::duration<double>(t_open - t0).count();
      row.compute = std::chrono::duration<double>(t1 - t_open).count();
      row.e2e = std::chrono::duration<double>(t1 - t0).count();
      rows.push_back(row);
    }
    std::sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) { return a.e2e < b.e2e; });
    const Row& med = rows[rows.size() / 2];
    out[0] = med.disk;
    out[1] = med.copy;
    out[2] = med.share;
    out[3] = med.compute;
    out[4] = med.e2e;
    out[5] = med.open;
    if (touch_out) *touch_out = touch;
    if (dmn) {
      dmn->request_stop();
      dmn->join();
    }
    return 0;
  });
}

// The reference worker's request stream (harness.cpp:294-300,
// tools/mrm_bench.cpp:107-116): mt19937_64(seed), uniform_real over
// (nextafter(0,1), 1), model = pareto_rank(u, alpha, x_m, active) - 1.
int ref_pareto_trace(uint64_t seed, uint32_t n, double alpha, double x_m, uint32_t active, uint32_t* out) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> uni(std::nextafter(0.0, 1.0), 1.0);
    for (uint32_t i = 0; i < n; ++i) out[i] = uint32_t(bench::pareto_rank(uni(rng), alpha, x_m, active) - 1);
    return 0;
  });
}

// A request trace through the UNMODIFIED reference daemon + client (the
// harness worker loop, harness.cpp:297-322): open(force_shared) -> touch ->
// close per request, catalog keys zoo/<name>@1.0.0 in `dir`. names: one model
// name per line, trace: indices into names. out_s: per-request e2e seconds.
// stats: fast hits, fast misses, fast evictions, open_errors, disk_reads.
int ref_trace(const char* dir, const char* names_c, const uint32_t* trace, uint32_t n, uint64_t fast_cap,
              uint64_t host_cap, uint64_t disk_cap, double* out_s, uint64_t* stats) {
  return guarded([&] {
    std::vector<model::ModelKey> keys;
    std::istringstream is(names_c);
    std::string nm;
    while (is >> nm) keys.push_back({"zoo", nm, "1.0.0"});
    daemon::DaemonConfig cfg;
    cfg.listen_path = sock_path("trace");
    cfg.disk_cache_dir = dir;
    cfg.startup_calibration = false;
    cfg.workspace_headroom_fraction = 1.0;
    cfg.fast_capacity_bytes = fast_cap;
    cfg.host_capacity_bytes = host_cap;
    cfg.disk_capacity_bytes = disk_cap;
    daemon::Daemon dmn(cfg);
    dmn.start();
    client::ClientConfig cc;
    cc.endpoint = cfg.listen_path;
    cc.model_dirs = {dir};
    client::Client cli(cc);
    client::OpenOptions opts;
    opts.force_shared = true;
    for (uint32_t i = 0; i < n; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      client::ModelView v = cli.open(keys.at(trace[i]), opts);
      cli.touch(v);
      auto t1 = std::chrono::steady_clock::now();
      cli.close(v);
      out_s[i] = std::chrono::duration<double>(t1 - t0).count();
    }
    cache::StatsSnapshot st = dmn.stats();
    stats[0] = st.tiers[0].hits;
    stats[1] = st.tiers[0].misses;
    stats[2] = st.tiers[0].evictions;
    stats[3] = st.open_errors;
    stats[4] = st.disk_reads;
    dmn.request_stop();
    dmn.join();
    return 0;
  });
}

// A reference daemon (daemon::Daemon, daemon.cpp:398-601) running inside this
// process for external worker processes (ref_worker): the harness's
// run_workers setup (harness.cpp:275-349) without its CLI11 executable.
// Returns an opaque handle; the socket path is written to endpoint_out.
void* ref_daemon_start(const char* dir, uint64_t fast_cap, uint64_t host_cap, uint64_t disk_cap, int eager,
                       char* endpoint_out, uint64_t cap) {
  try {
    daemon::DaemonConfig cfg;
    cfg.listen_path = sock_path("srv");
    cfg.disk_cache_dir = dir;
    cfg.startup_calibration = false;
    cfg.workspace_headroom_fraction = 1.0;
    cfg.fast_capacity_bytes = fast_cap;
    cfg.host_capacity_bytes = host_cap;
    cfg.disk_capacity_bytes = disk_cap;
    cfg.eager_reclaim = eager != 0;
    auto d = std::make_unique<daemon::Daemon>(cfg);
    d->start();
    if (put_text(cfg.listen_path, endpoint_out, cap) != 0) return nullptr;
    return d.release();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_shim: %s\n", e.what());
    return nullptr;
  }
}

// Stops the daemon; stats: fast hits, fast misses, fast evictions,
// open_errors, disk_reads, fast used bytes.
int ref_daemon_stop(void* h, uint64_t* stats) {
  return guarded([&] {
    std::unique_ptr<daemon::Daemon> d(static_cast<daemon::Daemon*>(h));
    cache::StatsSnapshot st = d->stats();
    if (stats) {
      stats[0] = st.tiers[0].hits;
      stats[1] = st.tiers[0].misses;
      stats[2] = st.tiers[0].evictions;
      stats[3] = st.open_errors;
      stats[4] = st.disk_reads;
      stats[5] = st.tiers[0].used_bytes;
    }
    d->request_stop();
    d->join();
    return 0;
  });
}

// The reference worker's request loop (bench::run_worker, harness.cpp:297-322)
// for one model key: open(force_shared) -> touch -> close, `warmup` untimed
// then `n` timed requests. out_s[i] = open + touch seconds (the harness's
// total_ns); touch_out = the last touch value.
int ref_worker(const char* endpoint, const char* dir, const char* ns, const char* name, const char* version,
               uint32_t n, uint32_t warmup, double* out_s, uint64_t* touch_out) {
  return guarded([&] {
    client::ClientConfig cc;
    cc.endpoint = endpoint;
    cc.model_dirs = {dir};
    client::Client cli(cc);
    client::OpenOptions opts;
    opts.force_shared = true;
    model::ModelKey key{ns, name, version};
    for (uint32_t i = 0; i < warmup + n; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      client::ModelView v = cli.open(key, opts);
      const uint64_t t = cli.touch(v);
      auto t1 = std::chrono::steady_clock::now();
      cli.close(v);
      if (touch_out) *touch_out = t;
      if (i >= warmup) out_s[i - warmup] = std::chrono::duration<double>(t1 - t0).count();
    }
    return 0;
  });
}

// Client::open's placement decision (client.cpp:148-222) against a reference
// daemon configured with (fast_cap, headroom, startup_calibration): opens the
// key with the given granularity (kind 0 model / 1 layer / 2 block) and, when
// has_params, explicit CostModelParams; writes "shared" or "private <reason>"
// and the daemon's published stats (has_calibration, q, o, s).
int ref_client_decision(const char* dir, const char* ns, const char* name, const char* version, int gran_kind,
                        uint64_t block_bytes, int has_params, double q, double o, double s, uint64_t fast_cap,
                        double headroom, int calibrate, char* out, uint64_t cap, double* stats4) {
  return guarded([&] {
    daemon::DaemonConfig cfg;
    cfg.listen_path = sock_path("dec");
    cfg.disk_cache_dir = dir;
    cfg.startup_calibration = calibrate != 0;
    cfg.workspace_headroom_fraction = headroom;
    cfg.fast_capacity_bytes = fast_cap;
    cfg.host_capacity_bytes = fast_cap;
    cfg.disk_capacity_bytes = 64ull << 30;
    daemon::Daemon dmn(cfg);
    dmn.start();
    client::ClientConfig cc;
    cc.endpoint = cfg.listen_path;
    cc.model_dirs = {dir};
    client::Client cli(cc);
    client::OpenOptions opts;
    opts.granularity = gran_kind == 0   ? shm::ShareGranularity::model()
                       : gran_kind == 1 ? shm::ShareGranularity::layer()
                                        : shm::ShareGranularity::block(block_bytes);
    if (has_params) opts.params = client::CostModelParams{q, o, s};
    std::string res;
    {
      client::ModelView v = cli.open({ns, name, version}, opts);
      res = v.origin() == client::Origin::Shared ? "shared"
                                                 : std::string("private ") + client::fallback_reason_name(
                                                                                 v.fallback_reason());
      cli.close(v);
    }
    wire::StatsResponse st = cli.stats();
    stats4[0] = st.has_calibration ? 1 : 0;
    stats4[1] = st.calib_q;
    stats4[2] = st.calib_o;
    stats4[3] = st.calib_s;
    dmn.request_stop();
    dmn.join();
    return put_text(res, out, cap);
  });
}

// wire_protocol.cpp:319-357 encode/decode through the text form
int ref_wire_encode_text(const char* text, uint8_t* out, uint64_t cap, uint64_t* n) {
  return guarded([&] {
    std::vector<uint8_t> f = wire::encode(wire_from_text(text));
    *n = f.size();
    if (f.size() > cap) return -2;
    std::memcpy(out, f.data(), f.size());
    return 0;
  });
}

int ref_wire_decode_text(const uint8_t* frame, uint64_t n, char* out, uint64_t cap) {
  return guarded([&] { return put_text(wire_to_text(wire::decode({frame, size_t(n)})), out, cap); });
}

// One request over the reference FramedSocket (wire_protocol.cpp:395-492) to a
// daemon at `endpoint`; the reply's text form in `out`.
int ref_wire_request(const char* endpoint, const char* text, char* out, uint64_t cap) {
  return guarded([&] {
    wire::FramedSocket sock = wire::FramedSocket::connect(wire::parse_endpoint(endpoint));
    return put_text(wire_to_text(sock.request(wire_from_text(text))), out, cap);
  });
}

}  // extern "C"

