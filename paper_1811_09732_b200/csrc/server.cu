// server.cu — the wire-protocol daemon over a trims_store: the
// reference mrmd's serving loop (proj/src/daemon.cpp:398-560) on the B200
// store. One accept thread per endpoint, one thread per connection, lockstep
// request/reply frames (wire.hpp), a handle registry whose open handles are
// closed when their connection drops, errors collapsed onto the frozen wire
// codes. An OpenResponse's objects tile the RESIDENT blob of the sealed HBM
// segment (layout_for over the resident manifest) and the allocation's fd
// rides the frame as SCM_RIGHTS, so a client process maps the weights
// read-only with no copy.
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/trims.h"
#include "store_api.hpp"
#include "wire.hpp"

using namespace trims;

struct trims_server {
  trims_store* store{nullptr};
  int listen_fd{-1};
  bool unix_socket{false};
  std::string unix_path;
  std::atomic<bool> stopping{false};
  std::thread acceptor;
  std::mutex mu;  // connection fds + threads
  std::vector<int> conn_fds;
  std::vector<std::thread> conns;
  struct Handle {
    fmt::ModelKey key;
    uint64_t model_id{0}, conn{0};
  };
  std::mutex hmu;
  std::map<uint64_t, Handle> handles;
  std::atomic<uint64_t> next_handle{1}, next_conn{1};
  std::atomic<uint64_t> served{0};

  // daemon.cpp:452-476
  wire::OpenResp open(const wire::OpenReq& q, uint64_t conn, int* fd_out) {
    if (stopping) raise(Errc::Internal, "daemon is shutting down");
    const fmt::ModelKey key{q.ns, q.name, q.model_version};
    if (!fmt::valid_key(key)) raise(Errc::ProtocolError, "malformed model key");
    PlacementResult r = store_api::open(store, key, {GranKind(q.gran.kind), q.gran.block_bytes});
    const uint64_t handle = next_handle.fetch_add(1);
    {
      std::lock_guard lk(hmu);
      handles[handle] = {key, r.model_id, conn};
    }
    try {
      wire::OpenResp m;
      m.model_id = r.model_id;
      m.handle_id = handle;
      m.weights_bytes = r.weights_bytes;
      m.workspace_bytes = r.workspace_bytes;
      m.total_bytes = r.weights_bytes + r.workspace_bytes;
      std::copy(r.manifest_digest.begin(), r.manifest_digest.end(), m.digest.begin());
      if (r.segments.empty()) raise(Errc::Internal, "open returned no segment");
      const ExportedSegment& seg = r.segments[0];
      std::shared_ptr<FastRecord> rec = store_api::fast_record(store, r.model_id);
      if (!rec) raise(Errc::Internal, "published model has no fast record");
      // objects tile the resident blob that the segment holds
      const std::vector<ObjectSpan> objs = layout_for(rec->resident, {GranKind(q.gran.kind), q.gran.block_bytes});
      const std::string token = wire::make_token(
          {seg.token, seg.device, seg.alloc_bytes, seg.offset, seg.length});
      for (const ObjectSpan& o : objs) m.objects.push_back({o.name, token, seg.generation, o.offset, o.length});
      *fd_out = seg.fd;
      return m;
    } catch (...) {
      drop_handle(handle);
      throw;
    }
  }

  void drop_handle(uint64_t handle) {
    fmt::ModelKey key;
    {
      std::lock_guard lk(hmu);
      auto it = handles.find(handle);
      if (it == handles.end()) return;
      key = it->second.key;
      handles.erase(it);
    }
    try {
      store_api::close(store, key);
    } catch (const Error&) {
    }
  }

  // daemon.cpp:478-492: any connection may close a handle it learned of
  wire::CloseResp close(const wire::CloseReq& q) {
    fmt::ModelKey key;
    {
      std::lock_guard lk(hmu);
      auto it = handles.find(q.handle_id);
      if (it == handles.end()) raise(Errc::NotOpen, "handle " + std::to_string(q.handle_id));
      if (it->second.model_id != q.model_id) raise(Errc::NotOpen, "handle/model mismatch on close");
      key = it->second.key;
      handles.erase(it);
    }
    return {q.model_id, store_api::close(store, key)};
  }

  // daemon.cpp:515-542, with the store's workspace headroom and its startup
  // calibration (measured on the B200 path at store creation)
  wire::StatsResp stats() {
    const StatsSnapshot st = store_api::stats(store);
    wire::StatsResp m;
    for (int t = 0; t < kTiers; ++t)
      m.tiers[size_t(t)] = {st.tiers[t].hits, st.tiers[t].misses, st.tiers[t].evictions, st.tiers[t].used_bytes,
                            st.tiers[t].capacity_bytes};
    for (const ModelStats& x : st.models)
      m.models.push_back({x.key.ns, x.key.name, x.key.version, x.refcount, x.use_count, x.residency});
    m.open_requests = st.open_requests;
    m.open_errors = st.open_errors;
    m.disk_reads = st.disk_reads;
    m.remote_fetches = st.remote_fetches;
    m.fetch_ns = st.cumulative.fetch_ns;
    m.disk_read_ns = st.cumulative.disk_read_ns;
    m.copy_ns = st.cumulative.host_to_fast_copy_ns;
    m.export_ns = st.cumulative.handle_export_ns;
    m.workspace_headroom = store_api::workspace_headroom(store);
    if (const auto cal = store_api::calibration(store)) {
      m.has_calibration = true;
      m.calib_q = cal->q;
      m.calib_o = cal->o;
      m.calib_s = cal->s;
    }
    return m;
  }

  // daemon.cpp:418-442
  void serve(int fd) {
    const uint64_t conn = next_conn.fetch_add(1);
    try {
      for (;;) {
        auto frame = wire::recv_frame(fd);
        if (!frame) break;
        int pass_fd = -1;
        wire::Msg reply;
        try {
          wire::Msg req = wire::decode(frame->data(), frame->size());
          if (auto* o = std::get_if<wire::OpenReq>(&req)) reply = open(*o, conn, &pass_fd);
          else if (auto* c = std::get_if<wire::CloseReq>(&req)) reply = close(*c);
          else if (std::holds_alternative<wire::StatsReq>(req)) reply = stats();
          else raise(Errc::ProtocolError, "unexpected message type in request position");
        } catch (const Error& e) {
          reply = wire::ErrorResp{uint16_t(wire_code(e.code())), e.what()};
          pass_fd = -1;
        } catch (const std::exception& e) {
          reply = wire::ErrorResp{uint16_t(Errc::Internal), e.what()};
          pass_fd = -1;
        }
        wire::send_frame(fd, wire::encode(reply), unix_socket ? pass_fd : -1);
        served.fetch_add(1);
      }
    } catch (const Error&) {
      // torn down mid-frame: fall through to the handle cleanup
    }
    std::vector<uint64_t> mine;
    {
      std::lock_guard lk(hmu);
      for (const auto& [h, v] : handles)
        if (v.conn == conn) mine.push_back(h);
    }
    for (uint64_t h : mine) drop_handle(h);
    std::lock_guard lk(mu);
    conn_fds.erase(std::remove(conn_fds.begin(), conn_fds.end(), fd), conn_fds.end());
    ::close(fd);
  }

  void accept_loop() {
    while (!stopping) {
      pollfd p{listen_fd, POLLIN, 0};
      if (::poll(&p, 1, 100) <= 0) continue;
      const int fd = ::accept4(listen_fd, nullptr, nullptr, SOCK_CLOEXEC);
      if (fd < 0) continue;
      std::lock_guard lk(mu);
      if (stopping) {
        ::close(fd);
        break;
      }
      conn_fds.push_back(fd);
      conns.emplace_back([this, fd] { serve(fd); });
    }
  }
};

namespace {
template <class F>
int sguard(F&& f) {
  try {
    store_api::set_last_error("");
    return f();
  } catch (const Error& e) {
    store_api::set_last_error(e.what());
    return int(e.code());
  } catch (const std::exception& e) {
    store_api::set_last_error(e.what());
    return int(Errc::Internal);
  }
}
}  // namespace

extern "C" {

int trims_server_start(trims_store* store, const char* endpoint, trims_server** out) {
  return sguard([&] {
    if (!store || !endpoint || !out) raise(Errc::InvalidArgument, "null argument");
    auto s = std::make_unique<trims_server>();
    s->store = store;
    s->listen_fd = wire::listen_endpoint(endpoint, &s->unix_path);
    s->unix_socket = !s->unix_path.empty();
    trims_server* raw = s.get();
    s->acceptor = std::thread([raw] { raw->accept_loop(); });
    *out = s.release();
    return 0;
  });
}

// daemon.cpp:562-601: stop accepting, shut the connections down, join, and
// close every handle still open (their connections are gone).
void trims_server_stop(trims_server* s) {
  if (!s) return;
  s->stopping = true;
  if (s->acceptor.joinable()) s->acceptor.join();
  std::vector<std::thread> conns;
  {
    std::lock_guard lk(s->mu);
    for (int fd : s->conn_fds) ::shutdown(fd, SHUT_RDWR);
    conns.swap(s->conns);
  }
  for (auto& t : conns)
    if (t.joinable()) t.join();
  if (s->listen_fd >= 0) ::close(s->listen_fd);
  if (s->unix_socket) ::unlink(s->unix_path.c_str());
  delete s;
}

uint64_t trims_server_frames_served(trims_server* s) { return s ? s->served.load() : 0; }

// Codec entry points (parity tests against the reference's encoder/decoder):
// text form -> frame bytes, and frame bytes -> text form.
int trims_wire_encode_text(const char* text, uint8_t* out, uint64_t cap, uint64_t* n) {
  return sguard([&] {
    std::vector<uint8_t> f = wire::encode(wire::from_text(text ? text : ""));
    *n = f.size();
    if (f.size() > cap) raise(Errc::InvalidArgument, "output buffer too small");
    std::copy(f.begin(), f.end(), out);
    return 0;
  });
}

int trims_wire_decode_text(const uint8_t* frame, uint64_t n, char* out, uint64_t cap) {
  return sguard([&] {
    const std::string t = wire::to_text(wire::decode(frame, n));
    if (t.size() + 1 > cap) raise(Errc::InvalidArgument, "output buffer too small");
    std::copy(t.begin(), t.end(), out);
    out[t.size()] = '\0';
    return 0;
  });
}

}  // extern "C"
