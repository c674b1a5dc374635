// wire.cpp — v1 frame codec (byte layout of proj/src/wire_protocol.cpp:124-357)
// and the socket transport, with SCM_RIGHTS fd passing for the B200 store.
#include "wire.hpp"

#include <arpa/inet.h>
#include <netinet/in.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cerrno>
#include <cstdio>
#include <cstring>
#include <sstream>

namespace trims::wire {

namespace {

// ---- little-endian field writer / bounds-checked reader

struct Out {
  std::vector<uint8_t> b;
  template <class T>
  void le(T v, int bytes) {
    for (int i = 0; i < bytes; ++i) b.push_back(uint8_t(uint64_t(v) >> (8 * i)));
  }
  void u8(uint8_t v) { b.push_back(v); }
  void u16(uint16_t v) { le(v, 2); }
  void u32(uint32_t v) { le(v, 4); }
  void u64(uint64_t v) { le(v, 8); }
  void f64(double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    u64(u);
  }
  void str(const std::string& s) {
    if (s.size() > 0xffff) raise(Errc::ProtocolError, "string too long to encode");
    u16(uint16_t(s.size()));
    b.insert(b.end(), s.begin(), s.end());
  }
  void gran(const Gran& g) {
    u8(g.kind);
    if (g.kind == 2) u64(g.block_bytes);
  }
};

struct In {
  const uint8_t* p;
  size_t n, at{0};
  void need(size_t k) const {
    if (k > n - at) raise(Errc::TruncatedFrame, "payload ends mid-field");
  }
  uint64_t le(int bytes) {
    need(size_t(bytes));
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= uint64_t(p[at + i]) << (8 * i);
    at += size_t(bytes);
    return v;
  }
  uint8_t u8() { return uint8_t(le(1)); }
  uint16_t u16() { return uint16_t(le(2)); }
  uint32_t u32() { return uint32_t(le(4)); }
  uint64_t u64() { return le(8); }
  double f64() {
    uint64_t u = u64();
    double d;
    std::memcpy(&d, &u, 8);
    return d;
  }
  std::string str() {
    const uint16_t k = u16();
    need(k);
    std::string s(reinterpret_cast<const char*>(p + at), k);
    at += k;
    return s;
  }
  Gran gran() {
    Gran g;
    g.kind = u8();
    if (g.kind > 2) raise(Errc::ProtocolError, "bad granularity tag");
    if (g.kind == 2) {
      g.block_bytes = u64();
      if (g.block_bytes == 0 || g.block_bytes % 64) raise(Errc::ProtocolError, "bad block_bytes");
    }
    return g;
  }
  // list count whose minimal encoding must still fit in the payload
  uint32_t count(size_t min_elem) {
    const uint32_t c = u32();
    if (uint64_t(c) * min_elem > n - at) raise(Errc::TruncatedFrame, "list count exceeds payload");
    return c;
  }
  uint16_t version() {
    const uint16_t v = u16();
    if (v != kVersion) raise(Errc::BadVersion, "protocol_version " + std::to_string(v));
    return v;
  }
};

void put(Out& o, const OpenReq& m) {
  o.u16(m.version);
  o.str(m.ns);
  o.str(m.name);
  o.str(m.model_version);
  o.gran(m.gran);
  o.u64(m.client_id);
}
void put(Out& o, const OpenResp& m) {
  for (uint64_t v : {m.model_id, m.handle_id, m.weights_bytes, m.workspace_bytes, m.total_bytes}) o.u64(v);
  o.u32(uint32_t(m.objects.size()));
  for (const Object& x : m.objects) {
    o.str(x.name);
    o.str(x.token);
    for (uint64_t v : {x.generation, x.offset, x.length}) o.u64(v);
  }
  o.b.insert(o.b.end(), m.digest.begin(), m.digest.end());
}
void put(Out& o, const CloseReq& m) {
  o.u16(m.version);
  o.u64(m.model_id);
  o.u64(m.handle_id);
}
void put(Out& o, const CloseResp& m) {
  o.u64(m.model_id);
  o.u64(m.refcount);
}
void put(Out& o, const StatsReq& m) { o.u16(m.version); }
void put(Out& o, const StatsResp& m) {
  for (const TierRow& t : m.tiers)
    for (uint64_t v : {t.hits, t.misses, t.evictions, t.used_bytes, t.capacity_bytes}) o.u64(v);
  o.u32(uint32_t(m.models.size()));
  for (const ModelRow& r : m.models) {
    o.str(r.ns);
    o.str(r.name);
    o.str(r.version);
    o.u64(r.refcount);
    o.u64(r.use_count);
    o.u8(r.residency);
  }
  for (uint64_t v : {m.open_requests, m.open_errors, m.disk_reads, m.remote_fetches, m.fetch_ns, m.disk_read_ns,
                     m.copy_ns, m.export_ns})
    o.u64(v);
  o.f64(m.workspace_headroom);
  o.u8(m.has_calibration ? 1 : 0);
  if (m.has_calibration)
    for (double v : {m.calib_q, m.calib_o, m.calib_s}) o.f64(v);
}
void put(Out& o, const ErrorResp& m) {
  o.u16(m.code);
  o.str(m.detail);
}

Msg get(Type t, In& in) {
  switch (t) {
    case Type::OpenRequest: {
      OpenReq m;
      m.version = in.version();
      m.ns = in.str();
      m.name = in.str();
      m.model_version = in.str();
      m.gran = in.gran();
      m.client_id = in.u64();
      return m;
    }
    case Type::OpenResponse: {
      OpenResp m;
      m.model_id = in.u64();
      m.handle_id = in.u64();
      m.weights_bytes = in.u64();
      m.workspace_bytes = in.u64();
      m.total_bytes = in.u64();
      const uint32_t c = in.count(2 + 2 + 3 * 8);
      for (uint32_t i = 0; i < c; ++i) {
        Object x;
        x.name = in.str();
        x.token = in.str();
        x.generation = in.u64();
        x.offset = in.u64();
        x.length = in.u64();
        m.objects.push_back(std::move(x));
      }
      in.need(32);
      std::memcpy(m.digest.data(), in.p + in.at, 32);
      in.at += 32;
      return m;
    }
    case Type::CloseRequest: {
      CloseReq m;
      m.version = in.version();
      m.model_id = in.u64();
      m.handle_id = in.u64();
      return m;
    }
    case Type::CloseResponse: {
      CloseResp m;
      m.model_id = in.u64();
      m.refcount = in.u64();
      return m;
    }
    case Type::StatsRequest: {
      StatsReq m;
      m.version = in.version();
      return m;
    }
    case Type::StatsResponse: {
      StatsResp m;
      for (TierRow& r : m.tiers) {
        r.hits = in.u64();
        r.misses = in.u64();
        r.evictions = in.u64();
        r.used_bytes = in.u64();
        r.capacity_bytes = in.u64();
      }
      const uint32_t c = in.count(3 * 2 + 2 * 8 + 1);
      for (uint32_t i = 0; i < c; ++i) {
        ModelRow r;
        r.ns = in.str();
        r.name = in.str();
        r.version = in.str();
        r.refcount = in.u64();
        r.use_count = in.u64();
        r.residency = in.u8();
        m.models.push_back(std::move(r));
      }
      uint64_t* f[] = {&m.open_requests, &m.open_errors, &m.disk_reads, &m.remote_fetches,
                       &m.fetch_ns,      &m.disk_read_ns, &m.copy_ns,   &m.export_ns};
      for (uint64_t* v : f) *v = in.u64();
      m.workspace_headroom = in.f64();
      m.has_calibration = in.u8() != 0;
      if (m.has_calibration) {
        m.calib_q = in.f64();
        m.calib_o = in.f64();
        m.calib_s = in.f64();
      }
      return m;
    }
    case Type::Error: {
      ErrorResp m;
      m.code = in.u16();
      m.detail = in.str();
      return m;
    }
  }
  raise(Errc::UnknownMessageType, std::to_string(int(t)));
}

bool known(uint8_t t) { return (t >= 1 && t <= 6) || t == 0x7F; }

// ---- text form

std::string esc(const std::string& s) {
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
  return o.empty() ? "%" : o;  // "%" alone = empty string
}

std::string unesc(const std::string& s) {
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

std::string f64s(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

}  // namespace

Type type_of(const Msg& m) {
  static constexpr Type kTypes[] = {Type::OpenRequest,  Type::OpenResponse,  Type::CloseRequest, Type::CloseResponse,
                                    Type::StatsRequest, Type::StatsResponse, Type::Error};
  return kTypes[m.index()];
}

std::vector<uint8_t> encode(const Msg& m) {
  Out o;
  o.b.resize(5);
  std::visit([&](const auto& x) { put(o, x); }, m);
  const size_t len = o.b.size() - 5;
  if (len + 1 > kMaxFrame) raise(Errc::FrameTooLarge, "encoded frame too large");
  for (int i = 0; i < 4; ++i) o.b[i] = uint8_t(len >> (8 * i));
  o.b[4] = uint8_t(type_of(m));
  return std::move(o.b);
}

Msg decode(const uint8_t* frame, size_t n) {
  if (n < 5) raise(Errc::TruncatedFrame, "frame shorter than header");
  uint32_t len = 0;
  for (int i = 0; i < 4; ++i) len |= uint32_t(frame[i]) << (8 * i);
  if (len > kMaxFrame) raise(Errc::FrameTooLarge, std::to_string(len));
  if (uint64_t(len) + 5 != n) raise(Errc::TruncatedFrame, "declared length does not match the frame");
  if (!known(frame[4])) raise(Errc::UnknownMessageType, std::to_string(int(frame[4])));
  In in{frame + 5, len};
  Msg m = get(Type(frame[4]), in);
  if (in.at != in.n) raise(Errc::ProtocolError, "trailing bytes in frame");
  return m;
}

std::string to_text(const Msg& m) {
  std::ostringstream os;
  auto hex = [](const std::array<uint8_t, 32>& d) {
    std::string h;
    char b[3];
    for (uint8_t x : d) {
      std::snprintf(b, sizeof b, "%02x", x);
      h += b;
    }
    return h;
  };
  std::visit(
      [&](const auto& x) {
        using T = std::decay_t<decltype(x)>;
        if constexpr (std::is_same_v<T, OpenReq>) {
          os << "open " << x.version << ' ' << esc(x.ns) << ' ' << esc(x.name) << ' ' << esc(x.model_version) << ' '
             << int(x.gran.kind) << ' ' << x.gran.block_bytes << ' ' << x.client_id;
        } else if constexpr (std::is_same_v<T, OpenResp>) {
          os << "openresp " << x.model_id << ' ' << x.handle_id << ' ' << x.weights_bytes << ' ' << x.workspace_bytes
             << ' ' << x.total_bytes << ' ' << x.objects.size();
          for (const Object& o : x.objects)
            os << ' ' << esc(o.name) << ' ' << esc(o.token) << ' ' << o.generation << ' ' << o.offset << ' '
               << o.length;
          os << ' ' << hex(x.digest);
        } else if constexpr (std::is_same_v<T, CloseReq>) {
          os << "close " << x.version << ' ' << x.model_id << ' ' << x.handle_id;
        } else if constexpr (std::is_same_v<T, CloseResp>) {
          os << "closeresp " << x.model_id << ' ' << x.refcount;
        } else if constexpr (std::is_same_v<T, StatsReq>) {
          os << "stats " << x.version;
        } else if constexpr (std::is_same_v<T, StatsResp>) {
          os << "statsresp";
          for (const TierRow& t : x.tiers)
            os << ' ' << t.hits << ' ' << t.misses << ' ' << t.evictions << ' ' << t.used_bytes << ' '
               << t.capacity_bytes;
          os << ' ' << x.models.size();
          for (const ModelRow& r : x.models)
            os << ' ' << esc(r.ns) << ' ' << esc(r.name) << ' ' << esc(r.version) << ' ' << r.refcount << ' '
               << r.use_count << ' ' << int(r.residency);
          os << ' ' << x.open_requests << ' ' << x.open_errors << ' ' << x.disk_reads << ' ' << x.remote_fetches << ' '
             << x.fetch_ns << ' ' << x.disk_read_ns << ' ' << x.copy_ns << ' ' << x.export_ns << ' '
             << f64s(x.workspace_headroom) << ' ' << (x.has_calibration ? 1 : 0);
          if (x.has_calibration) os << ' ' << f64s(x.calib_q) << ' ' << f64s(x.calib_o) << ' ' << f64s(x.calib_s);
        } else {
          os << "error " << x.code << ' ' << esc(x.detail);
        }
      },
      m);
  return os.str();
}

Msg from_text(const std::string& text) {
  std::istringstream is(text);
  std::string kind;
  is >> kind;
  auto s = [&] {
    std::string t;
    if (!(is >> t)) raise(Errc::InvalidArgument, "message text ends early");
    return unesc(t);
  };
  auto u = [&] { return std::stoull(s()); };
  auto d = [&] { return std::stod(s()); };
  if (kind == "open") {
    OpenReq m;
    m.version = uint16_t(u());
    m.ns = s();
    m.name = s();
    m.model_version = s();
    m.gran.kind = uint8_t(u());
    m.gran.block_bytes = u();
    m.client_id = u();
    return m;
  }
  if (kind == "openresp") {
    OpenResp m;
    m.model_id = u();
    m.handle_id = u();
    m.weights_bytes = u();
    m.workspace_bytes = u();
    m.total_bytes = u();
    const uint64_t c = u();
    for (uint64_t i = 0; i < c; ++i) {
      Object o;
      o.name = s();
      o.token = s();
      o.generation = u();
      o.offset = u();
      o.length = u();
      m.objects.push_back(std::move(o));
    }
    const std::string h = s();
    if (h.size() != 64) raise(Errc::InvalidArgument, "digest must be 64 hex digits");
    for (int i = 0; i < 32; ++i) m.digest[size_t(i)] = uint8_t(std::stoi(h.substr(size_t(2 * i), 2), nullptr, 16));
    return m;
  }
  if (kind == "close") {
    CloseReq m;
    m.version = uint16_t(u());
    m.model_id = u();
    m.handle_id = u();
    return m;
  }
  if (kind == "closeresp") return CloseResp{u(), u()};
  if (kind == "stats") return StatsReq{uint16_t(u())};
  if (kind == "statsresp") {
    StatsResp m;
    for (TierRow& t : m.tiers) t = {u(), u(), u(), u(), u()};
    const uint64_t c = u();
    for (uint64_t i = 0; i < c; ++i) {
      ModelRow r;
      r.ns = s();
      r.name = s();
      r.version = s();
      r.refcount = u();
      r.use_count = u();
      r.residency = uint8_t(u());
      m.models.push_back(std::move(r));
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
    ErrorResp m;
    m.code = uint16_t(u());
    m.detail = s();
    return m;
  }
  raise(Errc::InvalidArgument, "unknown message kind " + kind);
}

std::string make_token(const TokenInfo& t) {
  return t.base + "?dev=" + std::to_string(t.device) + "&alloc=" + std::to_string(t.alloc_bytes) +
         "&seg=" + std::to_string(t.segment_offset) + "&payload=" + std::to_string(t.payload_bytes);
}

TokenInfo parse_token(const std::string& token) {
  TokenInfo t;
  const size_t q = token.find('?');
  t.base = token.substr(0, q);
  if (q == std::string::npos) raise(Errc::ProtocolError, "token carries no CUDA coordinates: " + token);
  std::istringstream is(token.substr(q + 1));
  std::string kv;
  int seen = 0;
  while (std::getline(is, kv, '&')) {
    const size_t eq = kv.find('=');
    if (eq == std::string::npos) continue;
    const std::string k = kv.substr(0, eq);
    const uint64_t v = std::stoull(kv.substr(eq + 1));
    if (k == "dev") t.device = int(v), seen |= 1;
    else if (k == "alloc") t.alloc_bytes = v, seen |= 2;
    else if (k == "seg") t.segment_offset = v, seen |= 4;
    else if (k == "payload") t.payload_bytes = v, seen |= 8;
  }
  if (seen != 15) raise(Errc::ProtocolError, "incomplete token " + token);
  return t;
}

// ---- transport

namespace {

bool is_tcp(const std::string& ep, std::string* host, uint16_t* port) {
  if (ep.rfind("tcp:", 0) != 0) return false;
  const std::string rest = ep.substr(4);
  const size_t c = rest.rfind(':');
  if (c == std::string::npos) raise(Errc::InvalidArgument, "tcp endpoint needs host:port");
  *host = rest.substr(0, c);
  *port = uint16_t(std::stoi(rest.substr(c + 1)));
  return true;
}

std::string unix_path_of(const std::string& ep) { return ep.rfind("unix:", 0) == 0 ? ep.substr(5) : ep; }

sockaddr_un unix_addr(const std::string& path) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  if (path.size() >= sizeof(a.sun_path)) raise(Errc::InvalidArgument, "socket path too long");
  std::memcpy(a.sun_path, path.c_str(), path.size() + 1);
  return a;
}

void read_exact(int sock, uint8_t* p, size_t n, bool eof_ok, bool* eof, int* fd_out) {
  size_t got = 0;
  while (got < n) {
    char ctl[CMSG_SPACE(sizeof(int))];
    iovec iov{p + got, n - got};
    msghdr mh{};
    mh.msg_iov = &iov;
    mh.msg_iovlen = 1;
    mh.msg_control = ctl;
    mh.msg_controllen = sizeof ctl;
    const ssize_t r = ::recvmsg(sock, &mh, MSG_CMSG_CLOEXEC);
    if (r < 0 && errno == EINTR) continue;
    if (r < 0) raise(Errc::ConnectionLost, std::string("recv: ") + std::strerror(errno));
    for (cmsghdr* c = CMSG_FIRSTHDR(&mh); c; c = CMSG_NXTHDR(&mh, c))
      if (c->cmsg_level == SOL_SOCKET && c->cmsg_type == SCM_RIGHTS) {
        int fd;
        std::memcpy(&fd, CMSG_DATA(c), sizeof fd);
        if (fd_out && *fd_out < 0) *fd_out = fd;
        else ::close(fd);
      }
    if (r == 0) {
      if (got == 0 && eof_ok) {
        *eof = true;
        return;
      }
      raise(Errc::ConnectionLost, "peer closed mid-frame");
    }
    got += size_t(r);
  }
}

}  // namespace

int listen_endpoint(const std::string& endpoint, std::string* unix_path) {
  std::string host;
  uint16_t port = 0;
  int fd = -1;
  if (is_tcp(endpoint, &host, &port)) {
    fd = ::socket(AF_INET, SOCK_STREAM | SOCK_CLOEXEC, 0);
    int one = 1;
    ::setsockopt(fd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
    sockaddr_in a{};
    a.sin_family = AF_INET;
    a.sin_port = htons(port);
    if (::inet_pton(AF_INET, host.c_str(), &a.sin_addr) != 1) {
      ::close(fd);
      raise(Errc::InvalidArgument, "bad host " + host);
    }
    if (::bind(fd, reinterpret_cast<sockaddr*>(&a), sizeof a) || ::listen(fd, 128)) {
      const int e = errno;
      ::close(fd);
      raise(Errc::Internal, "bind/listen " + endpoint + ": " + std::strerror(e));
    }
    if (unix_path) unix_path->clear();
    return fd;
  }
  const std::string path = unix_path_of(endpoint);
  ::unlink(path.c_str());
  fd = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  sockaddr_un a = unix_addr(path);
  if (::bind(fd, reinterpret_cast<sockaddr*>(&a), sizeof a) || ::listen(fd, 128)) {
    const int e = errno;
    ::close(fd);
    raise(Errc::Internal, "bind/listen " + path + ": " + std::strerror(e));
  }
  if (unix_path) *unix_path = path;
  return fd;
}

int connect_endpoint(const std::string& endpoint) {
  std::string host;
  uint16_t port = 0;
  int fd = -1;
  int rc = 0;
  if (is_tcp(endpoint, &host, &port)) {
    fd = ::socket(AF_INET, SOCK_STREAM | SOCK_CLOEXEC, 0);
    sockaddr_in a{};
    a.sin_family = AF_INET;
    a.sin_port = htons(port);
    if (::inet_pton(AF_INET, host.c_str(), &a.sin_addr) != 1) {
      ::close(fd);
      raise(Errc::DaemonUnreachable, "bad host " + host);
    }
    rc = ::connect(fd, reinterpret_cast<sockaddr*>(&a), sizeof a);
  } else {
    fd = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    sockaddr_un a = unix_addr(unix_path_of(endpoint));
    rc = ::connect(fd, reinterpret_cast<sockaddr*>(&a), sizeof a);
  }
  if (rc) {
    const int e = errno;
    ::close(fd);
    raise(Errc::DaemonUnreachable, "connect " + endpoint + ": " + std::strerror(e));
  }
  return fd;
}

void send_frame(int sock, const std::vector<uint8_t>& frame, int fd) {
  size_t sent = 0;
  bool fd_pending = fd >= 0;
  while (sent < frame.size()) {
    iovec iov{const_cast<uint8_t*>(frame.data()) + sent, frame.size() - sent};
    msghdr mh{};
    mh.msg_iov = &iov;
    mh.msg_iovlen = 1;
    char ctl[CMSG_SPACE(sizeof(int))];
    if (fd_pending) {  // the fd rides the first bytes of the frame
      std::memset(ctl, 0, sizeof ctl);
      mh.msg_control = ctl;
      mh.msg_controllen = sizeof ctl;
      cmsghdr* c = CMSG_FIRSTHDR(&mh);
      c->cmsg_level = SOL_SOCKET;
      c->cmsg_type = SCM_RIGHTS;
      c->cmsg_len = CMSG_LEN(sizeof(int));
      std::memcpy(CMSG_DATA(c), &fd, sizeof fd);
    }
    const ssize_t r = ::sendmsg(sock, &mh, MSG_NOSIGNAL);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) raise(Errc::ConnectionLost, std::string("send: ") + std::strerror(errno));
    fd_pending = false;
    sent += size_t(r);
  }
}

std::optional<std::vector<uint8_t>> recv_frame(int sock, int* fd_out) {
  if (fd_out) *fd_out = -1;
  uint8_t head[5];
  bool eof = false;
  read_exact(sock, head, 5, true, &eof, fd_out);
  if (eof) return std::nullopt;
  uint32_t len = 0;
  for (int i = 0; i < 4; ++i) len |= uint32_t(head[i]) << (8 * i);
  if (len > kMaxFrame) raise(Errc::FrameTooLarge, std::to_string(len));
  std::vector<uint8_t> frame(5 + size_t(len));
  std::memcpy(frame.data(), head, 5);
  if (len) read_exact(sock, frame.data() + 5, len, false, &eof, fd_out);
  return frame;
}

}  // namespace trims::wire
