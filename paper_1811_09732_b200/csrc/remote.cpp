// remote.cpp — see remote.hpp.
//
// Structure: a fetch is "produce the bytes into a private staging file, then
// admit it". Producing is the backend's job (DirSource copies, HttpSource runs
// one GET over a plain socket); admission is one place (StagedFile::admit):
// a full artifact verification, then an atomic rename onto the canonical name.
// A StagedFile that is not admitted deletes itself, so no error path can leave
// a half-written or unverified file in the disk cache
// (behaviour of proj/src/remote_store.cpp:74-120).
#include "remote.hpp"

#include <fcntl.h>
#include <netdb.h>
#include <sys/socket.h>
#include <sys/stat.h>
#include <sys/time.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <filesystem>
#include <optional>
#include <vector>

#include "errc.hpp"

namespace trims::remote {

namespace fs = std::filesystem;

namespace {

// The verification verdict of an artifact on disk: nullopt = valid, else the
// error a full read_artifact_info raised.
std::optional<Error> verdict(const fs::path& p) {
  try {
    fmt::read_artifact_info(p.string(), /*full_verify=*/true);
    return std::nullopt;
  } catch (const Error& e) {
    return e;
  } catch (const std::exception& e) {
    return Error(Errc::CorruptManifest, e.what());
  }
}

class UniqueFd {
 public:
  explicit UniqueFd(int fd = -1) : fd_(fd) {}
  UniqueFd(const UniqueFd&) = delete;
  UniqueFd& operator=(const UniqueFd&) = delete;
  ~UniqueFd() { reset(); }
  void reset(int fd = -1) {
    if (fd_ >= 0) ::close(fd_);
    fd_ = fd;
  }
  int get() const { return fd_; }

 private:
  int fd_;
};

// `<dest_dir>/<file>.part.<pid>`: the only place a download is written to.
class StagedFile {
 public:
  StagedFile(const fs::path& dest_dir, const std::string& filename)
      : path_(dest_dir / (filename + ".part." + std::to_string(::getpid()))), dest_(dest_dir / filename) {}
  ~StagedFile() {
    if (!admitted_) {
      std::error_code ec;
      fs::remove(path_, ec);
    }
  }
  const fs::path& path() const { return path_; }

  int open_for_write() {
    int fd = ::open(path_.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
    if (fd < 0) raise(Errc::TransportError, "cannot write " + path_.string());
    return fd;
  }
  void append(int fd, const char* p, size_t n) {
    for (size_t done = 0; done < n;) {
      const ssize_t w = ::write(fd, p + done, n - done);
      if (w > 0) {
        done += size_t(w);
      } else if (!(w < 0 && errno == EINTR)) {
        raise(Errc::TransportError, "cannot write " + path_.string());
      }
    }
  }

  // Verify, then rename onto the canonical name. A download that does not
  // verify is reported as ChecksumMismatch whatever the parser's complaint.
  fs::path admit() {
    if (auto bad = verdict(path_)) {
      if (bad->code() == Errc::ChecksumMismatch) throw *bad;
      raise(Errc::ChecksumMismatch, std::string("fetched artifact invalid: ") + bad->what());
    }
    std::error_code ec;
    fs::rename(path_, dest_, ec);
    if (ec) raise(Errc::TransportError, "rename to " + dest_.string() + ": " + ec.message());
    admitted_ = true;
    return dest_;
  }

 private:
  fs::path path_, dest_;
  bool admitted_{false};
};

// ---- dir: backend ----------------------------------------------------------

void produce_from_dir(const std::string& root, const std::string& filename, StagedFile& staged) {
  const fs::path src = fs::path(root) / filename;
  std::error_code ec;
  if (!fs::exists(src, ec)) raise(Errc::RemoteNotFound, src.string());
  fs::copy_file(src, staged.path(), fs::copy_options::overwrite_existing, ec);
  if (ec) raise(Errc::TransportError, "copy " + src.string() + ": " + ec.message());
}

// ---- http:// backend -------------------------------------------------------

struct Endpoint {
  std::string authority;  // host[:port], as sent in the Host header
  std::string host, port{"80"};
  std::string prefix;  // path prefix without a trailing '/'
};

Endpoint parse_http_url(const std::string& url) {
  constexpr std::string_view kScheme = "http://";
  if (url.compare(0, kScheme.size(), kScheme) != 0) raise(Errc::InvalidArgument, "expected http:// url");
  const std::string rest = url.substr(kScheme.size());
  Endpoint ep;
  const size_t path_at = rest.find('/');
  ep.authority = rest.substr(0, path_at);
  if (path_at != std::string::npos) {
    ep.prefix = rest.substr(path_at);
    ep.prefix.erase(ep.prefix.find_last_not_of('/') + 1);
  }
  ep.host = ep.authority;
  const size_t colon = ep.authority.rfind(':');
  const bool bracketed_v6 = ep.authority.find(']') != std::string::npos;
  if (colon != std::string::npos && !bracketed_v6) {
    ep.host = ep.authority.substr(0, colon);
    ep.port = ep.authority.substr(colon + 1);
  }
  return ep;
}

int dial(const Endpoint& ep, const std::string& what) {
  addrinfo hints{};
  hints.ai_family = AF_UNSPEC;
  hints.ai_socktype = SOCK_STREAM;
  addrinfo* found = nullptr;
  if (int rc = ::getaddrinfo(ep.host.c_str(), ep.port.c_str(), &hints, &found); rc != 0)
    raise(Errc::TransportError, what + ": resolve " + ep.host + ": " + gai_strerror(rc));
  int fd = -1;
  for (addrinfo* ai = found; ai && fd < 0; ai = ai->ai_next) {
    fd = ::socket(ai->ai_family, ai->ai_socktype | SOCK_CLOEXEC, ai->ai_protocol);
    if (fd >= 0 && ::connect(fd, ai->ai_addr, ai->ai_addrlen) != 0) {
      ::close(fd);
      fd = -1;
    }
  }
  ::freeaddrinfo(found);
  if (fd < 0) raise(Errc::TransportError, what + ": connection to " + ep.authority + " failed");
  timeval tv{60, 0};  // a stalled server fails the fetch after 60 s of silence
  ::setsockopt(fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));
  return fd;
}

// Response reader: a 64 KiB window over the socket.
class Reader {
 public:
  explicit Reader(int fd) : fd_(fd), win_(1 << 16) {}

  std::string line() {
    std::string s;
    for (;;) {
      if (!more()) raise(Errc::TransportError, "connection closed in the response head");
      const char* b = win_.data() + at_;
      const char* nl = static_cast<const char*>(std::memchr(b, '\n', end_ - at_));
      const size_t take = nl ? size_t(nl - b) : end_ - at_;
      s.append(b, take);
      at_ += take + (nl ? 1 : 0);
      if (s.size() > 16384) raise(Errc::TransportError, "response line too long");
      if (nl) {
        if (!s.empty() && s.back() == '\r') s.pop_back();
        return s;
      }
    }
  }
  // Moves `n` body bytes (all remaining bytes when n is nullopt) into `sink`.
  template <class Sink>
  void body(std::optional<uint64_t> n, Sink&& sink) {
    uint64_t left = n.value_or(~0ull);
    while (left) {
      if (!more()) {
        if (!n) return;
        raise(Errc::TransportError, "connection closed mid-body");
      }
      const size_t take = size_t(std::min<uint64_t>(left, end_ - at_));
      sink(win_.data() + at_, take);
      at_ += take;
      if (n) left -= take;
    }
  }

 private:
  bool more() {
    while (at_ == end_) {
      const ssize_t r = ::recv(fd_, win_.data(), win_.size(), 0);
      if (r < 0 && errno == EINTR) continue;
      if (r < 0) raise(Errc::TransportError, std::string("recv: ") + std::strerror(errno));
      if (r == 0) return false;
      at_ = 0;
      end_ = size_t(r);
    }
    return true;
  }
  int fd_;
  std::vector<char> win_;
  size_t at_{0}, end_{0};
};

struct ResponseHead {
  int status{0};
  std::optional<uint64_t> content_length;
  bool chunked{false};
};

ResponseHead read_head(Reader& in, const std::string& what) {
  ResponseHead h;
  const std::string status = in.line();  // "HTTP/1.x NNN reason"
  if (status.compare(0, 5, "HTTP/") != 0 || status.size() < 12 || std::sscanf(status.c_str() + 9, "%d", &h.status) != 1)
    raise(Errc::TransportError, what + ": bad status line");
  for (std::string field = in.line(); !field.empty(); field = in.line()) {
    const size_t colon = field.find(':');
    if (colon == std::string::npos) continue;
    std::string name = field.substr(0, colon), value = field.substr(colon + 1);
    for (auto& ch : name) ch = char(std::tolower(static_cast<unsigned char>(ch)));
    value.erase(0, value.find_first_not_of(' '));
    if (name == "content-length") {
      h.content_length = std::stoull(value);
    } else if (name == "transfer-encoding") {
      for (auto& ch : value) ch = char(std::tolower(static_cast<unsigned char>(ch)));
      h.chunked = value.find("chunked") != std::string::npos;
    }
  }
  return h;
}

void produce_from_http(const std::string& url, const std::string& filename, StagedFile& staged) {
  const Endpoint ep = parse_http_url(url);
  const std::string what = "GET " + filename;
  UniqueFd sock(dial(ep, what));
  const std::string request = "GET " + ep.prefix + "/" + filename + " HTTP/1.1\r\nHost: " + ep.authority +
                              "\r\nAccept: */*\r\nConnection: close\r\n\r\n";
  for (size_t sent = 0; sent < request.size();) {
    const ssize_t w = ::send(sock.get(), request.data() + sent, request.size() - sent, MSG_NOSIGNAL);
    if (w <= 0) raise(Errc::TransportError, what + ": send failed");
    sent += size_t(w);
  }
  Reader in(sock.get());
  const ResponseHead head = read_head(in, what);
  if (head.status == 404) raise(Errc::RemoteNotFound, filename);
  if (head.status != 200) raise(Errc::TransportError, what + ": http " + std::to_string(head.status));

  UniqueFd out(staged.open_for_write());
  auto sink = [&](const char* p, size_t n) { staged.append(out.get(), p, n); };
  if (!head.chunked) {
    in.body(head.content_length, sink);
    return;
  }
  for (;;) {  // chunk-size line, chunk, CRLF ... until the 0-size chunk
    const uint64_t n = std::stoull(in.line(), nullptr, 16);
    if (n == 0) return;
    in.body(n, sink);
    in.line();
  }
}

}  // namespace

RemoteRef make_ref(const std::string& url, const fmt::ModelKey& key) {
  RemoteRef ref;
  ref.key = key;
  const bool http = url.compare(0, 7, "http://") == 0;
  ref.backend = http ? RemoteRef::Backend::Http : RemoteRef::Backend::Dir;
  ref.base = (!http && url.compare(0, 4, "dir:") == 0) ? url.substr(4) : url;
  return ref;
}

std::string fetch(const RemoteRef& ref, const std::string& dest_dir) {
  const std::string filename = fmt::canonical_filename(ref.key);
  const fs::path cached = fs::path(dest_dir) / filename;
  std::error_code ec;
  if (fs::exists(cached, ec) && !verdict(cached)) return cached.string();  // reuse a valid copy

  fs::create_directories(dest_dir, ec);
  StagedFile staged(dest_dir, filename);
  if (ref.backend == RemoteRef::Backend::Http)
    produce_from_http(ref.base, filename, staged);
  else
    produce_from_dir(ref.base, filename, staged);
  return staged.admit().string();
}

}  // namespace trims::remote
