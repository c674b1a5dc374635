// remote.cpp — see remote.hpp.
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
#include <vector>

#include "errc.hpp"

namespace trims::remote {

namespace fs = std::filesystem;

namespace {

// remote_store.cpp:15-22: a full verify succeeding is what makes a file valid
bool file_valid(const fs::path& p) {
  try {
    fmt::read_artifact_info(p.string(), /*full_verify=*/true);
    return true;
  } catch (...) {
    return false;
  }
}

// remote_store.cpp:24-33
void verify_or_remove(const fs::path& tmp) {
  try {
    fmt::read_artifact_info(tmp.string(), /*full_verify=*/true);
  } catch (const Error& e) {
    std::error_code ec;
    fs::remove(tmp, ec);
    if (e.code() == Errc::ChecksumMismatch) throw;
    raise(Errc::ChecksumMismatch, std::string("fetched artifact invalid: ") + e.what());
  }
}

struct Fd {
  int fd{-1};
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

void write_all(int fd, const char* p, size_t n, const fs::path& what) {
  while (n) {
    ssize_t w = ::write(fd, p, n);
    if (w < 0 && errno == EINTR) continue;
    if (w <= 0) raise(Errc::TransportError, "cannot write " + what.string());
    p += w;
    n -= size_t(w);
  }
}

// A buffered reader over the socket (status line, headers, chunked bodies).
struct Conn {
  int fd;
  std::vector<char> buf = std::vector<char>(1 << 16);
  size_t lo = 0, hi = 0;
  bool fill() {
    if (lo < hi) return true;
    for (;;) {
      ssize_t r = ::recv(fd, buf.data(), buf.size(), 0);
      if (r < 0 && errno == EINTR) continue;
      if (r < 0) raise(Errc::TransportError, std::string("recv: ") + std::strerror(errno));
      lo = 0;
      hi = size_t(r);
      return r > 0;
    }
  }
  std::string line() {
    std::string s;
    for (;;) {
      if (!fill()) raise(Errc::TransportError, "connection closed in the response head");
      while (lo < hi) {
        char c = buf[lo++];
        if (c == '\n') {
          if (!s.empty() && s.back() == '\r') s.pop_back();
          return s;
        }
        s.push_back(c);
        if (s.size() > 16384) raise(Errc::TransportError, "response line too long");
      }
    }
  }
  // copies n bytes (or to EOF when n == npos) into fd
  void body(int out, uint64_t n, const fs::path& what) {
    while (n) {
      if (!fill()) {
        if (n == ~0ull) return;
        raise(Errc::TransportError, "connection closed mid-body");
      }
      size_t take = size_t(std::min<uint64_t>(n, hi - lo));
      write_all(out, buf.data() + lo, take, what);
      lo += take;
      if (n != ~0ull) n -= take;
    }
  }
};

std::string lower(std::string s) {
  for (auto& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

// remote_store.cpp:35-56 (split_http) + the GET of :92-112, on a plain socket
void http_get(const std::string& base, const std::string& filename, const fs::path& tmp) {
  const std::string scheme = "http://";
  if (base.rfind(scheme, 0) != 0) raise(Errc::InvalidArgument, "expected http:// url");
  size_t slash = base.find('/', scheme.size());
  std::string host_port = base.substr(scheme.size(), slash == std::string::npos ? std::string::npos
                                                                                : slash - scheme.size());
  std::string prefix = slash == std::string::npos ? "" : base.substr(slash);
  while (!prefix.empty() && prefix.back() == '/') prefix.pop_back();
  std::string host = host_port, port = "80";
  if (size_t c = host_port.rfind(':'); c != std::string::npos && host_port.find(']') == std::string::npos) {
    host = host_port.substr(0, c);
    port = host_port.substr(c + 1);
  }

  addrinfo hints{}, *res = nullptr;
  hints.ai_family = AF_UNSPEC;
  hints.ai_socktype = SOCK_STREAM;
  if (int rc = ::getaddrinfo(host.c_str(), port.c_str(), &hints, &res); rc != 0)
    raise(Errc::TransportError, "GET " + filename + ": resolve " + host + ": " + gai_strerror(rc));
  Fd s;
  for (addrinfo* ai = res; ai; ai = ai->ai_next) {
    s.fd = ::socket(ai->ai_family, ai->ai_socktype | SOCK_CLOEXEC, ai->ai_protocol);
    if (s.fd < 0) continue;
    if (::connect(s.fd, ai->ai_addr, ai->ai_addrlen) == 0) break;
    ::close(s.fd);
    s.fd = -1;
  }
  ::freeaddrinfo(res);
  if (s.fd < 0) raise(Errc::TransportError, "GET " + filename + ": connection to " + host_port + " failed");
  timeval tv{60, 0};  // client.set_read_timeout(60, 0)
  ::setsockopt(s.fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));

  const std::string req = "GET " + prefix + "/" + filename + " HTTP/1.1\r\nHost: " + host_port +
                          "\r\nAccept: */*\r\nConnection: close\r\n\r\n";
  for (size_t at = 0; at < req.size();) {
    ssize_t w = ::send(s.fd, req.data() + at, req.size() - at, MSG_NOSIGNAL);
    if (w <= 0) raise(Errc::TransportError, "GET " + filename + ": send failed");
    at += size_t(w);
  }
  Conn c{s.fd};
  std::string status = c.line();  // HTTP/1.x NNN reason
  int code = 0;
  if (status.rfind("HTTP/", 0) != 0 || status.size() < 12 || std::sscanf(status.c_str() + 9, "%d", &code) != 1)
    raise(Errc::TransportError, "GET " + filename + ": bad status line");
  uint64_t length = ~0ull;
  bool chunked = false;
  for (std::string h; !(h = c.line()).empty();) {
    size_t colon = h.find(':');
    if (colon == std::string::npos) continue;
    std::string k = lower(h.substr(0, colon)), v = h.substr(colon + 1);
    while (!v.empty() && v.front() == ' ') v.erase(v.begin());
    if (k == "content-length") length = std::stoull(v);
    if (k == "transfer-encoding" && lower(v).find("chunked") != std::string::npos) chunked = true;
  }
  if (code == 404) raise(Errc::RemoteNotFound, filename);
  if (code != 200) raise(Errc::TransportError, "GET " + filename + ": http " + std::to_string(code));

  Fd out;
  out.fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (out.fd < 0) raise(Errc::TransportError, "cannot write " + tmp.string());
  if (chunked) {
    for (;;) {
      uint64_t n = std::stoull(c.line(), nullptr, 16);
      if (!n) break;
      c.body(out.fd, n, tmp);
      c.line();  // CRLF after the chunk
    }
  } else {
    c.body(out.fd, length, tmp);
  }
}

}  // namespace

RemoteRef make_ref(const std::string& url, const fmt::ModelKey& key) {
  RemoteRef ref;
  ref.key = key;
  if (url.rfind("http://", 0) == 0) {
    ref.backend = RemoteRef::Backend::Http;
    ref.base = url;
  } else {
    ref.backend = RemoteRef::Backend::Dir;
    ref.base = url.rfind("dir:", 0) == 0 ? url.substr(4) : url;
  }
  return ref;
}

std::string fetch(const RemoteRef& ref, const std::string& dest_dir) {
  const std::string filename = fmt::canonical_filename(ref.key);
  const fs::path dest = fs::path(dest_dir) / filename;
  std::error_code ec;
  if (fs::exists(dest, ec) && file_valid(dest)) return dest.string();

  fs::create_directories(dest_dir, ec);
  const fs::path tmp = fs::path(dest_dir) / (filename + ".part." + std::to_string(::getpid()));
  if (ref.backend == RemoteRef::Backend::Dir) {
    const fs::path src = fs::path(ref.base) / filename;
    if (!fs::exists(src, ec)) raise(Errc::RemoteNotFound, src.string());
    fs::copy_file(src, tmp, fs::copy_options::overwrite_existing, ec);
    if (ec) raise(Errc::TransportError, "copy " + src.string() + ": " + ec.message());
  } else {
    try {
      http_get(ref.base, filename, tmp);
    } catch (...) {
      fs::remove(tmp, ec);
      throw;
    }
  }
  verify_or_remove(tmp);
  fs::rename(tmp, dest, ec);
  if (ec) {
    std::error_code ec2;
    fs::remove(tmp, ec2);
    raise(Errc::TransportError, "rename to " + dest.string() + ": " + ec.message());
  }
  return dest.string();
}

}  // namespace trims::remote
