// format.cpp — .trms reader/writer, manifest JSON, ingest plan.
// Behaviour follows proj/src/model_format.cpp (cited per function); the JSON
// code is ours (no nlohmann): a writer that reproduces nlohmann's dump() bytes
// for the manifest schema and a strict recursive-descent parser.
#include "format.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <variant>

#include "pread.hpp"
#include "sha256.hpp"

namespace trims::fmt {

uint64_t element_size(DType t) {
  switch (t) {
    case DType::F64: return 8;
    case DType::F32: return 4;
    case DType::F16: return 2;
    case DType::I8: return 1;
    case DType::BF16: return 2;
  }
  return 0;
}

const char* dtype_name(DType t) {
  switch (t) {
    case DType::F64: return "f64";
    case DType::F32: return "f32";
    case DType::F16: return "f16";
    case DType::I8: return "i8";
    case DType::BF16: return "bf16";
  }
  return "?";
}

std::optional<DType> dtype_from_name(std::string_view s) {
  if (s == "f64") return DType::F64;
  if (s == "f32") return DType::F32;
  if (s == "f16") return DType::F16;
  if (s == "i8") return DType::I8;
  if (s == "bf16") return DType::BF16;
  return std::nullopt;
}

namespace {

// \d+(\.\d+)*  (model_format.cpp:30-48)
bool version_ok(std::string_view v) {
  if (v.empty() || v.front() == '.' || v.back() == '.') return false;
  char prev = '.';
  for (char c : v) {
    if (c == '.') {
      if (prev == '.') return false;
    } else if (c < '0' || c > '9') {
      return false;
    }
    prev = c;
  }
  return true;
}

bool clean(const std::string& s) {
  return s.find('/') == std::string::npos && s.find('\0') == std::string::npos &&
         s.find("__") == std::string::npos;
}

}  // namespace

bool valid_key(const ModelKey& k) {
  if (k.ns.empty() || k.name.empty() || k.version.empty()) return false;
  return clean(k.ns) && clean(k.name) && version_ok(k.version);
}

std::string to_string(const ModelKey& k) { return k.ns + "/" + k.name + "@" + k.version; }

std::string canonical_filename(const ModelKey& k) {
  return k.ns + "__" + k.name + "__" + k.version + ".trms";
}

std::optional<ModelKey> key_from_filename(std::string_view f) {
  constexpr std::string_view ext = ".trms";
  if (f.size() <= ext.size() || f.substr(f.size() - ext.size()) != ext) return std::nullopt;
  std::string_view stem = f.substr(0, f.size() - ext.size());
  size_t a = stem.find("__");
  if (a == std::string_view::npos) return std::nullopt;
  size_t b = stem.find("__", a + 2);
  if (b == std::string_view::npos) return std::nullopt;
  ModelKey k{std::string(stem.substr(0, a)), std::string(stem.substr(a + 2, b - a - 2)),
             std::string(stem.substr(b + 2))};
  if (!valid_key(k)) return std::nullopt;
  return k;
}

uint64_t blob_span(const std::vector<TensorSpec>& t) {
  uint64_t end = 0;
  for (const auto& x : t) end = std::max(end, x.offset + x.nbytes);
  return align_up(end);
}

uint64_t checked_product(const std::vector<uint64_t>& dims) {
  uint64_t p = 1;
  for (uint64_t d : dims) {
    if (d == 0) raise(Errc::CorruptManifest, "tensor dim must be positive");
    if (p > UINT64_MAX / d) raise(Errc::CorruptManifest, "dims overflow");
    p *= d;
  }
  return p;
}

void validate_manifest(const Manifest& m) {
  if (!valid_key(m.key)) raise(Errc::CorruptManifest, "invalid model key " + to_string(m.key));
  uint64_t prev_end = 0;
  for (size_t i = 0; i < m.tensors.size(); ++i) {
    const auto& t = m.tensors[i];
    if (t.name.empty()) raise(Errc::CorruptManifest, "tensor name empty");
    if (t.dims.empty()) raise(Errc::CorruptManifest, "tensor dims empty: " + t.name);
    if (t.nbytes != checked_product(t.dims) * element_size(t.dtype))
      raise(Errc::CorruptManifest, "tensor " + t.name + " nbytes != dims product");
    if (t.offset % kAlign) raise(Errc::CorruptManifest, "tensor " + t.name + " offset not 64-aligned");
    if (t.offset < prev_end)
      raise(Errc::CorruptManifest, "tensors overlap or are not sorted by offset at " + t.name);
    prev_end = t.offset + t.nbytes;
    for (size_t j = 0; j < i; ++j)
      if (m.tensors[j].name == t.name) raise(Errc::CorruptManifest, "duplicate tensor name " + t.name);
  }
  if (m.blob_bytes != blob_span(m.tensors)) raise(Errc::CorruptManifest, "blob_bytes != span");
}

uint64_t weights_bytes(const Manifest& m) {
  uint64_t w = 0;
  for (const auto& t : m.tensors) w += checked_product(t.dims) * element_size(t.dtype);
  return w;
}

Manifest make_manifest(ModelKey key, const std::vector<TensorDecl>& decls, uint64_t workspace) {
  Manifest m;
  m.key = std::move(key);
  m.workspace_bytes = workspace;
  uint64_t off = 0;
  for (const auto& d : decls) {
    TensorSpec t{d.name, d.dims, d.dtype, off, checked_product(d.dims) * element_size(d.dtype), d.layout};
    off = align_up(off + t.nbytes);
    m.tensors.push_back(std::move(t));
  }
  m.blob_bytes = blob_span(m.tensors);
  validate_manifest(m);
  return m;
}

// ---------------------------------------------------------------------------
// JSON. Writer: nlohmann dump() conventions (sorted keys, no spaces, escapes
// \" \\ \b \f \n \r \t and \u00xx for other control bytes, UTF-8 verbatim).

namespace {

void put_str(std::string& o, std::string_view s) {
  static const char* hex = "0123456789abcdef";
  o.push_back('"');
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          o += "\\u00";
          o.push_back(hex[c >> 4]);
          o.push_back(hex[c & 15]);
        } else {
          o.push_back(char(c));
        }
    }
  }
  o.push_back('"');
}

}  // namespace

std::string manifest_to_json(const Manifest& m) {
  std::string o;
  o.reserve(96 + m.tensors.size() * 96);
  o += "{\"name\":";
  put_str(o, m.key.name);
  o += ",\"namespace\":";
  put_str(o, m.key.ns);
  o += ",\"tensors\":[";
  for (size_t i = 0; i < m.tensors.size(); ++i) {
    const auto& t = m.tensors[i];
    if (i) o.push_back(',');
    o += "{\"dims\":[";
    for (size_t d = 0; d < t.dims.size(); ++d) {
      if (d) o.push_back(',');
      o += std::to_string(t.dims[d]);
    }
    o += "],\"dtype\":";
    put_str(o, dtype_name(t.dtype));
    if (t.layout == Layout::KRSC) o += ",\"layout\":\"krsc\"";
    o += ",\"name\":";
    put_str(o, t.name);
    o += ",\"nbytes\":" + std::to_string(t.nbytes) + ",\"offset\":" + std::to_string(t.offset) + "}";
  }
  o += "],\"version\":";
  put_str(o, m.key.version);
  o += ",\"workspace_bytes\":" + std::to_string(m.workspace_bytes) + "}";
  return o;
}

namespace {

struct JVal;
using JObj = std::map<std::string, std::shared_ptr<JVal>>;
using JArr = std::vector<std::shared_ptr<JVal>>;
struct JNum {
  bool is_float{false}, negative{false};
  uint64_t u{0};
  double d{0};
};
struct JVal {
  std::variant<std::nullptr_t, bool, JNum, std::string, JArr, JObj> v;
};

class Parser {
 public:
  explicit Parser(std::string_view s) : s_(s) {}
  std::shared_ptr<JVal> parse_document() {
    auto v = value(0);
    ws();
    if (p_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const char* what) {
    raise(Errc::CorruptManifest, std::string("manifest JSON parse failed: ") + what + " at " + std::to_string(p_));
  }
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\t' || s_[p_] == '\n' || s_[p_] == '\r')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < s_.size() && s_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  std::shared_ptr<JVal> value(int depth) {
    if (depth > 64) fail("nesting too deep");
    ws();
    if (p_ >= s_.size()) fail("unexpected end");
    auto out = std::make_shared<JVal>();
    char c = s_[p_];
    if (c == '{') {
      ++p_;
      JObj o;
      if (!eat('}')) {
        do {
          ws();
          if (p_ >= s_.size() || s_[p_] != '"') fail("object key");
          std::string k = str();
          if (!eat(':')) fail("':'");
          o[k] = value(depth + 1);
        } while (eat(','));
        if (!eat('}')) fail("'}'");
      }
      out->v = std::move(o);
    } else if (c == '[') {
      ++p_;
      JArr a;
      if (!eat(']')) {
        do {
          a.push_back(value(depth + 1));
        } while (eat(','));
        if (!eat(']')) fail("']'");
      }
      out->v = std::move(a);
    } else if (c == '"') {
      out->v = str();
    } else if (s_.compare(p_, 4, "true") == 0) {
      p_ += 4;
      out->v = true;
    } else if (s_.compare(p_, 5, "false") == 0) {
      p_ += 5;
      out->v = false;
    } else if (s_.compare(p_, 4, "null") == 0) {
      p_ += 4;
      out->v = nullptr;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      out->v = num();
    } else {
      fail("unexpected character");
    }
    return out;
  }
  static void put_utf8(std::string& o, uint32_t cp) {
    if (cp < 0x80) {
      o.push_back(char(cp));
    } else if (cp < 0x800) {
      o.push_back(char(0xC0 | (cp >> 6)));
      o.push_back(char(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      o.push_back(char(0xE0 | (cp >> 12)));
      o.push_back(char(0x80 | ((cp >> 6) & 0x3F)));
      o.push_back(char(0x80 | (cp & 0x3F)));
    } else {
      o.push_back(char(0xF0 | (cp >> 18)));
      o.push_back(char(0x80 | ((cp >> 12) & 0x3F)));
      o.push_back(char(0x80 | ((cp >> 6) & 0x3F)));
      o.push_back(char(0x80 | (cp & 0x3F)));
    }
  }
  uint32_t hex4() {
    if (p_ + 4 > s_.size()) fail("short \\u escape");
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) {
      char h = s_[p_++];
      v <<= 4;
      if (h >= '0' && h <= '9') v |= uint32_t(h - '0');
      else if (h >= 'a' && h <= 'f') v |= uint32_t(h - 'a' + 10);
      else if (h >= 'A' && h <= 'F') v |= uint32_t(h - 'A' + 10);
      else fail("bad hex digit");
    }
    return v;
  }
  std::string str() {
    ++p_;  // opening quote
    std::string o;
    while (true) {
      if (p_ >= s_.size()) fail("unterminated string");
      unsigned char c = static_cast<unsigned char>(s_[p_++]);
      if (c == '"') break;
      if (c < 0x20) fail("control character in string");
      if (c != '\\') {
        o.push_back(char(c));
        continue;
      }
      if (p_ >= s_.size()) fail("dangling escape");
      char e = s_[p_++];
      switch (e) {
        case '"': o.push_back('"'); break;
        case '\\': o.push_back('\\'); break;
        case '/': o.push_back('/'); break;
        case 'b': o.push_back('\b'); break;
        case 'f': o.push_back('\f'); break;
        case 'n': o.push_back('\n'); break;
        case 'r': o.push_back('\r'); break;
        case 't': o.push_back('\t'); break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (p_ + 2 > s_.size() || s_[p_] != '\\' || s_[p_ + 1] != 'u') fail("lone surrogate");
            p_ += 2;
            uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            fail("lone low surrogate");
          }
          put_utf8(o, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    return o;
  }
  JNum num() {
    size_t start = p_;
    JNum n;
    if (s_[p_] == '-') {
      n.negative = true;
      ++p_;
    }
    if (p_ >= s_.size() || s_[p_] < '0' || s_[p_] > '9') fail("digit expected");
    if (s_[p_] == '0' && p_ + 1 < s_.size() && s_[p_ + 1] >= '0' && s_[p_ + 1] <= '9') fail("leading zero");
    while (p_ < s_.size() && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
    if (p_ < s_.size() && (s_[p_] == '.' || s_[p_] == 'e' || s_[p_] == 'E')) {
      n.is_float = true;
      if (s_[p_] == '.') {
        ++p_;
        if (p_ >= s_.size() || s_[p_] < '0' || s_[p_] > '9') fail("fraction digit expected");
        while (p_ < s_.size() && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
      }
      if (p_ < s_.size() && (s_[p_] == 'e' || s_[p_] == 'E')) {
        ++p_;
        if (p_ < s_.size() && (s_[p_] == '+' || s_[p_] == '-')) ++p_;
        if (p_ >= s_.size() || s_[p_] < '0' || s_[p_] > '9') fail("exponent digit expected");
        while (p_ < s_.size() && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
      }
    }
    std::string tok(s_.substr(start, p_ - start));
    if (n.is_float) {
      n.d = std::strtod(tok.c_str(), nullptr);
    } else {
      errno = 0;
      if (n.negative) {
        long long v = std::strtoll(tok.c_str(), nullptr, 10);
        if (errno == ERANGE) {
          n.is_float = true;
          n.d = std::strtod(tok.c_str(), nullptr);
        } else {
          n.u = uint64_t(v);
        }
      } else {
        unsigned long long v = std::strtoull(tok.c_str(), nullptr, 10);
        if (errno == ERANGE) {
          n.is_float = true;
          n.d = std::strtod(tok.c_str(), nullptr);
        } else {
          n.u = v;
        }
      }
    }
    return n;
  }

  std::string_view s_;
  size_t p_{0};
};

[[noreturn]] void field_error(const std::string& what) {
  raise(Errc::CorruptManifest, "manifest field error: " + what);
}

const JVal& at(const JObj& o, const char* k) {
  auto it = o.find(k);
  if (it == o.end()) field_error(std::string("key '") + k + "' not found");
  return *it->second;
}
const JObj& as_obj(const JVal& v, const char* what) {
  if (auto* o = std::get_if<JObj>(&v.v)) return *o;
  field_error(std::string(what) + " is not an object");
}
const JArr& as_arr(const JVal& v, const char* what) {
  if (auto* a = std::get_if<JArr>(&v.v)) return *a;
  field_error(std::string(what) + " is not an array");
}
std::string as_str(const JVal& v, const char* what) {
  if (auto* s = std::get_if<std::string>(&v.v)) return *s;
  field_error(std::string(what) + " is not a string");
}
// nlohmann get<uint64_t>: any number converts by static_cast; others throw.
uint64_t as_u64(const JVal& v, const char* what) {
  if (auto* n = std::get_if<JNum>(&v.v)) return n->is_float ? uint64_t(n->d) : n->u;
  field_error(std::string(what) + " is not a number");
}

}  // namespace

Manifest manifest_from_json(std::string_view text) {
  std::shared_ptr<JVal> doc = Parser(text).parse_document();
  const JObj& j = as_obj(*doc, "manifest");
  Manifest m;
  m.key.ns = as_str(at(j, "namespace"), "namespace");
  m.key.name = as_str(at(j, "name"), "name");
  m.key.version = as_str(at(j, "version"), "version");
  m.workspace_bytes = as_u64(at(j, "workspace_bytes"), "workspace_bytes");
  const JVal& tv = at(j, "tensors");
  // nlohmann iterates objects' values too; the reference only ever writes arrays.
  const JArr& arr = as_arr(tv, "tensors");
  for (const auto& tp : arr) {
    const JObj& to = as_obj(*tp, "tensor");
    TensorSpec t;
    t.name = as_str(at(to, "name"), "name");
    for (const auto& d : as_arr(at(to, "dims"), "dims")) t.dims.push_back(as_u64(*d, "dim"));
    auto dt = dtype_from_name(as_str(at(to, "dtype"), "dtype"));
    if (!dt) raise(Errc::CorruptManifest, "unknown dtype in manifest");
    t.dtype = *dt;
    t.offset = as_u64(at(to, "offset"), "offset");
    t.nbytes = as_u64(at(to, "nbytes"), "nbytes");
    if (auto it = to.find("layout"); it != to.end()) {
      std::string l = as_str(*it->second, "layout");
      if (l == "krsc") t.layout = Layout::KRSC;
      else raise(Errc::CorruptManifest, "unknown layout " + l);
    }
    m.tensors.push_back(std::move(t));
  }
  m.blob_bytes = blob_span(m.tensors);
  validate_manifest(m);
  return m;
}

uint64_t blob_file_offset(uint64_t manifest_len) { return align_up(16 + manifest_len); }

// ---------------------------------------------------------------------------
// Artifact I/O (model_format.cpp:235-429).

namespace {

uint64_t get_u64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
  return v;
}
uint32_t get_u32(const uint8_t* p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

// parse_header (model_format.cpp:336-355)
ArtifactInfo parse_head(const uint8_t* head, uint64_t head_len, uint64_t total) {
  if (head_len < 16) raise(Errc::BadMagic, "stream shorter than header");
  if (std::memcmp(head, "TRMS", 4) != 0) raise(Errc::BadMagic, "bad magic");
  uint32_t ver = get_u32(head + 4);
  if (ver != kFormatVersion) raise(Errc::UnsupportedVersion, "format version " + std::to_string(ver));
  uint64_t mlen = get_u64(head + 8);
  if (mlen > (64ull << 20)) raise(Errc::CorruptManifest, "manifest_len implausibly large");
  if (16 + mlen > head_len) raise(Errc::CorruptManifest, "stream truncated inside the manifest section");
  ArtifactInfo a;
  a.manifest_len = mlen;
  a.manifest = manifest_from_json(std::string_view(reinterpret_cast<const char*>(head + 16), size_t(mlen)));
  a.blob_offset = blob_file_offset(mlen);
  a.file_bytes = total;
  uint64_t need = a.blob_offset + a.manifest.blob_bytes + 32;
  if (total < need)
    raise(Errc::CorruptManifest, "stream truncated: need " + std::to_string(need) + " bytes, have " +
                                     std::to_string(total));
  return a;
}

struct Fd {
  int fd{-1};
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

void pread_all(int fd, uint8_t* dst, uint64_t n, uint64_t off) {
  while (n) {
    ssize_t r = ::pread(fd, dst, size_t(std::min<uint64_t>(n, 1ull << 30)), off_t(off));
    if (r <= 0) raise(Errc::CorruptManifest, "short read");
    dst += r;
    n -= uint64_t(r);
    off += uint64_t(r);
  }
}

}  // namespace

ArtifactInfo parse_artifact(const uint8_t* bytes, uint64_t n, bool full_verify) {
  ArtifactInfo a = parse_head(bytes, n, n);
  std::memcpy(a.manifest.checksum.data(), bytes + a.blob_offset + a.manifest.blob_bytes, 32);
  if (full_verify) {
    Digest d = Sha256::of(bytes + a.blob_offset, a.manifest.blob_bytes);
    if (d != a.manifest.checksum) raise(Errc::ChecksumMismatch, to_string(a.manifest.key));
  }
  return a;
}

ArtifactInfo read_artifact_info(const std::string& path, bool full_verify) {
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) raise(Errc::NotFound, path);
  struct stat st {};
  if (::fstat(f.fd, &st) != 0) raise(Errc::NotFound, path);
  uint64_t total = uint64_t(st.st_size);
  uint8_t hdr[16];
  if (total < 16) raise(Errc::BadMagic, "file shorter than header");
  pread_all(f.fd, hdr, 16, 0);
  uint64_t mlen = get_u64(hdr + 8);
  if (std::memcmp(hdr, "TRMS", 4) != 0) raise(Errc::BadMagic, "bad magic");
  if (mlen > (64ull << 20)) raise(Errc::CorruptManifest, "manifest_len implausibly large");
  uint64_t head_len = std::min<uint64_t>(total, 16 + mlen);
  std::vector<uint8_t> head(head_len);
  pread_all(f.fd, head.data(), head_len, 0);
  ArtifactInfo a = parse_head(head.data(), head_len, total);
  pread_all(f.fd, a.manifest.checksum.data(), 32, a.blob_offset + a.manifest.blob_bytes);
  if (full_verify) {
    Sha256 h;  // readers ahead of one in-order hasher (pread.hpp)
    pipelined_read(f.fd, a.blob_offset, a.manifest.blob_bytes, nullptr, 8, &h);
    if (h.finish() != a.manifest.checksum) raise(Errc::ChecksumMismatch, path);
  }
  return a;
}

void write_artifact(const std::string& path, const Manifest& m, const uint8_t* blob) {
  validate_manifest(m);
  std::string j = manifest_to_json(m);
  std::string head("TRMS", 4);
  for (int i = 0; i < 4; ++i) head.push_back(char(uint8_t(kFormatVersion >> (8 * i))));
  for (int i = 0; i < 8; ++i) head.push_back(char(uint8_t(uint64_t(j.size()) >> (8 * i))));
  head += j;
  head.resize(blob_file_offset(j.size()), '\0');
  Digest d = Sha256::of(blob, m.blob_bytes);
  Fd f;
  f.fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (f.fd < 0) raise(Errc::Internal, "cannot open " + path + " for writing");
  auto put = [&](const void* p, uint64_t n) {
    const uint8_t* c = static_cast<const uint8_t*>(p);
    while (n) {
      ssize_t w = ::write(f.fd, c, size_t(std::min<uint64_t>(n, 1ull << 30)));
      if (w <= 0) raise(Errc::Internal, "artifact write failed");
      c += w;
      n -= uint64_t(w);
    }
  };
  put(head.data(), head.size());
  put(blob, m.blob_bytes);
  put(d.data(), 32);
}

Manifest resident_manifest(const Manifest& src, const Plan& plan) {
  if (plan.identity()) return src;
  std::vector<TensorDecl> decls;
  for (const auto& t : src.tensors) {
    TensorDecl d{t.name, t.dims, t.dtype, t.layout};
    bool floating = t.dtype == DType::F64 || t.dtype == DType::F32 || t.dtype == DType::F16 ||
                    t.dtype == DType::BF16;
    if (plan.convert && floating) d.dtype = plan.out_dtype;
    if (plan.permute_4d && t.dims.size() == 4 && t.layout == Layout::Native) {
      d.dims = {t.dims[0], t.dims[2], t.dims[3], t.dims[1]};
      d.layout = Layout::KRSC;
    }
    decls.push_back(std::move(d));
  }
  return make_manifest(src.key, decls, src.workspace_bytes);
}

}  // namespace trims::fmt
