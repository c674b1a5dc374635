// format.hpp — the .trms artifact (deserialise step of ingest) and the
// resident-manifest plan. Byte-compatible with proj/include/mrm/model_format.hpp:
//   "TRMS" | u32 1 | u64 manifest_len | manifest JSON | zero pad to 64
//   | blob | SHA-256(blob)
// The manifest JSON is emitted byte-identically to nlohmann::json::dump()
// (keys sorted, compact) — the reference's manifest digest and blob offset
// depend on those bytes.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "errc.hpp"

namespace trims::fmt {

inline constexpr uint32_t kFormatVersion = 1;
inline constexpr uint64_t kAlign = 64;
using Digest = std::array<uint8_t, 32>;

// F64..I8 as in model_format.hpp:26; BF16 is the B200 resident type.
enum class DType : uint8_t { F64 = 0, F32 = 1, F16 = 2, I8 = 3, BF16 = 4 };
uint64_t element_size(DType t);
const char* dtype_name(DType t);
std::optional<DType> dtype_from_name(std::string_view s);

// Resident layout tag of a tensor. KRSC is the NHWC-style conv weight layout
// produced by the ingest transform from the artifact's KCRS.
enum class Layout : uint8_t { Native = 0, KRSC = 1 };

struct ModelKey {
  std::string ns, name, version;
  bool operator==(const ModelKey&) const = default;
  auto operator<=>(const ModelKey&) const = default;
};
bool valid_key(const ModelKey& k);                 // model_format.cpp:82-92
std::string to_string(const ModelKey& k);          // ns/name@version
std::string canonical_filename(const ModelKey& k);  // <ns>__<name>__<version>.trms
std::optional<ModelKey> key_from_filename(std::string_view f);

struct TensorSpec {
  std::string name;
  std::vector<uint64_t> dims;
  DType dtype{DType::F64};
  uint64_t offset{0};
  uint64_t nbytes{0};
  Layout layout{Layout::Native};
  bool operator==(const TensorSpec&) const = default;
};

struct Manifest {
  ModelKey key;
  std::vector<TensorSpec> tensors;
  uint64_t workspace_bytes{0};
  uint64_t blob_bytes{0};
  Digest checksum{};
};

inline uint64_t align_up(uint64_t v, uint64_t a = kAlign) { return (v + a - 1) / a * a; }
uint64_t blob_span(const std::vector<TensorSpec>& t);
uint64_t checked_product(const std::vector<uint64_t>& dims);
void validate_manifest(const Manifest& m);  // model_format.cpp:123-148
uint64_t weights_bytes(const Manifest& m);  // estimate_footprint().weights_bytes

struct TensorDecl {
  std::string name;
  std::vector<uint64_t> dims;
  DType dtype{DType::F64};
  Layout layout{Layout::Native};
};
// model_format.cpp:158-177: sequential align64 offsets in declaration order.
Manifest make_manifest(ModelKey key, const std::vector<TensorDecl>& decls, uint64_t workspace);

std::string manifest_to_json(const Manifest& m);
Manifest manifest_from_json(std::string_view text);

uint64_t blob_file_offset(uint64_t manifest_len);

struct ArtifactInfo {
  Manifest manifest;
  uint64_t manifest_len{0};
  uint64_t blob_offset{0};  // file offset of the blob
  uint64_t file_bytes{0};
};
// Header + manifest + trailer; with full_verify also streams the blob through
// SHA-256 (model_format.cpp:370-409). Throws NotFound/BadMagic/... as the reference.
ArtifactInfo read_artifact_info(const std::string& path, bool full_verify);
ArtifactInfo parse_artifact(const uint8_t* bytes, uint64_t n, bool full_verify);

// Writes an artifact; `blob` is the full blob (blob_bytes, padding included).
void write_artifact(const std::string& path, const Manifest& m, const uint8_t* blob);

// ---- ingest plan: artifact manifest -> resident manifest -------------------
// out_dtype: DType to convert floating tensors to (F64/F32/F16 -> out_dtype);
// keep = no conversion. permute_4d: KCRS -> KRSC for every 4-D tensor.
struct Plan {
  bool convert{false};
  DType out_dtype{DType::BF16};
  bool permute_4d{false};
  bool identity() const { return !convert && !permute_4d; }
};
// The resident manifest of `src` under `plan`. Identity plans return `src`
// unchanged (same offsets, bit-identical blob); otherwise offsets are
// re-assigned with make_manifest's align64 rule.
Manifest resident_manifest(const Manifest& src, const Plan& plan);

}  // namespace trims::fmt
