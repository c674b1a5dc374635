// wire.hpp — the daemon protocol, byte-compatible with the reference's frozen
// v1 framing (proj/include/mrm/wire_protocol.hpp:15-163,
// proj/src/wire_protocol.cpp:124-357): frame = u32 LE payload length | u8
// message type | payload; LE integers, u16-length strings, u32-count lists,
// granularity = u8 tag (+ u64 block bytes for Block), 16 MiB frame cap.
//
// The B200 store rides v1 unchanged: an ObjectRef's segment_token names the
// exported cuMem allocation and carries its CUDA coordinates as a query
// ("trims.<pid>.arena<dev>?dev=D&alloc=A&seg=O&payload=P"), and the
// allocation's fd travels with the OpenResponse frame as SCM_RIGHTS ancillary
// data on a Unix socket (a reference v1 decoder sees an ordinary frame).
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <string>
#include <variant>
#include <vector>

#include "errc.hpp"

namespace trims::wire {

inline constexpr uint16_t kVersion = 1;
inline constexpr uint32_t kMaxFrame = 16u << 20;

enum class Type : uint8_t {
  OpenRequest = 0x01,
  OpenResponse = 0x02,
  CloseRequest = 0x03,
  CloseResponse = 0x04,
  StatsRequest = 0x05,
  StatsResponse = 0x06,
  Error = 0x7F,
};

struct Gran {
  uint8_t kind{0};  // 0 model, 1 layer, 2 block
  uint64_t block_bytes{0};
};

struct OpenReq {
  uint16_t version{kVersion};
  std::string ns, name, model_version;
  Gran gran;
  uint64_t client_id{0};
};

struct Object {
  std::string name, token;
  uint64_t generation{0}, offset{0}, length{0};
};

struct OpenResp {
  uint64_t model_id{0}, handle_id{0};
  uint64_t weights_bytes{0}, workspace_bytes{0}, total_bytes{0};
  std::vector<Object> objects;
  std::array<uint8_t, 32> digest{};
};

struct CloseReq {
  uint16_t version{kVersion};
  uint64_t model_id{0}, handle_id{0};
};

struct CloseResp {
  uint64_t model_id{0}, refcount{0};
};

struct StatsReq {
  uint16_t version{kVersion};
};

struct TierRow {
  uint64_t hits{0}, misses{0}, evictions{0}, used_bytes{0}, capacity_bytes{0};
};

struct ModelRow {
  std::string ns, name, version;
  uint64_t refcount{0}, use_count{0};
  uint8_t residency{0};
};

struct StatsResp {
  std::array<TierRow, 4> tiers{};  // fast, host, disk, remote
  std::vector<ModelRow> models;
  uint64_t open_requests{0}, open_errors{0}, disk_reads{0}, remote_fetches{0};
  uint64_t fetch_ns{0}, disk_read_ns{0}, copy_ns{0}, export_ns{0};
  double workspace_headroom{0.25};
  bool has_calibration{false};
  double calib_q{0}, calib_o{0}, calib_s{0};
};

struct ErrorResp {
  uint16_t code{0};
  std::string detail;
};

using Msg = std::variant<OpenReq, OpenResp, CloseReq, CloseResp, StatsReq, StatsResp, ErrorResp>;

Type type_of(const Msg& m);
std::vector<uint8_t> encode(const Msg& m);
// Decodes one whole frame; never reads out of bounds on arbitrary bytes.
// Throws TruncatedFrame / FrameTooLarge / UnknownMessageType / BadVersion /
// ProtocolError exactly where the reference decoder does.
Msg decode(const uint8_t* frame, size_t n);

// Text form of a message (tests and the reference-parity harness): one line,
// space-separated fields in wire order, strings percent-escaped, digest hex.
std::string to_text(const Msg& m);
Msg from_text(const std::string& text);

// CUDA coordinates carried in an ObjectRef token.
struct TokenInfo {
  std::string base;  // trims.<pid>.arena<dev> / trims.<pid>.<gen>.<name>
  int device{0};
  uint64_t alloc_bytes{0}, segment_offset{0}, payload_bytes{0};
};
std::string make_token(const TokenInfo& t);
TokenInfo parse_token(const std::string& token);

// ---- transport: "unix:<path>" / bare path, or "tcp:<ipv4>:<port>"
int listen_endpoint(const std::string& endpoint, std::string* unix_path);
int connect_endpoint(const std::string& endpoint);
// One frame; `fd` >= 0 is attached as SCM_RIGHTS (Unix sockets only).
void send_frame(int sock, const std::vector<uint8_t>& frame, int fd = -1);
// nullopt on a clean EOF at a frame boundary; a received fd (if any) goes
// to *fd_out (else it is closed).
std::optional<std::vector<uint8_t>> recv_frame(int sock, int* fd_out = nullptr);

}  // namespace trims::wire
