// store_api.hpp — the in-library C++ surface of a trims_store (capi.cu) for
// components that sit above it, the wire-protocol daemon (server.cu): the
// same calls the reference daemon makes on its CacheCore
// (proj/src/daemon.cpp:452-560), with the store's logical clock.
#pragma once

#include <memory>
#include <optional>

#include "backend.hpp"
#include "cache_core.hpp"

struct trims_store;

namespace trims::store_api {

// CacheCore::open_model with the next logical clock tick (daemon.cpp:457).
PlacementResult open(trims_store* s, const fmt::ModelKey& key, const Granularity& g);
uint64_t close(trims_store* s, const fmt::ModelKey& key);
StatsSnapshot stats(trims_store* s);
// The published fast-tier record (resident manifest, segment coordinates).
std::shared_ptr<FastRecord> fast_record(trims_store* s, uint64_t model_id);
// DaemonConfig::workspace_headroom_fraction and the startup calibration the
// daemon publishes in StatsResponse (daemon.cpp:535-539).
double workspace_headroom(trims_store* s);
std::optional<Calibration> calibration(trims_store* s);
// The C ABI's per-thread error text (trims_last_error).
void set_last_error(const std::string& what);

}  // namespace trims::store_api
