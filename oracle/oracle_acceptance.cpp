// oracle_acceptance.cpp — TEST INFRASTRUCTURE ONLY (ours).
//
// Compiles the reference's proj/src/bench/oracle.cpp UNMODIFIED, read in place
// (this file #includes it; oracle/Makefile builds this TU instead of that one),
// so the trace generator in its anonymous namespace (random_trace,
// oracle.cpp:136-196) is reachable from the same translation unit. One extra
// C entry point dumps the exact trace set of the reference's acceptance
// criterion C2 (proj/tests/acceptance.cpp:49-73: 1000 traces, seed 20250808,
// <= 64 models, <= 10000 ops, LRU/LCU alternating as run_oracle does at
// oracle.cpp:204-211) as ref_replay / trims_replay spec texts.
#include "src/bench/oracle.cpp"

#include <cstring>
#include <sstream>

extern "C" int ref_acceptance_specs(uint64_t seed, uint32_t traces, uint32_t max_models, uint32_t max_ops, char* out,
                                    uint64_t cap) {
  try {
    mrm::bench::OracleParams params;
    params.traces = traces;
    params.seed = seed;
    params.max_models = max_models;
    params.max_ops = max_ops;
    std::mt19937_64 rng(params.seed);
    const mrm::cache::Policy policies[2] = {mrm::cache::Policy::LRU, mrm::cache::Policy::LCU};
    std::ostringstream os;
    for (uint32_t t = 0; t < params.traces; ++t) {
      mrm::bench::TraceSetup s = mrm::bench::random_trace(rng, params, policies[t % 2]);
      os << "cfg " << s.cfg.fast_capacity << ' ' << s.cfg.host_capacity << ' ' << s.cfg.disk_capacity << ' '
         << int(s.cfg.policy) << ' ' << (s.cfg.eager_reclaim ? 1 : 0) << '\n';
      for (const auto& m : s.models)
        os << "model " << m.weights_bytes << ' ' << m.file_bytes << ' ' << (m.on_disk ? 1 : 0) << ' '
           << (m.on_remote ? 1 : 0) << '\n';
      for (const auto& op : s.trace)
        os << "op " << (op.kind == mrm::bench::sim::TraceOp::Kind::Open ? 'o' : 'c') << ' ' << op.model << '\n';
      os << "end\n";
    }
    const std::string text = os.str();
    if (!out || text.size() + 1 > cap) return -2;
    std::memcpy(out, text.data(), text.size() + 1);
    return 0;
  } catch (...) {
    return -1;
  }
}
