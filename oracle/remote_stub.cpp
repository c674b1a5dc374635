// remote_stub.cpp — stands in for proj/src/remote_store.cpp, which needs
// cpp-httplib (absent from the image). The remote tier is out of scope
// (SURVEY.md §2 row 14); the oracle never configures a remote_url, so these
// are unreachable. TEST INFRASTRUCTURE ONLY.
#include "mrm/remote_store.hpp"

namespace mrm::remote {

RemoteRef make_ref(const std::string& url, const model::ModelKey& key) {
  RemoteRef r;
  r.base = url;
  r.key = key;
  return r;
}

std::filesystem::path fetch(const RemoteRef& ref, const std::filesystem::path&) {
  raise(Errc::TransportError, "remote tier not built in the oracle (" + ref.base + ")");
}

}  // namespace mrm::remote
