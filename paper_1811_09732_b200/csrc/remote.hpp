// remote.hpp — the remote tier feeding the disk cache: the
// reference's remote::make_ref / fetch (proj/src/remote_store.cpp:58-120,
// remote_store.hpp). A `dir:<path>` (or bare path) store is copied, an
// `http://host[:port][/prefix]` store is fetched with a plain HTTP/1.1 GET
// (our own client: the reference links cpp-httplib, absent here). Either way
// the download lands as `<file>.part.<pid>`, must pass a full verify, and is
// renamed to its canonical name; a valid file already there is reused.
#pragma once

#include <string>

#include "format.hpp"

namespace trims::remote {

struct RemoteRef {
  enum class Backend { Dir, Http };
  Backend backend{Backend::Dir};
  std::string base;  // directory, or http://host[:port][/prefix]
  fmt::ModelKey key;
};

RemoteRef make_ref(const std::string& url, const fmt::ModelKey& key);  // remote_store.cpp:58-72
// remote_store.cpp:74-120. Returns the canonical path under dest_dir.
// RemoteNotFound (missing remotely / HTTP 404), TransportError (I/O, HTTP
// status, connection), ChecksumMismatch (the download failed verification).
std::string fetch(const RemoteRef& ref, const std::string& dest_dir);

}  // namespace trims::remote
