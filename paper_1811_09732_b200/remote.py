"""The remote tier feeding the disk cache: remote::make_ref / remote::fetch
(proj/src/remote_store.cpp:58-120), implemented in csrc/remote.cpp.

`url` is the daemon's `remote_url` (proj/include/mrm/daemon.hpp:26):
"dir:<path>" (or a bare path) is copied, "http://host[:port][/prefix]" is
fetched with an HTTP/1.1 GET. The download lands as `<file>.part.<pid>`, must
pass a full verify (the artifact trailer SHA-256), and is renamed to the
canonical `<ns>__<name>__<version>.trms`; a valid file already there is reused.
A Store with `StoreOptions(remote_url=...)` calls this on a miss that is not on
disk (outcome "remote_fetch")."""
from __future__ import annotations

import ctypes

from . import format as F
from ._lib import check, lib


def fetch(url: str, key: F.ModelKey, dest_dir: str) -> tuple[str, int]:
    """-> (canonical path under dest_dir, file bytes). Raises TrimsError with
    RemoteNotFound / TransportError / ChecksumMismatch as the reference."""
    buf = ctypes.create_string_buffer(4096)
    n = ctypes.c_uint64()
    check(lib.trims_remote_fetch(url.encode(), key.ns.encode(), key.name.encode(), key.version.encode(),
                                 dest_dir.encode(), buf, 4096, ctypes.byref(n)))
    return buf.value.decode(), n.value
