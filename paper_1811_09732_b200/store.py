"""The model store: CacheCore + CudaTierBackend behind the C ABI.

``Store`` plays the reference daemon's role in-process (proj/src/daemon.cpp:
298-603 minus the sockets): it owns the HBM fast tier, the pinned host tier
and the disk-cache registry of one GPU, and answers open/close with an
``Export`` — the reference's PlacementResult + ObjectRef, carrying a cuMem
fd instead of a shm segment name.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass

from . import format as F
from ._lib import Errc, Export, StoreConfig, TrimsError, check, lib, text_call

OUTCOMES = {0: "fast_hit", 1: "host_hit", 2: "disk_load", 3: "remote_fetch", 4: "peer_hit", 5: "peer_map"}
LRU, LCU = 0, 1
FAST, HOST, DISK = 0, 1, 2


@dataclass
class StoreOptions:
    """DaemonConfig (proj/include/mrm/daemon.hpp:19-34) + the B200 ingest plan."""
    disk_cache_dir: str
    fast_capacity_bytes: int = 1 << 30
    host_capacity_bytes: int = 2 << 30
    disk_capacity_bytes: int = 16 << 30
    policy: int = LRU
    eager_reclaim: bool = False
    full_verify: bool = False
    remote_url: str | None = None      # daemon.hpp:26: "http://host:port/prefix" or "dir:<path>"
    device: int = 0
    convert_to: str | None = None      # e.g. "bf16": floating tensors converted at ingest
    permute_4d: bool = False           # KCRS -> KRSC (NHWC conv weights) at ingest
    pinned_pool_bytes: int = 0         # 0 = host_capacity_bytes
    scan_disk: bool = True
    read_threads: int = 8
    arena_bytes: int = 0               # 0 = auto (fast capacity + slack), 1 = one allocation per model
    # multi-GPU: stores of one node share a residency directory
    directory: str | None = None       # /dev/shm name; None = single GPU
    rank: int = 0
    world: int = 1
    directory_slots: int = 0           # 0 = 1024 per rank
    workspace_headroom_fraction: float = 0.25  # daemon.hpp:29 (published to clients in stats)
    startup_calibration: bool = True   # daemon.hpp:33: q/o/s measured at creation, published in stats
    direct_io: str = "auto"            # cold-load reads: "buffered", "direct" (O_DIRECT) or "auto"
    peer_serve: str = "copy"           # multi-GPU miss held by a peer: "copy" (PeerHit) or "map" (serve in place)

    @property
    def plan_flags(self) -> int:
        return (F.PLAN_CONVERT if self.convert_to else 0) | (F.PLAN_PERMUTE_4D if self.permute_4d else 0)


class Store:
    def __init__(self, opts: StoreOptions):
        self.opts = opts
        cfg = StoreConfig()
        cfg.fast_capacity_bytes = opts.fast_capacity_bytes
        cfg.host_capacity_bytes = opts.host_capacity_bytes
        cfg.disk_capacity_bytes = opts.disk_capacity_bytes
        cfg.policy = opts.policy
        cfg.eager_reclaim = int(opts.eager_reclaim)
        cfg.full_verify = int(opts.full_verify)
        cfg.device = opts.device
        self._dir = opts.disk_cache_dir.encode()
        cfg.disk_cache_dir = self._dir
        cfg.plan_flags = opts.plan_flags
        cfg.out_dtype = F.DTYPE_CODE[opts.convert_to or "bf16"]
        cfg.pinned_pool_bytes = opts.pinned_pool_bytes
        cfg.scan_disk = int(opts.scan_disk)
        cfg.read_threads = opts.read_threads
        cfg.direct_io = {"buffered": 0, "direct": 1, "auto": 2}[opts.direct_io]
        cfg.peer_map = {"copy": 0, "map": 1}[opts.peer_serve]
        cfg.arena_bytes = opts.arena_bytes
        self._dirname = opts.directory.encode() if opts.directory else None
        cfg.directory = self._dirname
        cfg.rank = opts.rank
        cfg.world = opts.world
        cfg.directory_slots = opts.directory_slots
        self._remote = opts.remote_url.encode() if opts.remote_url else None
        cfg.remote_url = self._remote
        cfg.workspace_headroom_fraction = opts.workspace_headroom_fraction
        cfg.startup_calibration = int(opts.startup_calibration)
        h = ctypes.c_void_p()
        check(lib.trims_store_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h

    # -- lifecycle
    def close_store(self) -> None:
        if self._h:
            lib.trims_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close_store()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close_store()

    # -- CacheCore surface (cache_core.hpp:129-196)
    def open(self, key: F.ModelKey, granularity: int = F.MODEL, block_bytes: int = 2 << 20) -> Export:
        ex = Export()
        check(lib.trims_store_open(self._h, *key.b(), granularity, block_bytes, ctypes.byref(ex)))
        return ex

    def fast_resident(self, key: F.ModelKey) -> bool:
        out = ctypes.c_int()
        check(lib.trims_store_fast_resident(self._h, *key.b(), ctypes.byref(out)))
        return bool(out.value)

    def close(self, key: F.ModelKey) -> int:
        rc = ctypes.c_uint64()
        check(lib.trims_store_close(self._h, *key.b(), ctypes.byref(rc)))
        return rc.value

    def reclaim(self, tier: int, nbytes: int, policy: int = LRU) -> list[str]:
        txt = text_call(lambda o, c: lib.trims_store_reclaim(self._h, tier, nbytes, policy, o, c))
        return txt.split()

    def register_disk_file(self, key: F.ModelKey, path: str, nbytes: int) -> None:
        check(lib.trims_store_register_disk_file(self._h, *key.b(), path.encode(), nbytes))

    def drop_all(self) -> None:
        check(lib.trims_store_drop_all(self._h))

    def stats(self) -> dict:
        return json.loads(text_call(lambda o, c: lib.trims_store_stats_json(self._h, o, c)))

    def resident_manifest(self, model_id: int) -> str:
        return text_call(lambda o, c: lib.trims_store_resident_json(self._h, model_id, o, c), cap=1 << 22)

    def ingest_stats(self, model_id: int) -> dict:
        out = (ctypes.c_double * 7)()
        check(lib.trims_store_ingest_stats(self._h, model_id, out))
        return {"h2d_ms": out[0], "total_ms": out[1], "read_ms": out[2], "h2d_bytes": int(out[3]),
                "launches": int(out[4]), "alloc_ms": out[5], "seal_ms": out[6]}

    def checksums(self, model_id: int) -> list[int]:
        cap = 1 << 16
        buf = (ctypes.c_uint64 * cap)()
        n = ctypes.c_uint64()
        check(lib.trims_store_checksums(self._h, model_id, buf, cap, ctypes.byref(n)))
        return list(buf[: n.value])


def outcome_name(code: int) -> str:
    return OUTCOMES.get(code, "?")


def is_not_found(e: Exception) -> bool:
    return isinstance(e, TrimsError) and e.code in (Errc.NotFound, Errc.RemoteNotFound)


def device_count() -> int:
    return lib.trims_device_count()


def default_cache_dir() -> str:
    return os.environ.get("TRIMS_CACHE_DIR", "/tmp/trims-cache")
