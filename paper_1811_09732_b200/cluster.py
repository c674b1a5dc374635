"""Multi-GPU node: one store per GPU process, a shared residency directory,
and NVLink peer serve (builder-defined, the reference runs one
daemon per node and has no peer tier).

The directory lives in csrc/directory.cpp (POSIX shared memory, one seqlocked
row per rank); the peer open is csrc/directory.cpp:open_with_peers and the pull
is CudaTierBackend::publish_from_peer (one fused copy+checksum kernel reading
the peer's segment over NVLink). This module is the ctypes surface plus the
launcher glue that derives rank/world from torchrun's environment.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

from . import format as F
from ._lib import DirCoords, check, lib
from .store import Store, StoreOptions


def peer_score(key: str, rank: int) -> int:
    """Rendezvous weight of (key "ns/name@version", rank): a requester pulls
    from the holder with the highest weight."""
    return lib.trims_peer_score(key.encode(), rank)


class Directory:
    """A rank's handle on the node directory (diagnostics and tests; stores
    open their own through StoreOptions.directory)."""

    def __init__(self, name: str, world: int, rank: int, slots: int = 0):
        self.name, self.world, self.rank = name, world, rank
        h = ctypes.c_void_p()
        check(lib.trims_dir_open(name.encode(), world, rank, slots, ctypes.byref(h)))
        self._h = h

    def close(self) -> None:
        if self._h:
            lib.trims_dir_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @staticmethod
    def unlink(name: str) -> None:
        check(lib.trims_dir_unlink(name.encode()))

    def publish(self, key: F.ModelKey, **coords) -> None:
        c = DirCoords(**coords)
        check(lib.trims_dir_publish(self._h, *key.b(), ctypes.byref(c)))

    def retract(self, key: F.ModelKey) -> None:
        check(lib.trims_dir_retract(self._h, *key.b()))

    def holders(self, key: F.ModelKey, cap: int = 64) -> list[dict]:
        buf = (DirCoords * cap)()
        n = ctypes.c_uint64()
        check(lib.trims_dir_holders(self._h, *key.b(), buf, cap, ctypes.byref(n)))
        return [{f: getattr(buf[i], f) for f, _ in DirCoords._fields_} for i in range(min(cap, n.value))]


def node_env() -> tuple[int, int, int]:
    """(rank, world, local device) from torchrun's environment (1 node)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def node_store(opts: StoreOptions, job: str | None = None) -> Store:
    """The store of this GPU process: device = LOCAL_RANK, and — for world > 1
    — the directory "trims.<job>" shared by the node's ranks (job defaults to
    torchrun's MASTER_PORT so concurrent jobs do not collide)."""
    rank, world, local = node_env()
    o = dataclasses.replace(opts, device=local, rank=rank, world=world)
    if world > 1 and not o.directory:
        o.directory = f"trims.{job or os.environ.get('MASTER_PORT', 'job')}"
    return Store(o)
