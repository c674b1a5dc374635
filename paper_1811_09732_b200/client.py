"""Client SDK: open / close / touch / forward on shared (or private) weights.

Mirrors proj/include/mrm/client.hpp:97-119 and proj/src/client.cpp:
``open`` makes the rho = b/q - n(o+s) decision (client.cpp:16-18, 148-222),
attaches the store's exported HBM segment read-only and slices it into
device ``TensorView``s (client.cpp:243-315); it falls back to a private load
(client.cpp:224-241) exactly where the reference does. ``touch`` is the
reference's FNV-1a compute stand-in (client.cpp:338-359), kept as a parity
check; the B200 compute on the shared weights is ``models.forward``.
"""
from __future__ import annotations

import ctypes
import json
import os
import time
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import format as F
from ._lib import Errc, TrimsError, check, lib, text_call

SHARED, PRIVATE = "shared", "private"


@dataclass
class CostModelParams:
    q: float = 200e6    # disk bytes/s      (client.cpp:70 kDefaultParams)
    o: float = 2.5e-4   # export s/object
    s: float = 2.5e-4   # attach s/object


def share_benefit(nbytes: float, n_objects: float, p: CostModelParams) -> float:
    """client.cpp:16-18."""
    return nbytes / p.q - n_objects * (p.o + p.s)


@dataclass
class TensorView:
    name: str
    dims: list
    dtype: str
    layout: str
    offset: int
    nbytes: int
    dev_ptr: int
    _keep: object = field(default=None, repr=False, compare=False)  # what keeps dev_ptr's bytes valid

    def torch(self, device=None):
        """Zero-copy torch view of the (read-only) device bytes."""
        import torch
        typestr = {"f64": "<f8", "f32": "<f4", "f16": "<f2", "i8": "|i1", "bf16": "<i2"}[self.dtype]

        class _CAI:
            pass

        obj = _CAI()
        obj.__cuda_array_interface__ = {"shape": tuple(int(d) for d in self.dims), "typestr": typestr,
                                        "data": (int(self.dev_ptr), False), "version": 2, "strides": None}
        t = torch.as_tensor(obj, device=device or f"cuda:{torch.cuda.current_device()}")
        return t.view(torch.bfloat16) if self.dtype == "bf16" else t


@dataclass
class OpenTimings:  # client.hpp:53-57
    rpc_s: float = 0.0
    attach_s: float = 0.0
    private_load_s: float = 0.0


@dataclass
class ModelView:
    key: F.ModelKey
    origin: str
    fallback_reason: str
    manifest_json: str              # resident manifest
    base_ptr: int
    tensors: list = field(default_factory=list)
    model_id: int = 0
    generation: int = 0
    outcome: str = ""
    export: object = None
    timings: OpenTimings = field(default_factory=OpenTimings)
    is_open: bool = True
    _import: object = None          # trims_import* for imported mappings
    _private: object = None         # owning torch buffer of a private view
    _hold: object = None            # ViewHold of a shared view (keeps its bytes valid)
    _release: object = None

    @property
    def manifest(self) -> dict:
        return json.loads(self.manifest_json)

    def tensor(self, name: str) -> TensorView:
        for t in self.tensors:
            if t.name == name:
                return t
        raise KeyError(name)

    def blob_bytes(self) -> int:
        m = self.manifest
        end = max((t["offset"] + t["nbytes"] for t in m["tensors"]), default=0)
        return (end + 63) // 64 * 64


_PARSED: dict = {}  # manifest JSON -> parsed tensor records (manifests are immutable)


class TensorViews(Sequence):
    """The views of one attached model, built on first access: a warm open of
    a new generation then costs no per-tensor Python objects (267 for
    ResNet-50) until a caller actually walks the tensors."""

    __slots__ = ("_recs", "_base", "_made", "_keep")

    def __init__(self, recs, base_ptr: int, keep=None):
        self._recs, self._base, self._made, self._keep = recs, base_ptr, {}, keep

    def held_by(self, keep) -> "TensorViews":
        """The same views for one open, holding that open's pin / lease."""
        return TensorViews(self._recs, self._base, keep)

    def __len__(self):
        return len(self._recs)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self._recs)))]
        if i < 0:
            i += len(self._recs)
        v = self._made.get(i)
        if v is None:
            n, d, dt, lay, off, nb = self._recs[i]
            v = self._made[i] = TensorView(n, d, dt, lay, off, nb, self._base + off, self._keep)
        return v

    def __eq__(self, other):
        return list(self) == list(other)


def slice_tensors(manifest_json: str, base_ptr: int) -> TensorViews:
    """client.cpp:60-65 with device pointers; the parse is cached per manifest
    (client.cpp:293-307 caches it by digest), so a new generation of a model
    only re-bases the views."""
    recs = _PARSED.get(manifest_json)
    if recs is None:
        recs = [(t["name"], t["dims"], t["dtype"], t.get("layout", "native"), t["offset"], t["nbytes"])
                for t in json.loads(manifest_json)["tensors"]]
        if len(_PARSED) > 256:
            _PARSED.clear()
        _PARSED[manifest_json] = recs
    return TensorViews(recs, base_ptr)


class ViewHold:
    """Keeps an attached view's bytes valid for as long as any object that can
    read them (the ModelView, its TensorViews, a BoundNet) is alive — also
    after close() and after the store evicts the model, as an attached POSIX
    shm view outlives its owner (proj/tests/test_shared_segment.cpp:99-110):
    an in-process pin on the published record, or a lease row in the owner's
    arena lease table (trims_store_pin / trims_lease_acquire)."""

    __slots__ = ("_h", "_release")

    def __init__(self, h, release):
        self._h, self._release = h, release

    @classmethod
    def pin(cls, store, model_id: int, generation: int) -> "ViewHold":
        h = ctypes.c_void_p()
        check(lib.trims_store_pin(store._h, model_id, generation, ctypes.byref(h)))
        return cls(h, lib.trims_pin_release)

    @classmethod
    def lease(cls, token: str, offset: int, generation: int) -> "ViewHold":
        h = ctypes.c_void_p()
        check(lib.trims_lease_acquire(token.encode(), offset, generation, ctypes.byref(h)))
        return cls(h if h.value else None, lib.trims_lease_release)

    def release(self) -> None:
        if self._h:
            self._release(self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class ImportCache:
    """Per-process attach state. One read-only mapping per exported allocation
    (token: the store's arena, or a dedicated segment), and per attached model
    (token, offset, generation) its manifest + views, so re-opening a hot
    model costs neither a map nor a digest check (the reference caches
    manifests by digest, client.cpp:293-307)."""

    def __init__(self):
        self.maps = {}    # token -> (trims_import*, base)
        self.models = {}  # (token, offset, generation) -> (ptr, json, digest, views)

    def clear(self):
        for imp, _ in self.maps.values():
            lib.trims_import_close(imp)
        self.maps.clear()
        self.models.clear()


def map_allocation(device: int, fd: int, alloc_bytes: int):
    """Map an exported allocation read-only (shared_segment.cpp:212-232)."""
    imp = ctypes.c_void_p()
    base = ctypes.c_void_p()
    check(lib.trims_import_open(device, fd, alloc_bytes, ctypes.byref(imp), ctypes.byref(base)))
    return imp, int(base.value)


def attach_segment(imp, offset: int, generation: int, payload_bytes: int, digest: bytes):
    """Validate one model segment of a mapping (tail, generation, seal) and its
    manifest digest (client.cpp:284-291); returns (device ptr, resident JSON)."""
    ptr = ctypes.c_void_p()
    dig = (ctypes.c_uint8 * 32).from_buffer_copy(bytes(digest))
    json_txt = text_call(lambda o, c: lib.trims_import_attach(imp, offset, generation, payload_bytes, dig,
                                                               ctypes.byref(ptr), o, c))
    return int(ptr.value), json_txt


def import_segment(device: int, fd: int, alloc_bytes: int, offset: int, generation: int, payload_bytes: int,
                   digest: bytes):
    """map_allocation + attach_segment in one call (used by one-shot importers)."""
    imp, _ = map_allocation(device, fd, alloc_bytes)
    try:
        ptr, js = attach_segment(imp, offset, generation, payload_bytes, digest)
    except Exception:
        lib.trims_import_close(imp)
        raise
    return imp, ptr, js


class Client:
    """In-process client of a ``Store`` (or of a ``ipc.RemoteStore`` endpoint)."""

    def __init__(self, store=None, model_dirs=(), granularity: int = F.MODEL, params: CostModelParams | None = None,
                 disabled: bool | None = None, attach_via_import: bool = False, device: int = 0,
                 plan_flags: int | None = None, out_dtype: str | None = None):
        self.store = store
        self.model_dirs = list(model_dirs)
        env_dirs = os.environ.get("MRM_MODEL_DIR")  # client.cpp:81-91
        if env_dirs:
            self.model_dirs += [d for d in env_dirs.split(":") if d]
        self.granularity = granularity
        self.params = params
        self.disabled = disabled if disabled is not None else os.environ.get("MRM_DISABLE") == "1"
        self.attach_via_import = attach_via_import
        self.device = device
        opts = getattr(store, "opts", None)
        self.plan_flags = plan_flags if plan_flags is not None else (opts.plan_flags if opts else 0)
        self.out_dtype = out_dtype or (opts.convert_to if opts and opts.convert_to else "bf16")
        self.imports = ImportCache()
        self.cached_stats = None  # client.hpp cached_stats_: the last StatsResponse
        self._local = {}  # (model_id, generation) -> (resident json, digest, tensor views)

    # client.cpp:94-106
    def resolve_local(self, key: F.ModelKey, local_path: str | None = None) -> str | None:
        if local_path:
            return local_path if os.path.exists(local_path) else None
        for d in self.model_dirs:
            p = os.path.join(d, key.filename)
            if os.path.exists(p):
                return p
        return None

    # client.cpp:124-135
    def stats(self) -> dict:
        """Fetch (and cache) the store's stats: tiers, counters, the workspace
        headroom and the published calibration."""
        st = self.store.stats()
        self.cached_stats = st
        return st

    # client.cpp:137-142
    def effective_params(self, params: CostModelParams | None = None) -> CostModelParams:
        if params:
            return params
        if self.params:
            return self.params
        cs = self.cached_stats
        if cs and cs.get("has_calibration"):
            return CostModelParams(cs["calib_q"], cs["calib_o"], cs["calib_s"])
        return CostModelParams()

    def decide(self, key: F.ModelKey, local: str | None, force_private: bool = False, force_shared: bool = False,
               granularity: int | None = None, params: CostModelParams | None = None,
               block_bytes: int = 2 << 20) -> tuple[str, object]:
        """The placement decision of Client::open (client.cpp:148-205), before
        any data moves: (PRIVATE, fallback reason) or (SHARED, granularity).
        1. forced / disabled -> private;
        2. with a local artifact and no force_shared: rho = b/q - n(o+s) with
           the caller's params, else the store's published calibration (stats
           fetched once; unreachable -> private), else kDefaultParams; Layer
           falls back to Model when only that pays; rho <= 0 -> private;
        3. workspace reservation: the artifact's workspace_bytes must fit the
           store's advertised headroom (workspace_headroom x fast capacity),
           else private."""
        if force_private:
            return PRIVATE, "forced"
        if self.disabled:
            return PRIVATE, "disabled"
        if self.store is None:
            return PRIVATE, "daemon_unreachable"
        g = self.granularity if granularity is None else granularity
        if local and not force_shared:
            info = F.read_manifest(local)
            manifest = json.loads(info.manifest_json)
            b = os.path.getsize(local)
            if not params and not self.params and self.cached_stats is None:
                try:
                    self.stats()
                except (TrimsError, OSError):
                    return PRIVATE, "daemon_unreachable"
            p = self.effective_params(params)
            n = len(F.layout_for(info.manifest_json, g, block_bytes))
            if share_benefit(b, n, p) <= 0:
                if g == F.LAYER and share_benefit(b, 1, p) > 0:
                    g = F.MODEL
                else:
                    return PRIVATE, "benefit_non_positive"
            ws = int(manifest.get("workspace_bytes", 0))
            if ws > 0 and self.cached_stats is None:
                try:
                    self.stats()
                except (TrimsError, OSError):
                    return PRIVATE, "daemon_unreachable"
            cs = self.cached_stats
            if cs is not None and "workspace_headroom" in cs:
                headroom = cs["workspace_headroom"] * float(cs["tiers"][0]["capacity_bytes"])
                if float(ws) > headroom:
                    return PRIVATE, "workspace_reservation"
        return SHARED, g

    def open(self, key: F.ModelKey, force_private: bool = False, force_shared: bool = False,
             granularity: int | None = None, params: CostModelParams | None = None,
             local_path: str | None = None, block_bytes: int = 2 << 20) -> ModelView:
        """client.cpp:148-222."""
        local = self.resolve_local(key, local_path)
        origin, what = self.decide(key, local, force_private, force_shared, granularity, params, block_bytes)
        if origin == PRIVATE:
            if not local:
                raise TrimsError(Errc.NotFound, "NotFound", f"{key} (no daemon, no local artifact)")
            return self.open_private(key, local, what)
        try:
            return self.open_shared(key, what, block_bytes)
        except TrimsError as e:
            if local and e.code in (Errc.NotFound, Errc.RemoteNotFound, Errc.NoEvictableSpace,
                                    Errc.TooLargeForFast, Errc.Internal, Errc.DaemonUnreachable,
                                    Errc.ConnectionLost):
                return self.open_private(key, local, "daemon_error")
            raise

    def calibrate(self, sample: F.ModelKey) -> CostModelParams:
        """Client::calibrate (client.cpp:361-423): q = one sequential read of the
        sample artifact; o = the store's export time per open (handle_export
        counter deltas) and s = the local attach time, medians of 32 warm
        force-shared opens."""
        local = self.resolve_local(sample)
        if not local:
            raise TrimsError(Errc.NotFound, "NotFound", "calibration sample not found locally")
        t0 = time.perf_counter()
        total = 0
        with open(local, "rb", buffering=0) as f:
            while True:
                chunk = f.read(1 << 20)
                if not chunk:
                    break
                total += len(chunk)
        dt = time.perf_counter() - t0
        if dt <= 0 or total == 0:
            raise TrimsError(Errc.Internal, "Internal", "calibration read failed")
        q = total / dt
        exports, attaches = [], []
        before = self.stats()
        prev_export, prev_opens = before["export_ns"], before["open_requests"]
        for _ in range(32):
            v = self.open(sample, force_shared=True)
            if v.origin != SHARED:
                raise TrimsError(Errc.DaemonUnreachable, "DaemonUnreachable", "calibration needs the store")
            attaches.append(v.timings.attach_s)
            self.close(v)
            after = self.stats()
            if after["open_requests"] > prev_opens:
                exports.append((after["export_ns"] - prev_export) / 1e9 / (after["open_requests"] - prev_opens))
            prev_export, prev_opens = after["export_ns"], after["open_requests"]
        med = lambda v: sorted(v)[len(v) // 2] if v else 0.0
        return CostModelParams(q, med(exports), med(attaches))

    def open_shared(self, key: F.ModelKey, granularity: int = F.MODEL, block_bytes: int = 2 << 20) -> ModelView:
        """client.cpp:243-315: RPC, attach, digest, slice."""
        t0 = time.perf_counter()
        ex = self.store.open(key, granularity, block_bytes)
        t1 = time.perf_counter()
        token = ex.token.decode() if isinstance(ex.token, bytes) else ex.token
        remote = getattr(ex, "remote", False)
        digest = bytes(ex.manifest_digest)
        if remote or self.attach_via_import:
            mkey = (token, ex.segment_offset, ex.generation)
            hit = self.imports.models.get(mkey)
            if hit is None:
                mapping = self.imports.maps.get(token)
                if mapping is None:
                    fd = ex.fd if remote else os.dup(ex.fd)
                    try:
                        mapping = map_allocation(ex.device, fd, ex.alloc_bytes)
                    finally:
                        os.close(fd)
                    self.imports.maps[token] = mapping
                elif remote and ex.fd >= 0:
                    os.close(ex.fd)
                ptr, mjson = attach_segment(mapping[0], ex.segment_offset, ex.generation, ex.payload_bytes, digest)
                hit = (ptr, mjson, digest, slice_tensors(mjson, ptr))
                self.imports.models[mkey] = hit
            elif remote and ex.fd >= 0:
                os.close(ex.fd)
            base, mjson, seen, tensors = hit
            hold = ViewHold.lease(token, ex.segment_offset, ex.generation)
        else:
            # same process: the segment is already mapped; the manifest is
            # fetched, digest-checked and sliced once per (model, generation)
            base = int(ex.dev_ptr)
            hit = self._local.get((ex.model_id, ex.generation))
            if hit is None:
                mjson = self.store.resident_manifest(ex.model_id)
                if F.sha256(mjson.encode()) != digest:
                    raise TrimsError(Errc.Corrupt, "Corrupt", "manifest digest mismatch on attach")
                hit = (mjson, digest, slice_tensors(mjson, base))
                self._local[(ex.model_id, ex.generation)] = hit
            mjson, seen, tensors = hit
            hold = ViewHold.pin(self.store, ex.model_id, ex.generation)
        if seen != digest:
            raise TrimsError(Errc.Corrupt, "Corrupt", "manifest digest mismatch on attach")
        view = ModelView(key, SHARED, "none", mjson, base, tensors.held_by(hold), ex.model_id, ex.generation,
                         outcome=_outcome(ex.outcome), export=ex)
        view._hold = hold
        view.timings.rpc_s = t1 - t0
        view.timings.attach_s = time.perf_counter() - t1
        return view

    def open_private(self, key: F.ModelKey, path: str, reason: str) -> ModelView:
        """client.cpp:224-241: read the artifact and ingest it into private HBM
        with the same plan, so shared and private views are byte-identical."""
        import torch
        t0 = time.perf_counter()
        info = F.read_manifest(path)
        if json.loads(info.manifest_json)["name"] != key.name:
            raise TrimsError(Errc.Corrupt, "Corrupt", f"artifact at {path} holds another model")
        host = torch.empty(max(info.blob_bytes, 1), dtype=torch.uint8, pin_memory=True)
        with open(path, "rb") as f:
            f.seek(info.blob_offset)
            f.readinto(memoryview(host.numpy())[: info.blob_bytes])
        rj = F.resident_manifest(info.manifest_json, self.plan_flags, self.out_dtype)
        rb = json.loads(rj)
        rbytes = max((t["offset"] + t["nbytes"] for t in rb["tensors"]), default=0)
        rbytes = max((rbytes + 63) // 64 * 64, 1)
        dev = torch.empty(rbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        cs = ctypes.c_uint64()
        check(lib.trims_ingest_host(self.device, host.data_ptr(), info.manifest_json.encode(), self.plan_flags,
                                    F.DTYPE_CODE[self.out_dtype], dev.data_ptr(), ctypes.byref(cs), None))
        view = ModelView(key, PRIVATE, reason, rj, dev.data_ptr(), slice_tensors(rj, dev.data_ptr()).held_by(dev))
        view._private = dev
        view.timings.private_load_s = time.perf_counter() - t0
        return view

    def close(self, view: ModelView) -> None:
        """client.cpp:317-336: idempotent."""
        if not view.is_open:
            return
        view.is_open = False
        if view.origin == SHARED:
            try:
                self.store.close(view.key)
            except TrimsError:
                pass
        view._private = None
        view.tensors = []

    def touch(self, view: ModelView) -> int:
        """client.cpp:338-359 over a device->host copy of the view."""
        import torch
        n = view.blob_bytes()
        host = torch.empty(max(n, 1), dtype=torch.uint8)
        if n:
            src = TensorView("blob", [n], "i8", "native", 0, n, view.base_ptr).torch(f"cuda:{self.device}")
            host[:n].copy_(src.view(torch.uint8))
        return F.touch_host(host.numpy()[:n], view.manifest_json)

    def close_all_imports(self):
        self.imports.clear()


def _outcome(code: int) -> str:
    from .store import outcome_name
    return outcome_name(code)
