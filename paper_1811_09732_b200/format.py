"""Artifact format helpers over the C ABI (proj/include/mrm/model_format.hpp roles).

Everything here calls libtrims (format.cpp / sha256.cpp); Python only shapes
arguments. Manifests travel as their canonical JSON text — the same bytes the
reference's nlohmann dump() produces.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib, text_call

DTYPE_CODE = {"f64": 0, "f32": 1, "f16": 2, "i8": 3, "bf16": 4}
DTYPE_SIZE = {"f64": 8, "f32": 4, "f16": 2, "i8": 1, "bf16": 2}
NP_DTYPE = {"f64": np.float64, "f32": np.float32, "f16": np.float16, "i8": np.int8, "bf16": np.uint16}

PLAN_CONVERT = 1
PLAN_PERMUTE_4D = 2

MODEL, LAYER, BLOCK = 0, 1, 2  # ShareGranularity kinds (shared_segment.hpp:29)


@dataclass(frozen=True)
class ModelKey:
    ns: str
    name: str
    version: str

    def __str__(self) -> str:  # model_format.cpp:94-96
        return f"{self.ns}/{self.name}@{self.version}"

    @property
    def filename(self) -> str:  # canonical_filename (model_format.cpp:98-100)
        return f"{self.ns}__{self.name}__{self.version}.trms"

    def b(self):
        return self.ns.encode(), self.name.encode(), self.version.encode()


@dataclass
class ArtifactInfo:
    manifest_json: str
    checksum: bytes
    blob_bytes: int
    blob_offset: int

    @property
    def manifest(self) -> dict:
        return json.loads(self.manifest_json)


def sha256(data) -> bytes:
    arr = np.frombuffer(data, np.uint8) if isinstance(data, (bytes, bytearray, memoryview)) else \
        np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    out = (ctypes.c_uint8 * 32)()
    check(lib.trims_sha256(arr.ctypes.data if arr.size else None, arr.size, out))
    return bytes(out)


def read_manifest(path: str, full_verify: bool = False) -> ArtifactInfo:
    """model::read_manifest(path, full_verify) (model_format.cpp:370-409)."""
    cs = (ctypes.c_uint8 * 32)()
    bb, bo = ctypes.c_uint64(), ctypes.c_uint64()
    js = text_call(lambda out, cap: lib.trims_read_manifest(path.encode(), int(full_verify), out, cap, cs,
                                                            ctypes.byref(bb), ctypes.byref(bo)), cap=1 << 22)
    return ArtifactInfo(js, bytes(cs), bb.value, bo.value)


def canonical(manifest_json: str) -> str:
    return text_call(lambda o, c: lib.trims_manifest_canonical(manifest_json.encode(), o, c), cap=1 << 22)


def decls_text(decls) -> bytes:
    return "".join(f"{n} {dt} {','.join(str(int(d)) for d in dims)}\n" for n, dt, dims in decls).encode()


def make_manifest(key: ModelKey, decls, workspace: int = 0) -> str:
    """model::make_manifest (model_format.cpp:158-177) -> canonical JSON."""
    return text_call(lambda o, c: lib.trims_make_manifest(*key.b(), decls_text(decls), workspace, o, c), cap=1 << 22)


def write_model(path: str, manifest_json: str, blob) -> None:
    """model::write_model_file: blob is the full padded blob (blob_bytes)."""
    arr = np.ascontiguousarray(blob).view(np.uint8).reshape(-1) if not isinstance(blob, (bytes, bytearray)) \
        else np.frombuffer(blob, np.uint8)
    check(lib.trims_write_model(path.encode(), manifest_json.encode(), arr.ctypes.data if arr.size else None))


def layout_for(manifest_json: str, kind: int = MODEL, block_bytes: int = 2 << 20):
    txt = text_call(lambda o, c: lib.trims_layout_for(manifest_json.encode(), kind, block_bytes, o, c), cap=1 << 22)
    rows = []
    for line in txt.splitlines():
        n, s, off, ln = line.split()
        rows.append((n, int(s), int(off), int(ln)))
    return rows


def resident_manifest(manifest_json: str, plan_flags: int = 0, out_dtype: str = "bf16") -> str:
    return text_call(lambda o, c: lib.trims_resident_manifest(manifest_json.encode(), plan_flags,
                                                              DTYPE_CODE[out_dtype], o, c), cap=1 << 22)


def plan_info(manifest_json: str, plan_flags: int = 0, out_dtype: str = "bf16") -> dict:
    out = (ctypes.c_uint64 * 4)()
    check(lib.trims_plan_info(manifest_json.encode(), plan_flags, DTYPE_CODE[out_dtype], out))
    return {"tiles": out[0], "buckets": out[1], "read_bytes": out[2], "write_bytes": out[3]}


def touch_host(blob: np.ndarray, manifest_json: str) -> int:
    """Client::touch (client.cpp:338-359) over a host copy of the blob."""
    arr = np.ascontiguousarray(blob).view(np.uint8).reshape(-1)
    out = ctypes.c_uint64()
    check(lib.trims_touch_host(arr.ctypes.data if arr.size else None, manifest_json.encode(), ctypes.byref(out)))
    return out.value


def checksum_host(data, word0: int = 0) -> int:
    arr = np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    out = ctypes.c_uint64()
    check(lib.trims_checksum_host(arr.ctypes.data if arr.size else None, arr.size, word0, ctypes.byref(out)))
    return out.value


def fnv1a(s: str) -> int:
    return lib.trims_fnv1a(s.encode())


def tensor_specs(manifest_json: str):
    m = json.loads(manifest_json)
    return m["tensors"]
