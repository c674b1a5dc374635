"""Synthetic model artifacts: the reference's catalogs and real-shape CNNs.

* ``small37`` / ``large8`` / ``tiny`` restate proj/src/bench/catalog.cpp:21-66
  (the paper's Table 2 / Table 4 rows) and ``catalog_manifest`` restates
  catalog.cpp:111-128: ``layers`` 1-D F64 tensors of raw splitmix64 words
  (``gen_catalog``, catalog.cpp:130-159, seed ^ fnv1a(name)). Blob bytes and
  trailers are bit-identical to the reference's (tests/test_format_parity.py).
* ``alexnet`` (the paper's Table-1 dims, proj/tests/test_model_format.cpp:24-44,
  grouped conv2/4/5), ``resnet50``, ``vgg16``, ``vgg19`` with real shapes and
  fp32 uniform init (our K5 definition): fan-in bound sqrt(6/fan_in) for
  weights, small ranges for biases and batch-norm statistics.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass

import numpy as np

from . import format as F
from ._lib import check, lib

NS = "zoo"          # catalog.hpp:35
VERSION = "1.0.0"   # catalog.hpp:36

from .catalog_tables import LARGE8, SMALL37  # noqa: E402


@dataclass(frozen=True)
class CatalogModel:
    name: str
    layers: int
    workspace_mb: float
    weights_mb: float


def catalog(name: str) -> tuple[list[CatalogModel], float]:
    if name == "small37":
        return [CatalogModel(*r) for r in SMALL37], 1.0
    if name == "large8":
        return [CatalogModel(*r) for r in LARGE8], 1.0
    if name == "tiny":
        return [CatalogModel(*r) for r in SMALL37], 64.0
    raise ValueError(f"unknown catalog {name} (small37|large8|tiny)")


def catalog_key(m: CatalogModel) -> F.ModelKey:
    return F.ModelKey(NS, m.name, VERSION)


def scaled_weights_bytes(m: CatalogModel, div: float) -> int:  # catalog.cpp:95-97
    return int(m.weights_mb * 1e6 / div) // 8 * 8


def scaled_workspace_bytes(m: CatalogModel, div: float) -> int:  # catalog.cpp:99-101
    return int(m.workspace_mb * 1e6 / div)


def catalog_manifest(m: CatalogModel, div: float) -> str:
    """catalog.cpp:111-128: `layers` F64 tensors, all but the last 8-element aligned."""
    total = scaled_weights_bytes(m, div) // 8
    layers = min(m.layers, max(total, 1))
    base = total // layers // 8 * 8
    decls, assigned = [], 0
    for i in range(layers):
        elems = total - assigned if i + 1 == layers else max(base, 8)
        assigned += elems
        decls.append((f"layer_{i:04d}", "f64", [elems]))
    return F.make_manifest(catalog_key(m), decls, scaled_workspace_bytes(m, div))


def catalog_blob(manifest_json: str, name: str, seed: int) -> np.ndarray:
    """Blob of a catalog model: value k = splitmix(seed ^ fnv1a(name), k), padding zero."""
    m = json.loads(manifest_json)
    blob_bytes = _blob_bytes(m)
    blob = np.zeros(blob_bytes // 8, np.uint64)
    stream = (seed ^ F.fnv1a(name)) & 0xFFFFFFFFFFFFFFFF
    k = 0
    for t in m["tensors"]:
        n = t["nbytes"] // 8
        view = blob[t["offset"] // 8: t["offset"] // 8 + n]
        check(lib.trims_fill_splitmix_host(view.ctypes.data, n, stream, k))
        k += n
    return blob.view(np.uint8)


def _blob_bytes(m: dict) -> int:
    end = max((t["offset"] + t["nbytes"] for t in m["tensors"]), default=0)
    return (end + 63) // 64 * 64


def gen_catalog(name: str, out_dir: str, seed: int = 1, only=None) -> list[str]:
    """bench::gen_catalog (catalog.cpp:130-159): one .trms per model."""
    models, div = catalog(name)
    os.makedirs(out_dir, exist_ok=True)
    paths = []
    for m in models:
        if only and m.name not in (only if isinstance(only, (list, tuple, set)) else [only]):
            continue
        mj = catalog_manifest(m, div)
        path = os.path.join(out_dir, catalog_key(m).filename)
        F.write_model(path, mj, catalog_blob(mj, m.name, seed))
        paths.append(path)
    return paths


# ---------------------------------------------------------------- real-shape CNNs

from .archs import ARCHS, Arch, Layer, alexnet, arch_key_tuple, arch_tensors, resnet50, vgg16, vgg19  # noqa: E402,F401


def arch_key(arch: Arch) -> F.ModelKey:
    return F.ModelKey(*arch_key_tuple(arch))


def arch_manifest(arch: Arch, workspace: int = 0) -> str:
    return F.make_manifest(arch_key(arch), [(n, "f32", d) for n, d, _ in arch_tensors(arch)], workspace)


def tensor_stream(seed: int, model: str, tensor: str) -> int:
    return (seed ^ F.fnv1a(f"{model}/{tensor}")) & 0xFFFFFFFFFFFFFFFF


def arch_blob(arch: Arch, seed: int = 1) -> tuple[str, np.ndarray]:
    """Manifest JSON + padded fp32 blob (host generator; bit-identical to the device K5)."""
    mj = arch_manifest(arch)
    m = json.loads(mj)
    blob = np.zeros(_blob_bytes(m) // 4, np.float32)
    ranges = {n: r for n, _, r in arch_tensors(arch)}
    for t in m["tensors"]:
        n = t["nbytes"] // 4
        view = blob[t["offset"] // 4: t["offset"] // 4 + n]
        lo, hi = ranges[t["name"]]
        check(lib.trims_fill_uniform_host(view.ctypes.data, n, tensor_stream(seed, arch.name, t["name"]), 0,
                                          float(np.float32(lo)), float(np.float32(hi))))
    return mj, blob.view(np.uint8)


def write_arch(arch: Arch, out_dir: str, seed: int = 1) -> str:
    os.makedirs(out_dir, exist_ok=True)
    mj, blob = arch_blob(arch, seed)
    path = os.path.join(out_dir, arch_key(arch).filename)
    F.write_model(path, mj, blob)
    return path
