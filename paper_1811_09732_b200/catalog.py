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

# name, layers, workspace MB, weights MB  (catalog.cpp:21-59)
SMALL37 = [
    ("alexnet", 16, 516, 238), ("googlenet", 116, 111, 27), ("caffenet", 16, 512, 233),
    ("rcnn-ilsvrc13", 16, 479, 221), ("dpn68", 361, 122, 49), ("dpn92", 481, 340, 145),
    ("inception-v3", 472, 257, 92), ("inception-v4", 747, 399, 164), ("inceptionbn-v2", 416, 313, 129),
    ("inceptionbn-v3", 416, 142, 44), ("inception-resnet-v2", 1102, 493, 214), ("locationnet", 514, 666, 285),
    ("nin", 24, 131, 29), ("resnet101", 526, 423, 170), ("resnet101-v2", 522, 428, 171),
    ("resnet152", 777, 548, 231), ("resnet152-11k", 769, 721, 311), ("resnet152-v2", 761, 340, 231),
    ("resnet18-v2", 99, 154, 45), ("resnet200-v2", 1009, 589, 248), ("resnet269-v2", 1346, 889, 391),
    ("resnet34-v2", 179, 222, 84), ("resnet50", 268, 270, 98), ("resnet50-v2", 259, 275, 98),
    ("resnext101", 526, 375, 170), ("resnext101-32x4d", 522, 378, 170), ("resnext26-32x4d", 147, 147, 59),
    ("resnext50", 271, 222, 96), ("resnext50-32x4d", 267, 224, 96), ("squeezenet-v1.0", 52, 34, 4.8),
    ("squeezenet-v1.1", 52, 28, 4.8), ("vgg16", 32, 1228, 528), ("vgg16-sod", 32, 1198, 514),
    ("vgg16-sos", 32, 1195, 513), ("vgg19", 38, 1270, 549), ("wrn50-v2", 267, 758, 264),
    ("xception", 236, 244, 88),
]
# catalog.cpp:62-66 (no workspace figures in the source table)
LARGE8 = [("alexnet-s1", 16, 0, 238), ("alexnet-s2", 16, 0, 770), ("alexnet-s3", 16, 0, 1694),
          ("alexnet-s4", 16, 0, 3010), ("vgg16-s1", 32, 0, 528), ("vgg16-s2", 32, 0, 1704),
          ("vgg16-s3", 32, 0, 3664), ("vgg16-s4", 32, 0, 6408)]


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

@dataclass
class Layer:
    """One op of a CNN graph over named manifest tensors."""
    kind: str          # conv | fc | pool_max | pool_avg | relu | add | flatten | lrn
    name: str = ""
    cin: int = 0
    cout: int = 0
    k: int = 1
    stride: int = 1
    pad: int = 0
    groups: int = 1
    bias: bool = False
    bn: bool = False
    relu: bool = False
    src: str = ""      # input activation name ("" = previous)
    res: str = ""      # residual input fused into the epilogue
    out: str = ""      # output activation name


@dataclass
class Arch:
    name: str
    input_hw: int
    layers: list
    classes: int = 1000


def alexnet() -> Arch:
    """Table-1 AlexNet (test_model_format.cpp:24-44): 227x227 input, grouped conv2/4/5."""
    L = [
        Layer("conv", "conv1", 3, 96, 11, 4, 0, 1, True, relu=True),
        Layer("pool_max", k=3, stride=2),
        Layer("conv", "conv2", 96, 256, 5, 1, 2, 2, True, relu=True),
        Layer("pool_max", k=3, stride=2),
        Layer("conv", "conv3", 256, 384, 3, 1, 1, 1, True, relu=True),
        Layer("conv", "conv4", 384, 384, 3, 1, 1, 2, True, relu=True),
        Layer("conv", "conv5", 384, 256, 3, 1, 1, 2, True, relu=True),
        Layer("pool_max", k=3, stride=2),
        Layer("flatten"),
        Layer("fc", "fc6", 9216, 4096, bias=True, relu=True),
        Layer("fc", "fc7", 4096, 4096, bias=True, relu=True),
        Layer("fc", "fc8", 4096, 1000, bias=True),
    ]
    return Arch("alexnet", 227, L)


def _vgg(cfg, name) -> Arch:
    L, cin, i = [], 3, 0
    for v in cfg:
        if v == "M":
            L.append(Layer("pool_max", k=2, stride=2))
        else:
            L.append(Layer("conv", f"features.{i}", cin, v, 3, 1, 1, 1, True, relu=True))
            cin = v
            i += 1  # conv, then its ReLU, occupy two features.* slots
        i += 1
    L.append(Layer("flatten"))
    L.append(Layer("fc", "classifier.0", 512 * 7 * 7, 4096, bias=True, relu=True))
    L.append(Layer("fc", "classifier.3", 4096, 4096, bias=True, relu=True))
    L.append(Layer("fc", "classifier.6", 4096, 1000, bias=True))
    return Arch(name, 224, L)


def vgg16() -> Arch:
    return _vgg([64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"], "vgg16")


def vgg19() -> Arch:
    return _vgg([64, 64, "M", 128, 128, "M", 256, 256, 256, 256, "M", 512, 512, 512, 512, "M",
                 512, 512, 512, 512, "M"], "vgg19")


def resnet50() -> Arch:
    """torchvision ResNet-50 (v1.5, stride on the 3x3) with its state_dict names."""
    L = [Layer("conv", "conv1", 3, 64, 7, 2, 3, bn=True, relu=True, out="stem"),
         Layer("pool_max", k=3, stride=2, pad=1, out="x")]
    cin = 64
    for li, (width, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)], 1):
        for b in range(blocks):
            p = f"layer{li}.{b}"
            s = stride if b == 0 else 1
            cout = width * 4
            if b == 0:
                L.append(Layer("conv", f"{p}.downsample.0", cin, cout, 1, s, 0, bn=True, src="x", out="sc"))
                res = "sc"
            else:
                res = "x"
            L.append(Layer("conv", f"{p}.conv1", cin, width, 1, 1, 0, bn=True, relu=True, src="x"))
            L.append(Layer("conv", f"{p}.conv2", width, width, 3, s, 1, bn=True, relu=True))
            L.append(Layer("conv", f"{p}.conv3", width, cout, 1, 1, 0, bn=True, relu=True, res=res, out="x"))
            cin = cout
    L.append(Layer("pool_avg", k=7, stride=1))
    L.append(Layer("flatten"))
    L.append(Layer("fc", "fc", 2048, 1000, bias=True))
    return Arch("resnet50", 224, L)


ARCHS = {"alexnet": alexnet, "resnet50": resnet50, "vgg16": vgg16, "vgg19": vgg19}


def arch_tensors(arch: Arch):
    """(name, dims, (lo, hi)) in manifest order for an architecture."""
    out = []
    for l in arch.layers:
        if l.kind == "conv":
            fan_in = (l.cin // l.groups) * l.k * l.k
            b = math.sqrt(6.0 / fan_in)
            out.append((f"{l.name}.weight", [l.cout, l.cin // l.groups, l.k, l.k], (-b, b)))
            if l.bias:
                bb = 1.0 / math.sqrt(fan_in)
                out.append((f"{l.name}.bias", [l.cout], (-bb, bb)))
            if l.bn:
                bn = l.name.replace("conv", "bn") if "downsample" not in l.name else l.name[:-1] + "1"
                out += [(f"{bn}.weight", [l.cout], (0.5, 1.0)), (f"{bn}.bias", [l.cout], (-0.1, 0.1)),
                        (f"{bn}.running_mean", [l.cout], (-0.1, 0.1)),
                        (f"{bn}.running_var", [l.cout], (0.5, 1.5))]
        elif l.kind == "fc":
            b = math.sqrt(6.0 / l.cin)
            out.append((f"{l.name}.weight", [l.cout, l.cin], (-b, b)))
            if l.bias:
                bb = 1.0 / math.sqrt(l.cin)
                out.append((f"{l.name}.bias", [l.cout], (-bb, bb)))
    return out


def arch_key(arch: Arch) -> F.ModelKey:
    return F.ModelKey("torchvision" if arch.name != "alexnet" else "mxnet", arch.name, VERSION)


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
