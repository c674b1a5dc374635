"""Real-shape CNN architectures (pure Python: no native library, so the
bench's reference arm can describe the same models without loading
libtrims.so).

``alexnet`` (the paper's Table-1 dims, proj/tests/test_model_format.cpp:24-44,
grouped conv2/4/5), ``resnet50``, ``vgg16``, ``vgg19`` with torchvision
state_dict names. ``arch_tensors`` gives the manifest tensors and their fp32
uniform-init ranges (our K5 definition): fan-in bound sqrt(6/fan_in) for
weights, small ranges for biases and batch-norm statistics.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

VERSION = "1.0.0"


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


def arch_key_tuple(arch: Arch) -> tuple[str, str, str]:
    """(namespace, name, version) of a real-shape model artifact."""
    return ("torchvision" if arch.name != "alexnet" else "mxnet", arch.name, VERSION)
