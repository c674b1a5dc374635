"""Inference on shared weights: the B200 compute step of load-and-serve.

The reference's compute stand-in is ``Client::touch`` (client.cpp:338-359), an
FNV-1a pass over the weight bytes. Here a client binds the store-lent resident
weights (bf16, conv filters KRSC) to a native network executor (csrc/net.cu):
tcgen05 GEMMs for every conv/FC contraction (im2col for k>1), bandwidth-bound
pooling/flatten/GEMV kernels, batch-norm folded at bind time into per-channel
fp32 epilogue scale/shift (the shared weights are never modified), and the
whole forward replayed as one CUDA graph.
"""
from __future__ import annotations

import ctypes

from . import catalog as C
from ._lib import check, lib


def arch_text(arch: C.Arch) -> str:
    lines = [f"input hw={arch.input_hw} c=3"]
    for l in arch.layers:
        if l.kind == "conv":
            lines.append(f"conv name={l.name} cin={l.cin} cout={l.cout} k={l.k} stride={l.stride} pad={l.pad} "
                         f"groups={l.groups} bias={int(l.bias)} bn={int(l.bn)} relu={int(l.relu)} src={l.src} "
                         f"res={l.res} out={l.out}")
        elif l.kind == "pool_max":
            lines.append(f"pool_max k={l.k} stride={l.stride} pad={l.pad} out={l.out}")
        elif l.kind == "pool_avg":
            lines.append(f"pool_avg k={l.k}")
        elif l.kind == "flatten":
            lines.append("flatten")
        elif l.kind == "fc":
            lines.append(f"fc name={l.name} cin={l.cin} cout={l.cout} bias={int(l.bias)} relu={int(l.relu)}")
        else:
            raise ValueError(l.kind)
    return "\n".join(lines) + "\n"


NET_MODES = {"latency": 0, "throughput": 1, "lean": 3}  # trims_net_create_ex flags


class BoundNet:
    """A network executor over one attached model view (weights stay shared)."""

    def __init__(self, view, arch: C.Arch | str, batch: int = 1, device: int = 0, mode: str = "latency"):
        """mode: "latency" (split-K layers: fastest single request), "throughput"
        (one CTA per output tile: many clients' forwards pack one GPU) or "lean"
        (throughput with GEMM variants that fit two CTAs per SM)."""
        arch = C.ARCHS[arch]() if isinstance(arch, str) else arch
        self.arch, self.batch, self.device, self.view, self.mode = arch, batch, device, view, mode
        h = ctypes.c_void_p()
        check(lib.trims_net_create_ex(device, arch_text(arch).encode(), view.manifest_json.encode(), view.base_ptr,
                                      batch, NET_MODES[mode], ctypes.byref(h)))
        self._h = h
        inp, lg = ctypes.c_void_p(), ctypes.c_void_p()
        classes, hw = ctypes.c_int(), ctypes.c_int()
        check(lib.trims_net_buffers(h, ctypes.byref(inp), ctypes.byref(lg), ctypes.byref(classes), ctypes.byref(hw)))
        self.input_ptr, self.logits_ptr = int(inp.value), int(lg.value)
        self.classes, self.input_hw = classes.value, hw.value
        info = (ctypes.c_double * 3)()
        check(lib.trims_net_info(h, info))
        self.flops, self.launches, self.workspace_bytes = info[0], int(info[1]), int(info[2])

    def input_view(self):
        """Zero-copy torch view of the net's fp32 NCHW input buffer."""
        from .client import TensorView
        n = self.batch * 3 * self.input_hw * self.input_hw
        return TensorView("input", [self.batch, 3, self.input_hw, self.input_hw], "f32", "native", 0, n * 4,
                          self.input_ptr).torch(f"cuda:{self.device}")

    def logits_view(self):
        from .client import TensorView
        return TensorView("logits", [self.batch, self.classes], "f32", "native", 0, self.batch * self.classes * 4,
                          self.logits_ptr).torch(f"cuda:{self.device}")

    def layer_count(self) -> int:
        return int(lib.trims_net_tap(self._h, -1, None, None, None))

    def tap(self, layer: int):
        """Device view of what architecture layer `layer` wrote in the last forward
        (NCHW-permuted torch view of the NHWC buffer; bf16, or fp32 logits), or
        None for a conv whose 2x2 max pool was fused into it (the next layer's
        tap is the pooled map)."""
        import torch
        from .client import TensorView
        p, dims, dt = ctypes.c_void_p(), (ctypes.c_int * 4)(), ctypes.c_int()
        check(lib.trims_net_tap(self._h, layer, ctypes.byref(p), dims, ctypes.byref(dt)))
        if dt.value == 2:  # a conv whose 2x2 max pool ran in its epilogue: the pool layer holds the result
            return None
        n, h, w, c = dims
        es = 4 if dt.value else 2
        t = TensorView(f"layer{layer}", [n * h * w * c * es], "i8", "native", 0, n * h * w * c * es,
                       int(p.value)).torch(f"cuda:{self.device}").view(torch.uint8)
        t = t.view(torch.float32 if dt.value else torch.bfloat16).view(n, h, w, c)
        return t.permute(0, 3, 1, 2)

    def rebind(self, view) -> None:
        """Follow the model to a new segment (same resident manifest, new generation)."""
        if view.manifest_json != self.view.manifest_json:
            raise ValueError("rebind needs the same resident manifest")
        check(lib.trims_net_rebind(self._h, view.base_ptr))
        self.view = view

    def run(self, stream=None, graph: bool = True) -> None:
        check(lib.trims_net_run(self._h, stream, int(graph)))

    def infer(self, x, out=None, stream=None, graph: bool = True):
        """One request through the C ABI (trims_net_forward_host): H2D of the
        host input, the forward (one CUDA graph launch), D2H of the logits,
        stream sync. x: fp32 NCHW host tensor/array (pinned for full PCIe
        rate); out: a host [batch, classes] fp32 buffer (allocated if None)."""
        import numpy as np
        for a, what in ((x, "x"), (out, "out")):
            if a is None:
                continue
            dt = str(getattr(a, "dtype", ""))
            if dt not in ("float32", "torch.float32"):
                raise ValueError(f"{what} must be float32, got {dt}")
            contig = a.is_contiguous() if hasattr(a, "is_contiguous") else a.flags["C_CONTIGUOUS"]
            if not contig:
                raise ValueError(f"{what} must be contiguous")
            if hasattr(a, "device") and getattr(a.device, "type", "cpu") != "cpu":
                raise ValueError(f"{what} must be a host buffer")
        if out is None:
            out = np.empty((self.batch, self.classes), np.float32)
        xp = x.data_ptr() if hasattr(x, "data_ptr") else x.ctypes.data
        op = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        n_in = self.batch * 3 * self.input_hw * self.input_hw
        n = x.numel() if hasattr(x, "numel") else x.size
        m = out.numel() if hasattr(out, "numel") else out.size
        if n != n_in or m != self.batch * self.classes:
            raise ValueError("input / output sizes do not match the bound net")
        check(lib.trims_net_forward_host(self._h, xp, op, stream, int(graph)))
        return out

    def forward(self, x, graph: bool = True):
        """x: fp32 NCHW (any device). Returns the fp32 logits on the GPU."""
        import torch
        self.input_view().copy_(x)
        s = torch.cuda.current_stream(self.device)
        self.run(s.cuda_stream, graph)
        return self.logits_view()

    def close(self):
        if self._h:
            lib.trims_net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
