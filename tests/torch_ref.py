"""CPU oracle of the forward pass (test infrastructure, never on the product path).

Two restatements, both on the SAME resident bf16 weights the GPU path reads
(widened exactly, KRSC permuted back to KCRS):

* ``forward`` — a plain PyTorch fp32 model (activations stay fp32). Kept as a
  coarse cross-check; the B200 path rounds to bf16 between layers, so the two
  differ by ~1e-2.
* ``forward_bf16`` — the B200 executor's arithmetic restated op by op
  (``csrc/net.cu`` / ``gemm.cu`` epilogue / ``nn_kernels.cu``): every rounding
  point the device has, at the same place, with the contraction itself done in
  fp64 (exact products, negligible summation error) and rounded once to fp32,
  as an exact fp32 accumulator would. What remains between this and the GPU is
  only the device's fp32 summation order, which flips an occasional bf16
  activation by one ulp; ``tests/test_gpu_forward.py`` states the tolerance
  that follows from it.

Rounding points restated (device file:line):
  input          fp32 -> bf16 RNE (``nn_kernels.cu`` input_prep / im2col_input)
  BN fold        s = g / sqrtf(v + eps), t = b - m*s in fp32 (``nn_kernels.cu`` bn_fold_batched_kernel)
  conv/GEMM      acc(fp32) -> fma(acc, s, t) [+ residual] [relu] -> bf16 (``gemm.cu`` epilogue)
  max pool       exact on bf16
  global avgpool fp32 sum / HW -> bf16
  FC (GEMV, batch <= 8, K % 256 == 0)  fp32 dot + bias, relu -> bf16 (hidden) / fp32 (logits)
  FC (GEMM otherwise)                  GEMM epilogue -> bf16; the logits are bf16 widened to fp32
"""
import json

import numpy as np
import torch
import torch.nn.functional as Fn


def weights_from_resident(res_json: str, blob: np.ndarray) -> dict:
    out = {}
    for t in json.loads(res_json)["tensors"]:
        raw = blob[t["offset"]:t["offset"] + t["nbytes"]]
        if t["dtype"] == "bf16":
            x = torch.from_numpy((raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32).copy())
        elif t["dtype"] == "f32":
            x = torch.from_numpy(raw.view(np.float32).copy())
        else:
            raise ValueError(t["dtype"])
        x = x.reshape(t["dims"])
        if t.get("layout") == "krsc":
            x = x.permute(0, 3, 1, 2).contiguous()  # [K,R,S,C] -> [K,C,R,S]
        out[t["name"]] = x
    return out


def bn_of(conv: str) -> str:
    if conv.endswith("downsample.0"):
        return conv[:-1] + "1"
    i = conv.rfind("conv")
    return conv[:i] + "bn" + conv[i + 4:]


def forward(arch, W: dict, x: torch.Tensor) -> torch.Tensor:
    x = x.to(torch.bfloat16).float()
    named, cur = {}, x
    for l in arch.layers:
        if l.kind == "conv":
            inp = named[l.src] if l.src else cur
            y = Fn.conv2d(inp, W[f"{l.name}.weight"], W.get(f"{l.name}.bias") if l.bias else None, stride=l.stride,
                          padding=l.pad, groups=l.groups)
            if l.bn:
                b = bn_of(l.name)
                y = Fn.batch_norm(y, W[f"{b}.running_mean"], W[f"{b}.running_var"], W[f"{b}.weight"], W[f"{b}.bias"],
                                  training=False, eps=1e-5)
            if l.res:
                y = y + named[l.res]
            if l.relu:
                y = torch.relu(y)
            cur = y
        elif l.kind == "pool_max":
            cur = Fn.max_pool2d(cur, l.k, l.stride, l.pad)
        elif l.kind == "pool_avg":
            cur = Fn.adaptive_avg_pool2d(cur, 1)
        elif l.kind == "flatten":
            cur = torch.flatten(cur, 1)
        elif l.kind == "fc":
            cur = Fn.linear(cur, W[f"{l.name}.weight"], W.get(f"{l.name}.bias") if l.bias else None)
            if l.relu:
                cur = torch.relu(cur)
        if l.out:
            named[l.out] = cur
    return cur


def _bf(t: torch.Tensor) -> torch.Tensor:
    """fp32 -> bf16 RNE -> fp32 (the device's cvt.rn.bf16x2.f32)."""
    return t.float().to(torch.bfloat16).float()


def _fma32(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor) -> torch.Tensor:
    """fmaf(a, b, c) on fp32 operands: the product is exact in fp64, one rounding to fp32."""
    return (a.double() * b.double() + c.double()).float()


def bn_fold(W: dict, conv: str, eps: float = 1e-5):
    """nn_kernels.cu bn_fold_batched_kernel: s = g / sqrtf(v + eps); t = b - m * s (contracted to one fma)."""
    b = bn_of(conv)
    g, beta, m, v = (W[f"{b}.{k}"].float() for k in ("weight", "bias", "running_mean", "running_var"))
    s = g / torch.sqrt(v + torch.tensor(eps, dtype=torch.float32))
    return s, _fma32(-m, s, beta)


def apply_layer_bf16(arch, i: int, W: dict, cur: torch.Tensor, named: dict, batch: int,
                     acc_dtype=torch.float64, pre_round: bool = False) -> torch.Tensor:
    """Layer ``i`` of ``arch`` as the device computes it, on fp32 tensors that
    hold bf16 values (``cur`` = previous output, ``named`` = named outputs).
    ``pre_round`` returns the fp32 value before the final bf16 rounding (diagnostics)."""
    bf = (lambda t: t.float()) if pre_round else _bf
    l = arch.layers[i]
    last_fc = max(j for j, m in enumerate(arch.layers) if m.kind == "fc")
    if l.kind == "conv":
        inp = named[l.src] if l.src else cur
        acc = Fn.conv2d(inp.to(acc_dtype), W[f"{l.name}.weight"].to(acc_dtype), None, stride=l.stride,
                        padding=l.pad, groups=l.groups).float()
        C = l.cout
        if l.bn:
            s, t = bn_fold(W, l.name)
        else:
            s = torch.ones(C)
            t = W[f"{l.name}.bias"].float() if l.bias else torch.zeros(C)
        y = _fma32(acc, s.view(1, C, 1, 1), t.view(1, C, 1, 1))
        if l.res:
            y = y + named[l.res]
        if l.relu:
            y = torch.relu(y)
        return bf(y)
    if l.kind == "pool_max":
        return Fn.max_pool2d(cur, l.k, l.stride, l.pad)
    if l.kind == "pool_avg":
        return bf((cur.double().sum(dim=(2, 3), keepdim=True) / (cur.shape[2] * cur.shape[3])).float())
    if l.kind == "flatten":
        return torch.flatten(cur, 1)
    if l.kind == "fc":
        acc = (cur.reshape(batch, -1).to(acc_dtype) @ W[f"{l.name}.weight"].to(acc_dtype).t()).float()
        if l.bias:
            acc = acc + W[f"{l.name}.bias"].float()
        if l.relu:
            acc = torch.relu(acc)
        gemv = batch <= 8 and l.cin % 256 == 0
        return acc if (i == last_fc and gemv) else bf(acc)
    raise ValueError(l.kind)


def forward_bf16(arch, W: dict, x: torch.Tensor, acc_dtype=torch.float64) -> torch.Tensor:
    """The B200 executor's arithmetic on CPU (see the module docstring). ``acc_dtype``
    = float64 is the oracle; float32 is a second summation order, used to size
    the tolerance."""
    named, cur = {}, _bf(x)
    for i, l in enumerate(arch.layers):
        cur = apply_layer_bf16(arch, i, W, cur, named, x.shape[0], acc_dtype)
        if l.out:
            named[l.out] = cur
    return cur


def resident_weights_cpu(arch, seed: int = 1) -> dict:
    """The resident bf16 weights the store would lend for ``arch`` at ``seed``
    (fp32 generator -> bf16 RNE; BN vectors too), without a GPU: for CPU-side
    tolerance sizing."""
    from paper_1811_09732_b200 import catalog as C
    mj, blob = C.arch_blob(arch, seed)
    W = {}
    for t in json.loads(mj)["tensors"]:
        v = torch.from_numpy(blob[t["offset"]:t["offset"] + t["nbytes"]].view(np.float32).copy())
        W[t["name"]] = _bf(v).reshape(t["dims"])
    return W
