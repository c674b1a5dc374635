"""Plain PyTorch fp32 reference of the forward pass (test infrastructure).

It runs on the SAME resident bf16 weights the GPU path reads (widened to
fp32, KRSC permuted back to KCRS) and on the bf16-rounded input, with every
op in fp32 — so the only differences to the B200 path are its bf16
activations between layers and its fp32 accumulation order.
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
