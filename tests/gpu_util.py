"""Helpers for the -m gpu tests: oracle-side expected resident blobs."""
import json

import numpy as np

import oracle


def expected_resident(src_json: str, src_blob: np.ndarray, res_json: str) -> np.ndarray:
    """CPU oracle of the ingest transform: per tensor convert (+ permute), zero pads."""
    P = oracle.port()
    s = json.loads(src_json)["tensors"]
    r = json.loads(res_json)["tensors"]
    end = max((t["offset"] + t["nbytes"] for t in r), default=0)
    out = np.zeros((end + 63) // 64 * 64, np.uint8)
    for ts, tr in zip(s, r):
        raw = src_blob[ts["offset"]:ts["offset"] + ts["nbytes"]]
        sd, dd = ts["dtype"], tr["dtype"]
        if sd == "f32":
            x = raw.view(np.float32)
        elif sd == "f64":
            x = raw.view(np.float64)
        elif sd == "f16":
            x = raw.view(np.uint16)
        else:
            x = raw
        if sd == dd:
            y = x.copy()
        elif (sd, dd) == ("f32", "bf16"):
            y = P.f32_to_bf16(x)
        elif (sd, dd) == ("f64", "f32"):
            y = P.f64_to_f32(x)
        elif (sd, dd) == ("f64", "bf16"):
            y = P.f64_to_bf16(x)
        elif (sd, dd) == ("f16", "f32"):
            y = P.f16_to_f32(x)
        elif (sd, dd) == ("f16", "bf16"):
            y = P.f32_to_bf16(P.f16_to_f32(x))
        else:
            raise ValueError((sd, dd))
        if tr.get("layout") == "krsc":
            K, C, R, S = ts["dims"]
            y = P.permute_kcrs_krsc(y.reshape(K, C, R, S))
        yb = np.ascontiguousarray(y).view(np.uint8).reshape(-1)
        assert yb.size == tr["nbytes"]
        out[tr["offset"]:tr["offset"] + tr["nbytes"]] = yb
    return out


def layer_checksums(res_json: str, blob: np.ndarray) -> list:
    """Per-tensor (layer object, padding included) oracle checksums + the leading-pad bucket."""
    P = oracle.port()
    r = json.loads(res_json)["tensors"]
    out = []
    for i, t in enumerate(r):
        end = r[i + 1]["offset"] if i + 1 < len(r) else blob.size
        out.append(P.block_checksum(blob[t["offset"]:end], t["offset"] // 8))
    lead = r[0]["offset"] if r else 0
    out.append(P.block_checksum(blob[:lead], 0) if lead else 0)
    return out
