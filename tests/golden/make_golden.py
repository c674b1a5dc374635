#!/usr/bin/env python3
"""Regenerates tests/golden/* from the UNMODIFIED reference (oracle/_ref/libmrm_ref.so).

Run here, in the container that has /root/reference (the GPU box does not):
    make -C oracle && python tests/golden/make_golden.py
Every vector below is produced by the reference's own code path, called
through oracle/ref_shim.cpp; nothing is computed by our port or product.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import simulator as sim  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

SMALL37 = ["alexnet", "googlenet", "caffenet", "rcnn-ilsvrc13", "dpn68", "dpn92", "inception-v3",
           "inception-v4", "inceptionbn-v2", "inceptionbn-v3", "inception-resnet-v2", "locationnet",
           "nin", "resnet101", "resnet101-v2", "resnet152", "resnet152-11k", "resnet152-v2",
           "resnet18-v2", "resnet200-v2", "resnet269-v2", "resnet34-v2", "resnet50", "resnet50-v2",
           "resnext101", "resnext101-32x4d", "resnext26-32x4d", "resnext50", "resnext50-32x4d",
           "squeezenet-v1.0", "squeezenet-v1.1", "vgg16", "vgg16-sod", "vgg16-sos", "vgg19", "wrn50-v2",
           "xception"]

# Table-1 AlexNet dims as pinned by proj/tests/test_model_format.cpp:24-44.
ALEXNET_T1 = [("conv1_bias", [96]), ("conv1_weight", [96, 3, 11, 11]), ("conv2_weight", [256, 48, 5, 5]),
              ("conv2_bias", [256]), ("conv3_weight", [384, 256, 3, 3]), ("conv3_bias", [384]),
              ("conv4_bias", [384]), ("conv4_weight", [384, 192, 3, 3]), ("conv5_weight", [256, 192, 3, 3]),
              ("conv5_bias", [256]), ("fc6_bias", [4096]), ("fc6_weight", [4096, 9216]),
              ("fc7_weight", [4096, 4096]), ("fc7_bias", [4096]), ("fc8_bias", [1000]),
              ("fc8_weight", [1000, 4096])]


def file_sha(path: str) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


def catalog_entries(R, catalog: str, names: list[str], seed: int, tmp: str) -> list[dict]:
    out = []
    for name in names:
        d = os.path.join(tmp, f"{catalog}-{name}")
        R.gen_catalog(catalog, d, seed, name)
        path = os.path.join(d, f"zoo__{name}__1.0.0.trms")
        rc, mjson, cs, blob = R.read_manifest(path, full_verify=True)
        assert rc == 0
        out.append({"name": name, "seed": seed, "manifest_json": mjson, "trailer": cs.hex(),
                    "blob_bytes": blob, "file_bytes": os.path.getsize(path), "file_sha256": file_sha(path),
                    "touch": R.touch_file(path)})
        os.remove(path)
        print(f"  {catalog}/{name}: {blob} B trailer {cs.hex()[:16]}…", flush=True)
    return out


def main() -> None:
    R = oracle.ref()
    rng = np.random.default_rng(20261017)
    big = "--big" in sys.argv
    with tempfile.TemporaryDirectory(prefix="trims-golden-") as tmp:
        # 1. SHA-256 KATs (test_model_format.cpp:69-81) + longer vectors.
        kat = {"": R.sha256(b"").hex(), "abc": R.sha256(b"abc").hex()}
        vec = {}
        for n in (1, 55, 56, 63, 64, 65, 119, 120, 1000, 100000):
            data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
            vec[data.hex() if n <= 1000 else f"seed:{n}"] = R.sha256(data).hex()
        big_data = np.random.default_rng(7).integers(0, 256, 100000, dtype=np.uint8).tobytes()
        vec = {k: v for k, v in vec.items() if not k.startswith("seed:")}
        vec["rng7_100000"] = R.sha256(big_data).hex()
        json.dump({"kat": kat, "vectors": vec}, open(os.path.join(OUT, "sha256.json"), "w"), indent=1)

        # 2. Catalogs: all of `tiny` (small37 / 64), seed 1 (harness seed) and 42 (CLI default).
        print("catalog tiny …", flush=True)
        tiny = catalog_entries(R, "tiny", SMALL37, 1, tmp)
        tiny42 = catalog_entries(R, "tiny", SMALL37[:4], 42, tmp)
        manif = {name: R.catalog_manifest_json("small37", name) for name in SMALL37}
        large8 = {name: R.catalog_manifest_json("large8", name) for name in
                  ["alexnet-s1", "alexnet-s2", "alexnet-s3", "alexnet-s4", "vgg16-s1", "vgg16-s2", "vgg16-s3", "vgg16-s4"]}
        doc = {"tiny_seed1": tiny, "tiny_seed42": tiny42, "small37_manifests": manif, "large8_manifests": large8}
        if big:
            print("catalog small37 (alexnet, resnet50, vgg16) …", flush=True)
            doc["small37_seed1"] = catalog_entries(R, "small37", ["alexnet", "resnet50", "vgg16"], 1, tmp)
        else:
            cpath = os.path.join(OUT, "catalog.json.gz")
            prev = json.load(gzip.open(cpath, "rt")) if os.path.exists(cpath) else {}
            if "small37_seed1" in prev:
                doc["small37_seed1"] = prev["small37_seed1"]
        with gzip.open(os.path.join(OUT, "catalog.json.gz"), "wt") as f:
            json.dump(doc, f)

        # 3. Artifact bytes: random manifests over every dtype, written by the
        #    reference writer (ModelFileWriter) with seeded payloads.
        print("artifacts …", flush=True)
        arts = []
        for trial in range(24):
            n = int(rng.integers(0, 6))
            decls = []
            for i in range(n):
                dt = ["f64", "f32", "f16", "i8"][int(rng.integers(0, 4))]
                rank = int(rng.integers(1, 4))
                decls.append((f"t{i}", dt, [int(rng.integers(1, 41)) for _ in range(rank)]))
            ws = int(rng.integers(0, 4096))
            key = ("prop", f"r{trial}", "1")
            esz = {"f64": 8, "f32": 4, "f16": 2, "i8": 1}
            total = sum(int(np.prod(d)) * esz[dt] for _, dt, d in decls)
            data_seed = int(rng.integers(0, 2**31))
            data = np.random.default_rng(data_seed).integers(0, 256, total, dtype=np.uint8).tobytes()
            path = os.path.join(tmp, f"art{trial}.trms")
            R.write_model(path, key, decls, ws, data)
            rc, mjson, cs, blob = R.read_manifest(path, True)
            arts.append({"key": key, "decls": decls, "workspace": ws, "data_seed": data_seed,
                         "manifest_json": mjson, "trailer": cs.hex(), "blob_bytes": blob,
                         "file_sha256": file_sha(path), "file_bytes": os.path.getsize(path)})
        t1 = [(n, "f64", d) for n, d in ALEXNET_T1]
        alex_json = R.make_manifest_json(("mxnet", "alexnet", "1.0.0"), t1, 516_000_000)
        t1_f32 = [(n, "f32", d) for n, d in ALEXNET_T1]
        alex_f32 = R.make_manifest_json(("mxnet", "alexnet", "1.0.0"), t1_f32, 516_000_000)
        json.dump({"artifacts": arts, "alexnet_table1_f64": alex_json, "alexnet_table1_f32": alex_f32},
                  open(os.path.join(OUT, "artifacts.json"), "w"), indent=1)

        # 4. layout_for (shared_segment.cpp:63-95) at every granularity.
        print("layouts …", flush=True)
        cases = {
            "unaligned3": [("a", "f64", [3]), ("b", "f64", [17]), ("c", "f64", [5])],
            "sixteen": [(f"l{i}", "f64", [64]) for i in range(16)],
            "blocks5MiB": [("w", "f64", [5 * 1024 * 1024 // 8])],
            "empty": [],
            "mixed": [("x", "f16", [7, 3]), ("y", "i8", [5]), ("z", "f32", [9, 9, 2])],
        }
        lays = {}
        for cname, decls in cases.items():
            path = os.path.join(tmp, f"lay-{cname}.trms")
            esz = {"f64": 8, "f32": 4, "f16": 2, "i8": 1}
            total = sum(int(np.prod(d)) * esz[dt] for _, dt, d in decls)
            R.write_model(path, ("t", cname, "1"), decls, 0, bytes(total))
            lays[cname] = {"decls": decls, "model": R.layout_for(path, 0), "layer": R.layout_for(path, 1),
                           "block2MiB": R.layout_for(path, 2, 2 << 20)}
            if total < 4096:
                lays[cname]["block64"] = R.layout_for(path, 2, 64)
                lays[cname]["block128"] = R.layout_for(path, 2, 128)
        json.dump(lays, open(os.path.join(OUT, "layouts.json"), "w"), indent=1)

        # 5. Decision traces: live reference CacheCore == reference simulator,
        #    per op (outcome, evictions, used bytes, refcount) + final stats.
        print("decisions …", flush=True)
        traces = []
        for t in range(120):
            cfg, models, trace = sim.random_trace(rng, max_models=24 if t % 3 else 48,
                                                  max_ops=600 if t % 4 else 1500, policy=t % 2)
            spec = sim.spec_text(cfg, models, trace)
            out = R.replay(spec)
            live = [l for l in out.splitlines() if l.startswith("live ")]
            simv = [l for l in out.splitlines() if l.startswith("sim ")]
            stats = [l for l in out.splitlines() if l.startswith("stats")][0]
            for a, b in zip(live, simv):
                la, lb = a.split()[1:], b.split()[1:]
                # closes: the simulator reports outcome 0 for a valid close; the live shim reports 0 too
                assert la == lb, (t, a, b)
            traces.append({"spec": spec, "events": live, "stats": stats})
        with gzip.open(os.path.join(OUT, "decisions.json.gz"), "wt") as f:
            json.dump(traces, f)
        run = R.run_oracle(60, 2025, 24, 800)
        json.dump({"run_oracle_seed2025_60x24x800": run}, open(os.path.join(OUT, "oracle_run.json"), "w"))
    pareto_golden(R)
    wire_golden(R)
    print("golden vectors written to", OUT)


def pareto_golden(R) -> None:
    """The reference worker's request streams (mt19937_64 + libstdc++
    uniform_real + pareto_rank), for workload.pareto_trace."""
    cases = []
    for seed, n, active, alpha in [(42, 1000, 37, 1.0), (1, 400, 10, 1.0), (42001127, 1000, 37, 1.0),
                                   (7, 300, 8, 2.5)]:
        cases.append({"seed": seed, "n": n, "active": active, "alpha": alpha, "x_m": 1.0,
                      "trace": R.pareto_trace(seed, n, alpha, 1.0, active)})
    json.dump(cases, open(os.path.join(OUT, "pareto_trace.json"), "w"))


# v1 wire messages (text form of csrc/wire.hpp / oracle/ref_shim.cpp) covering
# every message type, each granularity, escapes, lists and calibration.
WIRE_MESSAGES = [
    "open 1 zoo resnet50 1.0.0 0 0 7",
    "open 1 zoo vgg16 1.0.0 1 0 0",
    "open 1 zoo vgg16-s4 1.0.0 2 4194304 18446744073709551615",
    "open 1 my%20ns n%25ame v%C3%A9 2 64 1",
    "openresp 1 2 98000000 4000000 102000000 1 resnet50 trims.77.arena0?dev=0&alloc=4362076160&seg=0&payload=51248352 1 "
    "0 51220352 " + "0f" * 32,
    "openresp 9 10 64 0 64 3 a t 5 0 64 b t 5 64 64 c t 5 128 64 " + "00" * 32,
    "openresp 0 0 0 0 0 0 " + "ff" * 32,
    "close 1 5 9",
    "closeresp 5 2",
    "stats 1",
    "statsresp " + " ".join(str(i * 1000003) for i in range(20)) + " 2 zoo m 1.0 2 3 5 zoo n 2.0 0 1 4 "
    "1 2 3 4 5 6 7 8 0.25 1 1.5 0.0625 3.5",
    "statsresp " + " ".join("0" for _ in range(20)) + " 0 0 0 0 0 0 0 0 0 0.125 0",
    "error 4 handle%2017%20not%20open",
    "error 7 %",
]


def wire_golden(R) -> None:
    """Reference-encoded v1 frames and the reference decoder's verdict on a
    set of malformed frames (error code, or its text form)."""
    msgs = []
    for t in WIRE_MESSAGES:
        rc, frame = R.wire_encode(t)
        assert rc == 0, t
        msgs.append({"text": t, "frame": frame.hex()})
    rng = np.random.default_rng(20251017)
    bad = []
    base = [bytes.fromhex(m["frame"]) for m in msgs]
    hand = [b"", b"\x01\x00", b"\x00\x00\x00\x00\x01", b"\x02\x00\x00\x00\x01\x02\x00",
            (16 << 20 | 1).to_bytes(4, "little") + b"\x01", b"\x00\x00\x00\x00\x42",
            b"\x02\x00\x00\x00\x05\x01\x00", b"\x03\x00\x00\x00\x05\x01\x00\x00"]
    for f in hand:
        bad.append(f)
    for _ in range(400):  # mutations of valid frames: flips, truncations, extensions, length edits
        f = bytearray(base[int(rng.integers(len(base)))])
        op = int(rng.integers(4))
        if op == 0 and len(f) > 5:
            i = int(rng.integers(5, len(f)))
            f[i] ^= 1 << int(rng.integers(8))
        elif op == 1:
            f = f[: int(rng.integers(len(f)))]
        elif op == 2:
            f += bytes(rng.integers(0, 256, int(rng.integers(1, 9)), dtype=np.uint8))
        else:
            delta = int(rng.integers(-3, 4))
            n = max(0, int.from_bytes(f[:4], "little") + delta)
            f[:4] = n.to_bytes(4, "little")
        bad.append(bytes(f))
    cases = []
    for f in bad:
        rc, text = R.wire_decode(f)
        cases.append({"frame": f.hex(), "rc": rc, "text": text})
    json.dump({"messages": msgs, "decode_cases": cases}, open(os.path.join(OUT, "wire.json"), "w"), indent=0)


if __name__ == "__main__":
    if "--pareto-only" in sys.argv:
        pareto_golden(oracle.ref())
    elif "--wire-only" in sys.argv:
        wire_golden(oracle.ref())
    else:
        main()
