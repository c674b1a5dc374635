"""Cold (disk) opens with and without full_verify, ResNet-50 fp32 real-shape
artifact, bf16/KRSC plan: the verified open reads + hashes the blob once
(pipelined, pread.hpp). Also times the reference-style verify (a serial
1-thread read+hash pass, as model_format.cpp:370-409 + read_model's second
pass) for comparison, and the host SHA-256 rate.
    python scripts/verify_cold.py [arch] [reps]"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch  # noqa: F401

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.store import Store, StoreOptions

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
arch = C.ARCHS[name]()
d = tempfile.mkdtemp()
C.write_arch(arch, d, seed=1)
key = C.arch_key(arch)
path = os.path.join(d, key.filename)
info = F.read_manifest(path)
out = {"model": name, "blob_bytes": info.blob_bytes}
blob = np.fromfile(path, np.uint8, info.blob_bytes, offset=info.blob_offset)
t0 = time.perf_counter()
F.sha256(blob)
out["sha256_GBps"] = round(info.blob_bytes / (time.perf_counter() - t0) / 1e9, 3)
for verify in (False, True):
    ts = []
    with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=4 << 30, host_capacity_bytes=4 << 30,
                            convert_to="bf16", permute_4d=True, eager_reclaim=True, full_verify=verify)) as s:
        cli = Client(s)
        for i in range(reps + 1):
            t0 = time.perf_counter()
            v = cli.open(key, force_shared=True)
            ts.append(time.perf_counter() - t0)
            cli.close(v)
    out[f"cold_open_ms_verify={int(verify)}"] = round(1e3 * float(np.median(ts[1:])), 3)
# the reference's verified load: read_manifest(full_verify) streams the blob
# through SHA in chunks, then read_model(verify) reads + hashes it again
ts = []
for i in range(reps):
    t0 = time.perf_counter()
    for _ in range(2):
        with open(path, "rb") as f:
            f.seek(info.blob_offset)
            import hashlib
            h = hashlib.sha256()
            while chunk := f.read(1 << 20):
                h.update(chunk)
    ts.append(time.perf_counter() - t0)
out["reference_style_two_serial_passes_ms (hashlib)"] = round(1e3 * float(np.median(ts)), 3)
print(json.dumps(out))
