"""Per-launch timeline of K back-to-back transform launches, as bench.py's
value leg runs them (rotating buffer sets, one stream, PDL), diagnostic build:
    make -C paper_1811_09732_b200/csrc OBJ=build_trace OUT=../variants LIBNAME=libtrims_trace.so EXTRA=-DTRIMS_TRACE
    TRIMS_LIB=paper_1811_09732_b200/variants/libtrims_trace.so python scripts/transform_b2b_trace.py [arch] [K]
Per launch (µs, relative to the previous launch's last CTA end): first / last
CTA start, first stage ready (min/med/max), CTA end (min/med/max)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import lib
from paper_1811_09732_b200.ingest import IngestPlan

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 12
src_json, blob = C.arch_blob(C.ARCHS[arch](), seed=1)
plan = IngestPlan(src_json, F.PLAN_CONVERT | F.PLAN_PERMUTE_4D, "bf16")
R = max(2, -(-4 * (126 << 20) // (blob.size + plan.resident_bytes)))
srcs = [torch.from_numpy(blob).cuda() for _ in range(R)]
dsts = [torch.empty(plan.resident_bytes, dtype=torch.uint8, device="cuda") for _ in range(R)]
sums = [torch.zeros(plan.buckets, dtype=torch.int64, device="cuda") for _ in range(R)]
fn = lib.trims_debug_transform_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
st = torch.cuda.Stream()
buf = np.zeros(16384 * 10, np.uint64)
for i in range(R):
    plan.transform(srcs[i].data_ptr(), dsts[i].data_ptr(), sums[i].data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
fn(buf.ctypes.data, 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for i in range(K):
    plan.transform(srcs[i % R].data_ptr(), dsts[i % R].data_ptr(), sums[i % R].data_ptr(), st.cuda_stream)
e1.record(st)
torch.cuda.synchronize()
recs = fn(buf.ctypes.data, buf.size)
t = buf[: recs * 10].reshape(-1, 10).astype(np.int64)
# records are appended in CTA start order and every launch has one CTA per
# blockIdx: the k-th record of blockIdx b belongs to launch k
t = t[np.argsort(t[:, 0], kind="stable")]
occ = np.zeros(len(t), np.int64)
seen = {}
for i, b in enumerate(t[:, 9].tolist()):
    occ[i] = seen.get(b, 0)
    seen[b] = occ[i] + 1
t = np.concatenate([t, occ[:, None]], axis=1)
launch_ids = sorted(set(occ.tolist()))
q = lambda x: [round(float(np.min(x)), 2), round(float(np.median(x)), 2), round(float(np.max(x)), 2)]  # noqa: E731
print(json.dumps({"arch": arch, "K": K, "event_us_per_launch": round(e0.elapsed_time(e1) * 1e3 / K, 2),
                  "records": int(recs), "launches": len(launch_ids)}))
prev_end = None
for lid in launch_ids:
    L = t[t[:, 10] == lid]
    base = prev_end if prev_end is not None else L[:, 0].min()
    rel = lambda c: (L[:, c] - base) / 1e3  # noqa: E731
    print(json.dumps({"ctas": int(len(L)), "start": q(rel(0)), "first_ready": q(rel(1)), "static_issued": q(rel(6)),
                      "last_issue": q(rel(2)), "end": q(rel(3)), "span_us": round(float((L[:, 3].max() - L[:, 0].min()) / 1e3), 2)}))
    prev_end = L[:, 3].max()
