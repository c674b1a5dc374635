"""Fixed costs around one transform launch (diagnostic):
host enqueue time per call, event-timed tiny plan (one 4 KiB tensor), and
back-to-back ResNet-50 launches with the host enqueue measured alongside.
    python scripts/transform_overhead.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200.ingest import IngestPlan

s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}


def setup(src_json, blob):
    plan = IngestPlan(src_json, 3, "bf16")
    d_src = torch.from_numpy(blob).cuda()
    d_dst = torch.empty(max(plan.resident_bytes, 64), dtype=torch.uint8, device="cuda")
    d_sums = torch.zeros(max(plan.buckets, 1), dtype=torch.int64, device="cuda")
    return plan, (lambda: plan.transform(d_src.data_ptr(), d_dst.data_ptr(), d_sums.data_ptr(), s.cuda_stream))


def ev(fn, n=30, pre=True):
    ts = []
    for i in range(n + 3):
        if pre:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return round(float(np.median(ts)), 2)


tiny_json = F.make_manifest(F.ModelKey("t", "tiny", "1"), [("w", "f32", [16, 8, 3, 3])])
tiny_blob = np.zeros(4608 + 64, np.uint8)[:((4608 + 63) // 64) * 64]
_, tiny = setup(tiny_json, tiny_blob)
out["event_us_nothing"] = ev(lambda: None)
out["event_us_tiny_plan"] = ev(tiny)
src_json, blob = C.arch_blob(C.ARCHS["resnet50"](), seed=1)
plan, rn = setup(src_json, blob)
out["event_us_resnet50"] = ev(rn)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    tiny()
out["host_us_per_call_tiny"] = round((time.perf_counter() - t0) / 200 * 1e6, 2)
torch.cuda.synchronize()
K = 40
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    rn()
e1.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
out["back_to_back_resnet50_host_us_per_call"] = round((t1 - t0) / K * 1e6, 2)
out["back_to_back_resnet50_gpu_us_per_call"] = round(e0.elapsed_time(e1) / K * 1e3, 2)
print(json.dumps(out))
