"""bench.py's e2e leg alone (pinned host fp32 ResNet-50 artifact -> resident
bf16/KRSC through the C ABI, L2 flushed before every step):
    python scripts/e2e_ab.py [arch] [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200.ingest import IngestPlan

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src_json, blob = C.arch_blob(C.ARCHS[name](), seed=1)
plan = IngestPlan(src_json, F.PLAN_CONVERT | F.PLAN_PERMUTE_4D, "bf16", 0)
host = torch.from_numpy(blob).pin_memory()
dst = torch.empty(plan.resident_bytes, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    plan.ingest_host(host.data_ptr(), dst.data_ptr())
ts, h2d = [], []
for _ in range(steps):
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cs, st = plan.ingest_host(host.data_ptr(), dst.data_ptr())
    ts.append(time.perf_counter() - t0)
    h2d.append(st["h2d_ms"])
ts.sort()
h2d.sort()
print(json.dumps({"arch": name, "streams": os.environ.get("TRIMS_H2D_STREAMS", "2"),
                  "e2e_GBps_median": round(blob.size / ts[len(ts) // 2] / 1e9, 2),
                  "e2e_GBps_best": round(blob.size / ts[0] / 1e9, 2),
                  "h2d_GBps_median": round(blob.size / (h2d[len(h2d) // 2] / 1e3) / 1e9, 2)}))
