"""bench.py's value leg alone (HBM-resident transform, R rotating buffer sets,
K launches back to back between CUDA events), for A/B runs:
    python scripts/transform_value.py [arch] [K] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200.ingest import IngestPlan

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
src_json, blob = C.arch_blob(C.ARCHS[arch](), seed=1)
plan = IngestPlan(src_json, F.PLAN_CONVERT | F.PLAN_PERMUTE_4D, "bf16")
R = max(2, -(-4 * (126 << 20) // (blob.size + plan.resident_bytes)))
srcs = [torch.from_numpy(blob).cuda() for _ in range(R)]
dsts = [torch.empty(plan.resident_bytes, dtype=torch.uint8, device="cuda") for _ in range(R)]
sums = [torch.zeros(plan.buckets, dtype=torch.int64, device="cuda") for _ in range(R)]
st = torch.cuda.Stream()
for i in range(2 * R):
    plan.transform(srcs[i % R].data_ptr(), dsts[i % R].data_ptr(), sums[i % R].data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
alg = plan.read_bytes + plan.write_bytes
out = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(K):
        plan.transform(srcs[i % R].data_ptr(), dsts[i % R].data_ptr(), sums[i % R].data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    out.append(e0.elapsed_time(e1) * 1e3 / K)
us = sorted(out)[len(out) // 2]
print(json.dumps({"arch": arch, "us_per_launch": round(us, 2), "artifact_GBps": round(blob.size / us / 1e3, 1),
                  "algorithmic_GBps": round(alg / us / 1e3, 1), "all_us": [round(x, 2) for x in out]}))
