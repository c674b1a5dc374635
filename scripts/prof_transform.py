"""Runs only the HBM-resident transform (for ncu / quick timing):
    python scripts/prof_transform.py [arch] [reps] [plan_flags]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.ingest import IngestPlan

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 3
src_json, blob = C.arch_blob(C.ARCHS[arch](), seed=1)
plan = IngestPlan(src_json, flags, "bf16")
d_src = torch.from_numpy(blob).cuda()
d_dst = torch.empty(plan.resident_bytes, dtype=torch.uint8, device="cuda")
d_sums = torch.zeros(plan.buckets, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_r = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
flush_mode = os.environ.get("PROF_FLUSH", "writeread")  # write | writeread | none | rotate


def flush_l2():
    # write 256 MiB (evicts everything), then read another 256 MiB so the
    # dirty lines are written back before the timed region starts
    if flush_mode != "none":
        flush.zero_()
    if flush_mode == "writeread":
        flush_r.view(torch.int64).sum()

s = torch.cuda.current_stream()
for i in range(reps):
    d_sums.zero_()
    plan.transform(d_src.data_ptr(), d_dst.data_ptr(), d_sums.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
times = []
if flush_mode == "rotate":
    # no flush: R buffer sets used in turn, R x (src + dst) >= 4 x L2, so every
    # launch reads and writes memory last touched R-1 launches (>= 3 x L2 of
    # traffic) earlier; K launches back to back between one pair of events
    R = max(2, -(-4 * (126 << 20) // (plan.src_bytes + plan.resident_bytes)))
    srcs = [d_src] + [d_src.clone() for _ in range(R - 1)]
    dsts = [d_dst] + [torch.empty_like(d_dst) for _ in range(R - 1)]
    sums = [d_sums] + [torch.zeros_like(d_sums) for _ in range(R - 1)]
    K = int(os.environ.get("PROF_ITERS", "40"))
    for i in range(2 * R):
        plan.transform(srcs[i % R].data_ptr(), dsts[i % R].data_ptr(), sums[i % R].data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(K):
            plan.transform(srcs[i % R].data_ptr(), dsts[i % R].data_ptr(), sums[i % R].data_ptr(), s.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / K)
else:
    for i in range(int(os.environ.get("PROF_ITERS", "40"))):
        flush_l2()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.transform(d_src.data_ptr(), d_dst.data_ptr(), d_sums.data_ptr(), s.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
# event ticks are ~2 us on this box: report the mean (quantisation averages out)
ms = sum(times) / len(times)
print(json.dumps({"arch": arch, "flags": flags, "flush": flush_mode, "pdl": os.environ.get("TRIMS_TRANSFORM_PDL", "1"),
                  "tiles": plan.tiles, "ms": round(ms, 4), "ms_median": round(sorted(times)[len(times) // 2], 4),
                  "GBps_algo": round((plan.read_bytes + plan.write_bytes) / ms / 1e6, 1),
                  "GBps_src": round(plan.src_bytes / ms / 1e6, 1)}))
