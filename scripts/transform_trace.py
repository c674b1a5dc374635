"""Per-CTA timeline of one HBM-resident transform launch (diagnostic build):
    make -C paper_1811_09732_b200/csrc OBJ=build_trace OUT=../variants LIBNAME=libtrims_trace.so EXTRA=-DTRIMS_TRACE
    TRIMS_LIB=paper_1811_09732_b200/variants/libtrims_trace.so python scripts/transform_trace.py [arch] [launches]
Prints, in µs from the earliest CTA start: CTA start spread, first-stage-ready
latency, the producer's last issue, CTA end distribution, and staged bytes /
tiles per CTA (min/median/max), for L2-flushed launches."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200._lib import lib
from paper_1811_09732_b200.ingest import IngestPlan

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
src_json, blob = C.arch_blob(C.ARCHS[arch](), seed=1)
plan = IngestPlan(src_json, 3, "bf16")
d_src = torch.from_numpy(blob).cuda()
d_dst = torch.empty(plan.resident_bytes, dtype=torch.uint8, device="cuda")
d_sums = torch.zeros(plan.buckets, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_r = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
fn = lib.trims_debug_transform_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
carve = lib.trims_debug_carveout
carve.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
prewarm = os.environ.get("PREWARM", "0") == "1"  # empty big-smem launch after the flush
s = torch.cuda.current_stream()
buf = np.zeros(16384 * 10, np.uint64)
evms = []
for i in range(n + 2):
    flush.zero_()
    flush_r.view(torch.int64).sum()
    if prewarm:
        carve(3 * ((64 << 10) + 128), 148, s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(buf.ctypes.data, 0)  # reset the record counter
    e0.record()
    plan.transform(d_src.data_ptr(), d_dst.data_ptr(), d_sums.data_ptr(), s.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    if i < 2:
        continue
    evms.append(e0.elapsed_time(e1) * 1e3)
    recs = fn(buf.ctypes.data, buf.size)  # records of this launch (the counter resets per call)
    assert recs > 0
    t = buf[: recs * 10].reshape(-1, 10).astype(np.int64)
    t0 = t[:, 0].min()
    rel = lambda c: (t[:, c] - t0) / 1e3  # noqa: E731
    q = lambda x: [round(float(np.min(x)), 2), round(float(np.median(x)), 2), round(float(np.max(x)), 2)]  # noqa: E731
    print(json.dumps({"arch": arch, "prewarm": prewarm, "event_us": round(evms[-1], 2),
                      "ctas": int(len(t)), "span_us": round(float(rel(3).max()), 2),
                      "start_us[min,med,max]": q(rel(0)), "first_ready_us": q(rel(1)),
                      "last_issue_us": q(rel(2)), "end_us": q(rel(3)),
                      "staged_KB": q(t[:, 4] / 1024), "tiles": q(t[:, 5]),
                      "static_issued_us": q(rel(6)), "dyn_tiles": q(t[:, 7]),
                      "corr_end_vs_static_issued": round(float(np.corrcoef(rel(3), rel(6))[0, 1]), 3),
                      "late_ctas(end>p90)": [{"cta": int(i), "static_us": round(float(rel(6)[i]), 2),
                                              "dyn": int(t[i, 7]), "KB": int(t[i, 4] // 1024)}
                                             for i in np.argsort(-rel(3))[:5]],
                      "end_hist_us": np.histogram(rel(3), bins=8)[1].round(1).tolist(),
                      "end_hist_n": np.histogram(rel(3), bins=8)[0].tolist()}))
