"""Per-layer timeline of one graph-replayed forward pass (diagnostic build):
    make -C paper_1811_09732_b200/csrc OBJ=build_gtrace OUT=../variants LIBNAME=libtrims_gtrace.so EXTRA=-DTRIMS_GEMM_TRACE
    TRIMS_LIB=paper_1811_09732_b200/variants/libtrims_gtrace.so python scripts/gemm_trace.py [arch] [batch]
For every GEMM launch of the forward (in order), in µs relative to the previous
GEMM's last CTA end: first CTA start, last CTA start, producer past
griddepcontrol.wait (median / max), first stage full (max), accumulator full
(max), last CTA end; plus grid and shape. Non-GEMM kernels between GEMMs show
up as gaps."""
import ctypes
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200._lib import lib
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.models import BoundNet
from paper_1811_09732_b200.store import Store, StoreOptions

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
fn = lib.trims_debug_gemm_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
arch = C.ARCHS[name]()
d = tempfile.mkdtemp()
C.write_arch(arch, d, seed=1)
with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=4 << 30, host_capacity_bytes=4 << 30,
                        convert_to="bf16", permute_4d=True)) as s:
    cli = Client(s)
    v = cli.open(C.arch_key(arch), force_shared=True)
    net = BoundNet(v, arch, batch)
    x = torch.randn(batch, 3, arch.input_hw, arch.input_hw)
    st = torch.cuda.current_stream()
    for _ in range(10):
        net.forward(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    fn(None, 0, 1)
    e0.record()
    for _ in range(reps):
        net.run(st.cuda_stream, True)
    e1.record()
    torch.cuda.synchronize()
    fwd_ms = e0.elapsed_time(e1) / reps
    cap = 16384
    buf = np.zeros(cap * 16, np.uint64)
    n = fn(buf.ctypes.data, cap, 1)
    rec = buf[: min(n, cap) * 16].reshape(-1, 16).astype(np.int64)
    # launches = runs of CTAs with the same (M,N,K) signature in start order
    rec = rec[np.argsort(rec[:, 2])]
    per_fwd = len(rec) // reps
    rec = rec[-per_fwd:]  # the last forward
    groups = []
    for r in rec:
        sig = (int(r[0]), int(r[1]) >> 32)
        if groups and groups[-1]["sig"] == sig and r[2] <= groups[-1]["end"]:
            g = groups[-1]
        else:
            g = {"sig": sig, "rows": [], "end": 0}
            groups.append(g)
        g["rows"].append(r)
        g["end"] = max(g["end"], int(r[6]))
    t0 = int(rec[:, 2].min())
    prev_end = t0
    out = []
    for g in groups:
        R = np.array(g["rows"])
        us = lambda v: round((float(v) - prev_end) / 1e3, 2)
        row = {"M": int(R[0, 0] >> 32), "N": int(R[0, 0] & 0xffffffff), "K": int(R[0, 1] >> 32),
               "ctas": len(R), "first_start": us(R[:, 2].min()), "last_start": us(R[:, 2].max()),
               "wait_med": us(np.median(R[:, 3])), "wait_max": us(R[:, 3].max()),
               "full_max": us(R[:, 4].max()), "accum_max": us(R[:, 5].max()),
               "opnd_max": us(R[:, 8].max()), "epi_ready_max": us(R[:, 9].max()) if R[:, 9].max() else None,
               "stored_max": us(R[:, 10].max()) if R[:, 10].max() else None,
               "parked_max": us(R[:, 11].max()) if R[:, 11].max() else None,
               "csync1_max": us(R[:, 12].max()) if R[:, 12].max() else None,
               "reduced_max": us(R[:, 13].max()) if R[:, 13].max() else None,
               "ldtm_cyc_med": float(np.median(R[:, 15])), "finish_cyc_med": float(np.median(R[:, 13])),
               "finish_again_cyc_med": float(np.median(R[:, 14])),
               "end_max": us(R[:, 6].max()), "splits": int(R[:, 1].max() >> 16 & 0xffff) + 1,
               "at_us": round((float(R[:, 2].min()) - t0) / 1e3, 2)}
        out.append(row)
        prev_end = int(R[:, 6].max())
    print(json.dumps({"arch": name, "batch": batch, "fwd_ms": round(fwd_ms, 4), "gemm_launches": len(out),
                      "span_us": round((prev_end - t0) / 1e3, 2)}))
    for r in out:
        print(json.dumps(r))
    # per-CTA phase durations (median over the launch's CTAs, µs): split
    # launches mma | stage partials | bar | bulk issue | recv wait | reduce+store | tail
    for g in groups:
        R = np.array(g["rows"])
        med = lambda a, b: round(float(np.median(R[:, b] - R[:, a])) / 1e3, 3)
        sig = [int(R[0, 0] >> 32), int(R[0, 0] & 0xffffffff), int(R[0, 1] >> 32)]
        if (R[:, 1] >> 16 & 0xffff).max() > 0:
            print(json.dumps({"split_phases": sig, "splits": int(R[:, 1].max() >> 16 & 0xffff) + 1,
                              "wait_to_full": med(3, 4), "mma": med(4, 5), "stage": med(5, 14), "bar": med(14, 15),
                              "issue": med(15, 11), "recv_wait": med(11, 12), "reduce_store": med(12, 13),
                              "tail": med(13, 6), "cta_total": med(2, 6)}))
        else:
            print(json.dumps({"phases": sig, "wait_to_full": med(3, 4), "mma": med(4, 5),
                              "epi": med(5, 10), "epi_ready": med(5, 9), "ldtm_finish": med(9, 14),
                              "bar": med(14, 15), "copy_out": med(15, 10), "tail": med(10, 6),
                              "ldtm_cyc": float(np.median(R[:, 12])), "finish_cyc": float(np.median(R[:, 13])),
                              "cta_total": med(2, 6)}))
