"""Forward-pass timing on store-lent weights: graph replay vs eager, and the
hot/warm/cold request latency around it. python scripts/time_forward.py [arch] [batch]"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.models import BoundNet
from paper_1811_09732_b200.store import Store, StoreOptions

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
arch = C.ARCHS[name]()
d = tempfile.mkdtemp()
C.write_arch(arch, d, seed=1)
with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=4 << 30, host_capacity_bytes=4 << 30,
                        convert_to="bf16", permute_4d=True)) as s:
    cli = Client(s)
    v = cli.open(C.arch_key(arch), force_shared=True)
    net = BoundNet(v, arch, batch, mode=os.environ.get("TRIMS_NET_MODE", "latency"))
    x = torch.randn(batch, 3, arch.input_hw, arch.input_hw).pin_memory()
    st = torch.cuda.current_stream()
    for _ in range(5):
        net.forward(x)
    torch.cuda.synchronize()
    res = {"arch": name, "batch": batch, "launches": net.launches, "gflop": net.flops / 1e9}
    for graph in (True, False):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            net.run(st.cuda_stream, graph)
        e1.record()
        torch.cuda.synchronize()
        res["fwd_ms_graph" if graph else "fwd_ms_eager"] = e0.elapsed_time(e1) / 50
    # hot request: open (HBM hit) + H2D input + forward + D2H logits + close
    out = torch.empty(batch, net.classes).pin_memory()
    ts = []
    for _ in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        w = cli.open(C.arch_key(arch), force_shared=True)
        net.input_view().copy_(x, non_blocking=True)
        net.run(st.cuda_stream, True)
        out.copy_(net.logits_view(), non_blocking=True)
        st.synchronize()
        cli.close(w)
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    res["hot_request_ms_p50"] = ts[len(ts) // 2]
    ts = []
    for _ in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        net.input_view().copy_(x, non_blocking=True)
        net.run(st.cuda_stream, True)
        out.copy_(net.logits_view(), non_blocking=True)
        st.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    res["compute_only_request_ms_p50"] = ts[len(ts) // 2]
    res["tflops_graph"] = net.flops / (res["fwd_ms_graph"] / 1e3) / 1e12
    print(json.dumps({k: (round(x, 4) if isinstance(x, float) else x) for k, x in res.items()}))
    net.close()
    cli.close(v)
