"""Cost of rebinding an executor to a new weights generation (BoundNet.rebind):
    python scripts/time_rebind.py [arch]"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.models import BoundNet
from paper_1811_09732_b200.store import Store, StoreOptions

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
arch = C.ARCHS[name]()
d = tempfile.mkdtemp()
C.write_arch(arch, d, seed=1)
with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=4 << 30, host_capacity_bytes=4 << 30,
                        convert_to="bf16", permute_4d=True)) as s:
    cli = Client(s)
    v = cli.open(C.arch_key(arch), force_shared=True)
    net = BoundNet(v, arch, 1)
    x = torch.randn(1, 3, arch.input_hw, arch.input_hw)
    net.forward(x)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        net.rebind(v)
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    print(json.dumps({"arch": name, "rebind_ms_p50": round(ts[10], 4), "rebind_ms_min": round(ts[0], 4)}))
    net.close()
    cli.close(v)
