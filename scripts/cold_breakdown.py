"""Where a cold (disk) / warm (host) open of a catalog model spends its time:
    python scripts/cold_breakdown.py [arch] [reps]"""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.store import Store, StoreOptions

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
arch = C.ARCHS[name]()
d = tempfile.mkdtemp()
C.write_arch(arch, d, seed=1)
key = C.arch_key(arch)
for mode in ("cold", "warm"):
    with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=4 << 30, host_capacity_bytes=4 << 30,
                            convert_to="bf16", permute_4d=True, eager_reclaim=(mode == "cold"),
                            read_threads=int(os.environ.get("RT", "8")))) as s:
        cli = Client(s)
        if mode == "warm":
            cli.close(cli.open(key, force_shared=True))
        for i in range(reps):
            if mode == "warm":
                s.reclaim(0, 4 << 30)
            t0 = time.perf_counter()
            v = cli.open(key, force_shared=True)
            t1 = time.perf_counter()
            ex = v.export
            print(mode, i, f"open {1e3 * (t1 - t0):.3f} ms  rpc {1e3 * v.timings.rpc_s:.3f}  attach "
                  f"{1e3 * v.timings.attach_s:.3f}  core[fetch,disk_read,h2fast,export] "
                  f"{[round(x / 1e6, 3) for x in ex.timings_ns]}  {s.ingest_stats(v.model_id)}")
            cli.close(v)
