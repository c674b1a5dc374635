"""Two stores in a row, cold opens with the streamed prestage (debug aid)."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.store import Store, StoreOptions

arch = C.ARCHS["resnet50"]()
d = tempfile.mkdtemp()
C.write_arch(arch, d, seed=1)
key = C.arch_key(arch)
base = dict(disk_cache_dir=d, fast_capacity_bytes=4 << 30, host_capacity_bytes=4 << 30, convert_to="bf16",
            permute_4d=True)
for rnd in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    for eager in (True, False):
        with Store(StoreOptions(eager_reclaim=eager, **base)) as s:
            cli = Client(s)
            for i in range(3):
                v = cli.open(key, force_shared=True)
                cli.close(v)
                if not eager:
                    s.reclaim(0, 4 << 30)
    print("round", rnd, "ok", flush=True)
