"""One ResNet-50/VGG-16/AlexNet forward on store-lent weights, for ncu:
    python scripts/prof_forward.py [arch] [batch] [reps]"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.models import BoundNet
from paper_1811_09732_b200.store import Store, StoreOptions

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
arch = C.ARCHS[name]()
d = tempfile.mkdtemp()
C.write_arch(arch, d, seed=1)
with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=4 << 30, host_capacity_bytes=4 << 30,
                        convert_to="bf16", permute_4d=True)) as s:
    cli = Client(s)
    v = cli.open(C.arch_key(arch), force_shared=True)
    net = BoundNet(v, arch, batch)
    st = torch.cuda.current_stream()
    for _ in range(reps):
        net.run(st.cuda_stream, False)  # eager: one launch per kernel
    torch.cuda.synchronize()
    net.close()
    cli.close(v)
