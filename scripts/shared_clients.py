"""bench.py's shared-clients leg alone (BASELINE configs[1]): one ResNet-50
copy served by the daemon to 1 client, 16 time-sliced clients and 16 MPS
clients. python scripts/shared_clients.py [n_clients] [n_reqs]"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1811_09732_b200 import catalog as C  # noqa: E402

if __name__ == "__main__":  # client processes are spawned: they re-import this module
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    reqs = int(sys.argv[2]) if len(sys.argv) > 2 else 250
    work = tempfile.mkdtemp()
    arch = C.ARCHS["resnet50"]()
    C.write_arch(arch, work, seed=1)
    r = bench.shared_clients(work, arch, 0, n, reqs)
    r.pop("logits", None)
    print(json.dumps(r))
