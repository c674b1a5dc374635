"""The oversubscription grid on the tiny or the full small37
catalog: python scripts/grid.py [out.json] [requests] [tiny|small37]"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.grid import run_grid

out = sys.argv[1] if len(sys.argv) > 1 else None
reqs = int(sys.argv[2]) if len(sys.argv) > 2 else 400
cat = sys.argv[3] if len(sys.argv) > 3 else "tiny"
models, div = C.catalog(cat)
keys = [C.catalog_key(m) for m in models]
total = sum(C.scaled_weights_bytes(m, div) for m in models)
d = tempfile.mkdtemp()
C.gen_catalog(cat, d, seed=1)
res = run_grid(d, keys, total, requests=reqs)
res["catalog"] = ("tiny (small37 / 64)" if cat == "tiny" else cat) + ", seed 1"
txt = json.dumps(res, indent=1)
print(txt)
if out:
    open(out, "w").write(txt)
