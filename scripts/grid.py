"""The oversubscription grid on the tiny or the full small37
catalog: python scripts/grid.py [out.json] [requests] [tiny|small37] [mps|nomps] [worlds] [concurrencies]
(worlds / concurrencies comma-separated, defaults 1,2,4 and 1,4)."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.grid import run_grid


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    reqs = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    cat = sys.argv[3] if len(sys.argv) > 3 else "tiny"
    mps = len(sys.argv) > 4 and sys.argv[4] == "mps"
    worlds = tuple(int(x) for x in sys.argv[5].split(",")) if len(sys.argv) > 5 else (1, 2, 4)
    concs = tuple(int(x) for x in sys.argv[6].split(",")) if len(sys.argv) > 6 else (1, 4)
    models, div = C.catalog(cat)
    keys = [C.catalog_key(m) for m in models]
    total = sum(C.scaled_weights_bytes(m, div) for m in models)
    d = tempfile.mkdtemp()
    C.gen_catalog(cat, d, seed=1)
    res = run_grid(d, keys, total, requests=reqs, worlds=worlds, concurrencies=concs, mps=mps)
    res["catalog"] = ("tiny (small37 / 64)" if cat == "tiny" else cat) + ", seed 1"
    txt = json.dumps(res, indent=1)
    print(txt)
    if out:
        open(out, "w").write(txt)


if __name__ == "__main__":  # worker processes are spawned: they re-import this module
    main()
