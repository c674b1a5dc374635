"""View lifetime across eviction and arena reuse (proj/tests/test_shared_segment.cpp:99-110:
"attached view survives owner destruction"). Every model lives in one HBM
arena, so a retained view is protected by a pin (same process) or a lease
row in the arena's lease table (another process): the owner retires the
range instead of handing it to the next model, and reuses it only after the
last reader lets go (or dies)."""
import gc
import multiprocessing as mp
import os

import pytest

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from tests.golden_data import load

pytestmark = pytest.mark.gpu
MB = 1_000_000


@pytest.fixture(scope="module")
def tiny_dir(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("life"))
    C.gen_catalog("tiny", d, seed=1, only=["alexnet", "resnet50", "googlenet"])
    return d


def key(name):
    return F.ModelKey("zoo", name, "1.0.0")


def _sha(view):
    import torch
    from paper_1811_09732_b200.client import TensorView
    n = view.blob_bytes()
    t = TensorView("b", [n], "i8", "native", 0, n, view.base_ptr).torch("cuda:0").view(torch.uint8).cpu().numpy()
    return F.sha256(t).hex()


def test_in_process_view_outlives_eviction_and_blocks_reuse(tiny_dir):
    import torch
    from paper_1811_09732_b200.client import Client
    from paper_1811_09732_b200.store import Store, StoreOptions
    g = {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=5 * MB, host_capacity_bytes=64 * MB)) as s:
        cli = Client(s)
        v = cli.open(key("alexnet"), force_shared=True)
        w = v.tensors[3]                           # a tensor view retained by the caller
        ref = w.torch("cuda:0").view(torch.uint8).clone()
        cli.close(v)
        b = cli.open(key("resnet50"), force_shared=True)  # 3.7 + 1.5 MB > 5 MB: alexnet is evicted
        assert s.stats()["tiers"][0]["used_bytes"] == b.export.weights_bytes  # only resnet50 is resident
        assert b.export.segment_offset != v.export.segment_offset   # the range is retired, not reused
        assert _sha(v) == g["alexnet"]["trailer"]                   # the retained view still reads alexnet
        assert torch.equal(w.torch("cuda:0").view(torch.uint8), ref)
        old = v.export.segment_offset
        cli.close(b)
        del v, w, b
        gc.collect()                                 # the last reader lets go: the range is free again
        s.reclaim(0, 5 * MB)
        c = cli.open(key("googlenet"), force_shared=True)
        assert c.export.segment_offset == old
        assert _sha(c) == g["googlenet"]["trailer"]
        cli.close(c)


def _reader(endpoint, q, go):
    """Another process: opens alexnet over the daemon, closes its handle,
    keeps the view, waits for the owner to load another model, reads."""
    try:
        from paper_1811_09732_b200.client import Client
        from paper_1811_09732_b200.daemon import RemoteStore
        cli = Client(RemoteStore(endpoint), attach_via_import=True)
        v = cli.open(key("alexnet"), force_shared=True)
        cli.close(v)
        q.put(("closed", v.export.segment_offset))
        go.get(timeout=120)
        q.put(("sha", _sha(v)))
    except Exception as e:  # reported to the parent
        q.put(("error", repr(e)))


def test_cross_process_view_outlives_eviction_and_reader_death(tiny_dir):
    from paper_1811_09732_b200.daemon import serve
    from paper_1811_09732_b200.store import Store, StoreOptions
    g = {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}
    ctx = mp.get_context("spawn")
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=5 * MB, host_capacity_bytes=64 * MB)) as s:
        ep = os.path.join(tiny_dir, "life.sock")
        with serve(s, ep):
            q, go = ctx.Queue(), ctx.Queue()
            p = ctx.Process(target=_reader, args=(ep, q, go))
            p.start()
            kind, old = q.get(timeout=180)
            assert kind == "closed", old
            b = s.open(key("resnet50"))                 # evicts alexnet; its range is leased by the reader
            assert b.segment_offset != old
            go.put("read")
            kind, sha = q.get(timeout=120)
            assert (kind, sha) == ("sha", g["alexnet"]["trailer"])
            p.join(60)                                   # the reader exits: its lease row is dead
            s.close(key("resnet50"))
            s.reclaim(0, 5 * MB)
            c = s.open(key("googlenet"))
            assert c.segment_offset == old               # reused once no live reader holds it
            s.close(key("googlenet"))
