"""Concurrent clients on one GPU store under memory pressure: threads open /
verify / close catalog models at random while the fast and host tiers evict
(disk loads, host hits, fast hits, single-flight waits, prestage contention,
verified reads). Every view's bytes must reproduce the reference's `touch`
(client.cpp:338-359) for that model, and at the end no refcount or reserved
byte may leak (cache_core.cpp accounting)."""
import random
import threading

import pytest

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import Errc, TrimsError
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.store import Store, StoreOptions
from tests.golden_data import load

pytestmark = pytest.mark.gpu
MB = 1_000_000
NAMES = ["alexnet", "caffenet", "resnet50", "googlenet", "inception-v3", "dpn92", "squeezenet-v1.1", "resnet152"]


@pytest.fixture(scope="module")
def tiny_dir(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("tinyc"))
    C.gen_catalog("tiny", d, seed=1, only=NAMES)
    return d


@pytest.mark.parametrize("verify,eager", [(False, False), (True, False), (False, True)])
def test_concurrent_clients_under_pressure(tiny_dir, verify, eager):
    gold = {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}
    errors, counts = [], {"ok": 0, "busy": 0}
    lock = threading.Lock()
    # fast tier ~ 2-3 models, host tier ~ 4: constant eviction traffic
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=8 * MB, host_capacity_bytes=12 * MB,
                            full_verify=verify, eager_reclaim=eager, scan_disk=False)) as s:

        def worker(wi):
            rng = random.Random(wi * 7919 + int(verify) * 13 + int(eager))
            cli = Client(s)
            try:
                for _ in range(30):
                    name = rng.choice(NAMES)
                    key = F.ModelKey("zoo", name, "1.0.0")
                    try:
                        v = cli.open(key, force_shared=True)
                    except TrimsError as e:
                        if e.code == Errc.NoEvictableSpace:  # every resident model pinned by the others
                            with lock:
                                counts["busy"] += 1
                            continue
                        raise
                    try:
                        assert cli.touch(v) == gold[name]["touch"], name
                    finally:
                        cli.close(v)
                    with lock:
                        counts["ok"] += 1
            except Exception as e:  # reported below
                errors.append(repr(e))

        ts = [threading.Thread(target=worker, args=(i,)) for i in range(6)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors, errors[:3]
        st = s.stats()
        assert all(m["refcount"] == 0 for m in st["models"])
        assert st["tiers"][0]["used_bytes"] <= 8 * MB and st["tiers"][1]["used_bytes"] <= 12 * MB
        assert st["open_requests"] == counts["ok"] and counts["ok"] >= 120
        if eager:
            assert st["tiers"][0]["used_bytes"] == 0  # eager reclaim: nothing resident once closed


def _blob_sha(cli, v):
    import torch
    from paper_1811_09732_b200.client import TensorView
    n = v.blob_bytes()
    t = torch.empty(n, dtype=torch.uint8)
    t.copy_(TensorView("b", [n], "i8", "native", 0, n, v.base_ptr).torch("cuda:0").view(torch.uint8))
    return F.sha256(t.numpy())


def test_concurrent_converting_store(tiny_dir):
    """The same under a converting plan (f64 -> bf16 at ingest), so host hits
    reload the resident-form host copy (async D2H after each publish) while
    other threads evict and publish: every view must equal a single-threaded
    load of the same model."""
    opts = dict(disk_cache_dir=tiny_dir, convert_to="bf16", scan_disk=False)
    want = {}
    with Store(StoreOptions(fast_capacity_bytes=64 * MB, host_capacity_bytes=64 * MB, **opts)) as s:
        cli = Client(s)
        for name in NAMES:
            v = cli.open(F.ModelKey("zoo", name, "1.0.0"), force_shared=True)
            want[name] = _blob_sha(cli, v)
            cli.close(v)
    errors = []
    with Store(StoreOptions(fast_capacity_bytes=5 * MB, host_capacity_bytes=7 * MB, **opts)) as s:

        def worker(wi):
            rng = random.Random(wi)
            cli = Client(s)
            try:
                for _ in range(30):
                    name = rng.choice(NAMES)
                    try:
                        v = cli.open(F.ModelKey("zoo", name, "1.0.0"), force_shared=True)
                    except TrimsError as e:
                        if e.code == Errc.NoEvictableSpace:
                            continue
                        raise
                    try:
                        assert _blob_sha(cli, v) == want[name], name
                    finally:
                        cli.close(v)
            except Exception as e:  # reported below
                errors.append(repr(e))

        ts = [threading.Thread(target=worker, args=(i,)) for i in range(6)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors, errors[:3]
        st = s.stats()
        assert all(m["refcount"] == 0 for m in st["models"])
        assert st["tiers"][1]["hits"] > 0 and st["tiers"][0]["evictions"] > 0
