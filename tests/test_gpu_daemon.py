"""The wire-protocol daemon (csrc/server.cu) over a GPU store: v1 frames on a
Unix socket, the allocation fd passed with the OpenResponse, handles closed
when a connection drops (proj/src/daemon.cpp:398-560), and live interop with
the REFERENCE's own FramedSocket + decoder (oracle/_ref) against our daemon."""
import multiprocessing as mp
import os

import pytest

import oracle
from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import TrimsError
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.daemon import RemoteStore, serve
from paper_1811_09732_b200.store import Store, StoreOptions
from tests.golden_data import load

pytestmark = pytest.mark.gpu
MB = 1_000_000


@pytest.fixture(scope="module")
def tiny_dir(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("tinyd"))
    C.gen_catalog("tiny", d, seed=1, only=["alexnet", "resnet50", "vgg16"])
    return d


def key(name):
    return F.ModelKey("zoo", name, "1.0.0")


def _remote_client(endpoint, name, q):
    """Another process: open over the socket, map the passed fd, read bytes."""
    try:
        import torch
        from paper_1811_09732_b200.client import TensorView
        cli = Client(RemoteStore(endpoint), attach_via_import=True)
        v = cli.open(key(name), force_shared=True)
        n = v.blob_bytes()
        t = torch.empty(n, dtype=torch.uint8)
        t.copy_(TensorView("b", [n], "i8", "native", 0, n, v.base_ptr).torch("cuda:0").view(torch.uint8))
        sha = F.sha256(t.numpy()).hex()
        st = cli.store.stats()
        cli.close(v)
        q.put(("ok", sha, v.generation, st["tiers"][0]["used_bytes"]))
    except Exception as e:  # reported to the test
        q.put(("error", repr(e)))


def test_remote_process_attaches_over_the_wire(tiny_dir, tmp_path):
    g = {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}
    ep = "unix:" + str(tmp_path / "mrmd.sock")
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=20 * MB, host_capacity_bytes=64 * MB)) as s:
        with serve(s, ep) as srv:
            ctx = mp.get_context("spawn")
            q = ctx.Queue()
            p = ctx.Process(target=_remote_client, args=(ep, "alexnet", q))
            p.start()
            msg = q.get(timeout=300)
            p.join(60)
            assert msg[0] == "ok", msg
            _, sha, gen, used = msg
            assert sha == g["alexnet"]["trailer"]  # the bytes the reference wrote, read through our daemon
            assert used == 3_718_744
            st = s.stats()
            assert st["disk_reads"] == 1 and st["open_requests"] == 1
            assert all(m["refcount"] == 0 for m in st["models"])  # the client closed its handle
            assert srv.frames_served() >= 3


def test_reference_framedsocket_talks_to_our_daemon(tiny_dir, tmp_path):
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    R = oracle.ref()
    ep = str(tmp_path / "mrmd2.sock")
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=20 * MB, host_capacity_bytes=64 * MB)) as s:
        with serve(s, ep):
            rc, txt = R.wire_request(ep, "stats 1")
            assert rc == 0 and txt.startswith("statsresp")
            rc, txt = R.wire_request(ep, "open 1 zoo resnet50 1.0.0 1 0 42")  # Layer granularity
            assert rc == 0, rc
            t = txt.split()
            assert t[0] == "openresp"
            nobj = int(t[6])
            res = s.resident_manifest(int(t[1]))
            assert nobj == len(F.layout_for(res, F.LAYER))      # one object per resident tensor
            assert "?dev=0&alloc=" in t[8]                        # token with CUDA coordinates
            # the reference client's connection closed after its request: handle auto-closed
            st = s.stats()
            assert st["open_requests"] == 1
            assert all(m["refcount"] == 0 for m in st["models"])
            rc, txt = R.wire_request(ep, "open 1 zoo no-such-model 1.0.0 0 0 1")
            assert rc == 0 and txt.startswith("error 1 ")         # NotFound, as an ErrorMsg frame
            rc, txt = R.wire_request(ep, "close 1 99 12345")
            assert rc == 0 and txt.startswith("error 4 ")         # NotOpen


def test_connection_drop_closes_handles(tiny_dir, tmp_path):
    ep = str(tmp_path / "mrmd3.sock")
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=20 * MB, host_capacity_bytes=64 * MB)) as s:
        with serve(s, ep):
            rs = RemoteStore(ep)
            ex1 = rs.open(key("vgg16"))
            ex2 = rs.open(key("vgg16"))
            assert ex1.fd >= 0 and ex2.fd >= 0 and ex1.generation == ex2.generation
            os.close(ex1.fd)
            os.close(ex2.fd)
            rcs = {m["key"]: m["refcount"] for m in rs.stats()["models"]}
            assert rcs["zoo/vgg16@1.0.0"] == 2 and sum(rcs.values()) == 2
            assert rs.close(key("vgg16")) == 1
            rs.open(key("alexnet"))
            rs.close_connection()  # drop with vgg16 x1 and alexnet x1 still open
            import time
            for _ in range(100):
                if all(m["refcount"] == 0 for m in s.stats()["models"]):
                    break
                time.sleep(0.02)
            assert all(m["refcount"] == 0 for m in s.stats()["models"])
            with pytest.raises(TrimsError):
                RemoteStore(ep).close(key("vgg16"))


def test_concurrent_connections_under_pressure(tiny_dir, tmp_path):
    """8 connections at once (one daemon thread each) opening and closing
    models while the fast tier evicts; half of them drop the connection with
    handles still open. Afterwards every refcount is back to 0."""
    import random
    import threading
    ep = str(tmp_path / "mrmd4.sock")
    names = ["alexnet", "resnet50", "vgg16"]
    errors = []
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=13 * MB, host_capacity_bytes=16 * MB)) as s:
        with serve(s, ep) as srv:

            def worker(wi):
                rng = random.Random(wi)
                try:
                    rs = RemoteStore(ep)
                    held = []
                    for _ in range(40):
                        k = key(rng.choice(names))
                        if held and rng.random() < 0.5:
                            rs.close(held.pop())
                            continue
                        try:
                            ex = rs.open(k)
                        except TrimsError as e:
                            if e.code in (2, 3):  # TooLargeForFast / NoEvictableSpace: all pinned by others
                                continue
                            raise
                        os.close(ex.fd)
                        held.append(k)
                    if wi % 2:
                        for k in held:
                            rs.close(k)
                    rs.close_connection()  # odd workers closed everything; even ones drop with handles open
                except Exception as e:  # reported below
                    errors.append(repr(e))

            ts = [threading.Thread(target=worker, args=(i,)) for i in range(8)]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
            assert not errors, errors[:3]
            import time
            for _ in range(200):
                if all(m["refcount"] == 0 for m in s.stats()["models"]):
                    break
                time.sleep(0.02)
            st = s.stats()
            assert all(m["refcount"] == 0 for m in st["models"]), st["models"]
            assert st["tiers"][0]["used_bytes"] <= 13 * MB
            assert srv.frames_served() > 100
