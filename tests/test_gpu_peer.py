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
