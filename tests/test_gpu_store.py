"""GPU store path end to end: disk -> pinned host -> HBM ingest, export/import,
decisions with the real CudaTierBackend, views surviving eviction, and the
multi-process one-copy dedup (proj/tests/acceptance.cpp:76-153 on B200)."""
import json
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import oracle
from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import Errc, TrimsError
from paper_1811_09732_b200.client import Client, import_segment
from paper_1811_09732_b200.store import Store, StoreOptions
from tests.golden_data import load
from tests.gpu_util import expected_resident

pytestmark = pytest.mark.gpu
MB = 1_000_000


@pytest.fixture(scope="module")
def tiny_dir(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("tiny"))
    C.gen_catalog("tiny", d, seed=1, only=["alexnet", "resnet50", "vgg16", "googlenet", "squeezenet-v1.1"])
    return d


def key(name):
    return F.ModelKey("zoo", name, "1.0.0")


def d2h(view, torch):
    n = view.blob_bytes()
    t = torch.empty(n, dtype=torch.uint8)
    from paper_1811_09732_b200.client import TensorView
    t.copy_(TensorView("b", [n], "i8", "native", 0, n, view.base_ptr).torch("cuda:0").view(torch.uint8))
    return t.numpy()


def test_disk_fast_host_hits_and_parity(tiny_dir):
    import torch
    g = {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=10 * MB, host_capacity_bytes=64 * MB)) as s:
        cli = Client(s, model_dirs=[tiny_dir])
        v = cli.open(key("alexnet"), force_shared=True)
        assert v.outcome == "disk_load" and v.origin == "shared"
        blob = d2h(v, torch)
        assert F.sha256(blob).hex() == g["alexnet"]["trailer"]        # bytes == the reference's blob
        assert cli.touch(v) == g["alexnet"]["touch"]                   # touch == the reference's touch
        assert v.export.ingest_checksum == oracle.port().block_checksum(blob)
        v2 = cli.open(key("alexnet"), force_shared=True)
        assert v2.outcome == "fast_hit" and v2.base_ptr == v.base_ptr
        st = s.stats()
        assert st["disk_reads"] == 1 and st["tiers"][0]["used_bytes"] == 3_718_744  # weights, not padded blob
        cli.close(v)
        cli.close(v2)
        cli.close(v2)  # idempotent
        # vgg16 (8.25 MB) does not fit next to alexnet in 10 MB: alexnet evicted from fast, kept on host
        w = cli.open(key("vgg16"), force_shared=True)
        assert w.outcome == "disk_load"
        cli.close(w)
        v3 = cli.open(key("alexnet"), force_shared=True)
        assert v3.outcome == "host_hit"
        assert F.sha256(d2h(v3, torch)).hex() == g["alexnet"]["trailer"]
        cli.close(v3)
        st = s.stats()
        assert st["tiers"][1]["hits"] == 1 and st["tiers"][0]["evictions"] >= 1


def test_errors_and_no_budget_leak(tiny_dir):
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=5 * MB, host_capacity_bytes=64 * MB)) as s:
        with pytest.raises(TrimsError) as ei:
            s.open(key("vgg16"))
        assert ei.value.code == Errc.TooLargeForFast
        with pytest.raises(TrimsError) as ei:
            s.open(key("absent"))
        assert ei.value.code == Errc.NotFound
        s.open(key("alexnet"))  # pinned (refcount 1), 3.7 MB
        with pytest.raises(TrimsError) as ei:
            s.open(key("resnet50"))  # 1.53 MB more needs eviction of a pinned model
        assert ei.value.code == Errc.NoEvictableSpace
        assert s.stats()["tiers"][0]["used_bytes"] == 3_718_744  # failed opens leak no budget
        s.close(key("alexnet"))
        with pytest.raises(TrimsError) as ei:
            s.close(key("alexnet"))
        assert ei.value.code == Errc.NotOpen


def test_stream_from_file_without_host_staging(tiny_dir):
    import torch
    g = {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}
    # host tier smaller than the model: publish_fast streams file -> pinned bounce -> HBM
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=64 * MB, host_capacity_bytes=1 * MB)) as s:
        cli = Client(s)
        v = cli.open(key("vgg16"), force_shared=True)
        assert F.sha256(d2h(v, torch)).hex() == g["vgg16"]["trailer"]
        assert s.stats()["tiers"][1]["used_bytes"] == 0
        cli.close(v)


def test_converting_store_bit_exact_and_import_path(tmp_path):
    import torch
    d = str(tmp_path)
    arch = C.ARCHS["resnet50"]()
    C.write_arch(arch, d, seed=1)
    src_json, blob = C.arch_blob(arch, seed=1)
    opts = StoreOptions(disk_cache_dir=d, fast_capacity_bytes=1 << 30, host_capacity_bytes=1 << 30,
                        convert_to="bf16", permute_4d=True)
    with Store(opts) as s:
        k = C.arch_key(arch)
        direct = Client(s, model_dirs=[d])
        via_fd = Client(s, attach_via_import=True)
        a = direct.open(k, force_shared=True)
        b = via_fd.open(k, force_shared=True)
        assert a.manifest_json == b.manifest_json
        got_a, got_b = d2h(a, torch), d2h(b, torch)
        want = expected_resident(src_json, blob, a.manifest_json)
        assert np.array_equal(got_a, want) and np.array_equal(got_b, want)
        assert a.tensor("conv1.weight").dims == [64, 7, 7, 3] and a.tensor("conv1.weight").dtype == "bf16"
        priv = direct.open(k, force_private=True)
        assert priv.origin == "private" and np.array_equal(d2h(priv, torch), want)
        direct.close(a)
        via_fd.close(b)
        direct.close(priv)
        via_fd.close_all_imports()


def _child_attach(conn, device: int, alloc: int, offset: int, gen: int, payload: int, digest: bytes, q):
    try:
        import ctypes
        from multiprocessing.reduction import recv_handle

        from paper_1811_09732_b200._lib import lib
        fd = recv_handle(conn)  # SCM_RIGHTS over the pipe: the fd of the cuMem allocation
        imp, ptr, mj = import_segment(device, fd, alloc, offset, gen, payload, digest)
        os.close(fd)
        cs = ctypes.c_uint64()
        rc = lib.trims_import_verify(imp, offset, gen, payload, ctypes.byref(cs))
        ro = lib.trims_import_read_only(imp)
        q.put((rc, cs.value, ro, len(mj)))
        lib.trims_import_close(imp)
    except Exception as e:  # report instead of dying silently
        q.put((-1, repr(e), 0, 0))


def test_multiprocess_one_copy(tiny_dir):
    """8 client processes attach one HBM copy (acceptance.cpp:76-153): one disk
    read, fast tier holds one copy, max refcount 8, every child verifies the
    resident checksum on its own mapping."""
    ctx = mp.get_context("spawn")
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=64 * MB, host_capacity_bytes=64 * MB)) as s:
        q = ctx.Queue()
        procs, exps = [], []
        from multiprocessing.reduction import send_handle
        for i in range(8):
            ex = s.open(key("vgg16"))
            exps.append(ex)
            parent, child = ctx.Pipe()
            p = ctx.Process(target=_child_attach, args=(child, ex.device, ex.alloc_bytes, ex.segment_offset,
                                                        ex.generation, ex.payload_bytes, bytes(ex.manifest_digest),
                                                        q))
            p.start()
            send_handle(parent, ex.fd, p.pid)
            procs.append((p, parent, child))
        res = [q.get(timeout=180) for _ in procs]
        for p, a, b in procs:
            p.join(60)
            a.close()
            b.close()
        st = s.stats()
        assert st["disk_reads"] == 1
        assert st["tiers"][0]["used_bytes"] == 8_250_000  # one copy (weights bytes)
        assert max(m["refcount"] for m in st["models"]) == 8
        assert len({e.generation for e in exps}) == 1
        for rc, cs, ro, jl in res:
            assert rc == 0 and cs == exps[0].ingest_checksum
        for _ in exps:
            s.close(key("vgg16"))


def test_views_survive_eviction(tiny_dir):
    import torch
    g = {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=64 * MB, host_capacity_bytes=64 * MB)) as s:
        cli = Client(s, attach_via_import=True)
        v = cli.open(key("googlenet"), force_shared=True)
        cli.close(v)  # refcount 0; the client keeps its mapping in the import cache
        s.reclaim(0, 64 * MB)  # evict everything evictable from the fast tier
        assert s.stats()["tiers"][0]["used_bytes"] == 0
        from paper_1811_09732_b200.client import TensorView
        n = v.blob_bytes()
        t = TensorView("b", [n], "i8", "native", 0, n, v.base_ptr).torch("cuda:0").view(torch.uint8).cpu().numpy()
        assert F.sha256(t).hex() == g["googlenet"]["trailer"]
        cli.close_all_imports()


def test_arena_reuse_is_detected_as_stale_generation(tiny_dir):
    """A freed arena range re-used by another model: attaching with the old
    generation fails with StaleGeneration (shared_segment.cpp:233-237)."""
    from paper_1811_09732_b200.client import attach_segment, map_allocation
    from paper_1811_09732_b200._lib import lib
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=5 * MB, host_capacity_bytes=64 * MB)) as s:
        a = s.open(key("alexnet"))
        s.close(key("alexnet"))
        fd = os.dup(a.fd)
        imp, base = map_allocation(a.device, fd, a.alloc_bytes)
        os.close(fd)
        ptr, js = attach_segment(imp, a.segment_offset, a.generation, a.payload_bytes, bytes(a.manifest_digest))
        assert ptr == base + a.segment_offset and json.loads(js)["name"] == "alexnet"
        b = s.open(key("resnet50"))  # 3.7 + 1.5 MB > 5 MB: alexnet evicted, its range reused
        assert b.segment_offset == a.segment_offset and b.generation != a.generation
        with pytest.raises(TrimsError) as ei:
            attach_segment(imp, a.segment_offset, a.generation, a.payload_bytes, bytes(a.manifest_digest))
        # scrubbed tail (NoSuchSegment) or a new tail at the same place (StaleGeneration)
        assert ei.value.code in (Errc.StaleGeneration, Errc.NoSuchSegment)
        ptr_b, js_b = attach_segment(imp, b.segment_offset, b.generation, b.payload_bytes, bytes(b.manifest_digest))
        assert json.loads(js_b)["name"] == "resnet50"
        lib.trims_import_close(imp)
        s.close(key("resnet50"))


def test_dedicated_segments_without_arena(tiny_dir):
    import torch
    g = {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=64 * MB, host_capacity_bytes=64 * MB,
                            arena_bytes=1)) as s:
        cli = Client(s, attach_via_import=True)
        v = cli.open(key("squeezenet-v1.1"), force_shared=True)
        assert v.export.segment_offset == 0
        assert F.sha256(d2h(v, torch)).hex() == g["squeezenet-v1.1"]["trailer"]
        cli.close(v)
        cli.close_all_imports()
