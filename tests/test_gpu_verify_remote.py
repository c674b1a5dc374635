"""Verified cold loads and the remote tier on the GPU store.

full_verify (daemon.hpp:32): read_manifest reads the blob into pinned memory
while one thread hashes it (pread.hpp) and the same open's stage_host /
publish_fast use those verified bytes, so the blob is read and hashed once
(the reference reads + hashes it twice, daemon.cpp:146 and :155). A corrupt
artifact fails in read_manifest, i.e. BEFORE any reclaim, as the reference
(cache_core.cpp:250 precedes the admission at :290-330): nothing is evicted.

remote_url (daemon.hpp:26): a model that is on neither tier is fetched into
the disk cache (remote.cpp) and loaded: outcome RemoteFetch, the
misses/hits accounting of cache_core.cpp:398-414, and the file registered in
the disk tier."""
import os
import shutil

import pytest

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import Errc, TrimsError
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.store import Store, StoreOptions
from tests.golden_data import load
from tests.test_gpu_store import d2h, key

pytestmark = pytest.mark.gpu
MB = 1_000_000


@pytest.fixture(scope="module")
def tiny_dir(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("tinyv"))
    C.gen_catalog("tiny", d, seed=1, only=["alexnet", "resnet50", "vgg16"])
    return d


@pytest.fixture(scope="module")
def gold():
    return {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}


def _o_direct_supported(d: str) -> bool:
    path = os.path.join(d, "odirect.probe")
    with open(path, "wb") as f:
        f.write(b"\0" * 8192)
    try:
        fd = os.open(path, os.O_RDONLY | os.O_DIRECT)
        os.close(fd)
        return True
    except OSError:
        return False
    finally:
        os.unlink(path)


@pytest.mark.parametrize("mode", ["direct", "buffered", "auto"])
@pytest.mark.parametrize("verify", [False, True])
def test_direct_io_cold_loads_bit_exact(tiny_dir, gold, mode, verify):
    """Cold loads with O_DIRECT reads into the pinned host tier (blob offsets
    are 64-aligned, not 4 KiB-aligned: the host buffer is placed congruent to
    the file offset and whole blocks are read around the blob): identical
    resident bytes, trailer SHA and touch; host-tier reloads identical too."""
    import torch
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=20 * MB, host_capacity_bytes=64 * MB,
                            full_verify=verify, direct_io=mode)) as s:
        cli = Client(s)
        for rnd in range(2):
            for name in ("alexnet", "resnet50", "vgg16"):
                v = cli.open(key(name), force_shared=True)
                assert v.outcome == ("disk_load" if rnd == 0 else "host_hit")
                assert F.sha256(d2h(v, torch)).hex() == gold[name]["trailer"]
                assert cli.touch(v) == gold[name]["touch"]
                cli.close(v)
            s.reclaim(0, 20 * MB)  # drop the fast tier: round 2 reloads from the host tier
        st = s.stats()
        assert st["open_errors"] == 0
        if mode == "direct" and _o_direct_supported(tiny_dir):
            assert st["direct_reads"] == 3
        if mode == "buffered":
            assert st["direct_reads"] == 0


@pytest.mark.parametrize("host_mb", [64, 1])  # 1 MB: host staging skipped, publish from the verified read
def test_full_verify_loads_bit_exact(tiny_dir, gold, host_mb):
    import torch
    with Store(StoreOptions(disk_cache_dir=tiny_dir, fast_capacity_bytes=20 * MB, host_capacity_bytes=host_mb * MB,
                            full_verify=True)) as s:
        cli = Client(s)
        for name in ("alexnet", "resnet50", "vgg16"):
            v = cli.open(key(name), force_shared=True)
            assert v.outcome == "disk_load"
            assert F.sha256(d2h(v, torch)).hex() == gold[name]["trailer"]
            assert cli.touch(v) == gold[name]["touch"]
            cli.close(v)
        st = s.stats()
        assert st["disk_reads"] == 3 and st["open_errors"] == 0
        weights = sum(t["nbytes"] for n in ("alexnet", "resnet50", "vgg16")
                      for t in F.read_manifest(os.path.join(tiny_dir, key(n).filename)).manifest["tensors"])
        assert st["tiers"][1]["used_bytes"] == (0 if host_mb == 1 else weights)


def test_full_verify_rejects_before_eviction(tiny_dir, tmp_path):
    d = str(tmp_path / "cache")
    shutil.copytree(tiny_dir, d)
    p = os.path.join(d, key("vgg16").filename)
    info = F.read_manifest(p)
    with open(p, "r+b") as f:  # one flipped blob byte
        f.seek(info.blob_offset + 12345)
        b = f.read(1)
        f.seek(info.blob_offset + 12345)
        f.write(bytes([b[0] ^ 0x40]))
    # fast tier fits alexnet (3.7 MB) or vgg16 (8.25 MB), not both
    with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=10 * MB, host_capacity_bytes=64 * MB,
                            full_verify=True)) as s:
        s.open(key("alexnet"))
        s.close(key("alexnet"))
        for _ in range(12):  # repeated failures leave no verified buffer behind
            with pytest.raises(TrimsError) as ei:
                s.open(key("vgg16"))
            assert ei.value.code == Errc.ChecksumMismatch
        st = s.stats()
        assert st["tiers"][0]["evictions"] == 0 and st["open_errors"] == 12
        assert s.open(key("alexnet")).outcome == 0  # FastHit: still resident: nothing was reclaimed
        s.close(key("alexnet"))
    with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=10 * MB, host_capacity_bytes=64 * MB)) as s:
        assert s.open(key("vgg16")).outcome == 2  # DiskLoad: without full_verify the bytes are taken as is


def test_remote_tier_fetch_into_disk_cache(tiny_dir, gold, tmp_path):
    import torch
    d = str(tmp_path / "disk")
    os.makedirs(d)
    with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=20 * MB, host_capacity_bytes=64 * MB,
                            remote_url="dir:" + tiny_dir, full_verify=True)) as s:
        cli = Client(s)
        v = cli.open(key("resnet50"), force_shared=True)
        assert v.outcome == "remote_fetch"
        assert F.sha256(d2h(v, torch)).hex() == gold["resnet50"]["trailer"]
        cli.close(v)
        assert os.listdir(d) == [key("resnet50").filename]
        st = s.stats()
        assert st["remote_fetches"] == 1 and st["disk_reads"] == 1
        assert st["tiers"][1]["misses"] == 1 and st["tiers"][2]["misses"] == 1 and st["tiers"][3]["hits"] == 1
        assert st["tiers"][2]["used_bytes"] == os.path.getsize(os.path.join(d, key("resnet50").filename))
        with pytest.raises(TrimsError) as ei:
            s.open(key("no-such-model"))
        assert ei.value.code == Errc.RemoteNotFound
        assert s.open(key("resnet50")).outcome == 0  # FastHit
        s.close(key("resnet50"))
