"""Drop-in at the TierBackend seam: the UNMODIFIED reference CacheCore
(compiled from /root/reference, oracle/_ref/libmrm_cuda.so) driving the B200
CudaTierBackend through the C ABI (integration/mrm_cuda_backend.cpp). Its
decisions must equal our own store's on the same trace and artifacts."""
import ctypes
import os

import pytest

import oracle
from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import TrimsError
from paper_1811_09732_b200.store import Store, StoreOptions

pytestmark = pytest.mark.gpu
SO = os.path.join(oracle.REF_DIR, "libmrm_cuda.so")
MB = 1_000_000

TRACE = ["o alexnet", "o alexnet", "c alexnet", "c alexnet", "o vgg16", "c vgg16", "o alexnet", "o resnet50",
         "c alexnet", "o googlenet", "c resnet50", "o vgg16", "c vgg16", "c googlenet", "o resnet50", "c resnet50",
         "c resnet50", "o absent"]


def ours(d, fast, host, eager, trace=TRACE, **kw):
    out = []
    with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=fast, host_capacity_bytes=host,
                            disk_capacity_bytes=1 << 40, eager_reclaim=eager, scan_disk=False, **kw)) as s:
        for line in trace:
            op, name = line.split()
            key = F.ModelKey("zoo", name, "1.0.0")
            outcome = 0
            try:
                if op == "o":
                    outcome = s.open(key).outcome
                else:
                    s.close(key)
            except TrimsError as e:
                outcome = 100 + e.code
            st = s.stats()
            rc = next((m["refcount"] for m in st["models"] if m["key"] == str(key)), 0)
            out.append((outcome, st["tiers"][0]["used_bytes"], st["tiers"][1]["used_bytes"], rc))
    return out


@pytest.mark.skipif(not os.path.exists(SO), reason="reference adapter not built (make -C oracle integration)")
@pytest.mark.parametrize("eager", [False, True])
def test_reference_cachecore_over_cuda_backend(tmp_path, eager):
    d = str(tmp_path)
    C.gen_catalog("tiny", d, seed=1, only=["alexnet", "resnet50", "vgg16", "googlenet"])
    L = ctypes.CDLL(SO)
    L.refcuda_replay.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_char_p,
                                 ctypes.c_char_p, ctypes.c_uint64]
    buf = ctypes.create_string_buffer(1 << 20)
    fast, host = 10 * MB, 13 * MB
    rc = L.refcuda_replay(d.encode(), fast, host, int(eager), "\n".join(TRACE).encode(), buf, len(buf))
    assert rc == 0
    lines = buf.value.decode().splitlines()
    ref = [tuple(int(x) for x in l.split()[:4]) for l in lines]
    tokens = [l.split()[4] for l in lines]
    assert ref == ours(d, fast, host, eager)
    assert any(t.startswith("trims.") and "@" in t for t in tokens)  # CUDA arena coordinates, not shm names


@pytest.mark.skipif(not os.path.exists(SO), reason="reference adapter not built (make -C oracle integration)")
def test_reference_cachecore_remote_tier_and_verify(tmp_path):
    """The reference CacheCore's RemoteFetch path (cache_core.cpp:230-285)
    through the adapter's fetch_remote -> remote.cpp, with full_verify on:
    same outcomes and tier usage as our store on the same trace."""
    remote = str(tmp_path / "remote")
    C.gen_catalog("tiny", remote, seed=1, only=["alexnet", "resnet50", "vgg16"])
    trace = ["o alexnet", "c alexnet", "o resnet50", "o vgg16", "c vgg16", "o alexnet", "c resnet50", "o absent",
             "c alexnet", "o vgg16", "c vgg16"]
    L = ctypes.CDLL(SO)
    L.refcuda_replay2.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64]
    buf = ctypes.create_string_buffer(1 << 20)
    fast, host = 10 * MB, 13 * MB
    url = "dir:" + remote
    d_ref, d_ours = str(tmp_path / "disk_ref"), str(tmp_path / "disk_ours")
    os.makedirs(d_ref)
    os.makedirs(d_ours)
    rc = L.refcuda_replay2(d_ref.encode(), url.encode(), 1, fast, host, 0, "\n".join(trace).encode(), buf, len(buf))
    assert rc == 0
    ref = [tuple(int(x) for x in l.split()[:4]) for l in buf.value.decode().splitlines()]
    got = ours(d_ours, fast, host, False, trace, remote_url=url, full_verify=True)
    assert ref == got
    assert [r[0] for r in ref[:4]] == [3, 0, 3, 3]  # RemoteFetch, -, RemoteFetch, RemoteFetch
    assert ref[7][0] == 100 + 140  # absent remotely: RemoteNotFound
    assert sorted(os.listdir(d_ref)) == sorted(os.listdir(d_ours)) == sorted(os.listdir(remote))
