"""GPU parity of the ingest kernels (K1..K5) against the CPU oracle — bit-exact."""
import ctypes
import json

import numpy as np
import pytest

import oracle
from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import check, lib
from tests.gpu_util import expected_resident, layer_checksums
from tests.golden_data import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    assert lib.trims_device_count() >= 1
    return t


def ingest(torch, src_json, blob, flags, out_dtype="bf16"):
    res_json = F.resident_manifest(src_json, flags, out_dtype)
    rb = json.loads(res_json)["tensors"]
    end = max((t["offset"] + t["nbytes"] for t in rb), default=0)
    rbytes = max((end + 63) // 64 * 64, 64)
    host = torch.from_numpy(np.ascontiguousarray(blob)).pin_memory() if blob.size else torch.zeros(1, dtype=torch.uint8).pin_memory()
    dev = torch.full((rbytes,), 0xCD, dtype=torch.uint8, device="cuda")
    cs = ctypes.c_uint64()
    st = (ctypes.c_double * 5)()
    check(lib.trims_ingest_host(0, host.data_ptr(), src_json.encode(), flags, F.DTYPE_CODE[out_dtype], dev.data_ptr(),
                                ctypes.byref(cs), st))
    torch.cuda.synchronize()
    end_b = (end + 63) // 64 * 64
    return res_json, dev[:end_b].cpu().numpy(), cs.value, list(st)


def test_identity_ingest_catalog_bytes_and_checksum(torch):
    g = load("catalog.json.gz")
    P = oracle.port()
    for e in g["tiny_seed1"][:8]:
        blob = C.catalog_blob(e["manifest_json"], e["name"], 1)
        res_json, out, cs, st = ingest(torch, e["manifest_json"], blob, 0)
        assert res_json == e["manifest_json"]
        assert F.sha256(out).hex() == e["trailer"], e["name"]        # == the reference's own trailer
        assert cs == P.block_checksum(out), e["name"]
        assert F.touch_host(out, res_json) == e["touch"]              # == the reference's own touch


@pytest.mark.parametrize("arch", ["alexnet", "resnet50", "vgg16", "vgg19"])
def test_convert_permute_bit_exact(torch, arch):
    """Every real-shape net the bench reports, fp32 KCRS -> bf16 KRSC. VGG's
    411 MB fc6 and its 512-channel k-slices take different tile paths from
    ResNet-50's (elementwise chunks vs whole k-slices vs the direct kernel)."""
    a = C.ARCHS[arch]()
    src_json, blob = C.arch_blob(a, seed=1)
    flags = F.PLAN_CONVERT | F.PLAN_PERMUTE_4D
    res_json, out, cs, st = ingest(torch, src_json, blob, flags)
    want = expected_resident(src_json, blob, res_json)
    assert out.size == want.size
    bad = np.nonzero(out != want)[0]
    assert bad.size == 0, f"{bad.size} bytes differ, first at {bad[:8]}"
    assert cs == oracle.port().block_checksum(want)


@pytest.mark.parametrize("flags,out_dtype", [(1, "bf16"), (1, "f32"), (2, "bf16"), (3, "f32"), (0, "bf16")])
def test_dtype_matrix_with_special_values(torch, flags, out_dtype):
    rng = np.random.default_rng(5)
    specials64 = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan, 1e-310, -1e-310, 1e300, -1e300,
                           3.4e38, 3.5e38, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 2 ** -133, 2 ** -134, 5e-324], np.float64)
    nan_payload = np.array([0x7ff0000000000001, 0xfff4000000000000], np.uint64).view(np.float64)
    x64 = np.concatenate([specials64, nan_payload, rng.standard_normal(997) * 10.0 ** rng.integers(-40, 40, 997)])
    x32 = np.concatenate([specials64.astype(np.float32), rng.standard_normal(1003).astype(np.float32)])
    x16 = np.concatenate([np.array([0, 0x8000, 0x7c00, 0xfc00, 0x7e01, 0x0001, 0x03ff, 0x8001], np.uint16),
                          rng.integers(0, 65536, 995, dtype=np.uint16)])
    i8 = rng.integers(0, 256, 77, dtype=np.uint8)
    conv = rng.standard_normal(5 * 3 * 3 * 3).astype(np.float32)
    decls = [("a64", "f64", [x64.size]), ("b32", "f32", [x32.size]), ("c16", "f16", [x16.size]),
             ("d8", "i8", [i8.size]), ("e4d", "f32", [5, 3, 3, 3]), ("f64x4", "f64", [7, 2, 1, 3])]
    mj = F.make_manifest(F.ModelKey("t", "dt", "1"), decls)
    m = json.loads(mj)
    blob = np.zeros((max(t["offset"] + t["nbytes"] for t in m["tensors"]) + 63) // 64 * 64, np.uint8)
    payloads = [x64.view(np.uint8), x32.view(np.uint8), x16.view(np.uint8), i8,
                conv.view(np.uint8), rng.standard_normal(42).view(np.uint8)]
    for t, p in zip(m["tensors"], payloads):
        blob[t["offset"]:t["offset"] + t["nbytes"]] = p
    res_json, out, cs, _ = ingest(torch, mj, blob, flags, out_dtype)
    want = expected_resident(mj, blob, res_json)
    assert np.array_equal(out, want)
    assert cs == oracle.port().block_checksum(want)


def test_per_tensor_checksums_sum_to_total(torch):
    a = C.ARCHS["alexnet"]()
    src_json, blob = C.arch_blob(a, seed=3)
    res_json, out, cs, _ = ingest(torch, src_json, blob, 3)
    parts = layer_checksums(res_json, out)
    assert sum(parts) % (1 << 64) == cs


def test_device_fills_match_host(torch):
    n = 1_000_003
    d = torch.empty(n, dtype=torch.int64, device="cuda")
    check(lib.trims_fill_splitmix_device(d.data_ptr(), n, 0x1234, 77, None))
    h = np.empty(n, np.uint64)
    check(lib.trims_fill_splitmix_host(h.ctypes.data, n, 0x1234, 77))
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy().view(np.uint64), h)
    assert np.array_equal(h[:1000], oracle.port().splitmix(0x1234, 77, 1000))
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    check(lib.trims_fill_uniform_device(f.data_ptr(), n, 99, 5, -0.25, 0.75, None))
    hf = np.empty(n, np.float32)
    check(lib.trims_fill_uniform_host(hf.ctypes.data, n, 99, 5, -0.25, 0.75))
    torch.cuda.synchronize()
    assert np.array_equal(f.cpu().numpy().view(np.uint32), hf.view(np.uint32))
    assert np.array_equal(hf[:1000], oracle.port().uniform_f32(99, 5, 1000, -0.25, 0.75))


def test_checksum_kernel_any_alignment(torch):
    rng = np.random.default_rng(11)
    data = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    d = torch.from_numpy(data).cuda()
    P = oracle.port()
    for off, n, w0 in [(0, 1 << 20, 0), (8, 12345, 3), (16, 64, 9), (0, 7, 0), (24, 1000000, 100)]:
        acc = torch.zeros(1, dtype=torch.int64, device="cuda")
        check(lib.trims_checksum_device(d.data_ptr() + off, n, w0, acc.data_ptr(), None))
        torch.cuda.synchronize()
        assert int(acc.cpu().numpy().view(np.uint64)[0]) == P.block_checksum(data[off:off + n], w0)
