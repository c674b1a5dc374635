"""Edge cases of the ingest transform vs the CPU oracle (bit-exact bytes and
checksum): the empty model and one-element tensors (zero dims are rejected,
model_format.cpp:123-148), ragged element counts (partial
resident words), 1x1 and 1-channel filters, k-slices larger than a ring stage
(the direct gather kernel), thousands of tiny tensors (static bins longer than
one shared-memory descriptor batch), every dtype pair, and the identity plan.
The same cases through the HBM-resident transform (trims_plan_transform)."""
import json

import numpy as np
import pytest

import oracle
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200.ingest import IngestPlan
from tests.gpu_util import expected_resident
from tests.test_gpu_ingest import ingest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def build(decls, seed):
    rng = np.random.default_rng(seed)
    mj = F.make_manifest(F.ModelKey("t", f"edge{seed}", "1"), decls)
    m = json.loads(mj)
    end = max((t["offset"] + t["nbytes"] for t in m["tensors"]), default=0)
    blob = np.zeros((end + 63) // 64 * 64, np.uint8)
    for t in m["tensors"]:
        n = t["nbytes"]
        if t["dtype"] == "f32":
            p = rng.standard_normal(n // 4).astype(np.float32).view(np.uint8)
        elif t["dtype"] == "f64":
            p = rng.standard_normal(n // 8).view(np.uint8)
        else:
            p = rng.integers(0, 256, n, dtype=np.uint8)
        blob[t["offset"]:t["offset"] + n] = p
    return mj, blob


CASES = {
    "single_elements": [("s0", "f32", [1]), ("a", "f32", [5]), ("s1", "f32", [1, 1, 3, 3]), ("b", "f64", [1])],
    "ragged_counts": [(f"r{i}", "f32", [n]) for i, n in enumerate([1, 2, 3, 5, 7, 9, 15, 17, 33, 1023, 4097])],
    "filters": [("c1", "f32", [64, 3, 7, 7]), ("pw", "f32", [128, 64, 1, 1]), ("one_c", "f32", [16, 1, 3, 3]),
                ("odd", "f32", [5, 7, 3, 5]), ("c96", "f32", [256, 96, 5, 5])],
    "oversize_slices": [("big", "f32", [4, 2048, 3, 3]), ("huge", "f32", [2, 4096, 5, 5]), ("tail", "f32", [3])],
    "f64_and_f16": [("d", "f64", [1001]), ("h", "f16", [1003]), ("dk", "f64", [9, 4, 3, 3]), ("hk", "f16", [8, 8, 3, 3])],
    "many_tiny": [(f"t{i}", "f32", [1 + (i * 7) % 13]) for i in range(3000)],
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("flags,out", [(3, "bf16"), (1, "f32"), (2, "bf16"), (0, "bf16")])
def test_edges_host_ingest_bit_exact(torch, name, flags, out):
    mj, blob = build(CASES[name], sum(map(ord, name)))
    res_json, got, cs, _ = ingest(torch, mj, blob, flags, out)
    want = expected_resident(mj, blob, res_json)
    assert got.size == want.size
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{name}: {bad.size} bytes differ, first at {bad[:8]}"
    assert cs == oracle.port().block_checksum(want)


@pytest.mark.parametrize("name", sorted(CASES))
def test_edges_hbm_resident_transform(torch, name):
    mj, blob = build(CASES[name], 7 + sum(map(ord, name)))
    plan = IngestPlan(mj, 3, "bf16")
    d_src = torch.from_numpy(blob if blob.size else np.zeros(64, np.uint8)).cuda()
    d_dst = torch.full((max(plan.resident_bytes, 64),), 0xCD, dtype=torch.uint8, device="cuda")
    d_sums = torch.zeros(plan.buckets, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(3):  # repeated launches: the scheduler's ticket bases must stay in step
        d_sums.zero_()
        plan.transform(d_src.data_ptr(), d_dst.data_ptr(), d_sums.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    want = expected_resident(mj, blob, plan.resident_json)
    got = d_dst[:want.size].cpu().numpy()
    assert np.array_equal(got, want), name
    total = int(d_sums.cpu().numpy().view(np.uint64).sum(dtype=np.uint64))
    assert total == oracle.port().block_checksum(want)


def test_empty_model(torch):
    mj = F.make_manifest(F.ModelKey("t", "empty", "1"), [])
    res_json, got, cs, _ = ingest(torch, mj, np.zeros(0, np.uint8), 3)
    assert json.loads(res_json)["tensors"] == [] and cs == 0
