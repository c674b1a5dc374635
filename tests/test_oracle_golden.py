"""Pins the CPU oracle (oracle/trims_oracle.c + oracle/simulator.py) against
vectors produced by the reference itself (tests/golden/, see make_golden.py)
and against the reference's own known-answer tests. CPU only."""
import json

import numpy as np
import pytest

import oracle
from oracle import simulator as sim
from tests.golden_data import load, manifest_tensors


@pytest.fixture(scope="module")
def P():
    return oracle.port()


def test_sha256_kats(P):
    g = load("sha256.json")
    # proj/tests/test_model_format.cpp:69-81
    assert P.sha256(b"").hex() == g["kat"][""] == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert P.sha256(b"abc").hex() == g["kat"]["abc"] == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    for k, v in g["vectors"].items():
        data = np.random.default_rng(7).integers(0, 256, 100000, dtype=np.uint8).tobytes() if k == "rng7_100000" \
            else bytes.fromhex(k)
        assert P.sha256(data).hex() == v


def catalog_blob(P, entry):
    """Rebuild a catalog blob with the port: k-th element = splitmix(seed ^ fnv1a(name), k)
    in manifest order, padding zero (catalog.cpp:130-159)."""
    m, tens = manifest_tensors(entry["manifest_json"])
    blob = np.zeros(entry["blob_bytes"], np.uint8)
    stream = P.catalog_stream(entry["seed"], entry["name"])
    k = 0
    for off, nb in tens:
        n = nb // 8
        blob[off:off + nb] = P.splitmix(stream, k, n).view(np.uint8)
        k += n
    return blob, tens


def test_tiny_catalog_blob_trailer_and_touch(P):
    g = load("catalog.json.gz")
    for entry in g["tiny_seed1"] + g["tiny_seed42"]:
        blob, tens = catalog_blob(P, entry)
        assert P.sha256(blob).hex() == entry["trailer"], entry["name"]
        assert P.touch(blob, [o for o, _ in tens], [n for _, n in tens]) == entry["touch"], entry["name"]


@pytest.mark.slow
def test_small37_alexnet_trailer(P):
    g = load("catalog.json.gz")
    entry = [e for e in g["small37_seed1"] if e["name"] == "alexnet"][0]
    # SURVEY.md §7 minimum-slice check 1
    assert entry["trailer"] == "b65080991db0dfab4cc84cd59e7f5423d7f469fdafa40ea4de38f9c290604aa4"
    blob, tens = catalog_blob(P, entry)
    assert P.sha256(blob).hex() == entry["trailer"]
    assert P.touch(blob, [o for o, _ in tens], [n for _, n in tens]) == entry["touch"] == 0xdbf1ed612dbadfbb


def test_share_benefit_examples(P):
    # proj/tests/test_client.cpp:28-42
    assert P.share_benefit(238e6, 1, 193.30e6, 0.001, 0.001) == pytest.approx(1.229, rel=0.01)
    assert P.share_benefit(4.8e6, 52, 521.32e6, 0.0005, 0.0005) == pytest.approx(-0.043, rel=0.01)
    assert P.share_benefit(0, 0, 193.30e6, 0.001, 0.001) == 0.0


def parse_spec(spec: str):
    cfg, models, trace = None, [], []
    for line in spec.splitlines():
        f = line.split()
        if f[0] == "cfg":
            cfg = sim.SimConfig(int(f[1]), int(f[2]), int(f[3]), int(f[4]), bool(int(f[5])))
        elif f[0] == "model":
            models.append(sim.SimModel(int(f[1]), int(f[2]), bool(int(f[3])), bool(int(f[4]))))
        elif f[0] == "op":
            trace.append((f[1], int(f[2])))
    return cfg, models, trace


def test_simulator_restatement_matches_reference_decisions():
    traces = load("decisions.json.gz")
    assert len(traces) >= 100
    n_ops = 0
    for t in traces:
        cfg, models, trace = parse_spec(t["spec"])
        ev = sim.simulate(cfg, models, trace)
        got = [e.line(i, "live") for i, e in enumerate(ev)]
        for a, b in zip(got, t["events"]):
            # closes: the reference live shim reports 0 for a valid close, 103 for invalid
            assert a == b, (a, b)
        n_ops += len(trace)
    assert n_ops > 30000


def test_new_transform_definitions(P):
    # fp32 -> bf16 RNE corner cases (our definition; parity unpinned vs reference)
    x = np.array([0.0, -0.0, 1.0, np.inf, -np.inf, np.nan, 3.4028235e38, 1.00390625, 1.01171875, 1e-40],
                 np.float32)
    b = P.f32_to_bf16(x)
    assert b[0] == 0x0000 and b[1] == 0x8000 and b[2] == 0x3F80
    assert b[3] == 0x7F80 and b[4] == 0xFF80 and (b[5] & 0x7FC0) == 0x7FC0
    assert b[6] == 0x7F80  # FLT_MAX rounds past the largest finite bf16 -> Inf
    assert b[7] == 0x3F80  # 1 + 2^-8: tie, round to even (down)
    assert b[8] == 0x3F82  # 1 + 3*2^-8: tie, round to even (up)
    # f64 -> bf16 single rounding agrees with f64->f32->bf16 whenever f32 is exact
    rng = np.random.default_rng(1)
    v = rng.standard_normal(10000).astype(np.float32).astype(np.float64)
    assert np.array_equal(P.f64_to_bf16(v), P.f32_to_bf16(v.astype(np.float32)))
    # permute
    w = rng.standard_normal((4, 3, 2, 5)).astype(np.float32)
    assert np.array_equal(P.permute_kcrs_krsc(w), np.transpose(w, (0, 2, 3, 1)))
    # checksum is additive over disjoint word ranges (a checksum of checksums)
    data = rng.integers(0, 256, 8 * 1000, dtype=np.uint8)
    whole = P.block_checksum(data)
    parts = (P.block_checksum(data[:4096], 0) + P.block_checksum(data[4096:], 512)) % (1 << 64)
    assert whole == parts
    # f16 -> f32 widening is exact
    h = rng.standard_normal(5000).astype(np.float16)
    assert np.array_equal(P.f16_to_f32(h.view(np.uint16)), h.astype(np.float32))
