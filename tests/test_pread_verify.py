"""The pipelined verify (csrc/pread.cpp through model::read_manifest with
full_verify, model_format.cpp:370-409): blobs around the 2 MiB piece and the
1 MiB final-wave boundaries and one larger than the verify ring (so ring slots
are reused), each accepted when intact and rejected (ChecksumMismatch) when one
byte anywhere -- first piece, middle, last fine piece, last byte -- is flipped.
CPU only."""
import os

import numpy as np
import pytest

from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import Errc, TrimsError

MiB = 1 << 20


def artifact(path, n_bytes, seed):
    rng = np.random.default_rng(seed)
    n = max(1, n_bytes // 8)
    mj = F.make_manifest(F.ModelKey("t", f"p{seed}", "1"), [("w", "f64", [n])])
    blob = np.zeros((n * 8 + 63) // 64 * 64, np.uint8)
    blob[:n * 8] = rng.integers(0, 256, n * 8, dtype=np.uint8)
    F.write_model(path, mj, blob)
    return F.read_manifest(path)


@pytest.mark.parametrize("n_bytes", [8, 2 * MiB - 64, 2 * MiB, 2 * MiB + 64, 17 * MiB + 8, 45 * MiB + 4096 + 8])
def test_verify_accepts_and_rejects(tmp_path, n_bytes):
    p = str(tmp_path / "m.trms")
    info = artifact(p, n_bytes, n_bytes % 1000)
    assert F.read_manifest(p, full_verify=True).checksum == info.checksum
    blob_end = info.blob_offset + info.blob_bytes
    spots = sorted({info.blob_offset, info.blob_offset + info.blob_bytes // 2,
                    max(info.blob_offset, blob_end - MiB // 2), blob_end - 1})
    for at in spots:
        with open(p, "r+b") as f:
            f.seek(at)
            b = f.read(1)
            f.seek(at)
            f.write(bytes([b[0] ^ 0x80]))
        with pytest.raises(TrimsError) as ei:
            F.read_manifest(p, full_verify=True)
        assert ei.value.code == Errc.ChecksumMismatch, at
        with open(p, "r+b") as f:
            f.seek(at)
            f.write(b)
    assert F.read_manifest(p, full_verify=True).checksum == info.checksum


def test_verify_truncated_blob(tmp_path):
    p = str(tmp_path / "m.trms")
    info = artifact(p, 9 * MiB, 3)
    os.truncate(p, info.blob_offset + info.blob_bytes // 2)
    with pytest.raises(TrimsError):
        F.read_manifest(p, full_verify=True)
