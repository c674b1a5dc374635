"""bench.py's reference arm: it must run the UNMODIFIED reference
(oracle/_ref/libmrm_ref.so) on the same inputs as our arm, with no product
code in its process (the driver voids the comparison if libtrims.so is mapped).
CPU only."""
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
def test_reference_writer_produces_our_artifact_bytes(tmp_path):
    """ref_write_arch (reference writer + oracle port generator) == catalog.write_arch (ours)."""
    import bench
    from paper_1811_09732_b200 import catalog as C
    from paper_1811_09732_b200 import format as F
    arch = C.ARCHS["resnet50"]()
    key, ref_path = bench.ref_write_arch(oracle.ref(), oracle.port(), bench._archs().ARCHS["resnet50"](),
                                         str(tmp_path / "ref"))
    ours = C.write_arch(arch, str(tmp_path / "ours"), seed=1)
    assert F.ModelKey(*key).filename == os.path.basename(ours)
    assert os.path.getsize(ours) == os.path.getsize(ref_path)
    with open(ours, "rb") as a, open(ref_path, "rb") as b:
        assert F.sha256(a.read()) == F.sha256(b.read())


def test_reference_arm_traces_equal_ours():
    import bench
    from paper_1811_09732_b200 import catalog as C
    from paper_1811_09732_b200 import workload as W
    assert bench.zipf_trace(42, 1000, 37, 1.1) == W.zipf_trace(42, 1000, 37, 1.1)
    assert [r[0] for r in bench._standalone("catalog_tables").SMALL37] == [m.name for m in C.catalog("small37")[0]]
    assert bench.nearest_rank([3, 1, 2, 4], 50) == W.percentile([3, 1, 2, 4], 50)
    if oracle.ref_available():
        assert oracle.ref().pareto_trace(42, 1000, 1.0, 1.0, 37) == W.pareto_trace(42, 1000, 37)


def test_both_arms_report_the_same_config():
    import bench
    assert bench.bench_config(1, 2) == bench.bench_config(1, 2)
    assert "workload" in bench.bench_config(1, 2)


@needs_ref
def test_reference_arm_process_maps_no_product_library(tmp_path):
    """Drive the reference arm's input writer, one run_latency and one worker
    in a fresh interpreter, then read its /proc/self/maps."""
    code = f"""
import os, sys
sys.path.insert(0, {ROOT!r})
import bench, oracle
R, P, A = oracle.ref(), oracle.port(), bench._archs()
key, path = bench.ref_write_arch(R, P, A.ARCHS["alexnet"](), {str(tmp_path)!r})
R.latency({str(tmp_path)!r}, key, "warm", 1)
r = bench.ref_workers(R, {str(tmp_path)!r}, key, 2, 2)
assert r["requests"] == 4 and r["identical_touch_across_clients"] and r["disk_reads"] == 1, r
maps = open("/proc/self/maps").read()
so = sorted({{l.split()[-1] for l in maps.splitlines() if l.split()[-1].startswith({ROOT!r}) and ".so" in l}})
print("\\n".join(so))
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    libs = [l for l in out.stdout.split() if l]
    assert libs and all("/oracle/_ref/" in l for l in libs), libs
    assert not any("libtrims.so" in l for l in libs)
