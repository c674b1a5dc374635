"""The C-ABI boundary: the library loads on a GPU-less host, exports every
symbol include/trims.h declares, and the product never imports the oracle."""
import os
import re

from paper_1811_09732_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "trims.h")).read()
    return sorted(set(re.findall(r"\b(trims_[a-z0-9_]+)\s*\(", hdr)))


def test_header_symbols_exported():
    names = declared_symbols()
    assert len(names) >= 39
    for n in names:
        assert hasattr(_lib.lib, n), n
    assert set(names) == set(_lib.exported_symbols())


def test_errc_values_and_wire_collapse():
    L = _lib.lib
    assert L.trims_errc_name(1) == b"NotFound"
    assert L.trims_errc_name(104) == b"ChecksumMismatch"
    assert L.trims_wire_code(104) == 5 and L.trims_wire_code(140) == 1 and L.trims_wire_code(120) == 4
    assert L.trims_wire_code(170) == 7


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1811_09732_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".hpp", ".h")):
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert not re.search(r'#include\s*[<"][^>"]*trims_oracle', src), f
                assert "libtrims_oracle" not in src and "libmrm_ref" not in src, f


def test_no_device_fails_loudly(tmp_path):
    import pytest
    from paper_1811_09732_b200.store import Store, StoreOptions, device_count
    if device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(_lib.TrimsError) as ei:
        Store(StoreOptions(disk_cache_dir=str(tmp_path)))
    assert ei.value.code == _lib.Errc.NoDevice
