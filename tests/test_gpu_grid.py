"""The oversubscription grid extended to N GPU stores (paper_1811_09732_b200/
grid.py, the reference's run_grid, harness.cpp:370-544): daemon per store,
worker processes on their own connections; every cell runs, the fast tier
stays at half the catalog, the recorded requests are the workers' post-warmup
streams, and with N = 2 misses are served as PeerHits."""
import pytest

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.grid import run_grid

pytestmark = pytest.mark.gpu


def test_small_grid(tmp_path):
    models, div = C.catalog("tiny")
    models = models[:12]
    keys = [C.catalog_key(m) for m in models]
    total = sum(C.scaled_weights_bytes(m, div) for m in models)
    C.gen_catalog("tiny", str(tmp_path), seed=1, only=[m.name for m in models])
    g = run_grid(str(tmp_path), keys, total, fractions=(0.5, 1.0), concurrencies=(1, 3), worlds=(1, 2),
                 requests=90)
    assert len(g["cells"]) == 8
    for c in g["cells"]:
        assert c["ok"], c["error"]
        assert c["requests"] == (90 // c["concurrency"]) * c["concurrency"]
        assert 0.0 <= c["fast_hit_rate"] <= 1.0 and c["geomean_p95_speedup"] > 0
        if c["gpus"] == 1:
            assert c["peer_hits"] == 0
    assert any(c["peer_hits"] > 0 for c in g["cells"] if c["gpus"] == 2)


def test_grid_workers_under_mps(tmp_path):
    """The same cell with the worker processes as MPS clients (when the host
    has MPS): same decisions (hit rate, evictions) as time-sliced workers for
    one worker; concurrent workers complete."""
    models, div = C.catalog("tiny")
    models = models[:8]
    keys = [C.catalog_key(m) for m in models]
    total = sum(C.scaled_weights_bytes(m, div) for m in models)
    C.gen_catalog("tiny", str(tmp_path), seed=1, only=[m.name for m in models])
    plain = run_grid(str(tmp_path), keys, total, fractions=(1.0,), concurrencies=(1,), worlds=(1,), requests=40)
    g = run_grid(str(tmp_path), keys, total, fractions=(1.0,), concurrencies=(1, 2), worlds=(1,), requests=40,
                 mps=True)
    for c in g["cells"]:
        assert c["ok"], c["error"]
    one = g["cells"][0]
    ref = plain["cells"][0]
    assert (one["fast_hit_rate"], one["evictions"], one["disk_reads"]) == \
        (ref["fast_hit_rate"], ref["evictions"], ref["disk_reads"])
