"""BASELINE configs[1] on the GPU: several client processes serve inference
from one HBM copy exported by the store (paper_1811_09732_b200/sharing.py).
Every client's logits equal the store process's own forward on the same
input (same weights bytes, same kernels); one copy, one disk read."""
import numpy as np
import pytest

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.models import BoundNet, arch_text
from paper_1811_09732_b200.sharing import SharedModel, run_clients
from paper_1811_09732_b200.store import Store, StoreOptions

pytestmark = pytest.mark.gpu


def test_four_clients_one_copy(tmp_path):
    import torch
    arch = C.ARCHS["resnet50"]()
    C.write_arch(arch, str(tmp_path), seed=1)
    opts = StoreOptions(disk_cache_dir=str(tmp_path), fast_capacity_bytes=1 << 30, convert_to="bf16",
                        permute_4d=True, scan_disk=False)
    with Store(opts) as s:
        ex = s.open(C.arch_key(arch))
        r = run_clients(SharedModel.from_export(ex, arch_text(arch)), ex.fd, n_clients=4, n_reqs=3, seed=5)
        st = s.stats()
        assert st["disk_reads"] == 1 and st["tiers"][0]["used_bytes"] == ex.weights_bytes
        assert r["requests"] == 12 and r["p50_ms"] > 0
        # the store process's own executor on the same bytes and input
        cli = Client(s, device=0)
        v = cli.open(C.arch_key(arch), force_shared=True)
        net = BoundNet(v, arch, batch=1)
        x = np.random.default_rng(5).standard_normal((1, 3, net.input_hw, net.input_hw)).astype(np.float32)
        want = net.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        for y in r["logits"]:
            assert np.array_equal(y, r["logits"][0])
            np.testing.assert_allclose(y, want, rtol=0, atol=1e-5)
        net.close()
        cli.close(v)
        s.close(C.arch_key(arch))


def test_daemon_clients_one_copy(tmp_path):
    """The same through the wire-protocol daemon: clients open over the
    socket (FastHits on the one copy) and close their handles at the end."""
    from paper_1811_09732_b200.daemon import serve
    from paper_1811_09732_b200.sharing import run_daemon_clients
    arch = C.ARCHS["resnet50"]()
    C.write_arch(arch, str(tmp_path), seed=1)
    opts = StoreOptions(disk_cache_dir=str(tmp_path), fast_capacity_bytes=1 << 30, convert_to="bf16",
                        permute_4d=True, scan_disk=False)
    ep = str(tmp_path / "mrmd.sock")
    with Store(opts) as s, serve(s, ep):
        ex = s.open(C.arch_key(arch))
        r = run_daemon_clients(ep, C.arch_key(arch), arch_text(arch), n_clients=4, n_reqs=3, seed=5)
        st = s.stats()
        assert st["disk_reads"] == 1 and st["tiers"][0]["used_bytes"] == ex.weights_bytes
        assert st["open_requests"] == 5 and st["tiers"][0]["hits"] == 4  # 4 client opens hit the one copy
        assert r["requests"] == 12
        assert all(np.array_equal(y, r["logits"][0]) for y in r["logits"])
        assert [m["refcount"] for m in st["models"]] == [1]  # only the store's own open remains
        s.close(C.arch_key(arch))
