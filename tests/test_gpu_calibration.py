"""SURVEY §8 row a13 on the device: the store measures the cost-model
calibration at creation (daemon.cpp:342-390) on the B200 path and publishes
it with the workspace headroom (StatsResponse, daemon.cpp:535-539), both in
process and over the wire daemon; Client.open uses it, and a model whose
workspace does not fit the advertised headroom is loaded privately
(client.cpp:192-204) with bytes identical to the shared copy."""
import os

import numpy as np
import pytest

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import Errc, TrimsError
from paper_1811_09732_b200.client import PRIVATE, SHARED, Client, TensorView
from paper_1811_09732_b200.daemon import RemoteStore, serve
from paper_1811_09732_b200.store import Store, StoreOptions

pytestmark = pytest.mark.gpu


def _bytes(v):
    import torch
    n = v.blob_bytes()
    return TensorView("b", [n], "i8", "native", 0, n, v.base_ptr).torch().view(torch.uint8).cpu().numpy()


def test_calibration_published_and_workspace_reservation(tmp_path):
    d = str(tmp_path)
    C.gen_catalog("tiny", d, seed=1, only=["alexnet", "resnet50"])
    key = F.ModelKey("zoo", "alexnet", "1.0.0")   # tiny alexnet: 3.7 MB weights, 8.06 MB workspace
    opts = StoreOptions(disk_cache_dir=d, fast_capacity_bytes=64 << 20, host_capacity_bytes=64 << 20,
                        workspace_headroom_fraction=0.1)   # headroom 6.7 MB < 8.06 MB
    with Store(opts) as s:
        st = s.stats()
        assert st["workspace_headroom"] == 0.1 and st["has_calibration"]
        assert st["calib_q"] > 1e6 and 0 < st["calib_o"] < 0.05 and 0 < st["calib_s"] < 0.05, st
        cli = Client(s, model_dirs=[d])
        v = cli.open(key)
        assert (v.origin, v.fallback_reason) == (PRIVATE, "workspace_reservation")
        assert cli.effective_params().q == st["calib_q"]   # the published calibration drives rho
        shared = cli.open(key, force_shared=True)
        assert shared.origin == SHARED
        assert np.array_equal(_bytes(v), _bytes(shared))
        cli.close(v)
        cli.close(shared)
        # Client::calibrate (client.cpp:361-423) against this store
        p = cli.calibrate(F.ModelKey("zoo", "resnet50", "1.0.0"))
        assert p.q > 1e6 and 0 <= p.o < 0.05 and 0 < p.s < 0.05
        # the same StatsResponse over the wire daemon
        ep = os.path.join(d, "mrmd.sock")
        with serve(s, ep):
            rs = RemoteStore(ep)
            rst = rs.stats()
            assert rst["workspace_headroom"] == 0.1 and rst["has_calibration"]
            assert rst["calib_q"] == st["calib_q"] and rst["calib_o"] == st["calib_o"]
            rcli = Client(rs, model_dirs=[d], attach_via_import=True)
            assert rcli.decide(key, rcli.resolve_local(key)) == (PRIVATE, "workspace_reservation")
            rs.close_connection()
    # a headroom that fits: shared
    with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=64 << 20, host_capacity_bytes=64 << 20,
                            startup_calibration=False)) as s:
        st = s.stats()
        assert st["workspace_headroom"] == 0.25 and not st["has_calibration"]
        cli = Client(s, model_dirs=[d])
        v = cli.open(key)
        assert v.origin == SHARED
        cli.close(v)
    with pytest.raises(TrimsError) as ei:
        Store(StoreOptions(disk_cache_dir=d, workspace_headroom_fraction=1.5))
    assert ei.value.code == Errc.InvalidArgument
