"""Client::open's placement decision (client.cpp:148-222) — the rho cost
model with the store's published calibration and the workspace-reservation
fallback — against the UNMODIFIED reference client + daemon (oracle/_ref).

For every case the reference daemon runs with the given fast capacity,
workspace headroom and startup calibration; its client opens the model and
reports Shared or Private + reason; the daemon's published calibration is
read back. Our ``Client.decide`` then sees the same StatsResponse values
(a stats-only stand-in store) and must reach the same decision. CPU only."""
import itertools
import json
import os

import pytest

import oracle
from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200.client import PRIVATE, SHARED, Client, CostModelParams

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")

MODELS = ["alexnet", "squeezenet-v1.0", "resnet152"]
GRANS = [(F.MODEL, 2 << 20), (F.LAYER, 2 << 20), (F.BLOCK, 64 << 10), (F.BLOCK, 2 << 20)]
PARAMS = [None, (2e9, 1e-4, 1e-4), (50e6, 1e-3, 1e-3)]


class _StatsOnly:
    """The daemon as the decision sees it: a StatsResponse."""

    def __init__(self, st):
        self.st = st

    def stats(self):
        return self.st


@pytest.fixture(scope="module")
def catalog_dir(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("dec"))
    C.gen_catalog("tiny", d, seed=1, only=MODELS)
    return d


@pytest.mark.parametrize("calibrate,headroom", [(False, 0.25), (True, 0.25), (False, 0.05), (True, 1.0)])
def test_decisions_match_reference_client(catalog_dir, calibrate, headroom):
    R = oracle.ref()
    fast_cap = 96 << 20
    seen = set()
    for name, (kind, block), params in itertools.product(MODELS, GRANS, PARAMS):
        key = F.ModelKey("zoo", name, "1.0.0")
        want, (has_cal, q, o, s) = R.client_decision(catalog_dir, (key.ns, key.name, key.version), kind, block,
                                                      params, fast_cap, headroom, calibrate)
        assert has_cal == calibrate  # the largest tiny artifact is >= 1 MiB
        st = {"tiers": [{"capacity_bytes": fast_cap}] + [{"capacity_bytes": 0}] * 3,
              "workspace_headroom": headroom, "has_calibration": has_cal}
        if has_cal:
            st.update(calib_q=q, calib_o=o, calib_s=s)
        cli = Client(_StatsOnly(st), model_dirs=[catalog_dir])
        origin, what = cli.decide(key, cli.resolve_local(key), granularity=kind, block_bytes=block,
                                  params=CostModelParams(*params) if params else None)
        got = "shared" if origin == SHARED else f"private {what}"
        assert got == want, (name, kind, block, params, calibrate, headroom, (q, o, s))
        seen.add(got)
    # the grid exercises every outcome of the decision
    want_seen = {"private benefit_non_positive"} | (
        {"private workspace_reservation"} if headroom < 0.1 else {"shared"})
    assert want_seen <= seen, seen


def test_workspace_reservation_and_calibrated_params_are_used(catalog_dir):
    key = F.ModelKey("zoo", "alexnet", "1.0.0")
    ws = json.loads(F.read_manifest(os.path.join(catalog_dir, key.filename)).manifest_json)["workspace_bytes"]
    base = {"tiers": [{"capacity_bytes": 4 * ws}] + [{"capacity_bytes": 0}] * 3, "has_calibration": False}
    fits = Client(_StatsOnly(dict(base, workspace_headroom=0.25)), model_dirs=[catalog_dir])
    assert fits.decide(key, fits.resolve_local(key)) == (SHARED, F.MODEL)
    tight = Client(_StatsOnly(dict(base, workspace_headroom=0.2)), model_dirs=[catalog_dir])
    assert tight.decide(key, tight.resolve_local(key)) == (PRIVATE, "workspace_reservation")
    # a published calibration that makes sharing not pay: slow export/attach
    slow = dict(base, workspace_headroom=1.0, has_calibration=True, calib_q=1e12, calib_o=1.0, calib_s=1.0)
    cli = Client(_StatsOnly(slow), model_dirs=[catalog_dir])
    assert cli.decide(key, cli.resolve_local(key)) == (PRIVATE, "benefit_non_positive")
    # explicit params win over the calibration (client.cpp:137-142)
    assert cli.decide(key, cli.resolve_local(key), params=CostModelParams()) == (SHARED, F.MODEL)
    # force_shared skips both checks
    assert cli.decide(key, cli.resolve_local(key), force_shared=True) == (SHARED, F.MODEL)
