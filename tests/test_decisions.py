"""Placement decisions of the product CacheCore (csrc/cache_core.cpp) replayed
through the C ABI (trims_replay) vs the reference live CacheCore + simulator
(tests/golden/decisions.json.gz): outcome, eviction lists, used bytes and
refcount per op, plus final stats — bit-exact."""
import numpy as np

from oracle import simulator as sim
from paper_1811_09732_b200._lib import lib, text_call
from tests.golden_data import load


def replay(spec: str) -> list[str]:
    return text_call(lambda o, c: lib.trims_replay(spec.encode(), o, c), cap=1 << 24).splitlines()


def test_recorded_traces_bit_exact():
    traces = load("decisions.json.gz")
    ops = 0
    for t in traces:
        got = replay(t["spec"])
        assert got[:-1] == t["events"]
        assert got[-1] == t["stats"]
        ops += len(t["events"])
    assert ops > 30000


def test_fresh_random_traces_vs_simulator_restatement():
    rng = np.random.default_rng(99)
    for _ in range(40):
        cfg, models, trace = sim.random_trace(rng, max_models=32, max_ops=800)
        got = replay(sim.spec_text(cfg, models, trace))[:-1]
        want = [e.line(i, "live") for i, e in enumerate(sim.simulate(cfg, models, trace))]
        assert got == want
