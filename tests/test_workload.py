"""Request-trace generators (paper_1811_09732_b200/workload.py): the Pareto
stream is the reference worker's, bit for bit (golden from the reference
build: tests/golden/pareto_trace.json); the Zipf stream is seeded and skewed."""
import json
import os

from paper_1811_09732_b200 import workload as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "pareto_trace.json")


def test_pareto_trace_is_the_reference_stream():
    for c in json.load(open(GOLDEN)):
        assert W.pareto_trace(c["seed"], c["n"], c["active"], c["alpha"], c["x_m"]) == c["trace"]


def test_pareto_rank_edges():
    assert W.pareto_rank(0.999999, 1.0, 1.0, 37) == 1
    assert W.pareto_rank(1e-9, 1.0, 1.0, 37) == 37
    assert W.pareto_rank(0.5, 1.0, 1.0, 37) == 2


def test_zipf_trace_seeded_and_skewed():
    a, b = W.zipf_trace(3, 1000, 37), W.zipf_trace(3, 1000, 37)
    assert a == b and min(a) >= 0 and max(a) < 37
    counts = [a.count(i) for i in range(37)]
    assert counts[0] > counts[5] > counts[30]


def test_percentile_nearest_rank():
    assert W.percentile([3, 1, 2, 4], 50) == 2
    assert W.percentile([3, 1, 2, 4], 100) == 4
    assert W.percentile([5], 1) == 5
