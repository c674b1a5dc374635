"""Loaders for the committed golden vectors (tests/golden/, made by make_golden.py)."""
import gzip
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rt") as f:
            return json.load(f)
    with open(path) as f:
        return json.load(f)


def manifest_tensors(mjson: str):
    m = json.loads(mjson)
    return m, [(t["offset"], t["nbytes"]) for t in m["tensors"]]
