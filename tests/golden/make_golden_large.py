#!/usr/bin/env python3
"""Golden vectors for the multi-GB large8 models, from the UNMODIFIED reference.

    make -C oracle && python tests/golden/make_golden_large.py [names...]

For each model the reference's own ``bench::gen_catalog`` writes the artifact
(seed 1, the harness seed, harness.cpp:100/371), ``read_manifest(full_verify)``
returns its trailer, ``touch_file`` its FNV touch; the file is then deleted.
Output: tests/golden/large8.json. The GPU test
``tests/test_gpu_large.py`` checks our 6.4 GB identity ingest against it.
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)
import oracle  # noqa: E402
from make_golden import catalog_entries  # noqa: E402


def main() -> None:
    names = sys.argv[1:] or ["vgg16-s4"]
    out_path = os.path.join(HERE, "large8.json")
    doc = json.load(open(out_path)) if os.path.exists(out_path) else {}
    with tempfile.TemporaryDirectory(prefix="trims-golden-large-", dir=os.environ.get("TMPDIR", "/tmp")) as tmp:
        for e in catalog_entries(oracle.ref(), "large8", names, 1, tmp):
            e.pop("manifest_json")  # pinned separately in catalog.json.gz (large8_manifests)
            doc[e["name"]] = e
    json.dump(doc, open(out_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
