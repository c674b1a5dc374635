"""Cold opens with buffered vs O_DIRECT reads into the pinned host tier, with
the artifact in the page cache ("cached") and evicted from it ("uncached":
fsync + posix_fadvise(DONTNEED) before every open):
    python scripts/direct_io_ab.py [arch ...]   (default resnet50 vgg19)
One JSON line per (arch, page cache state, read mode): median cold-open ms
over 5 opens and the artifact GB/s it implies."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200.client import Client
from paper_1811_09732_b200.store import Store, StoreOptions


def drop_cache(path: str) -> None:
    fd = os.open(path, os.O_RDONLY)
    try:
        os.fsync(fd)
        os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
    finally:
        os.close(fd)


def main():
    archs = sys.argv[1:] or ["resnet50", "vgg19"]
    d = tempfile.mkdtemp(dir=os.environ.get("TRIMS_AB_DIR"))
    for name in archs:
        arch = C.ARCHS[name]()
        C.write_arch(arch, d, seed=1)
        key = C.arch_key(arch)
        path = os.path.join(d, key.filename)
        size = os.path.getsize(path)
        for cache in ("cached", "uncached"):
            for mode in ("buffered", "direct"):
                with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=4 << 30, host_capacity_bytes=4 << 30,
                                        convert_to="bf16", permute_4d=True, eager_reclaim=True,
                                        direct_io=mode)) as s:
                    cli = Client(s)
                    ts = []
                    for _ in range(5):
                        if cache == "uncached":
                            drop_cache(path)
                        else:
                            with open(path, "rb") as f:  # make sure it is resident
                                while f.read(64 << 20):
                                    pass
                        t0 = time.perf_counter()
                        v = cli.open(key, force_shared=True)
                        ts.append((time.perf_counter() - t0) * 1e3)
                        cli.close(v)
                    st = s.stats()
                ts.sort()
                print(json.dumps({"arch": name, "artifact_bytes": size, "page_cache": cache, "reads": mode,
                                  "cold_open_ms_p50": round(ts[2], 3), "cold_open_ms_min": round(ts[0], 3),
                                  "artifact_GBps": round(size / ts[2] / 1e6, 2),
                                  "direct_reads": st.get("direct_reads"), "fs_dir": d}), flush=True)


if __name__ == "__main__":
    main()
