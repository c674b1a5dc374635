"""The oversubscription grid: the reference's run_grid
(proj/src/bench/harness.cpp:370-544) on the B200 store, extended to N GPUs.

For every cell (active fraction f of the catalog, c concurrent workers, N
GPU stores) the fast tier of each store holds half of the catalog's weights
(harness.cpp:448-452) and the stores of a cell share one residency directory,
so a miss on one GPU that another GPU holds is an NVLink PeerHit. Each worker
is a thread with its own Client, pinned to store (worker % N), replaying the
reference worker's Pareto request stream over the active models
(harness.cpp:275-300, seeds as harness.cpp:473) — open (force shared), the GPU
compute step over every weight byte, close. Per cell, as the reference: the
geomean over models of (private-load baseline / p95 latency), the mean latency
penalty against an all-resident warm reference, the fast-tier hit rate,
evictions, plus PeerHits. With one GPU the N stores share it (their NVLink
pulls become HBM copies); the decisions are the same.
"""
from __future__ import annotations

import math
import os
import threading
import time

import numpy as np

from . import workload as W
from .client import Client
from .store import Store, StoreOptions


def baselines(catalog_dir: str, keys, total_weights: int, device: int = 0, reps: int = 3) -> tuple[dict, dict]:
    """Private load + compute per model (harness.cpp:378-396) and the warm
    reference: open + compute with every model resident (harness.cpp:399-431)."""
    import torch

    from . import format as F
    touch = W.DeviceTouch(device)
    base = {}
    for k in keys:
        path = os.path.join(catalog_dir, k.filename)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            info = F.read_manifest(path)
            blob = np.fromfile(path, dtype=np.uint8, count=info.blob_bytes, offset=info.blob_offset)
            d = torch.from_numpy(blob).to(f"cuda:{device}")
            torch.cuda.current_stream(device).synchronize()  # the touch runs on its own stream
            touch(d.data_ptr(), d.numel())
            ts.append(time.perf_counter() - t0)
        base[k] = W.percentile(ts, 50)
    warm = {}
    cap = 2 * total_weights + (1 << 20)
    with Store(StoreOptions(disk_cache_dir=catalog_dir, fast_capacity_bytes=cap, host_capacity_bytes=cap,
                            device=device)) as s:
        cli = Client(s)
        for k in keys:
            cli.close(cli.open(k, force_shared=True))
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                v = cli.open(k, force_shared=True)
                touch(v.base_ptr, v.blob_bytes())
                cli.close(v)
                ts.append(time.perf_counter() - t0)
            warm[k] = W.percentile(ts, 50)
    return base, warm


def run_cell(catalog_dir: str, keys, total_weights: int, fraction: float, concurrency: int, world: int,
             base: dict, warm: dict, requests: int = 400, seed: int = 1, alpha: float = 1.0,
             devices: int = 1, tag: str = "grid") -> dict:
    active = min(len(keys), max(1, math.ceil(fraction * len(keys))))
    dirname = f"trims.{tag}.{os.getpid()}.{int(fraction * 1000)}.{concurrency}.{world}"
    stores = []
    try:
        for r in range(world):
            stores.append(Store(StoreOptions(
                disk_cache_dir=catalog_dir, fast_capacity_bytes=max(total_weights // 2, 1 << 20),
                host_capacity_bytes=total_weights + (1 << 20), disk_capacity_bytes=total_weights * 8 + (64 << 20),
                device=r % devices, directory=dirname if world > 1 else None, rank=r, world=world)))
        per_worker = max(1, requests // concurrency)
        lat = [[] for _ in keys]
        errors = []

        def worker(wi: int):
            try:
                store = stores[wi % world]
                cli = Client(store, device=store.opts.device)
                touch = W.DeviceTouch(store.opts.device)
                wseed = seed * 1000003 + int(fraction * 1000) * 131 + wi + 1  # harness.cpp:473
                for m in W.pareto_trace(wseed, per_worker, active, alpha):
                    t0 = time.perf_counter()
                    v = cli.open(keys[m], force_shared=True)
                    touch(v.base_ptr, v.blob_bytes())
                    cli.close(v)
                    lat[m].append(time.perf_counter() - t0)
            except Exception as e:  # reported in the cell
                errors.append(repr(e))

        threads = [threading.Thread(target=worker, args=(wi,)) for wi in range(concurrency)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        st = [s.stats() for s in stores]
    finally:
        for s in stores:
            s.close_store()
    hits = sum(x["tiers"][0]["hits"] for x in st)
    misses = sum(x["tiers"][0]["misses"] for x in st)
    speed, pen = [], []
    for i, v in enumerate(lat):
        if not v:
            continue
        speed.append(base[keys[i]] / W.percentile(v, 95))
        pen += [x / warm[keys[i]] - 1.0 for x in v]
    return {"fraction": fraction, "concurrency": concurrency, "gpus": world, "active_models": active,
            "ok": not errors, "error": errors[0] if errors else None,
            "requests": int(sum(len(v) for v in lat)),
            "geomean_p95_speedup": round(float(np.exp(np.mean(np.log(speed)))), 3) if speed else None,
            "mean_latency_penalty_vs_warm": round(float(np.mean(pen)), 3) if pen else None,
            "fast_hit_rate": round(hits / max(1, hits + misses), 4),
            "evictions": sum(x["tiers"][0]["evictions"] for x in st),
            "peer_hits": sum(x.get("peer_hits", 0) for x in st),
            "disk_reads": sum(x["disk_reads"] for x in st)}


def run_grid(catalog_dir: str, keys, total: int, fractions=(0.25, 0.5, 1.0), concurrencies=(1, 4),
             worlds=(1, 2, 4), requests: int = 400, seed: int = 1, device: int = 0) -> dict:
    """`total` = the catalog's weight bytes (harness.cpp:372)."""
    import torch
    devices = max(1, torch.cuda.device_count())
    base, warm = baselines(catalog_dir, keys, total, device)
    cells = [run_cell(catalog_dir, keys, total, f, c, n, base, warm, requests, seed, devices=devices)
             for n in worlds for f in fractions for c in concurrencies]
    return {"catalog_weight_bytes": total, "models": len(keys), "fast_capacity_per_gpu": total // 2,
            "devices": devices, "cells": cells}
