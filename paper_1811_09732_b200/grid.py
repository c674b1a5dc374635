"""The oversubscription grid: the reference's run_grid
(proj/src/bench/harness.cpp:370-544) on the B200 store, extended to N GPUs.

As the reference: per cell (active fraction f of the catalog, c concurrent
workers, N GPU stores) every store's fast tier holds half of the catalog's
weights (harness.cpp:448-452), a daemon serves each store on a Unix socket,
and c worker PROCESSES (posix_spawn'd in the reference, harness.cpp:323-344;
spawned Python processes here) each replay the reference worker's Pareto
request stream over the active models (harness.cpp:275-330: seeds as
harness.cpp:473, `warmup` unrecorded requests first) through their own
client connection: open (force shared) + the GPU compute step over every
weight byte (trims_touch_device) is the recorded latency, close excluded
(harness.cpp:302-313). The stores of a cell share one residency directory, so
a miss on one GPU that another GPU holds is an NVLink PeerHit; worker w talks
to store w % N. Per cell, as the reference: the geomean over models of
(private-load baseline / p95 latency), the mean latency penalty against the
all-resident warm reference (measured through the daemon by one worker, as
harness.cpp:399-431), the fast-tier hit rate and evictions; plus PeerHits.
With one GPU the N stores share it (their NVLink pulls become HBM copies);
the decisions are the same. `mps=True` runs the workers as MPS clients
(sharing.mps_session) so their kernels overlap instead of time-slicing.
"""
from __future__ import annotations

import ctypes
import math
import multiprocessing as mp
import os
import tempfile
import time

import numpy as np

from . import workload as W
from .store import Store, StoreOptions


def _key_tuple(k):
    return (k.ns, k.name, k.version)


def _worker_main(conn, endpoint: str, device: int, keys: list, active: int, n: int, warmup: int, seed: int,
                 alpha: float, mode: str) -> None:
    """One worker process (harness.cpp:275-330). mode "pareto": the Pareto
    stream; mode "warm": every active model once untimed, then 3 timed opens
    each (harness.cpp:412-429)."""
    try:
        from . import format as F
        from ._lib import check, lib
        from .client import SHARED, Client
        from .daemon import RemoteStore
        check(lib.trims_device_init(device))
        cli = Client(RemoteStore(endpoint), device=device)
        mk = [F.ModelKey(*k) for k in keys]
        out = ctypes.c_uint64()

        def request(m: int) -> tuple[float, float, bool]:
            t0 = time.perf_counter()
            v = cli.open(mk[m], force_shared=True)
            t_open = time.perf_counter()
            check(lib.trims_touch_device(device, v.base_ptr, v.blob_bytes(), ctypes.byref(out)))
            t1 = time.perf_counter()
            shared = v.origin == SHARED
            cli.close(v)
            return t1 - t0, t_open - t0, shared

        conn.send(("ready",))
        if conn.recv() != "go":
            return
        rec = []
        if mode == "warm":
            for m in range(active):
                request(m)
                ts = sorted(request(m)[0] for _ in range(3))
                rec.append((m, ts[1], 0.0, True))
        else:
            for i, m in enumerate(W.pareto_trace(seed, warmup + n, active, alpha)):
                total, opn, shared = request(m)
                if i >= warmup:
                    rec.append((m, total, opn, shared))
        conn.send(("done", rec))
    except Exception as e:  # reported to the parent
        conn.send(("error", repr(e)))
    finally:
        conn.close()


def _run_workers(specs: list[tuple], env: dict | None, timeout_s: float = 1800.0) -> list:
    """Spawn one process per spec (endpoint, device, keys, active, n, warmup,
    seed, alpha, mode); start them together; return their records."""
    from .sharing import _child_env
    ctx = mp.get_context("spawn")
    procs, conns = [], []
    with _child_env(env):
        for spec in specs:
            parent, child = ctx.Pipe()
            p = ctx.Process(target=_worker_main, args=(child, *spec), daemon=True)
            p.start()
            procs.append(p)
            conns.append(parent)
    try:
        for c in conns:
            if not c.poll(timeout_s):
                raise TimeoutError("grid worker did not start")
            msg = c.recv()
            if msg[0] != "ready":
                raise RuntimeError(f"grid worker failed: {msg}")
        for c in conns:
            c.send("go")
        recs = []
        for c in conns:
            if not c.poll(timeout_s):
                raise TimeoutError("grid worker did not finish")
            msg = c.recv()
            if msg[0] != "done":
                raise RuntimeError(f"grid worker failed: {msg}")
            recs.append(msg[1])
        return recs
    finally:
        for p in procs:
            p.join(30)
            if p.is_alive():
                p.kill()


def _store_opts(catalog_dir: str, fast: int, host: int, disk: int, device: int, directory=None, rank=0, world=1):
    return StoreOptions(disk_cache_dir=catalog_dir, fast_capacity_bytes=fast, host_capacity_bytes=host,
                        disk_capacity_bytes=disk, device=device, directory=directory, rank=rank, world=world)


def baselines(catalog_dir: str, keys, total_weights: int, device: int = 0, reps: int = 5,
              env: dict | None = None) -> tuple[dict, dict]:
    """Private load + compute per model, median of 5 (harness.cpp:378-396: the
    artifact read from disk, uploaded, touched on the GPU), and the warm
    reference: every model resident, open + compute through the daemon by one
    worker process (harness.cpp:399-431)."""
    import torch

    from . import format as F
    from .daemon import serve
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
    cap = 2 * total_weights + (1 << 20)
    sock = os.path.join(tempfile.mkdtemp(prefix="trims-grid-"), "warm.sock")
    with Store(_store_opts(catalog_dir, cap, cap, total_weights * 8 + (64 << 20), device)) as s:
        with serve(s, f"unix:{sock}"):
            rec = _run_workers([(f"unix:{sock}", device, [_key_tuple(k) for k in keys], len(keys), 0, 0, 0, 1.0,
                                 "warm")], env)[0]
    warm = {keys[m]: t for m, t, _, _ in rec}
    return base, warm


def run_cell(catalog_dir: str, keys, total_weights: int, fraction: float, concurrency: int, world: int,
             base: dict, warm: dict, requests: int = 200, seed: int = 1, alpha: float = 1.0, warmup: int = 10,
             devices: int = 1, tag: str = "grid", env: dict | None = None) -> dict:
    from .daemon import serve
    active = min(len(keys), max(1, math.ceil(fraction * len(keys))))
    dirname = f"trims.{tag}.{os.getpid()}.{int(fraction * 1000)}.{concurrency}.{world}"
    sockdir = tempfile.mkdtemp(prefix="trims-grid-")
    stores, servers = [], []
    errors = []
    recs = []
    try:
        for r in range(world):
            stores.append(Store(_store_opts(catalog_dir, max(total_weights // 2, 1 << 20), total_weights + (1 << 20),
                                            total_weights * 8 + (64 << 20), r % devices,
                                            dirname if world > 1 else None, r, world)))
            servers.append(serve(stores[-1], f"unix:{sockdir}/s{r}.sock"))
        per_worker = max(1, requests // concurrency)
        kt = [_key_tuple(k) for k in keys]
        specs = [(f"unix:{sockdir}/s{wi % world}.sock", stores[wi % world].opts.device, kt, active, per_worker, warmup,
                  seed * 1000003 + int(fraction * 1000) * 131 + wi + 1, alpha, "pareto")  # harness.cpp:473
                 for wi in range(concurrency)]
        try:
            recs = _run_workers(specs, env)
        except Exception as e:  # reported in the cell, as the reference's worker_failed
            errors.append(repr(e))
        st = [s.stats() for s in stores]
    finally:
        for sv in servers:
            sv.stop()
        for s in stores:
            s.close_store()
    lat = [[] for _ in keys]
    opens = []
    for rec in recs:
        for m, total, opn, _shared in rec:
            lat[m].append(total)
            opens.append(opn)
    hits = sum(x["tiers"][0]["hits"] for x in st)
    misses = sum(x["tiers"][0]["misses"] for x in st)
    speed, pen = [], []
    for i, v in enumerate(lat):
        if not v:
            continue
        speed.append(base[keys[i]] / W.percentile(v, 95))
        pen += [x / warm[keys[i]] - 1.0 for x in v]
    n_req = int(sum(len(v) for v in lat))
    return {"fraction": fraction, "concurrency": concurrency, "gpus": world, "active_models": active,
            "ok": not errors and n_req > 0, "error": errors[0] if errors else (None if n_req else "no_samples"),
            "requests": n_req,
            "geomean_p95_speedup": round(float(np.exp(np.mean(np.log(speed)))), 3) if speed else None,
            "mean_latency_penalty_vs_warm": round(float(np.mean(pen)), 3) if pen else None,
            "median_latency_penalty_vs_warm": round(float(np.median(pen)), 3) if pen else None,
            "open_ms_p50": round(W.percentile(opens, 50) * 1e3, 3) if opens else None,
            "fast_hit_rate": round(hits / max(1, hits + misses), 4),
            "evictions": sum(x["tiers"][0]["evictions"] for x in st),
            "peer_hits": sum(x.get("peer_hits", 0) for x in st),
            "disk_reads": sum(x["disk_reads"] for x in st)}


def run_grid(catalog_dir: str, keys, total: int, fractions=(0.25, 0.5, 1.0), concurrencies=(1, 4),
             worlds=(1, 2, 4), requests: int = 200, seed: int = 1, device: int = 0, warmup: int = 10,
             mps: bool = False) -> dict:
    """`total` = the catalog's weight bytes (harness.cpp:372). With `mps` the
    worker processes are MPS clients (when the host has MPS)."""
    import contextlib

    import torch

    from .sharing import mps_session
    devices = max(1, torch.cuda.device_count())
    with (mps_session() if mps else contextlib.nullcontext()) as env:
        base, warm = baselines(catalog_dir, keys, total, device, env=env)
        cells = [run_cell(catalog_dir, keys, total, f, c, n, base, warm, requests, seed, warmup=warmup,
                          devices=devices, env=env)
                 for n in worlds for f in fractions for c in concurrencies]
    return {"catalog_weight_bytes": total, "models": len(keys), "fast_capacity_per_gpu": total // 2,
            "devices": devices, "workers": "processes (one daemon connection each)",
            "mps": bool(mps and env is not None), "requests_per_cell": requests, "warmup_per_worker": warmup,
            "cells": cells}
