"""Request-trace workloads over the model store (BASELINE configs[2] and [4]).

* `pareto_trace` reproduces the reference worker's request stream exactly
  (harness.cpp:294-300, tools/mrm_bench.cpp:107-116): std::mt19937_64(seed),
  libstdc++ uniform_real_distribution over (nextafter(0, 1), 1), and
  bench::pareto_rank (stats_math.cpp:9-17). Pinned against the reference build
  by tests/test_workload.py (golden tests/golden/pareto_trace.json).
* `zipf_trace` is the builder-added FaaS trace (Zipf(s) over model ids,
  seeded numpy Generator); the reference has only Pareto ranks.
* `run_trace` replays a trace through a Store the way the reference's worker
  does (open force-shared -> compute -> close per request) with a GPU compute
  step in place of `touch`: one pass of the block-checksum kernel over the
  resident blob (reads every weight byte once, like touch), then reports the
  fast-tier hit rate, per-request latency percentiles and the harness's
  geomean p95 speedup against a private (no-store) load of each model.
"""
from __future__ import annotations

import ctypes
import math
import time

import numpy as np

from . import format as F
from ._lib import check, lib

_M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the standard 64-bit Mersenne Twister)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _M64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _M64
        self.i = 312

    def __call__(self) -> int:
        if self.i >= 312:
            mt = self.mt
            for k in range(312):
                y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                mt[k] = v
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64


def _canonical(rng: MT19937_64) -> float:
    """libstdc++ generate_canonical<double, 53> over a 64-bit engine."""
    r = float(rng()) / 18446744073709551616.0
    return r if r < 1.0 else math.nextafter(1.0, 0.0)


def pareto_rank(u: float, alpha: float, x_m: float, n: int) -> int:
    """stats_math.cpp:9-17."""
    if not (0.0 < u < 1.0) or not (alpha > 0 and x_m > 0) or n == 0:
        raise ValueError("pareto_rank: bad argument")
    x = x_m / math.pow(u, 1.0 / alpha)
    if x >= float(n):
        return n
    return max(int(math.floor(x)), 1)


def pareto_trace(seed: int, n: int, active: int, alpha: float = 1.0, x_m: float = 1.0) -> list[int]:
    """Model indices (0-based) of the reference worker's request stream."""
    rng = MT19937_64(seed)
    lo = math.nextafter(0.0, 1.0)
    out = []
    for _ in range(n):
        u = _canonical(rng) * (1.0 - lo) + lo
        out.append(pareto_rank(u, alpha, x_m, active) - 1)
    return out


def zipf_trace(seed: int, n: int, n_models: int, s: float = 1.1) -> list[int]:
    """Zipf(s) over model ids 0..n_models-1 (id 0 most popular), seeded."""
    w = 1.0 / np.arange(1, n_models + 1, dtype=np.float64) ** s
    return [int(i) for i in np.random.default_rng(seed).choice(n_models, size=n, p=w / w.sum())]


def percentile(xs, p: float) -> float:
    """Nearest rank, stats_math.cpp:19-27."""
    v = sorted(xs)
    k = max(1, int(math.ceil(p / 100.0 * len(v))))
    return v[k - 1]


class DeviceTouch:
    """The GPU compute step of a catalog request: the block checksum of the
    resident blob (every weight byte read once, as Client::touch does)."""

    def __init__(self, device: int = 0):
        import torch
        self.torch = torch
        self.out = torch.zeros(1, dtype=torch.int64, device=f"cuda:{device}")
        self.host = torch.zeros(1, dtype=torch.int64).pin_memory()
        # a stream of its own: concurrent workers (grid.py threads) must not
        # queue behind each other's kernels and synchronisations on one stream
        self.stream = torch.cuda.Stream(device)

    def __call__(self, dev_ptr: int, nbytes: int) -> int:
        with self.torch.cuda.stream(self.stream):
            self.out.zero_()
            check(lib.trims_checksum_device(ctypes.c_void_p(dev_ptr), nbytes, 0,
                                            ctypes.c_void_p(self.out.data_ptr()),
                                            ctypes.c_void_p(self.stream.cuda_stream)))
            self.host.copy_(self.out, non_blocking=True)
        self.stream.synchronize()  # the request includes the kernel
        return int(self.host.item()) & _M64


def run_trace(store, keys: list[F.ModelKey], trace: list[int], device: int = 0, private_baseline: dict | None = None,
              warmup: int = 0) -> dict:
    """Replay `trace` (indices into keys) through `store`; returns hit rate,
    latency percentiles (ms) and, with `private_baseline` (key -> seconds of a
    private load + compute), the harness's geomean p95 speedup
    (harness.cpp:508-521)."""
    touch = DeviceTouch(device)
    st0 = store.stats()
    per_model: dict[int, list[float]] = {}
    lat = []
    outcomes = [0] * 5
    for j, m in enumerate(trace):
        t0 = time.perf_counter()
        ex = store.open(keys[m])
        touch(ex.dev_ptr, ex.resident_blob_bytes)
        store.close(keys[m])
        dt = time.perf_counter() - t0
        if j < warmup:
            continue
        lat.append(dt)
        per_model.setdefault(m, []).append(dt)
        outcomes[ex.outcome] += 1
    st = store.stats()
    hits = st["tiers"][0]["hits"] - st0["tiers"][0]["hits"]
    misses = st["tiers"][0]["misses"] - st0["tiers"][0]["misses"]
    out = {"requests": len(lat), "fast_hit_rate": round(hits / max(1, hits + misses), 4),
           "outcomes": {"fast_hit": outcomes[0], "host_hit": outcomes[1], "disk_load": outcomes[2],
                        "peer_hit": outcomes[4]},
           "evictions": st["tiers"][0]["evictions"] - st0["tiers"][0]["evictions"],
           "p50_ms": round(percentile(lat, 50) * 1e3, 3), "p99_ms": round(percentile(lat, 99) * 1e3, 3),
           "mean_ms": round(float(np.mean(lat)) * 1e3, 3)}
    if private_baseline:
        sp = [private_baseline[keys[m]] / percentile(v, 95) for m, v in per_model.items() if keys[m] in private_baseline]
        out["geomean_p95_speedup_vs_private"] = round(float(np.exp(np.mean(np.log(sp)))), 3) if sp else None
    return out
