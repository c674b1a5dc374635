"""Many client processes serving inference from ONE HBM-resident copy of a
model (BASELINE configs[1]: ResNet-50, 16 concurrent clients sharing one copy
via IPC; the reference's acceptance C4, proj/tests/acceptance.cpp:76-153).

The store process owns the weights (a sealed segment of its cuMem arena). Each
client process receives the arena's POSIX fd over a Unix pipe (SCM_RIGHTS,
what the reference daemon's UDS would carry), maps it read-only
(trims_import_open), validates the segment tail + manifest digest
(trims_import_attach), binds an executor on the shared weights
(trims_net_create) and serves requests with trims_net_forward_host (input
H2D -> CUDA-graph forward -> logits D2H). No weight byte is copied per client.

Clients use only the C ABI through ctypes (no torch), so a client process
costs a CUDA context plus its activation workspace.
"""
from __future__ import annotations

import contextlib
import ctypes
import multiprocessing as mp
import os
import shutil
import subprocess
import tempfile
import time
from dataclasses import dataclass
from multiprocessing.reduction import recv_handle, send_handle

import numpy as np


@dataclass
class SharedModel:
    """What a client needs to attach one exported model (ObjectRef +
    manifest digest of the reference's OpenResponse, wire_protocol.hpp:44-62)."""
    device: int
    alloc_bytes: int
    offset: int
    generation: int
    payload_bytes: int
    digest: bytes
    arch_text: str

    @classmethod
    def from_export(cls, ex, arch_text: str) -> "SharedModel":
        return cls(ex.device, ex.alloc_bytes, ex.segment_offset, ex.generation, ex.payload_bytes,
                   bytes(ex.manifest_digest), arch_text)


def _serve(conn, sm: SharedModel, fd: int, batch: int, n_reqs: int, seed: int, on_exit=None,
           mode: str = "latency") -> None:
    """Attach `fd`'s segment, bind an executor, warm up, then serve n_reqs
    requests on the parent's "go"; reports latencies and the last logits."""
    from ._lib import check, lib
    from .client import import_segment
    try:
        t0 = time.perf_counter()
        imp, ptr, res_json = import_segment(sm.device, fd, sm.alloc_bytes, sm.offset, sm.generation,
                                            sm.payload_bytes, sm.digest)
        net = ctypes.c_void_p()
        from .models import NET_MODES
        check(lib.trims_net_create_ex(sm.device, sm.arch_text.encode(), res_json.encode(), ptr, batch,
                                      NET_MODES[mode], ctypes.byref(net)))
        classes, hw = ctypes.c_int(), ctypes.c_int()
        check(lib.trims_net_buffers(net, None, None, ctypes.byref(classes), ctypes.byref(hw)))
        attach_ms = (time.perf_counter() - t0) * 1e3
        shape_x, shape_y = (batch, 3, hw.value, hw.value), (batch, classes.value)
        pinned = []
        if os.environ.get("TRIMS_CLIENT_PINNED", "1") == "1":  # page-locked request buffers (A/B: =0)
            def host_array(shape):
                n = int(np.prod(shape)) * 4
                p = ctypes.c_void_p()
                check(lib.trims_host_alloc(n, ctypes.byref(p)))
                pinned.append(p)
                return np.ctypeslib.as_array((ctypes.c_float * (n // 4)).from_address(p.value)).reshape(shape)
            x, y = host_array(shape_x), host_array(shape_y)
        else:
            x, y = np.empty(shape_x, np.float32), np.empty(shape_y, np.float32)
        x[...] = np.random.default_rng(seed).standard_normal(shape_x).astype(np.float32)
        check(lib.trims_net_forward_host(net, x.ctypes.data, y.ctypes.data, None, 1))  # warm-up + graph capture
        conn.send(("ready", attach_ms))
        assert conn.recv() == "go"
        lat = []
        t_first = time.perf_counter()
        for _ in range(n_reqs):
            t = time.perf_counter()
            check(lib.trims_net_forward_host(net, x.ctypes.data, y.ctypes.data, None, 1))
            lat.append((time.perf_counter() - t) * 1e3)
        t_last = time.perf_counter()
        conn.send(("done", lat, t_first, t_last, y.copy()))
        for p in pinned:
            lib.trims_host_free(p)
        lib.trims_net_destroy(net)
        lib.trims_import_close(imp)
        if on_exit:
            on_exit()
    except Exception as e:  # reported to the parent
        conn.send(("error", repr(e)))
    finally:
        conn.close()


def _daemon_client_main(conn, endpoint: str, key: tuple, arch_text: str, batch: int, n_reqs: int,
                        seed: int, mode: str = "latency") -> None:
    """A client process of the wire-protocol daemon (daemon.py): opens the
    model over the socket (the allocation fd arrives with the OpenResponse),
    attaches, binds an executor and serves; closes its handle at the end."""
    try:
        from . import format as F
        from ._lib import check, lib
        from .client import import_segment
        from .daemon import RemoteStore
        rs = RemoteStore(endpoint)
        ex = rs.open(F.ModelKey(*key))
        check(lib.trims_device_init(ex.device))
        sm = SharedModel(ex.device, ex.alloc_bytes, ex.segment_offset, ex.generation, ex.payload_bytes,
                         ex.manifest_digest, arch_text)
        _serve(conn, sm, ex.fd, batch, n_reqs, seed, on_exit=lambda: rs.close(F.ModelKey(*key)), mode=mode)
    except Exception as e:
        if not conn.closed:
            conn.send(("error", repr(e)))
            conn.close()


def _client_main(conn, sm: SharedModel, batch: int, n_reqs: int, seed: int) -> None:
    try:
        from ._lib import check, lib
        check(lib.trims_device_init(sm.device))  # context creation is not part of the attach
        _serve(conn, sm, recv_handle(conn), batch, n_reqs, seed)
    except Exception as e:  # reported to the store process
        if not conn.closed:
            conn.send(("error", repr(e)))
            conn.close()


@contextlib.contextmanager
def mps_session():
    """An MPS control daemon for the CLIENT processes (the store process keeps
    its own context): with MPS the clients' kernels share the GPU
    concurrently instead of time-slicing 16 contexts. Yields the environment
    a client needs (pipe / log directories), or None when MPS is not
    available on this host (no nvidia-cuda-mps-control, or it fails to start;
    e.g. a GPU in exclusive-process mode owned by another process)."""
    exe = shutil.which("nvidia-cuda-mps-control")
    if not exe:
        yield None
        return
    root = tempfile.mkdtemp(prefix="trims-mps-")
    env = {"CUDA_MPS_PIPE_DIRECTORY": os.path.join(root, "pipe"), "CUDA_MPS_LOG_DIRECTORY": os.path.join(root, "log")}
    for d in env.values():
        os.makedirs(d, exist_ok=True)
    full = {**os.environ, **env}
    try:
        started = subprocess.run([exe, "-d"], env=full, timeout=30).returncode == 0
    except (OSError, subprocess.SubprocessError):
        started = False
    if not started:
        shutil.rmtree(root, ignore_errors=True)
        yield None
        return
    try:
        yield env
    finally:
        try:
            subprocess.run([exe], input=b"quit\n", env=full, timeout=60)
        except (OSError, subprocess.SubprocessError):
            pass
        shutil.rmtree(root, ignore_errors=True)


@contextlib.contextmanager
def _child_env(env: dict | None):
    """Environment inherited by processes spawned inside the block."""
    saved = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        yield
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def run_daemon_clients(endpoint: str, key, arch_text: str, n_clients: int = 16, n_reqs: int = 20, batch: int = 1,
                       seed: int = 2, timeout_s: float = 600.0, env: dict | None = None,
                       mode: str = "latency") -> dict:
    """As run_clients, but every client process gets the model from the
    daemon at `endpoint` (v1 OpenRequest over the socket, fd by SCM_RIGHTS).
    `env` (e.g. mps_session()'s) is set in the clients' environment; `mode`
    is the clients' executor mode (models.BoundNet)."""
    ctx = mp.get_context("spawn")
    procs, conns = [], []
    with _child_env(env):
        for i in range(n_clients):
            parent, child = ctx.Pipe()
            p = ctx.Process(target=_daemon_client_main,
                            args=(child, endpoint, (key.ns, key.name, key.version), arch_text, batch, n_reqs, seed,
                                  mode),
                            daemon=True)
            p.start()
            procs.append(p)
            conns.append(parent)
    return _collect(procs, conns, n_clients, batch, timeout_s)


def run_clients(sm: SharedModel, fd: int, n_clients: int = 16, n_reqs: int = 20, batch: int = 1,
                seed: int = 2, timeout_s: float = 600.0) -> dict:
    """Spawn `n_clients` processes on the shared model; all start serving at
    once. Returns per-request latency percentiles (ms), aggregate requests/s
    over the common serving window, attach cost, and every client's logits
    of the last request (same input in every client)."""
    ctx = mp.get_context("spawn")
    procs, conns = [], []
    for i in range(n_clients):
        parent, child = ctx.Pipe()
        p = ctx.Process(target=_client_main, args=(child, sm, batch, n_reqs, seed), daemon=True)
        p.start()
        send_handle(parent, fd, p.pid)
        procs.append(p)
        conns.append(parent)
    return _collect(procs, conns, n_clients, batch, timeout_s)


def _collect(procs, conns, n_clients: int, batch: int, timeout_s: float) -> dict:
    try:
        attach = []
        for c in conns:
            if not c.poll(timeout_s):
                raise TimeoutError("client did not become ready")
            msg = c.recv()
            if msg[0] != "ready":
                raise RuntimeError(f"client failed: {msg}")
            attach.append(msg[1])
        for c in conns:
            c.send("go")
        lat, starts, ends, logits = [], [], [], []
        for c in conns:
            if not c.poll(timeout_s):
                raise TimeoutError("client did not finish")
            msg = c.recv()
            if msg[0] != "done":
                raise RuntimeError(f"client failed: {msg}")
            lat += msg[1]
            starts.append(msg[2])
            ends.append(msg[3])
            logits.append(msg[4])
    finally:
        for p in procs:
            p.join(30)
            if p.is_alive():
                p.kill()
    lat.sort()
    pct = lambda q: lat[min(len(lat) - 1, max(0, int(np.ceil(q * len(lat))) - 1))]  # nearest rank
    window = max(ends) - min(starts)
    return {"clients": n_clients, "requests": len(lat), "batch": batch,
            "p50_ms": round(pct(0.50), 3), "p99_ms": round(pct(0.99), 3), "max_ms": round(lat[-1], 3),
            "requests_per_s": round(len(lat) / window, 1),
            "attach_ms_median": round(float(np.median(attach)), 2), "logits": logits}
