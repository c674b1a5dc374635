"""CPU oracle for the TrIMS load-and-serve path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline. The product package ``paper_1811_09732_b200`` never
imports it (tests/test_boundary.py greps for that).

Two layers:

* ``port``  — ``oracle/_ref/libtrims_oracle.so`` built from ``trims_oracle.c``:
  our C restatement of the reference's byte/integer algorithms (each function
  cites the reference file:line) plus the definitions of the new transforms.
  ``oracle.simulator`` is the Python restatement of the decision simulator.
* ``ref``   — ``oracle/_ref/libmrm_ref.so``: the UNMODIFIED reference compiled
  from /root/reference/proj by ``oracle/Makefile`` with ``ref_shim.cpp`` as its
  driver. Present wherever it was built (it travels to the GPU box as a built
  artefact); used to pin the port and, in bench.py, as the reference arm.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
PORT_SO = os.path.join(REF_DIR, "libtrims_oracle.so")
REF_SO = os.path.join(REF_DIR, "libmrm_ref.so")

_u8p = ctypes.POINTER(ctypes.c_uint8)


def _as_u8(data) -> np.ndarray:
    if isinstance(data, (bytes, bytearray, memoryview)):
        return np.frombuffer(data, np.uint8) if len(data) else np.zeros(0, np.uint8)
    return np.ascontiguousarray(data).view(np.uint8).reshape(-1)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build(ref: bool | None = None) -> None:
    """Compile the C port (always) and the reference (when /root/reference exists)."""
    targets = ["port"]
    if ref or (ref is None and os.path.isdir("/root/reference/proj")):
        targets.append("ref")
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_1811_09732_b200", "libtrims.so")):
            targets.append("integration")  # reference CacheCore over the B200 backend
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _load(path: str) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return ctypes.CDLL(path)


class _Port:
    def __init__(self) -> None:
        L = _load(PORT_SO)
        L.tro_sha256.argtypes = [ctypes.c_void_p, ctypes.c_uint64, _u8p]
        L.tro_fnv1a_str.argtypes = [ctypes.c_char_p]
        L.tro_fnv1a_str.restype = ctypes.c_uint64
        L.tro_splitmix_at.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.tro_splitmix_at.restype = ctypes.c_uint64
        L.tro_splitmix_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        L.tro_catalog_stream.argtypes = [ctypes.c_uint64, ctypes.c_char_p]
        L.tro_catalog_stream.restype = ctypes.c_uint64
        L.tro_touch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64]
        L.tro_touch.restype = ctypes.c_uint64
        L.tro_share_benefit.argtypes = [ctypes.c_double] * 5
        L.tro_share_benefit.restype = ctypes.c_double
        for fn in ("tro_f32_to_bf16", "tro_f64_to_f32", "tro_f64_to_bf16", "tro_f16_to_f32"):
            getattr(L, fn).argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        L.tro_permute_kcrs_krsc.argtypes = [ctypes.c_void_p] + [ctypes.c_uint64] * 5 + [ctypes.c_void_p]
        L.tro_block_checksum.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64]
        L.tro_block_checksum.restype = ctypes.c_uint64
        L.tro_uniform_fill_f32.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_float, ctypes.c_float, ctypes.c_void_p]
        self.L = L

    # -- reference restatements
    def sha256(self, data) -> bytes:
        arr = _as_u8(data)
        out = (ctypes.c_uint8 * 32)()
        self.L.tro_sha256(arr.ctypes.data, arr.size, out)
        return bytes(out)

    def fnv1a(self, s: str) -> int:
        return self.L.tro_fnv1a_str(s.encode())

    def catalog_stream(self, seed: int, name: str) -> int:
        return self.L.tro_catalog_stream(seed, name.encode())

    def splitmix(self, stream: int, k0: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.L.tro_splitmix_fill(stream, k0, n, out.ctypes.data)
        return out

    def touch(self, blob: np.ndarray, offsets, nbytes) -> int:
        blob = np.ascontiguousarray(blob, np.uint8)
        o = np.ascontiguousarray(offsets, np.uint64)
        n = np.ascontiguousarray(nbytes, np.uint64)
        return self.L.tro_touch(blob.ctypes.data, o.ctypes.data, n.ctypes.data, o.size)

    def share_benefit(self, b, n, q, o, s) -> float:
        return self.L.tro_share_benefit(b, n, q, o, s)

    # -- new transforms (our definitions)
    def f32_to_bf16(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(x.size, np.uint16)
        self.L.tro_f32_to_bf16(x.ctypes.data, x.size, out.ctypes.data)
        return out.reshape(x.shape)

    def f64_to_f32(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(x.size, np.float32)
        self.L.tro_f64_to_f32(x.ctypes.data, x.size, out.ctypes.data)
        return out.reshape(x.shape)

    def f64_to_bf16(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(x.size, np.uint16)
        self.L.tro_f64_to_bf16(x.ctypes.data, x.size, out.ctypes.data)
        return out.reshape(x.shape)

    def f16_to_f32(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.uint16)
        out = np.empty(x.size, np.float32)
        self.L.tro_f16_to_f32(x.ctypes.data, x.size, out.ctypes.data)
        return out.reshape(x.shape)

    def permute_kcrs_krsc(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x)
        K, C, R, S = x.shape
        out = np.empty((K, R, S, C), x.dtype)
        self.L.tro_permute_kcrs_krsc(x.ctypes.data, K, C, R, S, x.itemsize, out.ctypes.data)
        return out

    def block_checksum(self, b, word0: int = 0) -> int:
        arr = _as_u8(b)
        return self.L.tro_block_checksum(arr.ctypes.data, arr.size, word0)

    def uniform_f32(self, stream: int, j0: int, n: int, lo: float, hi: float) -> np.ndarray:
        out = np.empty(n, np.float32)
        self.L.tro_uniform_fill_f32(stream, j0, n, lo, hi, out.ctypes.data)
        return out


class _Ref:
    """ctypes view of oracle/_ref/libmrm_ref.so (the reference, unmodified)."""

    def __init__(self) -> None:
        L = _load(REF_SO)
        L.ref_sha256.argtypes = [ctypes.c_void_p, ctypes.c_uint64, _u8p]
        L.ref_gen_catalog.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p]
        L.ref_catalog_manifest_json.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64]
        L.ref_make_manifest_json.argtypes = [ctypes.c_char_p] * 4 + [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64]
        L.ref_write_model.argtypes = [ctypes.c_char_p] * 5 + [ctypes.c_uint64, ctypes.c_void_p]
        L.ref_read_manifest.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_uint64, _u8p, _u64p]
        L.ref_touch_file.argtypes = [ctypes.c_char_p, _u64p]
        L.ref_layout_for.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64]
        L.ref_replay.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64]
        L.ref_acceptance_specs.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.c_char_p, ctypes.c_uint64]
        L.ref_run_oracle.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, _u64p]
        L.ref_ingest.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        L.ref_latency.argtypes = [ctypes.c_char_p] * 5 + [ctypes.c_int, ctypes.POINTER(ctypes.c_double), _u64p]
        L.ref_pareto_trace.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]
        L.ref_trace.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint32,
                                ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double),
                                _u64p]
        L.ref_ingest_parallel.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        L.ref_wire_encode_text.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_uint64, _u64p]
        L.ref_wire_decode_text.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64]
        L.ref_wire_request.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64]
        L.ref_client_decision.argtypes = [ctypes.c_char_p] * 4 + [ctypes.c_int, ctypes.c_uint64, ctypes.c_int] + \
            [ctypes.c_double] * 3 + [ctypes.c_uint64, ctypes.c_double, ctypes.c_int, ctypes.c_char_p, ctypes.c_uint64,
                                     ctypes.POINTER(ctypes.c_double)]
        L.ref_daemon_start.restype = ctypes.c_void_p
        L.ref_daemon_start.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                       ctypes.c_char_p, ctypes.c_uint64]
        L.ref_daemon_stop.argtypes = [ctypes.c_void_p, _u64p]
        L.ref_worker.argtypes = [ctypes.c_char_p] * 5 + [ctypes.c_uint32, ctypes.c_uint32,
                                                         ctypes.POINTER(ctypes.c_double), _u64p]
        self.L = L

    # wire_protocol.cpp:319-357 through the shim's text form; (rc, value)
    def wire_encode(self, text: str):
        buf = ctypes.create_string_buffer(1 << 20)
        n = ctypes.c_uint64()
        rc = self.L.ref_wire_encode_text(text.encode(), buf, len(buf), ctypes.byref(n))
        return rc, (buf.raw[: n.value] if rc == 0 else None)

    def wire_decode(self, frame: bytes):
        out = ctypes.create_string_buffer(max(1 << 16, 4 * len(frame)))
        rc = self.L.ref_wire_decode_text(frame, len(frame), out, len(out))
        return rc, (out.value.decode() if rc == 0 else None)

    def wire_request(self, endpoint: str, text: str):
        out = ctypes.create_string_buffer(1 << 20)
        rc = self.L.ref_wire_request(endpoint.encode(), text.encode(), out, len(out))
        return rc, (out.value.decode() if rc == 0 else None)

    @staticmethod
    def _check(rc: int, what: str) -> None:
        if rc != 0:
            raise RuntimeError(f"reference {what} failed with code {rc}")

    def sha256(self, data: bytes) -> bytes:
        out = (ctypes.c_uint8 * 32)()
        self.L.ref_sha256(data, len(data), out)
        return bytes(out)

    def gen_catalog(self, catalog: str, out_dir: str, seed: int, only: str | None = None) -> None:
        self._check(self.L.ref_gen_catalog(catalog.encode(), out_dir.encode(), seed,
                                           only.encode() if only else None), "gen_catalog")

    def catalog_manifest_json(self, catalog: str, model: str) -> str:
        buf = ctypes.create_string_buffer(1 << 22)
        self._check(self.L.ref_catalog_manifest_json(catalog.encode(), model.encode(), buf, len(buf)), "catalog_manifest")
        return buf.value.decode()

    @staticmethod
    def _decls(decls) -> bytes:
        return "".join(f"{n} {dt} {','.join(str(d) for d in dims)}\n" for n, dt, dims in decls).encode()

    def make_manifest_json(self, key, decls, workspace: int) -> str:
        buf = ctypes.create_string_buffer(1 << 22)
        self._check(self.L.ref_make_manifest_json(*(k.encode() for k in key), self._decls(decls), workspace,
                                                  buf, len(buf)), "make_manifest")
        return buf.value.decode()

    def write_model(self, path: str, key, decls, workspace: int, data: bytes) -> None:
        arr = np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)
        self._check(self.L.ref_write_model(path.encode(), *(k.encode() for k in key), self._decls(decls),
                                           workspace, arr.ctypes.data), "write_model")

    def read_manifest(self, path: str, full_verify: bool = False):
        buf = ctypes.create_string_buffer(1 << 24)
        cs = (ctypes.c_uint8 * 32)()
        bb = ctypes.c_uint64()
        rc = self.L.ref_read_manifest(path.encode(), int(full_verify), buf, len(buf), cs, ctypes.byref(bb))
        if rc != 0:
            return rc, None, None, None
        return 0, buf.value.decode(), bytes(cs), bb.value

    def touch_file(self, path: str) -> int:
        out = ctypes.c_uint64()
        self._check(self.L.ref_touch_file(path.encode(), ctypes.byref(out)), "touch")
        return out.value

    def layout_for(self, path: str, kind: int, block_bytes: int = 2 << 20):
        buf = ctypes.create_string_buffer(1 << 22)
        self._check(self.L.ref_layout_for(path.encode(), kind, block_bytes, buf, len(buf)), "layout_for")
        rows = []
        for line in buf.value.decode().splitlines():
            n, s, o, l = line.split()
            rows.append((n, int(s), int(o), int(l)))
        return rows

    def replay(self, spec: str) -> str:
        buf = ctypes.create_string_buffer(1 << 26)
        self._check(self.L.ref_replay(spec.encode(), buf, len(buf)), "replay")
        return buf.value.decode()

    def replay_into(self, spec: bytes, buf) -> bytes:
        """ref_replay into a caller-owned buffer (no per-call 64 MiB zeroing)."""
        self._check(self.L.ref_replay(spec, buf, len(buf)), "replay")
        return buf.value

    def acceptance_specs(self, seed: int, traces: int, max_models: int, max_ops: int) -> list[str]:
        """The exact trace set run_oracle draws (oracle.cpp:136-211) as replay specs."""
        buf = ctypes.create_string_buffer(1 << 28)
        self._check(self.L.ref_acceptance_specs(seed, traces, max_models, max_ops, buf, len(buf)), "acceptance_specs")
        return [s for s in buf.value.decode().split("end\n") if s]

    def run_oracle(self, traces: int, seed: int, max_models: int, max_ops: int):
        out = (ctypes.c_uint64 * 6)()
        self._check(self.L.ref_run_oracle(traces, seed, max_models, max_ops, out), "run_oracle")
        return tuple(out)

    def ingest(self, path: str, reps: int = 3):
        out = (ctypes.c_double * 3)()
        self._check(self.L.ref_ingest(path.encode(), reps, out), "ingest")
        return {"stage_s": out[0], "publish_s": out[1], "blob_bytes": int(out[2])}

    def ingest_parallel(self, path: str, threads: int, reps: int = 3):
        out = (ctypes.c_double * 2)()
        rc = self.L.ref_ingest_parallel(path.encode(), threads, reps, out)
        return (out[0], int(out[1])) if rc == 0 else (None, 0)

    def latency(self, dir: str, key, mode: str, reps: int = 5):
        out = (ctypes.c_double * 6)()
        t = ctypes.c_uint64()
        self._check(self.L.ref_latency(dir.encode(), *(k.encode() for k in key), mode.encode(), reps, out,
                                       ctypes.byref(t)), "latency")
        names = ("load_disk_s", "init_copy_s", "share_overhead_s", "compute_s", "end_to_end_s", "open_s")
        d = dict(zip(names, list(out)))
        d["touch"] = t.value
        return d

    def pareto_trace(self, seed: int, n: int, alpha: float, x_m: float, active: int) -> list[int]:
        out = (ctypes.c_uint32 * n)()
        self._check(self.L.ref_pareto_trace(seed, n, alpha, x_m, active, out), "pareto_trace")
        return list(out)

    def trace(self, dir: str, names: list[str], trace: list[int], fast: int, host: int, disk: int):
        n = len(trace)
        tr = (ctypes.c_uint32 * n)(*trace)
        out = (ctypes.c_double * n)()
        st = (ctypes.c_uint64 * 5)()
        self._check(self.L.ref_trace(dir.encode(), "\n".join(names).encode(), tr, n, fast, host, disk, out, st),
                    "trace")
        return list(out), dict(zip(("fast_hits", "fast_misses", "fast_evictions", "open_errors", "disk_reads"),
                                   list(st)))

    def client_decision(self, dir: str, key, gran_kind: int, block_bytes: int, params, fast_cap: int,
                        headroom: float, calibrate: bool):
        """Client::open's origin / fallback reason against a reference daemon, + its published calibration."""
        buf = ctypes.create_string_buffer(256)
        st = (ctypes.c_double * 4)()
        q, o, s = params if params else (0.0, 0.0, 0.0)
        self._check(self.L.ref_client_decision(dir.encode(), *(k.encode() for k in key), gran_kind, block_bytes,
                                               int(params is not None), q, o, s, fast_cap, headroom, int(calibrate),
                                               buf, len(buf), st), "client_decision")
        return buf.value.decode(), (bool(st[0]), st[1], st[2], st[3])

    def daemon_start(self, dir: str, fast: int, host: int, disk: int, eager: bool = False) -> tuple:
        """A reference daemon inside this process: (handle, socket path)."""
        buf = ctypes.create_string_buffer(4096)
        h = self.L.ref_daemon_start(dir.encode(), fast, host, disk, int(eager), buf, len(buf))
        if not h:
            raise RuntimeError("ref_daemon_start failed")
        return h, buf.value.decode()

    def daemon_stop(self, h) -> dict:
        st = (ctypes.c_uint64 * 6)()
        self._check(self.L.ref_daemon_stop(h, st), "daemon_stop")
        return dict(zip(("fast_hits", "fast_misses", "fast_evictions", "open_errors", "disk_reads",
                         "fast_used_bytes"), list(st)))

    def worker(self, endpoint: str, dir: str, key, n: int, warmup: int = 1):
        """bench::run_worker's loop on one key: per-request open+touch seconds, last touch."""
        out = (ctypes.c_double * max(n, 1))()
        t = ctypes.c_uint64()
        self._check(self.L.ref_worker(endpoint.encode(), dir.encode(), *(k.encode() for k in key), n, warmup, out,
                                      ctypes.byref(t)), "worker")
        return list(out)[:n], t.value


_port = None
_ref = None


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)
