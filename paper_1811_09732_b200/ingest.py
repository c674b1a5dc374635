"""Compiled ingest plans (K1..K4) over the C ABI (trims_plan_*).

``publish_fast`` runs these inside the store; this handle exposes the same
pipeline to callers that manage their own buffers (bench, private loads).
"""
from __future__ import annotations

import ctypes
import json

from . import format as F
from ._lib import check, lib, text_call


class IngestPlan:
    def __init__(self, src_json: str, plan_flags: int, out_dtype: str = "bf16", device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        check(lib.trims_plan_create(device, src_json.encode(), plan_flags, F.DTYPE_CODE[out_dtype], ctypes.byref(h)))
        self._h = h
        out = (ctypes.c_uint64 * 8)()
        check(lib.trims_plan_describe(h, out))
        self.tiles, self.buckets, self.read_bytes, self.write_bytes = out[0], out[1], out[2], out[3]
        self.src_bytes, self.resident_bytes, self.chunks, self.pairs = out[4], out[5], out[6], out[7]
        self.resident_json = text_call(lambda o, c: lib.trims_plan_resident_json(h, o, c), cap=1 << 22)

    @property
    def resident(self) -> dict:
        return json.loads(self.resident_json)

    def transform(self, dev_src: int, dev_dst: int, d_sums: int, stream: int | None = None) -> int:
        """HBM raw blob -> resident blob, async on `stream`; returns kernel launches."""
        n = ctypes.c_uint32()
        check(lib.trims_plan_transform(self._h, dev_src, dev_dst, d_sums, stream, ctypes.byref(n)))
        return n.value

    def ingest_host(self, host_blob: int, dev_dst: int):
        """Host raw blob -> resident blob (chunked H2D overlapped with the transform);
        returns (checksum, {h2d_ms, total_ms, read_ms, h2d_bytes, launches})."""
        cs = ctypes.c_uint64()
        st = (ctypes.c_double * 5)()
        check(lib.trims_plan_ingest_host(self._h, host_blob, dev_dst, ctypes.byref(cs), st))
        return cs.value, {"h2d_ms": st[0], "total_ms": st[1], "read_ms": st[2], "h2d_bytes": int(st[3]),
                          "launches": int(st[4])}

    def close(self):
        if self._h:
            lib.trims_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
