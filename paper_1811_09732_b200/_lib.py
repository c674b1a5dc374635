"""ctypes binding of libtrims.so (include/trims.h).

The library is built in-tree (``make -C paper_1811_09732_b200/csrc``, or
``__graft_entry__.build()``). There is no fallback: importing the package
without it raises, and every device entry point fails loudly on a host
without a CUDA device.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TRIMS_LIB: an A/B variant build of the same library (scripts/ab_transform.sh)
LIB_PATH = os.environ.get("TRIMS_LIB") or os.path.join(HERE, "libtrims.so")


class TrimsError(RuntimeError):
    """A non-zero return of the C ABI; ``code`` is the reference Errc value."""

    def __init__(self, code: int, name: str, detail: str):
        super().__init__(f"{name}({code}): {detail}")
        self.code = code
        self.name = name
        self.detail = detail


# Errc values (proj/include/mrm/error.hpp:11-56), for callers that branch on them.
class Errc:
    NotFound = 1
    TooLargeForFast = 2
    NoEvictableSpace = 3
    NotOpen = 4
    Corrupt = 5
    ProtocolError = 6
    Internal = 7
    LengthMismatch = 100
    BadMagic = 101
    UnsupportedVersion = 102
    CorruptManifest = 103
    ChecksumMismatch = 104
    NoSuchSegment = 112
    StaleGeneration = 113
    NotSealed = 115
    UnknownModel = 120
    RemoteNotFound = 140
    TransportError = 141
    DaemonUnreachable = 150
    ConnectionLost = 151
    InvalidArgument = 160
    CudaError = 170
    OutOfDeviceMemory = 171
    NoDevice = 173


class StoreConfig(ctypes.Structure):
    _fields_ = [
        ("fast_capacity_bytes", ctypes.c_uint64),
        ("host_capacity_bytes", ctypes.c_uint64),
        ("disk_capacity_bytes", ctypes.c_uint64),
        ("policy", ctypes.c_uint32),
        ("eager_reclaim", ctypes.c_uint32),
        ("full_verify", ctypes.c_uint32),
        ("device", ctypes.c_int32),
        ("disk_cache_dir", ctypes.c_char_p),
        ("plan_flags", ctypes.c_uint32),
        ("out_dtype", ctypes.c_uint32),
        ("pinned_pool_bytes", ctypes.c_uint64),
        ("scan_disk", ctypes.c_uint32),
        ("read_threads", ctypes.c_uint32),
        ("arena_bytes", ctypes.c_uint64),
        ("directory", ctypes.c_char_p),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("directory_slots", ctypes.c_uint32),
        ("remote_url", ctypes.c_char_p),
        ("workspace_headroom_fraction", ctypes.c_double),
        ("startup_calibration", ctypes.c_uint32),
        ("direct_io", ctypes.c_uint32),
        ("peer_map", ctypes.c_uint32),
    ]


class DirCoords(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("pid", ctypes.c_int32),
        ("fd", ctypes.c_int32),
        ("arena", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("alloc_bytes", ctypes.c_uint64),
        ("offset", ctypes.c_uint64),
        ("payload_bytes", ctypes.c_uint64),
        ("resident_blob_bytes", ctypes.c_uint64),
        ("generation", ctypes.c_uint64),
        ("checksum", ctypes.c_uint64),
    ]


class Export(ctypes.Structure):
    _fields_ = [
        ("model_id", ctypes.c_uint64),
        ("outcome", ctypes.c_uint32),
        ("device", ctypes.c_int32),
        ("generation", ctypes.c_uint64),
        ("payload_bytes", ctypes.c_uint64),
        ("resident_blob_bytes", ctypes.c_uint64),
        ("alloc_bytes", ctypes.c_uint64),
        ("weights_bytes", ctypes.c_uint64),
        ("workspace_bytes", ctypes.c_uint64),
        ("ingest_checksum", ctypes.c_uint64),
        ("timings_ns", ctypes.c_uint64 * 4),
        ("manifest_digest", ctypes.c_uint8 * 32),
        ("dev_ptr", ctypes.c_void_p),
        ("fd", ctypes.c_int32),
        ("n_objects", ctypes.c_uint32),
        ("token", ctypes.c_char * 160),
        ("segment_offset", ctypes.c_uint64),
    ]


_c = ctypes
_u64 = _c.c_uint64
_u32 = _c.c_uint32
_p = _c.c_void_p
_s = _c.c_char_p

# name -> (restype, argtypes)
_SIGS = {
    "trims_errc_name": (_s, [_c.c_int]),
    "trims_wire_code": (_c.c_int, [_c.c_int]),
    "trims_last_error": (_s, []),
    "trims_device_count": (_c.c_int, []),
    "trims_device_init": (_c.c_int, [_c.c_int]),
    "trims_sha_hw": (_c.c_int, []),
    "trims_sha256": (_c.c_int, [_p, _u64, _p]),
    "trims_read_manifest": (_c.c_int, [_s, _c.c_int, _s, _u64, _p, _c.POINTER(_u64), _c.POINTER(_u64)]),
    "trims_manifest_canonical": (_c.c_int, [_s, _s, _u64]),
    "trims_make_manifest": (_c.c_int, [_s, _s, _s, _s, _u64, _s, _u64]),
    "trims_write_model": (_c.c_int, [_s, _s, _p]),
    "trims_layout_for": (_c.c_int, [_s, _u32, _u64, _s, _u64]),
    "trims_resident_manifest": (_c.c_int, [_s, _u32, _u32, _s, _u64]),
    "trims_fill_splitmix_host": (_c.c_int, [_p, _u64, _u64, _u64]),
    "trims_fill_uniform_host": (_c.c_int, [_p, _u64, _u64, _u64, _c.c_float, _c.c_float]),
    "trims_fnv1a": (_u64, [_s]),
    "trims_touch_host": (_c.c_int, [_p, _s, _c.POINTER(_u64)]),
    "trims_tile_plan_text": (_c.c_int, [_c.c_char_p, _c.c_uint32, _c.c_uint32, _c.c_int, _c.c_char_p, _u64]),
    "trims_server_start": (_c.c_int, [_p, _c.c_char_p, _c.POINTER(_p)]),
    "trims_server_stop": (None, [_p]),
    "trims_server_frames_served": (_u64, [_p]),
    "trims_wire_encode_text": (_c.c_int, [_c.c_char_p, _p, _u64, _c.POINTER(_u64)]),
    "trims_wire_decode_text": (_c.c_int, [_p, _u64, _c.c_char_p, _u64]),
    "trims_checksum_host": (_c.c_int, [_p, _u64, _u64, _c.POINTER(_u64)]),
    "trims_backend_create": (_c.c_int, [_c.POINTER(StoreConfig), _c.POINTER(_p)]),
    "trims_backend_destroy": (None, [_p]),
    "trims_backend_locate": (_c.c_int, [_p, _s, _s, _s, _s, _u64, _c.POINTER(_u64)]),
    "trims_backend_fetch_remote": (_c.c_int, [_p, _s, _s, _s, _s, _u64, _c.POINTER(_u64)]),
    "trims_backend_load_settled": (_c.c_int, [_p, _s, _s, _s]),
    "trims_remote_fetch": (_c.c_int, [_s, _s, _s, _s, _s, _s, _u64, _c.POINTER(_u64)]),
    "trims_backend_read_manifest": (_c.c_int, [_p, _s, _s, _s, _s, _s, _u64, _p]),
    "trims_backend_stage_host": (_c.c_int, [_p, _u64, _s, _p, _s]),
    "trims_backend_publish_fast": (_c.c_int, [_p, _u64, _s, _c.c_int, _s, _c.POINTER(Export)]),
    "trims_backend_evict_fast": (_c.c_int, [_p, _u64]),
    "trims_backend_evict_host": (_c.c_int, [_p, _u64]),
    "trims_backend_evict_disk": (_c.c_int, [_p, _s]),
    "trims_store_create": (_c.c_int, [_c.POINTER(StoreConfig), _c.POINTER(_p)]),
    "trims_store_destroy": (None, [_p]),
    "trims_store_open": (_c.c_int, [_p, _s, _s, _s, _u32, _u64, _c.POINTER(Export)]),
    "trims_store_close": (_c.c_int, [_p, _s, _s, _s, _c.POINTER(_u64)]),
    "trims_store_reclaim": (_c.c_int, [_p, _u32, _u64, _u32, _s, _u64]),
    "trims_store_register_disk_file": (_c.c_int, [_p, _s, _s, _s, _s, _u64]),
    "trims_store_drop_all": (_c.c_int, [_p]),
    "trims_store_stats_json": (_c.c_int, [_p, _s, _u64]),
    "trims_store_resident_json": (_c.c_int, [_p, _u64, _s, _u64]),
    "trims_store_ingest_stats": (_c.c_int, [_p, _u64, _c.POINTER(_c.c_double)]),
    "trims_store_checksums": (_c.c_int, [_p, _u64, _c.POINTER(_u64), _u64, _c.POINTER(_u64)]),
    "trims_store_fast_resident": (_c.c_int, [_p, _s, _s, _s, _c.POINTER(_c.c_int)]),
    "trims_dir_open": (_c.c_int, [_s, _c.c_int, _c.c_int, _u32, _c.POINTER(_p)]),
    "trims_dir_close": (None, [_p]),
    "trims_dir_unlink": (_c.c_int, [_s]),
    "trims_dir_publish": (_c.c_int, [_p, _s, _s, _s, _c.POINTER(DirCoords)]),
    "trims_dir_retract": (_c.c_int, [_p, _s, _s, _s]),
    "trims_dir_holders": (_c.c_int, [_p, _s, _s, _s, _c.POINTER(DirCoords), _u64, _c.POINTER(_u64)]),
    "trims_peer_score": (_u64, [_s, _c.c_int]),
    "trims_simcore_create": (_c.c_int, [_s, _s, _c.c_int, _c.c_int, _c.POINTER(_p)]),
    "trims_simcore_destroy": (None, [_p]),
    "trims_simcore_step": (_c.c_int, [_p, _c.c_char, _u32, _u64, _s, _u64]),
    "trims_import_open": (_c.c_int, [_c.c_int, _c.c_int, _u64, _c.POINTER(_p), _c.POINTER(_p)]),
    "trims_import_attach": (_c.c_int, [_p, _u64, _u64, _u64, _p, _c.POINTER(_p), _s, _u64]),
    "trims_import_read_only": (_c.c_int, [_p]),
    "trims_import_close": (None, [_p]),
    "trims_import_verify": (_c.c_int, [_p, _u64, _u64, _u64, _c.POINTER(_u64)]),
    "trims_ingest_host": (_c.c_int, [_c.c_int, _p, _s, _u32, _u32, _p, _c.POINTER(_u64), _c.POINTER(_c.c_double)]),
    "trims_transform_device": (_c.c_int, [_c.c_int, _p, _s, _u32, _u32, _p, _p, _p]),
    "trims_plan_info": (_c.c_int, [_s, _u32, _u32, _c.POINTER(_u64)]),
    "trims_plan_create": (_c.c_int, [_c.c_int, _s, _u32, _u32, _c.POINTER(_p)]),
    "trims_plan_destroy": (None, [_p]),
    "trims_plan_describe": (_c.c_int, [_p, _c.POINTER(_u64)]),
    "trims_plan_resident_json": (_c.c_int, [_p, _s, _u64]),
    "trims_plan_transform": (_c.c_int, [_p, _p, _p, _p, _p, _c.POINTER(_u32)]),
    "trims_plan_ingest_host": (_c.c_int, [_p, _p, _p, _c.POINTER(_u64), _c.POINTER(_c.c_double)]),
    "trims_checksum_device": (_c.c_int, [_p, _u64, _u64, _p, _p]),
    "trims_touch_device": (_c.c_int, [_c.c_int, _p, _u64, _c.POINTER(_u64)]),
    "trims_fill_splitmix_device": (_c.c_int, [_p, _u64, _u64, _u64, _p]),
    "trims_fill_uniform_device": (_c.c_int, [_p, _u64, _u64, _u64, _c.c_float, _c.c_float, _p]),
    "trims_replay": (_c.c_int, [_s, _s, _u64]),
    "trims_gemm_bf16": (_c.c_int, [_p, _u64, _u64, _u64, _p, _u64, _u64, _p, _u64, _p, _p, _p, _u64, _c.c_int,
                                   _c.c_int, _p]),
    "trims_gemm_bf16_split": (_c.c_int, [_p, _u64, _u64, _u64, _p, _u64, _u64, _p, _u64, _p, _p, _p, _u64,
                                         _c.c_int, _c.c_int, _c.c_int, _p]),
    "trims_gemm_bf16_ex": (_c.c_int, [_p, _u64, _u64, _u64, _p, _u64, _u64, _p, _u64, _p, _p, _p, _u64,
                                      _c.c_int, _c.c_int, _c.c_int, _c.c_int, _p]),
    "trims_host_alloc": (_c.c_int, [_u64, _c.POINTER(_p)]),
    "trims_host_free": (None, [_p]),
    "trims_net_create": (_c.c_int, [_c.c_int, _s, _s, _p, _c.c_int, _c.POINTER(_p)]),
    "trims_net_create_ex": (_c.c_int, [_c.c_int, _s, _s, _p, _c.c_int, _c.c_int, _c.POINTER(_p)]),
    "trims_net_destroy": (None, [_p]),
    "trims_net_buffers": (_c.c_int, [_p, _c.POINTER(_p), _c.POINTER(_p), _c.POINTER(_c.c_int),
                                     _c.POINTER(_c.c_int)]),
    "trims_net_run": (_c.c_int, [_p, _p, _c.c_int]),
    "trims_net_rebind": (_c.c_int, [_p, _p]),
    "trims_net_info": (_c.c_int, [_p, _c.POINTER(_c.c_double)]),
    "trims_net_forward_host": (_c.c_int, [_p, _p, _p, _p, _c.c_int]),
    "trims_store_pin": (_c.c_int, [_p, _u64, _u64, _c.POINTER(_p)]),
    "trims_pin_release": (None, [_p]),
    "trims_lease_acquire": (_c.c_int, [_s, _u64, _u64, _c.POINTER(_p)]),
    "trims_lease_release": (None, [_p]),
    "trims_net_tap": (_c.c_int, [_p, _c.c_int, _c.POINTER(_p), _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)]),
    "trims_softmax": (_c.c_int, [_p, _p, _c.c_int, _c.c_int, _p]),
}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `make -C {os.path.join(HERE, 'csrc')}` "
            "or `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc != 0:
        raise TrimsError(rc, lib.trims_errc_name(rc).decode(), lib.trims_last_error().decode())


_TEXT_BUFS: dict = {}


def text_call(fn, *args, cap: int = 1 << 16) -> str:
    """Call an entry point whose last two args are (char* out, uint64 cap).
    Output buffers are reused per size (allocating and zeroing a fresh
    multi-MiB buffer per call cost more than the call)."""
    import threading
    while True:
        k = (threading.get_ident(), cap)
        buf = _TEXT_BUFS.get(k)
        if buf is None:
            buf = _TEXT_BUFS[k] = ctypes.create_string_buffer(cap)
        rc = fn(*args, buf, cap)
        if rc == Errc.InvalidArgument and b"too small" in lib.trims_last_error() and cap < (1 << 30):
            cap *= 8
            continue
        check(rc)
        return buf.value.decode()


def exported_symbols() -> list[str]:
    return sorted(_SIGS)
