"""The wire-protocol daemon and its client transport.

``serve(store, endpoint)`` runs the reference mrmd's serving loop
(proj/src/daemon.cpp:398-560) natively (csrc/server.cu) over a ``Store``: the
reference's frozen v1 frames (proj/src/wire_protocol.cpp) on a Unix or TCP
socket, one thread per connection, handles auto-closed on disconnect.

``RemoteStore(endpoint)`` is the client side of that socket
(proj/src/client.cpp:243-336 with the reference FramedSocket's lockstep
request/reply): it offers the ``Store`` surface ``Client`` uses (open / close /
stats), so ``Client(RemoteStore(path))`` serves from another process's HBM
copy. Frames are encoded and decoded by the library's C++ codec; the exported
allocation's fd arrives with the OpenResponse (SCM_RIGHTS) and the token
carries its CUDA coordinates.
"""
from __future__ import annotations

import ctypes
import os
import socket
import struct
from dataclasses import dataclass, field

from . import format as F
from ._lib import Errc, TrimsError, check, lib

MAX_FRAME = 16 << 20
_ERRC_NAMES = {1: "NotFound", 2: "TooLargeForFast", 3: "NoEvictableSpace", 4: "NotOpen", 5: "Corrupt",
               6: "ProtocolError", 7: "Internal"}


def encode(text: str) -> bytes:
    """One message (text form, csrc/wire.hpp) -> v1 frame bytes."""
    buf = ctypes.create_string_buffer(1 << 20)
    n = ctypes.c_uint64()
    check(lib.trims_wire_encode_text(text.encode(), buf, len(buf), ctypes.byref(n)))
    return buf.raw[: n.value]


def decode(frame: bytes) -> str:
    """v1 frame bytes -> text form; raises TrimsError with the decoder's code."""
    out = ctypes.create_string_buffer(max(1 << 16, 4 * len(frame)))
    check(lib.trims_wire_decode_text(frame, len(frame), out, len(out)))
    return out.value.decode()


def esc(s: str) -> str:
    o = "".join(c if " " < c < "\x7f" and c != "%" else "".join(f"%{b:02X}" for b in c.encode()) for c in s)
    return o or "%"


def unesc(s: str) -> str:
    if s == "%":
        return ""
    raw, i = bytearray(), 0
    while i < len(s):
        if s[i] == "%" and i + 2 < len(s):
            raw.append(int(s[i + 1:i + 3], 16))
            i += 3
        else:
            raw += s[i].encode()
            i += 1
    return raw.decode()


class Server:
    """A running daemon over ``store`` at ``endpoint`` ("unix:<path>", a bare
    path, or "tcp:<ipv4>:<port>")."""

    def __init__(self, store, endpoint: str):
        self.store = store
        self.endpoint = endpoint
        self._h = ctypes.c_void_p()
        check(lib.trims_server_start(store._h, endpoint.encode(), ctypes.byref(self._h)))

    def frames_served(self) -> int:
        return lib.trims_server_frames_served(self._h) if self._h else 0

    def stop(self) -> None:
        if self._h:
            lib.trims_server_stop(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.stop()

    def __del__(self):
        try:
            self.stop()
        except Exception:
            pass


def serve(store, endpoint: str) -> Server:
    return Server(store, endpoint)


@dataclass
class RemoteExport:
    """An OpenResponse as ``Client.open_shared`` consumes it (the fields of the
    in-process ``Export`` it needs), plus the wire handle."""
    model_id: int
    handle_id: int
    generation: int
    token: str
    device: int
    alloc_bytes: int
    segment_offset: int
    payload_bytes: int
    manifest_digest: bytes
    fd: int
    weights_bytes: int
    workspace_bytes: int
    objects: list = field(default_factory=list)  # (name, offset, length) over the resident blob
    outcome: int = -1  # not on the v1 wire
    remote: bool = True


def parse_token(token: str) -> dict:
    base, _, q = token.partition("?")
    kv = dict(p.split("=", 1) for p in q.split("&") if "=" in p)
    return {"base": base, "device": int(kv["dev"]), "alloc_bytes": int(kv["alloc"]),
            "segment_offset": int(kv["seg"]), "payload_bytes": int(kv["payload"])}


class RemoteStore:
    """Client transport to a daemon: lockstep frames on one connection
    (client.hpp:131), the ``Store`` surface for ``Client``."""

    def __init__(self, endpoint: str, client_id: int = 0):
        self.endpoint = endpoint
        self.client_id = client_id
        if endpoint.startswith("tcp:"):
            host, port = endpoint[4:].rsplit(":", 1)
            self.sock = socket.create_connection((host, int(port)))
            self.unix = False
        else:
            path = endpoint[5:] if endpoint.startswith("unix:") else endpoint
            self.sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            self.sock.connect(path)
            self.unix = True
        self.handles: dict[tuple, list] = {}  # key -> [(model_id, handle_id)]

    # -- framing
    def _recv_exact(self, n: int, fds: list) -> bytes:
        out = bytearray()
        while len(out) < n:
            if self.unix:
                data, anc, _, _ = self.sock.recvmsg(n - len(out), socket.CMSG_SPACE(4))
                for level, typ, payload in anc:
                    if level == socket.SOL_SOCKET and typ == socket.SCM_RIGHTS:
                        fds += list(struct.unpack(f"{len(payload) // 4}i", payload[: len(payload) // 4 * 4]))
            else:
                data = self.sock.recv(n - len(out))
            if not data:
                raise TrimsError(Errc.ConnectionLost, "ConnectionLost", "daemon closed the connection")
            out += data
        return bytes(out)

    def request(self, text: str) -> tuple[str, int]:
        """Send one message, return (reply text, received fd or -1)."""
        self.sock.sendall(encode(text))
        fds: list[int] = []
        head = self._recv_exact(5, fds)
        n = int.from_bytes(head[:4], "little")
        if n > MAX_FRAME:
            raise TrimsError(Errc.ProtocolError, "FrameTooLarge", str(n))
        body = self._recv_exact(n, fds) if n else b""
        fd = fds.pop(0) if fds else -1
        for extra in fds:
            os.close(extra)
        reply = decode(head + body)
        if reply.startswith("error "):
            if fd >= 0:
                os.close(fd)
            _, code, detail = reply.split(" ", 2)
            code = int(code)
            raise TrimsError(code, _ERRC_NAMES.get(code, "Error"), unesc(detail))
        return reply, fd

    # -- Store surface (client.cpp:243-336)
    def open(self, key: F.ModelKey, granularity: int = F.MODEL, block_bytes: int = 2 << 20) -> RemoteExport:
        blk = block_bytes if granularity == F.BLOCK else 0
        reply, fd = self.request(f"open 1 {esc(key.ns)} {esc(key.name)} {esc(key.version)} {granularity} {blk} "
                                 f"{self.client_id}")
        t = reply.split()
        assert t[0] == "openresp", reply
        model_id, handle_id, wb, wsb, _tot, nobj = (int(x) for x in t[1:7])
        objs, at = [], 7
        for _ in range(nobj):
            name, token, gen, off, ln = t[at:at + 5]
            objs.append((unesc(name), unesc(token), int(gen), int(off), int(ln)))
            at += 5
        digest = bytes.fromhex(t[at])
        if not objs:
            raise TrimsError(Errc.ProtocolError, "ProtocolError", "OpenResponse without objects")
        tok = parse_token(objs[0][1])
        self.handles.setdefault((key.ns, key.name, key.version), []).append((model_id, handle_id))
        return RemoteExport(model_id, handle_id, objs[0][2], tok["base"], tok["device"], tok["alloc_bytes"],
                            tok["segment_offset"], tok["payload_bytes"], digest, fd, wb, wsb,
                            [(o[0], o[3], o[4]) for o in objs])

    def close(self, key: F.ModelKey) -> int:
        hs = self.handles.get((key.ns, key.name, key.version))
        if not hs:
            raise TrimsError(Errc.NotOpen, "NotOpen", f"{key} has no open handle on this connection")
        model_id, handle_id = hs.pop()
        reply, _ = self.request(f"close 1 {model_id} {handle_id}")
        return int(reply.split()[2])

    def stats(self) -> dict:
        reply, _ = self.request("stats 1")
        t = reply.split()[1:]
        tiers = [dict(zip(("hits", "misses", "evictions", "used_bytes", "capacity_bytes"),
                          (int(x) for x in t[5 * i:5 * i + 5]))) for i in range(4)]
        at = 20
        n = int(t[at])
        at += 1
        models = []
        for _ in range(n):
            ns, name, ver, rc, uc, res = t[at:at + 6]
            models.append({"key": f"{unesc(ns)}/{unesc(name)}@{unesc(ver)}", "refcount": int(rc),
                           "use_count": int(uc), "residency": int(res)})
            at += 6
        names = ("open_requests", "open_errors", "disk_reads", "remote_fetches", "fetch_ns", "disk_read_ns",
                 "copy_ns", "export_ns")
        out = {"tiers": tiers, "models": models}
        out.update({k: int(v) for k, v in zip(names, t[at:at + 8])})
        at += 8
        if at < len(t):  # wire_protocol.hpp StatsResponse tail: headroom, calibration
            out["workspace_headroom"] = float(t[at])
            out["has_calibration"] = t[at + 1] == "1"
            if out["has_calibration"]:
                out.update(zip(("calib_q", "calib_o", "calib_s"), (float(x) for x in t[at + 2:at + 5])))
        return out

    def close_connection(self) -> None:
        self.sock.close()


def main(argv=None) -> int:
    """``python -m paper_1811_09732_b200.daemon`` — the mrmd entry point
    (proj/tools/mrmd.cpp:35-136): a store on one GPU served on an endpoint
    until SIGINT/SIGTERM; SIGUSR1 prints the stats."""
    import argparse
    import json
    import signal
    import threading

    from .store import Store, StoreOptions, default_cache_dir
    ap = argparse.ArgumentParser(description=main.__doc__)
    ap.add_argument("--listen", default="unix:/tmp/trims-mrmd.sock")
    ap.add_argument("--disk-cache", default=default_cache_dir())
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--fast-capacity", type=int, default=8 << 30)
    ap.add_argument("--host-capacity", type=int, default=16 << 30)
    ap.add_argument("--disk-capacity", type=int, default=256 << 30)
    ap.add_argument("--policy", choices=["lru", "lcu"], default="lru")
    ap.add_argument("--convert-to", default="bf16", help="resident dtype of floating tensors ('' keeps them)")
    ap.add_argument("--no-permute", action="store_true", help="keep 4-D filters KCRS")
    ap.add_argument("--eager-reclaim", action="store_true")
    ap.add_argument("--full-verify", action="store_true", help="verify the blob SHA-256 on every disk load")
    ap.add_argument("--remote", default=None, help="remote store: http://host[:port][/prefix] or dir:<path>")
    a = ap.parse_args(argv)
    opts = StoreOptions(disk_cache_dir=a.disk_cache, fast_capacity_bytes=a.fast_capacity,
                        host_capacity_bytes=a.host_capacity, disk_capacity_bytes=a.disk_capacity,
                        policy=0 if a.policy == "lru" else 1, device=a.device,
                        convert_to=a.convert_to or None, permute_4d=not a.no_permute,
                        eager_reclaim=a.eager_reclaim, scan_disk=True, full_verify=a.full_verify,
                        remote_url=a.remote)
    stop = threading.Event()
    with Store(opts) as s, serve(s, a.listen):
        signal.signal(signal.SIGINT, lambda *_: stop.set())
        signal.signal(signal.SIGTERM, lambda *_: stop.set())
        signal.signal(signal.SIGUSR1, lambda *_: print(json.dumps(s.stats()), flush=True))
        print(f"mrmd: serving {a.disk_cache} on {a.listen} (device {a.device})", flush=True)
        stop.wait()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
