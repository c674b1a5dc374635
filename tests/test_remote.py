"""The remote tier (csrc/remote.cpp) against the reference's remote::fetch
(proj/src/remote_store.cpp:58-120): dir: and http:// stores, reuse of a valid
file already in the disk cache, re-fetch of an invalid one, RemoteNotFound for
a missing artifact (HTTP 404), TransportError for transport failures, and
ChecksumMismatch with no file left behind when the download fails its full
verify. CPU only: the fetch is host code (no device calls)."""
import functools
import hashlib
import http.server
import os
import shutil
import threading

import pytest

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200 import remote
from paper_1811_09732_b200._lib import Errc, TrimsError
from tests.golden_data import load

KEY = F.ModelKey("zoo", "alexnet", "1.0.0")
FILE = KEY.filename


@pytest.fixture(scope="module")
def store_dir(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("remote"))
    C.gen_catalog("tiny", os.path.join(d, "models"), seed=1, only=["alexnet", "vgg16"])
    return d


def code(fn):
    with pytest.raises(TrimsError) as ei:
        fn()
    return ei.value.code


def golden_trailer():
    return {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}["alexnet"]["trailer"]


def test_dir_store_fetch_verify_reuse(store_dir, tmp_path):
    dest = str(tmp_path / "cache")
    for url in ("dir:" + os.path.join(store_dir, "models"), os.path.join(store_dir, "models")):
        shutil.rmtree(dest, ignore_errors=True)
        p, n = remote.fetch(url, KEY, dest)
        assert p == os.path.join(dest, FILE) and n == os.path.getsize(p)
        assert F.read_manifest(p, full_verify=True).checksum.hex() == golden_trailer()
        assert os.listdir(dest) == [FILE]  # no .part left
        m0 = os.stat(p).st_mtime_ns
        assert remote.fetch(url, KEY, dest)[0] == p and os.stat(p).st_mtime_ns == m0  # valid: reused
    # an invalid file in the cache is replaced by a fresh download
    with open(p, "r+b") as f:
        f.seek(-40, 2)
        f.write(b"\xff")
    remote.fetch("dir:" + os.path.join(store_dir, "models"), KEY, dest)
    F.read_manifest(p, full_verify=True)


def test_dir_store_errors(store_dir, tmp_path):
    dest = str(tmp_path / "cache")
    assert code(lambda: remote.fetch("dir:" + store_dir, KEY, dest)) == Errc.RemoteNotFound
    bad = tmp_path / "bad"
    bad.mkdir()
    shutil.copy(os.path.join(store_dir, "models", FILE), bad / FILE)
    with open(bad / FILE, "r+b") as f:  # flip a blob byte: the trailer no longer matches
        f.seek(4096)
        b = f.read(1)
        f.seek(4096)
        f.write(bytes([b[0] ^ 1]))
    assert code(lambda: remote.fetch("dir:" + str(bad), KEY, dest)) == Errc.ChecksumMismatch
    assert os.listdir(dest) == []  # the .part was removed, nothing promoted


class _Chunked(http.server.SimpleHTTPRequestHandler):
    """Serves files with Transfer-Encoding: chunked (odd chunk sizes)."""
    protocol_version = "HTTP/1.1"

    def do_GET(self):
        path = self.translate_path(self.path)
        if not os.path.isfile(path):
            self.send_error(404)
            return
        data = open(path, "rb").read()
        self.send_response(200)
        self.send_header("Transfer-Encoding", "chunked")
        self.send_header("Connection", "close")
        self.end_headers()
        for i in range(0, len(data), 99991):
            c = data[i:i + 99991]
            self.wfile.write(b"%x\r\n" % len(c) + c + b"\r\n")
        self.wfile.write(b"0\r\n\r\n")

    def log_message(self, *a):
        pass


class _Quiet(http.server.SimpleHTTPRequestHandler):
    def log_message(self, *a):
        pass


@pytest.fixture(params=["content-length", "chunked"])
def http_store(request, store_dir):
    h = _Quiet if request.param == "content-length" else _Chunked
    srv = http.server.ThreadingHTTPServer(("127.0.0.1", 0), functools.partial(h, directory=store_dir))
    t = threading.Thread(target=srv.serve_forever, daemon=True)
    t.start()
    yield f"http://127.0.0.1:{srv.server_address[1]}"
    srv.shutdown()
    srv.server_close()


def test_http_store(http_store, store_dir, tmp_path):
    dest = str(tmp_path / "cache")
    for url in (http_store + "/models", http_store + "/models/"):
        shutil.rmtree(dest, ignore_errors=True)
        p, n = remote.fetch(url, KEY, dest)
        src = os.path.join(store_dir, "models", FILE)
        assert n == os.path.getsize(src)
        assert hashlib.sha256(open(p, "rb").read()).digest() == hashlib.sha256(open(src, "rb").read()).digest()
        assert os.listdir(dest) == [FILE]
    assert code(lambda: remote.fetch(http_store, KEY, dest + "2")) == Errc.RemoteNotFound  # 404
    assert os.listdir(dest + "2") == []


def test_http_transport_errors(tmp_path):
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()  # nothing listens there now
    assert code(lambda: remote.fetch(f"http://127.0.0.1:{port}/m", KEY, str(tmp_path))) == Errc.TransportError
    assert code(lambda: remote.fetch("http://no-such-host.invalid/m", KEY, str(tmp_path))) == Errc.TransportError
