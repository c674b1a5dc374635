"""Host logic of the transform's tile scheduler (csrc/ingest.cu build_tiles,
no device needed): the device image covers every logical tile exactly once,
each CTA's bin sits at a fixed stride padded with OP_END, the static bins are
balanced, and the dynamic tail holds the smallest tiles."""
import collections

import pytest

from paper_1811_09732_b200 import catalog as C
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import lib, text_call

OP_END = 255


def schedule(src_json, flags=3, out="bf16", sms=148):
    txt = text_call(lambda o, c: lib.trims_tile_plan_text(src_json.encode(), flags, F.DTYPE_CODE[out], sms, o, c),
                    cap=1 << 26)
    tiles, groups = [], []
    for line in txt.splitlines():
        f = line.split()
        if f[0] == "tile":
            tiles.append(tuple(int(x) for x in f[1:]))
        elif f[0] == "group":
            groups.append({"kind": int(f[1]), "tiles": int(f[2]), "nbins": int(f[3]), "stride": int(f[4]),
                           "tail": int(f[5]), "dev": []})
        else:
            groups[-1]["dev"].append(tuple(int(x) for x in f[1:]))
    return tiles, groups


def cost(t):
    op, src, dst, dbytes, n, tensor = t
    return 8192 + dbytes + n * 4  # kFixed + resident bytes + source bytes (fp32 sources)


@pytest.mark.parametrize("arch,sms", [("resnet50", 148), ("vgg16", 148), ("alexnet", 132), ("resnet50", 7)])
def test_device_image_covers_every_tile_once(arch, sms):
    src_json = C.arch_manifest(C.ARCHS[arch]())
    tiles, groups = schedule(src_json, sms=sms)
    image = [t for g in groups for t in g["dev"] if t[0] != OP_END]
    assert collections.Counter(image) == collections.Counter(tiles)
    for g in groups:
        if g["kind"] != 1:
            continue
        assert g["nbins"] == min(g["tiles"], sms)
        bins = [g["dev"][b * g["stride"]:(b + 1) * g["stride"]] for b in range(g["nbins"])]
        for b in bins:  # real tiles first, then padding only
            real = [t for t in b if t[0] != OP_END]
            assert b[:len(real)] == real and all(t[0] == OP_END for t in b[len(real):])
        tail = g["dev"][g["nbins"] * g["stride"]:]
        assert len(tail) == g["tail"] and all(t[0] != OP_END for t in tail)
        loads = [sum(cost(t) for t in b if t[0] != OP_END) for b in bins]
        biggest = max(cost(t) for t in tiles)
        assert max(loads) - min(loads) <= biggest  # LPT: spread within one tile
        if tail:  # the tail holds the smallest tiles
            assert max(cost(t) for t in tail) <= min(cost(t) for b in bins for t in b if t[0] != OP_END)


def test_identity_plan_has_hash_tiles_only():
    src_json = C.arch_manifest(C.ARCHS["alexnet"]())
    tiles, groups = schedule(src_json, flags=0)
    assert {t[0] for t in tiles} == {0} and all(g["kind"] == 0 and g["nbins"] == 0 for g in groups)
