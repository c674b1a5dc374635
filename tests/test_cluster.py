"""Multi-GPU placement (builder-defined) on CPU:

* the PeerHit step of the product CacheCore ('p' ops through trims_replay)
  equals the simulator restatement (oracle/simulator.py Core.step) on random
  traces;
* simulate_cluster with one rank is the reference simulator exactly (pinned on
  the reference's recorded traces);
* the shared-memory directory (csrc/directory.cpp) across real processes:
  visibility, rendezvous order, retract, and no torn reads under a writer;
* two ranks over gloo, each a real CacheCore + directory (trims_simcore), step
  through one global trace and match simulate_cluster decision for decision.
"""
import ctypes
import multiprocessing as mp
import os
import uuid

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

from oracle import simulator as sim
from paper_1811_09732_b200 import format as F
from paper_1811_09732_b200._lib import check, lib, text_call
from paper_1811_09732_b200.cluster import Directory, peer_score
from tests.golden_data import load


def replay(spec: str) -> list[str]:
    return text_call(lambda o, c: lib.trims_replay(spec.encode(), o, c), cap=1 << 24).splitlines()


def with_peer_ops(rng, trace, frac=0.3):
    return [("p" if k == "o" and rng.random() < frac else k, i) for k, i in trace]


def test_peer_step_matches_simulator():
    rng = np.random.default_rng(2024)
    peer_hits = 0
    for _ in range(40):
        cfg, models, trace = sim.random_trace(rng, max_models=24, max_ops=600)
        trace = with_peer_ops(rng, trace)
        got = replay(sim.spec_text(cfg, models, trace))[:-1]
        events = sim.simulate(cfg, models, trace)
        assert got == [e.line(i, "live") for i, e in enumerate(events)]
        peer_hits += sum(e.outcome == sim.PEER_HIT for e in events)
    assert peer_hits > 100


def test_cluster_of_one_is_the_reference():
    for t in load("decisions.json.gz")[:40]:
        lines = t["spec"].splitlines()
        c = lines[0].split()
        cfg = sim.SimConfig(int(c[1]), int(c[2]), int(c[3]), int(c[4]), c[5] == "1")
        models = [sim.SimModel(int(a), int(b), d == "1", r == "1")
                  for _, a, b, d, r in (l.split() for l in lines if l.startswith("model"))]
        trace = [(0, k, int(i)) for _, k, i in (l.split() for l in lines if l.startswith("op"))]
        got = [ev.line(s, "live") for s, (ev, peer) in enumerate(sim.simulate_cluster(cfg, models, 1, trace))]
        assert got == t["events"]


def test_peer_score_matches_restatement():
    for key in ["trace/m0@1", "zoo/resnet50@1.0.0", "a/b@c"]:
        for r in range(8):
            assert peer_score(key, r) == sim.peer_score(key, r)


# ---------------------------------------------------------------- directory

def _dir_child(name, q, mode, back=None):
    try:
        key = F.ModelKey("zoo", "resnet50", "1.0.0")
        with Directory(name, 3, 1) as d:
            if mode == "publish":
                d.publish(key, device=1, pid=os.getpid(), fd=7, arena=1, alloc_bytes=1 << 30, offset=4096,
                          payload_bytes=1000, resident_blob_bytes=900, generation=5, checksum=77)
                q.put("published")
                back.get()  # wait for the parent to look
                d.retract(key)
                q.put("retracted")
                back.get()
            elif mode == "churn":
                for g in range(1, 20001):
                    d.publish(key, generation=g, checksum=g * 3, payload_bytes=g * 5, resident_blob_bytes=g)
                    if g % 7 == 0:
                        d.retract(key)
                q.put("done")
        q.put("ok")
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(f"error {e!r}")


def test_directory_across_processes():
    name = f"trims.test.{uuid.uuid4().hex[:10]}"
    key = F.ModelKey("zoo", "resnet50", "1.0.0")
    ctx = mp.get_context("spawn")
    q, back = ctx.Queue(), ctx.Queue()
    try:
        with Directory(name, 3, 0) as d0, Directory(name, 3, 2) as d2:
            d2.publish(key, device=2, generation=9, checksum=1, payload_bytes=1000, resident_blob_bytes=900)
            p = ctx.Process(target=_dir_child, args=(name, q, "publish", back))
            p.start()
            assert q.get(timeout=60) == "published"
            hs = d0.holders(key)
            assert [h["rank"] for h in hs] == sorted([1, 2], key=lambda r: -peer_score(str(key), r))
            h1 = next(h for h in hs if h["rank"] == 1)
            assert (h1["device"], h1["pid"], h1["fd"], h1["arena"], h1["offset"], h1["generation"],
                    h1["checksum"]) == (1, p.pid, 7, 1, 4096, 5, 77)
            assert [h["rank"] for h in d2.holders(key)] == [1]  # a rank never lists itself
            back.put("go")
            assert q.get(timeout=60) == "retracted"
            assert [h["rank"] for h in d0.holders(key)] == [2]
            back.put("go")
            assert q.get(timeout=60) == "ok"
            p.join(60)
            # the child's row is cleared when its directory handle closes
            assert [h["rank"] for h in d0.holders(key)] == [2]
            assert d0.holders(F.ModelKey("zoo", "absent", "1")) == []
            with pytest.raises(Exception):
                Directory(name, 4, 0)  # world mismatch with the existing table
    finally:
        Directory.unlink(name)


def test_directory_reads_are_never_torn():
    name = f"trims.test.{uuid.uuid4().hex[:10]}"
    key = F.ModelKey("zoo", "resnet50", "1.0.0")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    try:
        with Directory(name, 3, 0) as d0:
            p = ctx.Process(target=_dir_child, args=(name, q, "churn"))
            p.start()
            seen = 0
            while q.empty():
                for h in d0.holders(key):
                    g = h["generation"]
                    assert (h["checksum"], h["payload_bytes"], h["resident_blob_bytes"]) == (3 * g, 5 * g, g)
                    seen += 1
            assert q.get(timeout=60) == "done"
            assert q.get(timeout=60) == "ok"
            p.join(60)
            assert seen > 0
    finally:
        Directory.unlink(name)


# ------------------------------------------------------------ gloo, world 2

def _cluster_rank(rank, world, port, name, spec, trace, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = ctypes.c_void_p()
    check(lib.trims_simcore_create(spec.encode(), name.encode(), world, rank, ctypes.byref(h)))
    lines = []
    buf = ctypes.create_string_buffer(256)
    for step, (r, kind, i) in enumerate(trace):
        dist.barrier()  # the directory reflects every earlier step of every rank
        if r == rank:
            check(lib.trims_simcore_step(h, kind.encode(), i, step + 1, buf, len(buf)))
            lines.append((step, buf.value.decode()))
    dist.barrier()
    gathered = [None] * world
    dist.all_gather_object(gathered, lines)
    if rank == 0:
        out.put(sorted(x for g in gathered for x in g))
    dist.barrier()
    lib.trims_simcore_destroy(h)
    dist.destroy_process_group()


def test_two_ranks_over_gloo_match_simulate_cluster():
    world = 2
    rng = np.random.default_rng(7)
    cfg, models, trace1 = sim.random_trace(rng, max_models=12, max_ops=300)
    cfg.disk_capacity = 1 << 40  # every rank keeps its artifacts (the peer path reads the local header)
    for m in models:
        m.on_disk = True
    trace = [(int(rng.integers(0, world)), k, i) for k, i in trace1]
    spec = sim.spec_text(cfg, models, [])
    name = f"trims.test.{uuid.uuid4().hex[:10]}"
    ctx = tmp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = 29500 + int(rng.integers(0, 2000))
    try:
        procs = [ctx.Process(target=_cluster_rank, args=(r, world, port, name, spec, trace, q)) for r in range(world)]
        for p in procs:
            p.start()
        got = q.get()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
    finally:
        Directory.unlink(name)
    want = sim.simulate_cluster(cfg, models, world, trace)
    assert len(got) == len(trace)
    for (step, line), (ev, peer) in zip(got, want):
        assert line == f"{ev.outcome} {ev.fast_used} {ev.host_used} {ev.refcount} {peer}", step
    assert sum(ev.outcome == sim.PEER_HIT for ev, _ in want) > 5
