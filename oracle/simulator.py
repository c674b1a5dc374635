"""Python restatement of the reference decision simulator — TEST INFRASTRUCTURE ONLY.

Follows proj/src/bench/simulator.cpp:131-254 (and the World helper at :22-120):
naive from-scratch scans per step, greedy policy-order reclaim with an
all-or-nothing feasibility check, LRU by last_access / LCU by use_count with
ties broken by insertion seq. It is the checker for the product CacheCore
(paper_1811_09732_b200/csrc/cache_core.cpp); its own pin is the reference
simulator + live CacheCore run through oracle/_ref (tests/golden/decisions*.json.gz).

Also carries the N>1 extension (builder-defined): per-GPU shards
with a host directory and NVLink peer-serve, which must reduce to the
reference exactly at N=1.
"""
from __future__ import annotations

from dataclasses import dataclass, field

LRU, LCU = 0, 1
FAST_HIT, HOST_HIT, DISK_LOAD, REMOTE_FETCH = 0, 1, 2, 3
PEER_HIT = 4  # N>1 extension only
ERR_NOT_FOUND, ERR_TOO_LARGE, ERR_NO_EVICTABLE, ERR_NOT_OPEN = 100, 101, 102, 103


@dataclass
class SimModel:
    weights_bytes: int
    file_bytes: int
    on_disk: bool = True
    on_remote: bool = False


@dataclass
class SimConfig:
    fast_capacity: int
    host_capacity: int
    disk_capacity: int
    policy: int = LRU
    eager_reclaim: bool = False


@dataclass
class SimEvent:
    outcome: int
    fast_used: int
    host_used: int
    refcount: int
    evicted_fast: list = field(default_factory=list)
    evicted_host: list = field(default_factory=list)
    evicted_disk: list = field(default_factory=list)

    def line(self, step: int, tag: str = "sim") -> str:
        f = lambda v: ",".join(map(str, v)) if v else "-"
        return (f"{tag} {step} {self.outcome} {self.fast_used} {self.host_used} {self.refcount} "
                f"f:{f(self.evicted_fast)} h:{f(self.evicted_host)} d:{f(self.evicted_disk)}")


class _World:
    # simulator.cpp:22-120
    def __init__(self, cfg: SimConfig, models: list[SimModel]):
        self.cfg, self.models = cfg, models
        n = len(models)
        self.has = [False] * n
        self.seq = [0] * n
        self.rc = [0] * n
        self.last = [0] * n
        self.uses = [0] * n
        self.res = [[False] * n for _ in range(3)]  # fast, host, disk
        self.used = [0, 0, 0]
        self.next_seq = 1
        for i, m in enumerate(models):
            if m.on_disk:
                self.has[i] = True
                self.seq[i] = self.next_seq
                self.next_seq += 1
                self.res[2][i] = True
                self.used[2] += m.file_bytes

    def touch_entry(self, i):
        if not self.has[i]:
            self.has[i] = True
            self.seq[i] = self.next_seq
            self.next_seq += 1

    def metric(self, i):
        return self.last[i] if self.cfg.policy == LRU else self.uses[i]

    def bytes(self, tier, i):
        return self.models[i].file_bytes if tier == 2 else self.models[i].weights_bytes

    def cap(self, tier):
        return (self.cfg.fast_capacity, self.cfg.host_capacity, self.cfg.disk_capacity)[tier]

    def evictable(self, tier, i):
        return self.has[i] and self.rc[i] == 0 and self.res[tier][i]

    def pick_victim(self, tier, loading):
        best = -1
        for i in range(len(self.models)):
            if i == loading or not self.evictable(tier, i):
                continue
            if best < 0 or self.metric(i) < self.metric(best) or (
                    self.metric(i) == self.metric(best) and self.seq[i] < self.seq[best]):
                best = i
        return best

    def drop(self, tier, i):
        self.used[tier] -= self.bytes(tier, i)
        self.res[tier][i] = False

    def reclaim(self, tier, need, evicted, loading):
        cap, used = self.cap(tier), self.used[tier]
        free = cap - used if cap > used else 0
        if need <= free:
            return True
        ev = sum(self.bytes(tier, i) for i in range(len(self.models))
                 if i != loading and self.evictable(tier, i))
        if free + ev < need:
            return False
        while free < need:
            v = self.pick_victim(tier, loading)
            free += self.bytes(tier, v)
            self.drop(tier, v)
            evicted.append(v)
        return True


class Core(_World):
    """One store's decision state, stepped one op at a time (simulate() below
    is the reference loop over it). Op kinds: "o" open, "c" close, and the
    multi-GPU extension "p": open with a peer copy available."""

    def step(self, kind: str, i: int, now: int) -> SimEvent:
        cfg, m, w = self.cfg, self.models[i], self
        ev = SimEvent(FAST_HIT, 0, 0, 0)

        def finish():
            ev.fast_used, ev.host_used, ev.refcount = w.used[0], w.used[1], w.rc[i]
            return ev

        if kind == "c":
            if not w.has[i] or w.rc[i] == 0:
                ev.outcome = ERR_NOT_OPEN
                return finish()
            w.rc[i] -= 1
            if cfg.eager_reclaim and w.rc[i] == 0:
                if w.res[0][i]:
                    w.drop(0, i)
                    ev.evicted_fast.append(i)
                if w.res[1][i]:
                    w.drop(1, i)
                    ev.evicted_host.append(i)
            return finish()

        if w.has[i] and w.res[0][i]:
            w.rc[i] += 1
            w.last[i] = now
            w.uses[i] += 1
            ev.outcome = FAST_HIT
            return finish()

        if kind == "p":
            # PeerHit (builder-defined, paper_1811_09732_b200/csrc/cache_core.cpp
            # open_model with a PeerSource): fast-tier admission only; host and
            # disk tiers untouched.
            w.touch_entry(i)
            if m.weights_bytes > cfg.fast_capacity:
                ev.outcome = ERR_TOO_LARGE
                return finish()
            if not w.reclaim(0, m.weights_bytes, ev.evicted_fast, i):
                ev.outcome = ERR_NO_EVICTABLE
                return finish()
            w.used[0] += m.weights_bytes
            w.res[0][i] = True
            w.rc[i] += 1
            w.last[i] = now
            w.uses[i] += 1
            ev.outcome = PEER_HIT
            return finish()

        host_hit = w.has[i] and w.res[1][i]
        fetched = False
        if not host_hit:
            have_disk = w.has[i] and w.res[2][i]
            if not have_disk and not m.on_remote:
                ev.outcome = ERR_NOT_FOUND
                return finish()
            fetched = not have_disk
        w.touch_entry(i)

        temp_file = False
        if fetched:
            if m.file_bytes <= cfg.disk_capacity and w.reclaim(2, m.file_bytes, ev.evicted_disk, i):
                w.res[2][i] = True
                w.used[2] += m.file_bytes
            else:
                temp_file = True

        if m.weights_bytes > cfg.fast_capacity:
            if temp_file:
                ev.evicted_disk.append(i)
            ev.outcome = ERR_TOO_LARGE
            return finish()
        if not w.reclaim(0, m.weights_bytes, ev.evicted_fast, i):
            if temp_file:
                ev.evicted_disk.append(i)
            ev.outcome = ERR_NO_EVICTABLE
            return finish()
        w.used[0] += m.weights_bytes

        staged = False
        if not host_hit and m.weights_bytes <= cfg.host_capacity and \
                w.reclaim(1, m.weights_bytes, ev.evicted_host, i):
            w.used[1] += m.weights_bytes
            staged = True
        if temp_file:
            ev.evicted_disk.append(i)
        w.res[0][i] = True
        if staged:
            w.res[1][i] = True
        w.rc[i] += 1
        w.last[i] = now
        w.uses[i] += 1
        ev.outcome = HOST_HIT if host_hit else (REMOTE_FETCH if fetched else DISK_LOAD)
        return finish()


def simulate(cfg: SimConfig, models: list[SimModel], trace: list[tuple[str, int]]) -> list[SimEvent]:
    """simulator.cpp:131-254. trace items are ("o"|"c", model_index); "p"
    (peer copy available) is the multi-GPU extension."""
    core = Core(cfg, models)
    return [core.step(kind, i, step + 1) for step, (kind, i) in enumerate(trace)]


# --- N > 1 (builder-defined extension) -----------------------

_GOLD = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def _mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _fnv1a(s: str) -> int:
    h = 0xCBF29CE484222325
    for c in s.encode():
        h = ((h ^ c) * 0x100000001B3) & _M64
    return h


def peer_score(key: str, rank: int) -> int:
    """Rendezvous weight of (key, rank) (csrc/directory.cpp:peer_score)."""
    return _mix64(_fnv1a(key) ^ (((rank + 1) * _GOLD) & _M64))


def trace_key(i: int) -> str:
    """Key string of model i in a replay spec (csrc/replay.cpp FakeBackend::key_of)."""
    return f"trace/m{i}@1"


def simulate_cluster(cfg: SimConfig, models: list[SimModel], world: int,
                     trace: list[tuple[int, str, int]]) -> list[tuple[SimEvent, int]]:
    """N stores (one per GPU) sharing a residency directory; trace items are
    (rank, "o"|"c", model). An open at rank r of a model that is not
    fast-resident at r, is fast-resident on another rank, and whose artifact
    is on r's disk tier, is a PeerHit served by the holder with the highest
    peer_score; anything else is the single-store step. Returns (event, peer
    rank or -1) per op. With world == 1 this is simulate() exactly."""
    cores = [Core(cfg, models) for _ in range(world)]
    out = []
    for step, (r, kind, i) in enumerate(trace):
        w = cores[r]
        peer = -1
        if kind == "o" and not (w.has[i] and w.res[0][i]) and w.has[i] and w.res[2][i]:
            holders = [h for h in range(world) if h != r and cores[h].has[i] and cores[h].res[0][i]]
            if holders:
                peer = max(holders, key=lambda h: peer_score(trace_key(i), h))
        ev = w.step("p" if peer >= 0 else kind, i, step + 1)
        if ev.outcome != PEER_HIT:
            peer = -1
        out.append((ev, peer))
    return out


def spec_text(cfg: SimConfig, models: list[SimModel], trace: list[tuple[str, int]]) -> str:
    """The trace spec format shared by oracle/ref_shim.cpp:ref_replay and libtrims' replay."""
    lines = [f"cfg {cfg.fast_capacity} {cfg.host_capacity} {cfg.disk_capacity} {cfg.policy} {int(cfg.eager_reclaim)}"]
    lines += [f"model {m.weights_bytes} {m.file_bytes} {int(m.on_disk)} {int(m.on_remote)}" for m in models]
    lines += [f"op {k} {i}" for k, i in trace]
    return "\n".join(lines) + "\n"


def random_trace(rng, max_models: int = 24, max_ops: int = 600, policy: int | None = None):
    """Our own seeded trace generator (numpy Generator); shaped like the
    reference's random_trace (oracle.cpp:136-196): capacities in 8-byte units,
    ~6% too-large models, disk/remote/both/neither sources, ~2% invalid closes."""
    n = int(rng.integers(1, max_models + 1))
    ops = int(rng.integers(10, max_ops + 1))
    fast = int(rng.integers(64, 4097)) * 8
    host = 0 if rng.integers(0, 100) < 15 else int(rng.integers(64, 4097)) * 8
    pol = int(rng.integers(0, 2)) if policy is None else policy
    eager = bool(rng.integers(0, 100) < 25)
    models, disk_seed = [], 0
    for _ in range(n):
        wb = int(rng.integers(1, 221)) * 8
        if rng.integers(0, 100) < 6:
            wb = fast + 8
        src = int(rng.integers(0, 100))
        m = SimModel(wb, wb + 64, src < 70, 55 <= src < 95)
        if m.on_disk:
            disk_seed += m.file_bytes
        models.append(m)
    disk = disk_seed + int(rng.integers(0, 4096 * 8 + 1))
    cfg = SimConfig(fast, host, disk, pol, eager)
    trace, open_models = [], []
    for _ in range(ops):
        r = int(rng.integers(0, 100))
        if r < 62 or not open_models:
            mi = int(rng.integers(0, n))
            if 60 <= r < 62:
                trace.append(("c", mi))
            else:
                trace.append(("o", mi))
                open_models.append(mi)
        else:
            at = int(rng.integers(0, len(open_models)))
            trace.append(("c", open_models.pop(at)))
    return cfg, models, trace
