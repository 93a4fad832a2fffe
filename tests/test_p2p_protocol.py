"""The fused z-slab exchange's ordering protocol, checked on CPU.

`slabs.run_step_p2p` / `DeviceSlabEngine.finish` emit, per rank, a stream of
`stkb_peer_wait(v)`, `stkb_launch_map_pull(map)` and `stkb_peer_signal(v)`
calls (plus host-side swaps).  Here those exact call streams are recorded
from the real functions (with `_lib.call` replaced by a recorder) and
replayed in many random interleavings, one in-order stream per rank, each
kernel an interval [start, end].  Every interleaving must

* never deadlock (a wait is eventually satisfied) — with the real flag encoding: a wait
  for launch v tests one bit of a word that only encodes the last two completions
  (v mod 3), which is sound only while neighbours stay within one launch,
* give each pulling launch c neighbour data exactly as a serial execution
  would (the neighbour's buffer was last written by its launch with the
  same index my own program last wrote it), and
* never overlap a kernel reading a neighbour's buffer with a neighbour
  kernel writing that buffer (no read/write race over NVLink),

and `finish()`'s halo fetch must see the neighbours' final buffers.
"""

from __future__ import annotations

import dataclasses
import random
from types import SimpleNamespace

import pytest

from paper_2309_04671_b200 import _lib, corpus
from paper_2309_04671_b200.front import stmt_kind
from paper_2309_04671_b200.slabs import (DeviceSlabEngine, SlabPlan, d0_read_reach, exchange_schedule,
                                         run_step_p2p, written)


class FakeEngine:
    """The attributes run_step_p2p / finish use, with a host-side binding."""

    def __init__(self, body, plan, names):
        self.body = tuple(body)
        self.plan = plan
        self.sched = exchange_schedule(self.body)
        self.map_index = {}
        for i, s in enumerate(self.body):
            if stmt_kind(s) == "BoundMap":
                self.map_index[i] = len(self.map_index)
        self.maps = [s for s in self.body if stmt_kind(s) == "BoundMap"]
        self.t = 0
        self.launches = 0
        self.peers_connected = True
        self.transport = "p2p"
        self.compute = SimpleNamespace(cuda_stream=1000 + plan.rank)
        self.dt = SimpleNamespace(h=plan.rank, order=4)
        self.names = list(names)
        self.bind = {n: k for k, n in enumerate(self.names)}
        self.ops = []

    def swap(self, a, b):
        self.bind[a], self.bind[b] = self.bind[b], self.bind[a]

    def launch(self, i, lo, hi):  # world == 1 only
        raise AssertionError("single-rank launch in a multi-rank test")

    def record(self, fn, *args):
        if fn == "stkb_peer_wait":
            self.ops.append(("wait", args[2].value))
        elif fn == "stkb_peer_signal":
            self.ops.append(("signal", args[2].value))
        elif fn == "stkb_launch_map_pull":
            m = self.maps[args[1]]
            reads = {self.bind[g] for g, r in d0_read_reach(m).items() if r > 0}
            writes = {self.bind[g] for g in written(m)}
            self.ops.append(("kernel", frozenset(reads), frozenset(writes)))
        elif fn == "stkb_peer_fetch_halo":
            self.ops.append(("fetch",))
        else:
            raise AssertionError(fn)


def record_streams(body, names, world, steps, monkeypatch):
    engines = [FakeEngine(body, SlabPlan(8 * world, world, r, 1), names) for r in range(world)]
    monkeypatch.setattr(_lib, "call", lambda fn, *a: engines[a[0]].record(fn, *a))
    for _ in range(steps):
        for e in engines:
            run_step_p2p(e)
    for e in engines:
        DeviceSlabEngine.finish(e, halo=True)
    return engines


def mask(v, mod=3):
    """stkb200.cu peer_mask: "launch v completed" as the bit pair {v mod 3, (v-1) mod 3}."""
    return (1 << (v % mod)) | (1 << ((v - 1) % mod))


def simulate(engines, rng, mod=3):
    world = len(engines)
    pc = [0] * world  # next op per rank
    flag = [mask(0, mod)] * world  # flag word rank r last wrote into its neighbours (initial: launch 0 done)
    active = {}  # rank -> (reads, writes) of its running kernel
    version = [dict() for _ in range(world)]  # rank -> {buffer: index of its last writing launch}
    launches = [0] * world
    nbrs = [[n for n in (r - 1, r + 1) if 0 <= n < world] for r in range(world)]
    while True:
        moves = []
        for r in range(world):
            if r in active:
                moves.append(("end", r))
                continue
            if pc[r] >= len(engines[r].ops):
                continue
            op = engines[r].ops[pc[r]]
            # stream wait AND: the bit of launch v (only the last two completions are encoded)
            if op[0] == "wait" and not all(flag[n] >> (op[1] % mod) & 1 for n in nbrs[r]):
                continue
            moves.append(("op", r))
        if not moves:
            assert all(pc[r] == len(engines[r].ops) for r in range(world)), "deadlock"
            return
        kind, r = rng.choice(moves)
        if kind == "end":
            reads, writes = active.pop(r)
            for b in writes:
                version[r][b] = launches[r]
            continue
        op = engines[r].ops[pc[r]]
        pc[r] += 1
        if op[0] == "signal":
            flag[r] = mask(op[1], mod)
        elif op[0] == "kernel":
            _, reads, writes = op
            launches[r] += 1
            mine = {b: v for b, v in version[r].items()}
            for n in nbrs[r]:
                for b in reads:
                    # serial semantics: the neighbour has applied exactly the launches I have
                    assert version[n].get(b, 0) == mine.get(b, 0), ("stale or early neighbour data", r, n, b)
                    assert not (n in active and b in active[n][1]), ("read while the neighbour writes", r, n, b)
                if n in active:
                    assert not (writes & active[n][0]), ("write while the neighbour reads", r, n)
            active[r] = (reads, writes)
        elif op[0] == "fetch":
            for n in nbrs[r]:
                assert version[n] == version[r], ("halo fetch before the neighbour finished", r, n)


def _two_map_body():
    bound, decls = corpus.config_target("star3d2r", (16, 16, 16), 1)
    m = bound.stmts[0].body[0]
    flipped = dataclasses.replace(m, grid_args=tuple((p, {"u": "v", "v": "u"}[g]) for p, g in m.grid_args))
    return (m, flipped), list(decls)


@pytest.mark.parametrize("case", ["star", "wave", "jacobi7", "two_maps"])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_p2p_protocol_is_race_free_in_every_interleaving(case, world, monkeypatch):
    if case == "two_maps":
        body, names = _two_map_body()
    else:
        builder = {"star": "star3d4r_norm", "wave": "wave", "jacobi7": "jacobi7"}[case]
        bound, decls = corpus.config_target(builder, (16, 16, 16), 1)
        body, names = bound.stmts[0].body, list(decls)
    engines = record_streams(body, names, world, steps=5, monkeypatch=monkeypatch)
    assert all(e.ops.count(("fetch",)) == 1 for e in engines)
    rng = random.Random(1234 + world)
    for _ in range(300):
        simulate(engines, rng)


def test_protocol_checker_catches_a_missing_wait(monkeypatch):
    """The checker is not vacuous: dropping the waits produces a detected race."""
    bound, decls = corpus.config_target("star3d4r_norm", (16, 16, 16), 1)
    engines = record_streams(bound.stmts[0].body, list(decls), 2, steps=4, monkeypatch=monkeypatch)
    for e in engines:
        e.ops = [op for op in e.ops if op[0] != "wait"]
    rng = random.Random(7)
    with pytest.raises(AssertionError):
        for _ in range(300):
            simulate(engines, rng)


def test_protocol_checker_catches_a_too_short_flag_cycle(monkeypatch):
    """Flags that encode launches mod 2 cannot tell 'one behind' from 'one ahead'."""
    bound, decls = corpus.config_target("star3d4r_norm", (16, 16, 16), 1)
    engines = record_streams(bound.stmts[0].body, list(decls), 3, steps=5, monkeypatch=monkeypatch)
    rng = random.Random(11)
    with pytest.raises(AssertionError):
        for _ in range(300):
            simulate(engines, rng, mod=2)
