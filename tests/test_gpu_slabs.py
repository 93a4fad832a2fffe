"""Device z-slab engine on one B200 (the NCCL transport replaced by a mailbox).

Two (or three) DeviceSlabEngines — the real per-rank GPU objects, with their
compute/comm streams, boundary-first launches, plane spans and swaps — run
on one GPU; a fake ``dist`` pairs each rank's sends with the peer's receives
and performs them as device copies once every rank has posted the step.  No
kernel ever waits on another rank's kernel.  Results are checked against
the unsplit CPU oracle (bitwise for precision="exact").
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle
from paper_2309_04671_b200 import compare, corpus
from paper_2309_04671_b200.grids import GridBuffer, fill_loguniform
from paper_2309_04671_b200.slabs import DeviceSlabEngine, SlabPlan

pytestmark = pytest.mark.gpu


class _Op:
    def __init__(self, fn, tensor, peer, group=None):
        self.fn, self.tensor, self.peer = fn, tensor, peer


class MailboxDist:
    """Collects P2P ops from all simulated ranks; `resolve` performs them."""

    P2POp = _Op

    def __init__(self):
        self.rank = 0
        self.posted = []

    def isend(self, *a):
        raise AssertionError("only batched P2P is used")

    def irecv(self, *a):
        raise AssertionError("only batched P2P is used")

    def batch_isend_irecv(self, ops):
        for op in ops:
            kind = "send" if op.fn == self.isend else "recv"
            self.posted.append((self.rank, kind, op.peer, op.tensor))
        return []

    def resolve(self):
        import torch

        torch.cuda.synchronize()
        sends = {(r, p): t for r, k, p, t in self.posted if k == "send"}
        for r, k, p, t in self.posted:
            if k == "recv":
                t.copy_(sends.pop((p, r)))
        assert not sends
        self.posted.clear()
        torch.cuda.synchronize()


def _case(builder, shape, steps, dtype="f32"):
    bound, decls = corpus.config_target(builder, shape, steps, dtype)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    if builder == "wave":
        corpus.wave_inputs(grids)
    else:
        fill_loguniform(grids["u"], 9)
    return bound, decls, grids


@pytest.mark.parametrize("world,builder,shape,steps,precision", [
    (2, "star3d4r_norm", (40, 36, 140), 6, "fast"),
    (3, "star3d4r", (37, 20, 64), 4, "exact"),
    (2, "wave", (32, 24, 72), 8, "fast"),
    (2, "wave", (24, 16, 40), 4, "exact"),
    (4, "jacobi7", (48, 30, 70), 10, "fast"),
])
def test_device_slabs_match_unsplit_oracle(world, builder, shape, steps, precision):
    bound, decls, grids = _case(builder, shape, steps)
    body = bound.stmts[0].body
    order = next(iter(decls.values())).order
    fake = MailboxDist()
    engines = []
    for r in range(world):
        plan = SlabPlan(shape[0], world, r, order)
        eng = DeviceSlabEngine(body, decls, plan, device=0, precision=precision)
        for n in decls:
            eng.dt.upload(n, np.ascontiguousarray(grids[n].data[plan.global_slice()]))
        engines.append(eng)
    for _ in range(steps):
        for r, eng in enumerate(engines):
            fake.rank = r
            eng.step(fake)
        fake.resolve()
    ref = oracle.run_target_c(bound, grids)
    for n in decls:
        parts = []
        for eng in engines:
            full = eng.dt.download(n)
            o = eng.dt.order
            parts.append(full[o:-o, o:-o, o:-o])
        got = GridBuffer(ref[n].dtype, ref[n].shape, ref[n].order, np.zeros_like(ref[n].data))
        got.interior[...] = np.concatenate(parts, axis=0)
        if precision == "exact":
            assert np.array_equal(got.data, ref[n].data), n
        else:
            assert compare(ref[n], got).max_relative <= 1e-5, (n, compare(ref[n], got).render())
    for eng in engines:
        eng.close()


def test_run_slab_single_rank_matches_run_gpu():
    from paper_2309_04671_b200 import run_gpu
    from paper_2309_04671_b200.planning import plan_gpu
    from paper_2309_04671_b200.slabs import run_slab

    bound, decls, grids = _case("star3d4r_norm", (36, 40, 72), 5)
    bmap = bound.stmts[0].body[0]
    plan = plan_gpu(bmap.info, {"template": "unroll", "computeCapability": "10.0"})
    slab = SlabPlan(36, 1, 0, 4)
    local = {n: GridBuffer(g.dtype, tuple(g.shape), g.order, g.data[slab.global_slice()].copy()) for n, g in grids.items()}
    got = run_slab(bound, plan, local, slab, dist=None, device=0)
    ref = run_gpu(bound, plan, grids, device=0)
    for n in grids:
        assert np.array_equal(got[n].data, ref[n].data), n
