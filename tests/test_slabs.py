"""Multi-GPU z-slab logic on CPU (gloo, world_size 2 and 3).

The slab plan, exchange schedule, message layout and the boundary-first /
overlap / join step order (paper_2309_04671_b200.slabs.run_step) are the
same code the GPU path runs; here the per-rank "kernel" is the oracle over
the rank's sub-box and the transport is gloo.  The gathered result must be
bit-identical to the unsplit oracle (SURVEY.md §8(e) test).
"""

from __future__ import annotations

import contextlib
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2309_04671_b200 import corpus
from paper_2309_04671_b200 import GridBuffer, fill_loguniform
from paper_2309_04671_b200.slabs import SlabPlan, exchange_schedule, localize, partition, run_step


def test_partition_even_and_ragged():
    assert partition(1024, 8) == [(128 * r, 128) for r in range(8)]
    assert partition(10, 3) == [(0, 4), (4, 3), (7, 3)]
    with pytest.raises(ValueError):
        partition(2, 3)


def test_exchange_schedule_forms():
    for builder, dst, r in (("star3d4r", "v", 4), ("star3d1r", "v", 1), ("wave", "up", 4), ("jacobi7", "v", 1)):
        bound, _ = corpus.config_target(builder, (16, 16, 16), 1)
        body = bound.stmts[0].body
        sched = exchange_schedule(body)
        assert sched[0] == {dst: r}, builder
        assert sched[1] == {}


def test_boundary_ranges_cover_the_slab_once():
    from paper_2309_04671_b200.slabs import boundary_ranges

    for n in (1, 3, 4, 7, 8, 9, 128):
        for r in (1, 2, 4):
            rng = boundary_ranges(n, r)
            covered = sorted(z for lo, hi in rng for z in range(lo, hi))
            assert covered == list(range(n)), (n, r, rng)
            assert rng[0][0] == 0


def test_messages_land_in_neighbour_halo():
    mid = SlabPlan(30, 3, 1, 4)
    assert mid.messages(4) == [("send", 0, 0, 4), ("recv", 0, -4, 4), ("send", 2, 6, 4), ("recv", 2, 10, 4)]
    assert SlabPlan(30, 3, 0, 4).messages(2) == [("send", 1, 8, 2), ("recv", 1, 10, 2)]


class CpuSlabEngine:
    """Oracle-backed stand-in for DeviceSlabEngine (same run_step driver)."""

    def __init__(self, body, local: dict, plan: SlabPlan):
        self.body, self.state, self.plan = tuple(body), local, plan
        self.sched = exchange_schedule(self.body)
        self.local_body = localize(self.body, plan.start, plan.size)

    def launch(self, i, lo0, hi0):
        if hi0 <= lo0:
            return
        bmap = self.local_body[i]
        m = oracle._Map(bmap, self.state)
        for reg in bmap.regions:
            b = list(reg.bounds)
            b[0] = (max(b[0][0], lo0), min(b[0][1], hi0))
            m.region(tuple(b))

    def swap(self, a, b):
        self.state[a], self.state[b] = self.state[b], self.state[a]

    def view(self, g, z0, n):
        buf = self.state[g]
        o = buf.order
        flat = torch.from_numpy(buf.data.reshape(-1))
        per = int(np.prod(buf.data.shape[1:]))
        return flat[(z0 + o) * per:(z0 + o + n) * per]

    def launch_with_boundary(self, i, r):
        from paper_2309_04671_b200.slabs import boundary_ranges

        for lo, hi in boundary_ranges(self.plan.size, r):
            self.launch(i, lo, hi)
        return None

    def comm_context(self, _):
        return contextlib.nullcontext()

    def join(self, works):
        for w in works:
            w.wait()


def _global_case(builder, shape, steps, width=0):
    bound, decls = corpus.config_target(builder, shape, steps, map_width=width)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    if builder == "wave":
        corpus.wave_inputs(grids)
    else:
        fill_loguniform(grids["u"], 5)
    return bound, grids


def _worker(rank, world, port, builder, shape, steps, outdir, width):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bound, grids = _global_case(builder, shape, steps, width)
        order = next(iter(grids.values())).order
        plan = SlabPlan(shape[0], world, rank, order)
        local = {}
        for n, g in grids.items():
            data = np.ascontiguousarray(g.data[plan.global_slice()])
            local[n] = GridBuffer(g.dtype, (plan.size,) + tuple(shape[1:]), order, data)
        eng = CpuSlabEngine(bound.stmts[0].body, local, plan)
        for _ in range(steps):
            run_step(eng, dist)
        for n, g in eng.state.items():
            np.save(os.path.join(outdir, f"{n}_{rank}.npy"), g.interior)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,builder,shape,steps,width", [
    (2, "star3d4r_norm", (20, 12, 16), 4, 0),
    (3, "star3d2r", (17, 9, 12), 3, 0),
    (2, "wave", (18, 10, 12), 5, 0),
    (3, "jacobi7", (10, 8, 8), 6, 0),
    (2, "star3d4r_norm", (22, 14, 12), 3, 3),  # PML-style regions clipped per slab
])
def test_slab_run_bitwise_equals_unsplit_oracle(world, builder, shape, steps, width):
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), builder, shape, steps, d, width), nprocs=world,
                           join=True, start_method="spawn")
        bound, grids = _global_case(builder, shape, steps, width)
        ref = oracle.run_target(bound, grids)
        for n, g in ref.items():
            parts = [np.load(os.path.join(d, f"{n}_{r}.npy")) for r in range(world)]
            assert np.array_equal(np.concatenate(parts, axis=0), g.interior), n
