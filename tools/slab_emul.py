"""Per-rank cost of the z-slab step on ONE GPU (development estimate, not a bench line).

Runs rank `r` of a `G`-way strong-scaling decomposition of a config with the
real DeviceSlabEngine.  transport nccl: single launch, boundary items first,
SM reservation, signal wait on the exchange stream, but a transport that
moves no bytes.  transport p2p: the fused exchange with the rank wired to
itself as both neighbours (the TMA reads the planes beyond the slab from its
own buffer, through HBM instead of NVLink; the step flags are its own).  Either way the measured step
time is the compute-side critical path of one rank.

    python tools/slab_emul.py c4 8 [steps] [strong|weak] [nccl|p2p]
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2309_04671_b200 import corpus  # noqa: E402
from paper_2309_04671_b200.slabs import DeviceSlabEngine, SlabPlan  # noqa: E402


class NullDist:
    class P2POp:
        def __init__(self, *a, **k):
            pass

    def isend(self, *a):
        pass

    def irecv(self, *a):
        pass

    def batch_isend_irecv(self, ops):
        return []


def main():
    cfg, world = sys.argv[1], int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    weak = len(sys.argv) > 4 and sys.argv[4] == "weak"
    transport = sys.argv[5] if len(sys.argv) > 5 else "p2p"
    builder, shape, dtype, bpp, _ = bench.CONFIGS[cfg]
    if weak:
        shape = (shape[0] * world,) + tuple(shape[1:])
    bound, decls = corpus.config_target(builder, shape, 1, dtype)
    body = bound.stmts[0].body
    order = next(iter(decls.values())).order
    rank = world // 2 if world > 1 else 0
    plan = SlabPlan(shape[0], world, rank, order)
    eng = DeviceSlabEngine(body, decls, plan, device=0, transport=transport)
    if transport == "p2p" and world > 1:
        import ctypes

        from paper_2309_04671_b200 import _lib as L

        bufs = []
        for b in range(len(eng.dt.names)):
            p = ctypes.c_void_p()
            L.call("stkb_buffer_ptr", eng.dt.h, b, ctypes.byref(p))
            bufs.append(p.value)
        f = ctypes.c_void_p()
        L.call("stkb_flags_ptr", eng.dt.h, ctypes.byref(f))
        arr = (ctypes.c_void_p * len(bufs))(*bufs)
        for side in (0, 1):
            L.call("stkb_set_peer", eng.dt.h, side, len(bufs), arr, f, ctypes.c_int64(plan.size))
        eng.peers_connected = True
    local = (plan.size,) + tuple(shape[1:])
    bench.fill_device(eng.dt, list(decls), local, builder)
    d = NullDist()
    eng.run(2 * eng.graph_period() if transport == "p2p" else 3, d)  # warm-up (captures the step graph)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(eng.compute)
    eng.run(steps, d)
    e.record(eng.compute)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    pts = plan.size * shape[1] * shape[2]
    print(json.dumps({"config": cfg, "transport": transport, "scaling": "weak" if weak else "strong", "world": world, "rank": rank, "slab_planes": plan.size, "ms_per_step": round(ms, 4),
                      "rank_gpts": round(pts / ms / 1e6, 1), "implied_job_gpts": round(pts * world / ms / 1e6, 1)}))
    eng.close()


if __name__ == "__main__":
    main()
