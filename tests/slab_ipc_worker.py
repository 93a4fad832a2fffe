"""One rank of the two-process fused-halo-exchange test (test_gpu_slabs.py).

Launched by torch.distributed.run with the gloo backend (only for the IPC
handle exchange and barriers: the halo planes are read by the compute
kernels' TMA straight from the neighbour's buffers).  Both ranks use cuda:0 — CUDA IPC between two
processes on one device — and each writes its final slab to <out>/rank<r>.npz.
"""

import os
import sys

import numpy as np


def main():
    builder, shape, steps, out = sys.argv[1], tuple(int(x) for x in sys.argv[2].split(",")), int(sys.argv[3]), sys.argv[4]
    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2309_04671_b200 import corpus
    from paper_2309_04671_b200 import GridBuffer, fill_loguniform
    from paper_2309_04671_b200 import plan_gpu
    from paper_2309_04671_b200.slabs import SlabPlan, run_slab

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    bound, decls = corpus.config_target(builder, shape, steps)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    if builder == "wave":
        corpus.wave_inputs(grids)
    else:
        fill_loguniform(grids["u"], 9)
    order = next(iter(decls.values())).order
    slab = SlabPlan(shape[0], world, rank, order)
    local = {n: GridBuffer(g.dtype, (slab.size,) + tuple(g.shape[1:]), g.order,
                           np.ascontiguousarray(g.data[slab.global_slice()])) for n, g in grids.items()}
    bmap = bound.stmts[0].body[0]
    plan = plan_gpu(bmap.info, {"template": "unroll", "computeCapability": "10.0"})
    got = run_slab(bound, plan, local, slab, dist, device=0)
    np.savez(os.path.join(out, f"rank{rank}.npz"), **{n: b.data for n, b in got.items()})
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
