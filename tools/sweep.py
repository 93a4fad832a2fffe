"""Quick device timing sweep (development tool): ms/step and HBM GB/s per config.

    python tools/sweep.py star3d4r_norm:1024,1024,1024:f32 wave:1024,1024,1024:f32 ...
Env STKB_LZ / STKB_CTAS override the work decomposition.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2309_04671_b200 import DeviceTarget, corpus  # noqa: E402


def time_one(builder, shape, dtype, steps=20, warm=3):
    bound, decls = corpus.config_target(builder, shape, steps, dtype)
    names = list(decls)
    body = bound.stmts[0].body
    dt = DeviceTarget({n: bench._decl_grid(d) for n, d in decls.items()}, names)
    bench.fill_device(dt, names, shape, builder)
    dt.set_program(body)
    dt.run(warm)
    dt.run(4)  # graphs and fused-sweep scratch for the timed run's start state
    dt.sync()
    dt.run(steps)
    dt.sync()
    ms = dt.elapsed_ms() / steps
    kind = dt.plans[0].kind
    dt.close()
    bpp = (16 if builder == "wave" else 8) * (2 if dtype == "f64" else 1)  # algorithmic bytes per point
    pts = int(np.prod(shape))
    return dict(builder=builder, shape=shape, dtype=dtype, kind=kind, ms=round(ms, 4),
                gpts=round(pts / ms / 1e6, 1), gbs=round(pts * bpp / ms / 1e6, 1))


if __name__ == "__main__":
    import os

    steps = int(os.environ.get("SWEEP_STEPS", "20"))
    for spec in sys.argv[1:]:
        b, s, d = spec.split(":")
        print(json.dumps(time_one(b, tuple(int(x) for x in s.split(",")), d, steps=steps)), flush=True)
