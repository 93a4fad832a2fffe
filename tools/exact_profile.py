"""Time precision='exact' on one configuration (development tool).

    python tools/exact_profile.py star3d4r_norm 512,512,512 f32 8
Canonical stars and boxes run on the exact streaming kernels (XSTAR / XBOX; 2-D too), other maps
on the bytecode kernel (XP_FORCE_EXPR=1: everything on the bytecode kernel, for comparison).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2309_04671_b200 import DeviceTarget, corpus  # noqa: E402

import os  # noqa: E402

import numpy as np  # noqa: E402

if os.environ.get("XP_FORCE_EXPR") == "1":  # the bytecode kernel, for comparison
    from paper_2309_04671_b200 import matcher  # noqa: E402

    def _no(*a, **k):
        raise matcher.MatchError("forced to the bytecode kernel")

    matcher.match_exact_star = matcher.match_exact_box = matcher.match_exact_wave = _no

builder = sys.argv[1] if len(sys.argv) > 1 else "star3d4r_norm"
shape = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "512,512,512").split(","))
dtype = sys.argv[3] if len(sys.argv) > 3 else "f32"
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
bound, decls = corpus.config_target(builder, shape, steps, dtype)
names = list(decls)
dt = DeviceTarget({n: bench._decl_grid(d) for n, d in decls.items()}, names, precision="exact")
bench.fill_device(dt, names, shape, builder)
dt.set_program(bound.stmts[0].body)
dt.run(2)
dt.run(4)  # the CUDA graph of the step program is captured here, outside the timed run
dt.sync()
dt.run(steps)
dt.sync()
ms = dt.elapsed_ms() / steps
n = int(np.prod(shape))
print(builder, dtype, dt.plans[0].kind, round(ms, 3), "ms/step", round(n / ms / 1e6, 1), "GPts/s")
