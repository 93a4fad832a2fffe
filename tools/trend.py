"""Per-segment step time over a long run (thermal/power drift check)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2309_04671_b200 import DeviceTarget, corpus  # noqa: E402

shape = (1024, 1024, 1024)
bound, decls = corpus.config_target("star3d4r_norm", shape, 1)
names = list(decls)
dt = DeviceTarget({n: bench._decl_grid(d) for n, d in decls.items()}, names)
bench.fill_device(dt, names, shape, "star3d4r_norm")
dt.set_program(bound.stmts[0].body)
dt.run(5)
dt.run(2)
dt.sync()
seg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nseg = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = []
with bench.ClockSampler(0) as clk:
    for i in range(nseg):
        dt.run(seg)
        dt.sync()
        out.append(round(dt.elapsed_ms() / seg, 4))
print("ms/step per segment:", out)
print("clocks:", clk.summary())
