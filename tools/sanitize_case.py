"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck)."""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2309_04671_b200 import corpus, fill_loguniform, run_gpu  # noqa: E402
from paper_2309_04671_b200 import GridBuffer  # noqa: E402
from paper_2309_04671_b200 import plan_gpu  # noqa: E402


def run(builder, shape, steps, precision="fast"):
    bound, decls = corpus.config_target(builder, shape, steps)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    if builder == "wave":
        corpus.wave_inputs(grids)
    else:
        fill_loguniform(grids["u"], 1)
    bmap = bound.stmts[0].body[0]
    plan = plan_gpu(bmap.info, {"template": "unroll", "computeCapability": "10.0"})
    run_gpu(bound, plan, grids, precision=precision)


if __name__ == "__main__":
    run("star3d4r", (20, 36, 136), 3)
    run("wave", (18, 30, 100), 3)
    run("j3d27pt", (12, 33, 70), 2)
    run("star2d4r", (40, 300), 3)
    run("star3d2r", (10, 12, 40), 2, precision="exact")
    print("sanitize cases ok")
