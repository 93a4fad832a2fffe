"""Randomised parity sweep on the GPU (development tool): random corpus kernel, shape, step
count, dtype and precision against the C oracle — exact bitwise, fast within tolerance.

    python tools/fuzz_parity.py [n_cases] [seed]
"""
from __future__ import annotations

import random
import sys
import traceback
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402
from paper_2309_04671_b200 import GridBuffer, compare, corpus, fill_loguniform, front, plan_gpu, run_gpu  # noqa: E402

TOL = {"f32": 1e-5, "f64": 1e-12}


def main(n: int, seed: int) -> int:
    rng = random.Random(seed)
    names = [k.name for k in front.module("corpus").TABLE_KERNELS] + ["wave", "star3d4r_norm", "jacobi7"]
    bad = 0
    for i in range(n):
        name = rng.choice(names)
        dims = 2 if "2d" in name else 3
        big = rng.random() < 0.3  # several x-tiles / y-tiles / z-chunks
        hi = (48, 64, 300) if big else (40, 40, 40)
        shape = tuple(rng.randint(1, h) for h in hi[3 - dims:])
        steps = rng.randint(1, 12 if big else 5)
        dtype = rng.choice(["f32", "f64"])
        precision = rng.choice(["exact", "fast"])
        width = rng.choice([0, 0, 0, 1, 3]) if dims == 3 and name != "wave" else 0
        try:
            bound, decls = corpus.config_target(name, shape, steps, dtype, map_width=width)
            grids = {k: GridBuffer.zeros(d.shape, d.order, d.dtype) for k, d in decls.items()}
            for j, k in enumerate(grids):
                fill_loguniform(grids[k], 100 + i + j)
            if "kap" in grids:
                grids["kap"].interior[...] = 0.01
            ref = oracle.run_target_c(bound, grids)
            bmap = next(s for s in bound.stmts[0].body if type(s).__name__ == "BoundMap")
            plan = plan_gpu(bmap.info, {"template": rng.choice(["unroll", "gmem", "shift"]), "computeCapability": "10.0"})
            got = run_gpu(bound, plan, grids, precision=precision)
            for k in ref:
                if precision == "exact":
                    ok = np.array_equal(ref[k].data, got[k].data)
                else:
                    ok = compare(ref[k], got[k]).max_relative <= TOL[dtype]
                if not ok:
                    bad += 1
                    print("MISMATCH", name, shape, steps, dtype, precision, width, k, compare(ref[k], got[k]).render())
        except Exception as e:  # noqa: BLE001
            msg = str(e)
            if type(e).__name__ in ("AnalysisError", "PlanError", "ParseError"):
                continue  # the reference itself refuses the generated program (e.g. regions wider than the grid)
            bad += 1
            print("ERROR", name, shape, steps, dtype, precision, width, type(e).__name__, msg[:200])
            traceback.print_exc(limit=2)
    print(f"{n - bad}/{n} cases ok")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]) if len(sys.argv) > 1 else 200, int(sys.argv[2]) if len(sys.argv) > 2 else 1))
