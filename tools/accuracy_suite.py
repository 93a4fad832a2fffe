#!/usr/bin/env python3
"""The reference's numerical-accuracy sweep, through the drop-in on the B200.

    python tools/accuracy_suite.py [--dtype f32 f64] [--precision exact fast] > profiles/r2_accuracy_suite.txt

The B200 counterpart of the reference's ``scripts/run_accuracy_suite.py:27-65``: every
corpus table kernel (``corpus.TABLE_KERNELS``; 16³ / 64² grids, 3 iterations, ``u``
log-uniform in [1e-4, 1e5] from seed 7) runs through the reference's own
``run_tile_plan`` with ``integrate.install()`` in place, for every GPU template
(``gmem smem f4 shift unroll`` + ``semi`` for stars), and is compared with the
reference's ``run_target`` by its own ``compare``. One line per kernel × template × dtype
× precision, with the reference's ``render()`` (max / RMSD relative).

Verdict per line: ``exact`` is held to the reference's 1e-7 max / 1e-8 RMSD relative
(the acceptance bar; it is bit-identical in practice, ``bitwise`` says so); ``fast`` to
the north-star tolerance (max relative 1e-5 fp32, 1e-12 fp64).  Exit code 1 if any
line fails.  Needs a GPU and ``baseline/_ref`` (the reference front end).
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_04671_b200 import front, integrate  # noqa: E402

sk_corpus = front.module("corpus")
sk_executor = front.module("executor")
sk_grids = front.module("grids")
sk_parser = front.module("parser")
sk_planning = front.module("planning")
sk_analysis = front.module("analysis")

MAX_TOL, RMSD_TOL = 1e-7, 1e-8
FAST_TOL = {"f32": 1e-5, "f64": 1e-12}
TEMPLATES = ("gmem", "smem", "f4", "shift", "unroll")


def _unit(kernel, dtype):
    shape = (64, 64) if kernel.dims == 2 else (16, 16, 16)
    unit = sk_parser.parse_source(sk_corpus.source_text(kernel.name, shape=shape, iters=3, dtype=dtype))
    assert not sk_parser.validate(unit)
    return unit


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", nargs="+", default=["f32", "f64"])
    ap.add_argument("--precision", nargs="+", default=["exact", "fast"])
    a = ap.parse_args()
    failures = total = 0
    start = time.perf_counter()
    for precision in a.precision:
        integrate.install(precision)
        try:
            for dtype in a.dtype:
                for kernel in sk_corpus.TABLE_KERNELS:
                    unit = _unit(kernel, dtype)
                    decls = {g.name: g for g in unit.grids}
                    info = sk_analysis.analyze_kernel(unit.kernels[0], {"u": decls["u"], "v": decls["v"]})
                    grids = {n: sk_grids.GridBuffer.zeros(g.shape, g.order, g.dtype) for n, g in decls.items()}
                    sk_grids.fill_loguniform(grids["u"], 7)
                    reference = sk_executor.run_target(unit, grids)
                    templates = TEMPLATES + (("semi",) if kernel.shape == "star" else ())
                    for template in templates:
                        plan = sk_planning.plan_gpu(info, {"template": template, "threadsPerBlock": (8, 4, 4)})
                        result = sk_executor.run_tile_plan(unit, plan, grids)
                        rep = sk_grids.compare(reference["u"], result["u"])
                        if precision == "exact":
                            ok = rep.max_relative <= MAX_TOL and rep.rmsd_relative <= RMSD_TOL
                        else:
                            ok = rep.max_relative <= FAST_TOL[dtype]
                        same = np.array_equal(reference["u"].data, result["u"].data)
                        total += 1
                        failures += 0 if ok else 1
                        print(f"{'ok ' if ok else 'FAIL'} {kernel.display:<11} gpu  {template:<7} {dtype} "
                              f"{precision:<5} {'bitwise' if same else '       '} max_rel={rep.max_relative:.3e} "
                              f"rmsd_rel={rep.rmsd_relative:.3e} | {rep.render()}", flush=True)
        finally:
            integrate.uninstall()
    elapsed = time.perf_counter() - start
    print(f"\n{total - failures}/{total} combinations within tolerance in {elapsed:.1f}s "
          f"(exact: max_rel <= {MAX_TOL:g}, rmsd_rel <= {RMSD_TOL:g}; fast: max_rel <= 1e-5 f32 / 1e-12 f64)")
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
