"""Install :func:`run_gpu` as the GPU branch of the reference's ``run_tile_plan``.

This is the drop-in of INTEGRATION.md applied at run time: after
:func:`install`, ``stencilkit.executor.run_tile_plan`` (executor.py:491-557)
sends every ``GpuPlan`` to the B200 backend and every other plan (``OmpPlan``)
to the reference's own emulation, unchanged.  The reference CLI
(``stencilkit.cli.cmd_run``, cli.py:246-283) calls the patched function too,
so ``stencilkit run --backend gpu ... --oracle`` executes on the device.

Precision: ``exact`` by default — float64 evaluation in parse order with one
rounding per store, bit-identical to ``run_target``, i.e. the contract the
reference's own GPU-plan tests assert (``array_equal`` / 1e-7 / 1e-8,
tests/test_executor.py:228-280).  ``precision="fast"`` (or
``STKB_PRECISION=fast``) selects the tuned streaming kernels in the grid
dtype, with the north-star tolerance (fp32 max relative error <= 1e-5).
"""

from __future__ import annotations

import os
from typing import Optional

from . import front
from .backend import run_gpu

_ORIGINAL: dict = {}


def precision_default() -> str:
    return os.environ.get("STKB_PRECISION", "exact")


def install(precision: Optional[str] = None):
    """Patch ``stencilkit.executor.run_tile_plan`` (and the CLI's reference to it)."""
    executor, cli, planning = front.module("executor"), front.module("cli"), front.module("planning")
    original = _ORIGINAL.setdefault("run_tile_plan", executor.run_tile_plan)

    def run_tile_plan(unit, plan, grids, bindings=None, target=None, args=None, scheme=None):
        if isinstance(plan, planning.GpuPlan):
            return run_gpu(unit, plan, grids, bindings, target, args, scheme,
                           precision=precision or precision_default())
        return original(unit, plan, grids, bindings, target, args, scheme)

    run_tile_plan.__wrapped__ = original
    run_tile_plan.__doc__ = original.__doc__
    executor.run_tile_plan = run_tile_plan
    cli.run_tile_plan = run_tile_plan
    return run_tile_plan


def uninstall() -> None:
    """Restore the reference's own ``run_tile_plan``."""
    if "run_tile_plan" in _ORIGINAL:
        original = _ORIGINAL["run_tile_plan"]
        front.module("executor").run_tile_plan = original
        front.module("cli").run_tile_plan = original


def installed() -> bool:
    return getattr(front.module("executor").run_tile_plan, "__wrapped__", None) is not None
