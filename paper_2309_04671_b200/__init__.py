"""B200-native backend for the StencilPy star-stencil time step (arXiv 2309.04671).

Drop-in for the reference's GPU execution path: ``run_gpu`` takes the same
arguments as ``stencilkit.executor.run_tile_plan`` and runs the bound target
on hand-written sm_100a kernels through the C-ABI in include/stkb200.h.
"""

from . import front
from .backend import DeviceTarget, ExecutionError, release_device_cache, run_gpu

# the reference's grid and plan types, re-exported (this package restates neither)
_grids = front.module("grids")
_planning = front.module("planning")
ComparisonReport, GridBuffer, compare = _grids.ComparisonReport, _grids.GridBuffer, _grids.compare
fill_loguniform, load_grid, save_grid = _grids.fill_loguniform, _grids.load_grid, _grids.save_grid
GpuPlan, PlanError, plan_gpu = _planning.GpuPlan, _planning.PlanError, _planning.plan_gpu

__version__ = "0.1.0"

__all__ = [
    "ComparisonReport", "DeviceTarget", "ExecutionError", "GpuPlan", "GridBuffer", "PlanError",
    "compare", "fill_loguniform", "load_grid", "plan_gpu", "release_device_cache", "run_gpu", "save_grid",
]
