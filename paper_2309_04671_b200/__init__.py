"""B200-native backend for the StencilPy star-stencil time step (arXiv 2309.04671).

Drop-in for the reference's GPU execution path: ``run_gpu`` takes the same
arguments as ``stencilkit.executor.run_tile_plan`` and runs the bound target
on hand-written sm_100a kernels through the C-ABI in include/stkb200.h.
"""

from .backend import DeviceTarget, ExecutionError, release_device_cache, run_gpu
from .grids import ComparisonReport, GridBuffer, compare, fill_loguniform, load_grid, save_grid
from .planning import GpuPlan, PlanError, plan_gpu

__version__ = "0.1.0"

__all__ = [
    "ComparisonReport", "DeviceTarget", "ExecutionError", "GpuPlan", "GridBuffer", "PlanError",
    "compare", "fill_loguniform", "load_grid", "plan_gpu", "release_device_cache", "run_gpu", "save_grid",
]
