"""GPU launch plans (mirror of planning.py:104-202 of the reference).

``plan_gpu`` resolves the DSL's ``st.cuda(...)``/``st.gpu(...)`` launch
parameters exactly as the reference does (same template set, defaults,
memType auto rule, asyncMemcpy capability gate, f4 divisibility rule and
fail-closed unknown keys), so a plan built here and one built by
``stencilkit.planning.plan_gpu`` are interchangeable inputs to
:func:`paper_2309_04671_b200.run_gpu`.

On B200 the template / block / plane fields are *hints*: every template
routes to the same tuned 2.5D streaming kernel for star forms (SURVEY.md
§8(b)1: "Treat template/threadsPerBlock/planeDims as hints").
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping

GPU_TEMPLATES = ("gmem", "smem", "f4", "shift", "unroll", "semi")
GPU_STREAMING_TEMPLATES = ("shift", "unroll", "semi")
DEFAULT_BLOCK = (16, 8, 8)
DEFAULT_PLANE = (32, 32)
ASYNC_MEMCPY_MIN_CAPABILITY = (8, 0)
B200_CAPABILITY = (10, 0)


class PlanError(ValueError):
    """A launch configuration that cannot be resolved (planning.py:28-29)."""


@dataclass(frozen=True)
class GpuPlan:
    template: str
    block: tuple
    plane: tuple
    mem_type: str
    prefetch: bool
    async_memcpy: bool
    compute_capability: str
    dims: int
    padding: int = 0
    warnings: tuple = field(default=(), compare=False)

    @property
    def is_streaming(self) -> bool:
        return self.template in GPU_STREAMING_TEMPLATES


def parse_capability(text) -> tuple:
    """'10.0' / '10.0a' / '10' -> (10, 0)."""
    try:
        parts = str(text).rstrip("aAfF").split(".")
        return int(parts[0]), (int(parts[1]) if len(parts) > 1 and parts[1] else 0)
    except (ValueError, IndexError):
        raise PlanError(f"malformed compute capability '{text}'") from None


def _ints(value, n: int, what: str) -> tuple:
    if isinstance(value, int):
        value = (value,)
    if not isinstance(value, tuple) or not all(isinstance(v, int) for v in value):
        raise PlanError(f"{what} must be a tuple of integers")
    if len(value) < n:
        raise PlanError(f"{what} needs at least {n} entries, got {value}")
    out = tuple(int(v) for v in value[:n])
    if any(v < 1 for v in out):
        raise PlanError(f"{what} entries must be >= 1, got {value}")
    return out


def plan_gpu(info, params: Mapping) -> GpuPlan:
    p = dict(params)
    p.pop("scheme", None)
    warnings = []
    template = str(p.pop("template", "gmem"))
    if template not in GPU_TEMPLATES:
        raise PlanError(f"unknown GPU template '{template}'; valid templates: {', '.join(GPU_TEMPLATES)}")
    if template == "semi" and info.shape != "star":
        raise PlanError("the semi template supports star-shaped stencils only")
    dims = info.dims
    block = _ints(p.pop("threadsPerBlock", DEFAULT_BLOCK), min(dims, 3), "threadsPerBlock")
    plane = _ints(p.pop("planeDims", DEFAULT_PLANE), max(dims - 1, 1), "planeDims")
    mem = str(p.pop("memType", "auto"))
    if mem not in ("auto", "registers", "shared"):
        raise PlanError(f"unknown memType '{mem}'")
    if mem == "auto":
        mem = "registers" if info.shape == "star" else "shared"
    cap_text = str(p.pop("computeCapability", "8.0"))
    cap = parse_capability(cap_text)
    async_memcpy = bool(p.pop("asyncMemcpy", False))
    if async_memcpy and cap < ASYNC_MEMCPY_MIN_CAPABILITY:
        raise PlanError("asyncMemcpy requires compute capability >= 8.0, got " + cap_text)
    prefetch = bool(p.pop("prefetch", False))
    padding = int(p.pop("padding", 0))
    if padding:
        warnings.append("padding is accepted but not applied by the generator")
    if template == "f4":
        if info.dest_extents is None:
            raise PlanError("f4 template needs known grid extents to check divisibility")
        if info.dest_extents[-1] % 4 != 0:
            raise PlanError(
                f"f4 template requires the innermost extent to be divisible by 4, got {info.dest_extents[-1]}")
    if p:
        raise PlanError(f"unknown GPU parameters: {', '.join(sorted(map(str, p)))}")
    return GpuPlan(template, block, plane, mem, prefetch, async_memcpy, cap_text, dims, padding, tuple(warnings))
