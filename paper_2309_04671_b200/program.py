"""Bound stencil programs: the input contract of the B200 backend.

The backend consumes the reference's *bound* program model — a
``BoundTarget`` whose statements are ``BoundFor`` / ``BoundMap`` /
``BoundSwap`` (analysis.py:383-415), each ``BoundMap`` carrying the kernel's
expression tree (dsl.py:24-74), its ``StencilInfo`` (analysis.py:42-57) and its
region decomposition (analysis.py:322-376).  Objects produced by the reference
front end (``stencilkit.analysis.bind_target``) are accepted as they are, by
attribute name.  This module restates the same model so programs can be
built where the reference package is absent (the GPU box): expression nodes
with Python operator overloading (so ``2.0 * u.at(0,0,0) - p.at(0,0,0)``
builds exactly the left-associated tree the reference parser builds,
parser.py:279-321), ``analyze_kernel``, ``decompose_regions`` and a small
``bind`` that assembles a BoundTarget.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import Optional, Sequence, Union


class AnalysisError(ValueError):
    """Malformed map specs / program structure (analysis.py:34-35)."""


# ---------------------------------------------------------------------------
# expressions (attribute names of dsl.py:24-74)


class Expr:
    __slots__ = ()

    def _wrap(self, other) -> "Expr":
        if isinstance(other, Expr):
            return other
        if isinstance(other, (int, float)):
            return Const(float(other))
        raise TypeError(f"cannot combine an expression with {other!r}")

    def __add__(self, o): return Binary("+", self, self._wrap(o))
    def __radd__(self, o): return Binary("+", self._wrap(o), self)
    def __sub__(self, o): return Binary("-", self, self._wrap(o))
    def __rsub__(self, o): return Binary("-", self._wrap(o), self)
    def __mul__(self, o): return Binary("*", self, self._wrap(o))
    def __rmul__(self, o): return Binary("*", self._wrap(o), self)
    def __truediv__(self, o): return Binary("/", self, self._wrap(o))
    def __rtruediv__(self, o): return Binary("/", self._wrap(o), self)

    def __neg__(self):
        # the parser folds negated literals (parser.py:284-290)
        if isinstance(self, Const):
            return Const(-self.value)
        return Unary("neg", self)


@dataclass(frozen=True, eq=True)
class Const(Expr):
    value: float


@dataclass(frozen=True, eq=True)
class Read(Expr):
    grid: str
    offset: tuple


@dataclass(frozen=True, eq=True)
class Var(Expr):
    name: str


@dataclass(frozen=True, eq=True)
class Unary(Expr):
    op: str
    operand: Expr


@dataclass(frozen=True, eq=True)
class Binary(Expr):
    op: str
    left: Expr
    right: Expr


class GridRef:
    """``u.at(o1, o2[, o3])`` builder for kernel bodies."""

    def __init__(self, name: str):
        self.name = name

    def at(self, *offset: int) -> Read:
        return Read(self.name, tuple(int(o) for o in offset))


def node_kind(node) -> str:
    """Class name of an expression node from either model."""
    return type(node).__name__


def walk(expr):
    """Pre-order, iterative (expanded corpus kernels nest hundreds deep)."""
    stack = [expr]
    while stack:
        n = stack.pop()
        yield n
        k = node_kind(n)
        if k == "Unary":
            stack.append(n.operand)
        elif k == "Binary":
            stack.append(n.right)
            stack.append(n.left)


# ---------------------------------------------------------------------------
# declarations and the bound model


@dataclass(frozen=True)
class GridDecl:
    name: str
    dtype: str
    shape: tuple
    order: int


@dataclass(frozen=True)
class Update:
    dest: str
    offset: tuple
    expr: Expr


@dataclass(frozen=True)
class KernelDecl:
    name: str
    params: tuple  # (name, "grid" | "f32" | "f64" | "i32")
    locals: tuple  # (name, Expr)
    updates: tuple  # Update

    def dims(self) -> int:
        return len(self.updates[0].offset) if self.updates else 0


@dataclass(frozen=True)
class StencilInfo:
    dims: int
    radius: int
    shape: str  # star | box | other
    offsets: tuple  # ((grid, (offsets...)), ...)
    flops_per_point: int
    dest: str
    dest_extents: Optional[tuple] = None
    dtype: str = "f32"

    def all_offsets(self) -> tuple:
        return tuple(sorted({o for _, offs in self.offsets for o in offs}))


@dataclass(frozen=True)
class Region:
    bounds: tuple  # ((lo, hi), ...) half open, interior coordinates
    tag: str

    @property
    def extents(self) -> tuple:
        return tuple(hi - lo for lo, hi in self.bounds)

    @property
    def size(self) -> int:
        n = 1
        for e in self.extents:
            n *= e
        return n


@dataclass(frozen=True)
class BoundMap:
    kernel: KernelDecl
    info: StencilInfo
    grid_args: tuple  # (kernel param, module grid name)
    scalar_args: tuple  # (kernel param, value)
    spec: tuple  # per-dim (a0, a1, a2, a3)
    regions: tuple


@dataclass(frozen=True)
class BoundFor:
    var: str
    count: Union[int, str]
    body: tuple


@dataclass(frozen=True)
class BoundSwap:
    first: str
    second: str


@dataclass(frozen=True)
class BoundTarget:
    name: str
    stmts: tuple
    grid_params: tuple  # (target param, module grid name)
    scalar_params: tuple
    scheme: str
    warnings: tuple = field(default=())


def stmt_kind(stmt) -> str:
    return type(stmt).__name__


# ---------------------------------------------------------------------------
# analysis (restates analysis.py:60-104)


def _classify(offsets, dims: int, radius: int) -> str:
    if all(sum(1 for c in o if c) <= 1 for o in offsets):
        return "star"
    cube = set(itertools.product(range(-radius, radius + 1), repeat=dims))
    return "box" if set(offsets) == cube else "other"


def analyze_kernel(kernel, grids: Optional[dict] = None) -> StencilInfo:
    per_grid: dict = {}
    flops = 0
    exprs = [e for _, e in kernel.locals] + [u.expr for u in kernel.updates]
    for e in exprs:
        for n in walk(e):
            k = node_kind(n)
            if k == "Read":
                per_grid.setdefault(n.grid, set()).add(tuple(n.offset))
            elif k in ("Binary", "Unary"):
                flops += 1
    union = sorted({o for offs in per_grid.values() for o in offs})
    dims = kernel.dims() or (len(union[0]) if union else 0)
    radius = max((max(abs(c) for c in o) for o in union), default=0)
    shape = _classify(union, dims, radius) if union else "star"
    dest = kernel.updates[0].dest if kernel.updates else ""
    extents, dtype = None, "f32"
    if grids and dest in grids:
        extents, dtype = tuple(grids[dest].shape), grids[dest].dtype
    offsets = tuple((g, tuple(sorted(o))) for g, o in sorted(per_grid.items()))
    return StencilInfo(dims, radius, shape, offsets, flops, dest, extents, dtype)


# ---------------------------------------------------------------------------
# map domains and regions (restates analysis.py:133-376)


def map_spec(extents: Sequence[int], width: int = 0) -> tuple:
    """``map(e=extents[, w=width])`` -> per-dim (a0, a1, a2, a3), validated as
    MapSpec.concrete does (analysis.py:133-160)."""
    spec = tuple((0, width, e - width, e) for e in extents) if width else tuple((0, 0, e, e) for e in extents)
    for axis, (a0, a1, a2, a3) in enumerate(spec):
        if not (0 <= a0 <= a1 and a2 <= a3) or a1 > a3 or a2 < a0:
            raise AnalysisError(f"map bounds for dimension {'ijk'[axis]} are out of order: {(a0, a1, a2, a3)}")
    return spec


SCHEMES = ("unified", "cross_product", "slab7")


def decompose_regions(spec: Sequence[tuple], scheme: str = "cross_product") -> list:
    """Disjoint regions covering the map domain, inner first, then boundary
    regions sorted by tag (analysis.py:322-376)."""
    if scheme not in SCHEMES:
        raise AnalysisError(f"unknown decomposition scheme '{scheme}'")
    dims = [tuple(int(v) for v in d) for d in spec]
    if scheme == "unified":
        b = tuple((a0, a3) for a0, _, _, a3 in dims)
        return [] if any(hi <= lo for lo, hi in b) else [Region(b, "inner")]
    if scheme == "cross_product":
        axes = []
        for a0, a1, a2, a3 in dims:
            top = max(a1, a2)  # an oversized width empties the middle interval
            axes.append([iv for iv in ((a0, a1, "0"), (a1, a2, "1"), (top, a3, "2")) if iv[1] > iv[0]])
        regions = []
        for combo in itertools.product(*axes):
            code = "".join(c for _, _, c in combo)
            tag = "inner" if set(code) == {"1"} else f"boundary:{code}"
            regions.append(Region(tuple((lo, hi) for lo, hi, _ in combo), tag))
        inner = [r for r in regions if r.tag == "inner"]
        return inner + sorted((r for r in regions if r.tag != "inner"), key=lambda r: r.tag)
    if len(dims) != 3:
        raise AnalysisError("slab7 decomposition requires a 3D map")
    (x0, x1, x2, x3), (y0, y1, y2, y3), (z0, z1, z2, z3) = dims
    hx, hy, hz = max(x1, x2), max(y1, y2), max(z1, z2)
    fx, fy = (x0, x3), (y0, y3)
    mx, my, mz = (x1, x2), (y1, y2), (z1, z2)
    cands = [
        Region((mx, my, mz), "inner"),
        Region(((x0, x1), my, mz), "boundary:x0"),
        Region(((hx, x3), my, mz), "boundary:x1"),
        Region((fx, (y0, y1), mz), "boundary:y0"),
        Region((fx, (hy, y3), mz), "boundary:y1"),
        Region((fx, fy, (z0, z1)), "boundary:z0"),
        Region((fx, fy, (hz, z3)), "boundary:z1"),
    ]
    kept = [r for r in cands if all(hi > lo for lo, hi in r.bounds)]
    inner = [r for r in kept if r.tag == "inner"]
    return inner + sorted((r for r in kept if r.tag != "inner"), key=lambda r: r.tag)


# ---------------------------------------------------------------------------
# assembling a bound target without the reference front end


def bind_map(kernel: KernelDecl, grid_args: Sequence[tuple], decls: dict, *, scalar_args=(),
             width: int = 0, scheme: str = "cross_product", extents=None) -> BoundMap:
    """One ``st.map(e=<first grid>.shape[, w=width])(kernel)(args)`` call."""
    kgrids = {p: decls[g] for p, g in grid_args}
    info = analyze_kernel(kernel, kgrids)
    if extents is None:
        extents = decls[grid_args[0][1]].shape
    spec = map_spec(extents, width)
    return BoundMap(kernel, info, tuple(grid_args), tuple(scalar_args), spec,
                    tuple(decompose_regions(spec, scheme)))


def time_loop(name: str, maps: Sequence[BoundMap], swaps: Sequence[tuple], iters: Union[int, str],
              grid_params: Sequence[tuple], scheme: str = "cross_product",
              scalar_params: Sequence[tuple] = ()) -> BoundTarget:
    """``for _t in range(iters): <maps>; (b, a) = (a, b) ...`` as a BoundTarget."""
    body = tuple(maps) + tuple(BoundSwap(a, b) for a, b in swaps)
    return BoundTarget(name, (BoundFor("_t", iters, body),), tuple(grid_params), tuple(scalar_params), scheme)


# ---------------------------------------------------------------------------
# source text and canonical dumps


_PREC = {"+": 1, "-": 1, "*": 2, "/": 2}


def expr_source(e) -> str:
    """DSL text whose parse (parser.py:279-321) is exactly the tree ``e``."""
    k = node_kind(e)
    if k == "Const":
        return repr(float(e.value))
    if k == "Read":
        return f"{e.grid}.at({', '.join(str(int(c)) for c in e.offset)})"
    if k == "Var":
        return e.name
    if k == "Unary":
        inner = expr_source(e.operand)
        return f"-({inner})" if node_kind(e.operand) in ("Binary", "Unary") else f"-{inner}"
    p = _PREC[e.op]
    left = expr_source(e.left)
    if node_kind(e.left) == "Binary" and _PREC[e.left.op] < p:
        left = f"({left})"
    right = expr_source(e.right)
    if node_kind(e.right) == "Binary" and _PREC[e.right.op] <= p:
        right = f"({right})"
    elif node_kind(e.right) == "Const" and e.right.value < 0:
        right = f"({right})"
    if node_kind(e.left) == "Const" and e.left.value < 0 and p == 2:
        left = f"({left})"  # (-c) * x parses to Const(-c) either way; keep it explicit
    return f"{left} {e.op} {right}"


def expr_dump(e) -> str:
    """Fully parenthesised prefix dump, identical for both object models."""
    out, stack = [], [e]
    while stack:
        n = stack.pop()
        if isinstance(n, str):
            out.append(n)
            continue
        k = node_kind(n)
        if k == "Const":
            out.append(repr(float(n.value)))
        elif k == "Read":
            out.append(f"{n.grid}{tuple(int(c) for c in n.offset)}")
        elif k == "Var":
            out.append(f"${n.name}")
        elif k == "Unary":
            stack += [")", n.operand, "(neg "]
        else:
            stack += [")", n.right, " ", n.left, f"({n.op} "]
    return "".join(out)


def dump(bound) -> str:
    """Canonical text of a bound target (statements, maps, kernels, regions)."""
    lines = [f"target {bound.name} scheme={bound.scheme} grids={tuple(tuple(p) for p in bound.grid_params)}"]

    def rec(stmts, ind):
        for s in stmts:
            k = stmt_kind(s)
            if k == "BoundSwap":
                lines.append(f"{ind}swap {s.first} {s.second}")
            elif k == "BoundFor":
                lines.append(f"{ind}for {s.count}")
                rec(s.body, ind + "  ")
            else:
                kern = s.kernel
                lines.append(f"{ind}map {kern.name} args={tuple(tuple(a) for a in s.grid_args)} "
                             f"scalars={tuple(tuple(a) for a in s.scalar_args)}")
                for name, e in kern.locals:
                    lines.append(f"{ind}  local {name} = {expr_dump(e)}")
                for u in kern.updates:
                    lines.append(f"{ind}  update {u.dest}{tuple(u.offset)} = {expr_dump(u.expr)}")
                info = s.info
                lines.append(f"{ind}  info dims={info.dims} radius={info.radius} shape={info.shape} "
                             f"flops={info.flops_per_point}")
                for r in s.regions:
                    lines.append(f"{ind}  region {r.tag} {tuple(tuple(b) for b in r.bounds)}")

    rec(bound.stmts, "  ")
    return "\n".join(lines) + "\n"
