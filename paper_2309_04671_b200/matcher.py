"""Kernel matcher: BoundMap -> one C-ABI map descriptor.

Decides which device kernel evaluates a bound map and extracts its
parameters.  The reference's own term collection for additive kernels is the
pattern (``split_semi_terms`` / ``peel_constant_divisor``, executor.py:149-188):
here the update expression is expanded into a polynomial over grid reads
(constants folded in float64) and matched against

  STAR  v[0] = (sum_k c_k * u[o_k]) [/ d]      star offsets, radius 1..4, 3-D
  WAVE  w[0] = a*u[0] + b*p[0] + k[0] * (sum_k c_k * u[o_k])
  BOX   v[0] = (sum over the dense (2R+1)^3 cube) [/ d]   box / "other", R <= 2

With ``precision="exact"`` a 3-D map whose update is literally the corpus star
(corpus.py:77-120: ``c0*u.at(0,0,0) + c1*u.at(o1) + ...`` left-associated, every star
offset once, the centre first and the rest sorted, optionally ``/ D``) matches

  XSTAR the same float64 operations in the same order on the exact streaming kernel
        (csrc/star_exact.cuh): bit-identical to run_target at streaming speed

Everything else — larger box/"other" shapes, several updates, 2-D maps,
in-place Jacobi updates, offset destinations, or ``precision="exact"`` —
compiles to EXPR bytecode, which the device evaluates in float64 in parse
order with one rounding per store (bit-identical to run_target).
"""

from __future__ import annotations

import itertools

from dataclasses import dataclass, field
from typing import Optional

from .front import node_kind

MAX_FAST_RADIUS = 4
MAX_BOX_RADIUS = 4


class MatchError(ValueError):
    pass


@dataclass
class MapPlan:
    kind: str  # "star" | "wave" | "box" | "xstar" | "xbox" | "xwave" | "expr"
    radius: int = 0
    src: Optional[str] = None  # module grid names
    dst: Optional[str] = None
    prev: Optional[str] = None
    vel: Optional[str] = None
    coef: list = field(default_factory=list)  # star: 6R+1, C-ABI layout; box: (2R+1)^3 dense cube
    divisor: float = 0.0
    wave_a: float = 0.0
    wave_b: float = 0.0
    box: tuple = ()  # ((lo, hi), ...) interior coordinates
    # EXPR
    args: list = field(default_factory=list)  # module grid name per kernel grid param
    code: list = field(default_factory=list)  # [op, a, b, c, d] * n
    consts: list = field(default_factory=list)
    reason: str = ""  # why the fast path was not taken


def coef_index(offset: tuple, radius: int) -> int:
    """Slot of a star offset in the C-ABI coefficient table."""
    nz = [(a, c) for a, c in enumerate(offset) if c]
    if not nz:
        return 0
    (axis, c), = nz
    return 1 + axis * 2 * radius + 2 * (abs(c) - 1) + (1 if c > 0 else 0)


# ---------------------------------------------------------------------------
# polynomial expansion (fast-path matching only; evaluation order is not kept)


def _mul(p: dict, q: dict) -> dict:
    out: dict = {}
    for ka, va in p.items():
        for kb, vb in q.items():
            key = tuple(sorted(ka + kb))
            if len(key) > 2:
                raise MatchError("expression is not of degree <= 2 in grid reads")
            out[key] = out.get(key, 0.0) + va * vb
    return out


def _add(p: dict, q: dict, sign: float = 1.0) -> dict:
    out = dict(p)
    for k, v in q.items():
        out[k] = out.get(k, 0.0) + sign * v
    return out


def expand(expr, locals_: dict, scalars: dict) -> dict:
    """Polynomial {(read, ...): coefficient}; a read is (grid param, offset)."""
    k = node_kind(expr)
    if k == "Const":
        return {(): float(expr.value)}
    if k == "Read":
        return {((expr.grid, tuple(expr.offset)),): 1.0}
    if k == "Var":
        if expr.name in locals_:
            return locals_[expr.name]
        if expr.name in scalars:
            return {(): float(scalars[expr.name])}
        raise MatchError(f"unbound name '{expr.name}' in kernel expression")
    if k == "Unary":
        return {kk: -v for kk, v in expand(expr.operand, locals_, scalars).items()}
    if k == "Binary":
        a = expand(expr.left, locals_, scalars)
        b = expand(expr.right, locals_, scalars)
        if expr.op == "+":
            return _add(a, b)
        if expr.op == "-":
            return _add(a, b, -1.0)
        if expr.op == "*":
            return _mul(a, b)
        if set(b) == {()}:
            return {kk: v / b[()] for kk, v in a.items()}
        raise MatchError("division by a grid-dependent expression")
    raise MatchError(f"unsupported expression node {k}")


def _drop_zeros(p: dict) -> dict:
    return {k: v for k, v in p.items() if v != 0.0}


def _is_star(offsets, dims: int) -> bool:
    return all(len(o) == dims and sum(1 for c in o if c) <= 1 for o in offsets)


# ---------------------------------------------------------------------------


def map_box(bmap) -> tuple:
    """Union box of a map's regions; they are an exact cover of it
    (analysis.py:322-376), and every region evaluates the same expression
    against the same pre-map snapshot, so one launch over the box computes
    exactly what the per-region loop of run_target does."""
    regions = list(bmap.regions)
    if not regions:
        return ()
    nd = len(regions[0].bounds)
    box = tuple((min(r.bounds[d][0] for r in regions), max(r.bounds[d][1] for r in regions)) for d in range(nd))
    vol = 1
    for lo, hi in box:
        vol *= hi - lo
    if sum(r.size for r in regions) != vol:
        raise MatchError("map regions do not form an exact cover of their bounding box")
    return box


def match_map(bmap, *, exact: bool = False) -> MapPlan:
    """Choose the device kernel for one bound map."""
    params = dict(bmap.grid_args)  # kernel grid param -> module grid
    box = map_box(bmap)
    if exact:
        why = []
        for m in (match_exact_star, match_exact_box, match_exact_wave):
            try:
                return m(bmap, params, box)
            except MatchError as e:
                why.append(str(e))
        p = compile_expr(bmap)
        p.box, p.reason = box, "precision='exact': " + "; ".join(why)
        return p
    try:
        return _match_fast(bmap, params, box)
    except MatchError as why:
        p = compile_expr(bmap)
        p.box, p.reason = box, str(why)
        return p


def _match_fast(bmap, params: dict, box: tuple) -> MapPlan:
    kern = bmap.kernel
    if len(kern.updates) != 1:
        raise MatchError("several updates in one kernel")
    upd = kern.updates[0]
    dims = len(upd.offset)
    if dims not in (2, 3):
        raise MatchError(f"{dims}-D kernel (the streaming kernels are 2-D and 3-D)")
    if any(upd.offset):
        raise MatchError("destination offset is not the centre")
    scalars = {n: float(v) for n, v in bmap.scalar_args}
    loc: dict = {}
    for name, e in kern.locals:
        loc[name] = expand(e, loc, scalars)
    expr = upd.expr
    divisor = 0.0
    if node_kind(expr) == "Binary" and expr.op == "/" and node_kind(expr.right) == "Const":
        divisor = float(expr.right.value)  # executor.py:149-153
        expr = expr.left
        if divisor == 0.0:
            raise MatchError("division by zero constant")
    poly = _drop_zeros(expand(expr, loc, scalars))
    if () in poly:
        raise MatchError("constant term")
    dst = params[upd.dest]
    deg1 = {k: v for k, v in poly.items() if len(k) == 1}
    deg2 = {k: v for k, v in poly.items() if len(k) == 2}

    if not deg2:
        grids = {k[0][0] for k in deg1}
        if len(grids) != 1:
            raise MatchError("weighted sum over several grids")
        src_param = grids.pop()
        offs = [k[0][1] for k in deg1]
        r = max(max(abs(c) for c in o) for o in offs)
        if dims == 2 and not _is_star(offs, 2):
            if r < 1 or r > MAX_FAST_RADIUS:
                raise MatchError(f"2-D box/other shape of radius {r} outside 1..{MAX_FAST_RADIUS}")
            src = params[src_param]
            if src == dst:
                raise MatchError("in-place update (reads and writes the same grid)")
            n = 2 * r + 1
            square = [0.0] * n * n
            for k, v in deg1.items():
                dy, dx = k[0][1]
                square[(dy + r) * n + (dx + r)] = v
            return MapPlan("box", r, src, dst, coef=square, divisor=divisor, box=box)
        if dims == 3 and not _is_star(offs, 3):
            if r > MAX_BOX_RADIUS:
                raise MatchError(f"box/other shape of radius {r} (dense streaming kernel covers <= {MAX_BOX_RADIUS})")
            src = params[src_param]
            if src == dst:
                raise MatchError("in-place update (reads and writes the same grid)")
            n = 2 * r + 1
            cube = [0.0] * n ** 3
            for k, v in deg1.items():
                dz, dy, dx = k[0][1]
                cube[((dz + r) * n + (dy + r)) * n + (dx + r)] = v
            return MapPlan("box", r, src, dst, coef=cube, divisor=divisor, box=box)
        if r < 1 or r > MAX_FAST_RADIUS:
            raise MatchError(f"radius {r} outside 1..{MAX_FAST_RADIUS}")
        src = params[src_param]
        if src == dst:
            raise MatchError("in-place update (reads and writes the same grid)")
        coef = [0.0] * (6 * r + 1)
        for k, v in deg1.items():
            coef[coef_index(k[0][1], r)] = v
        return MapPlan("star", r, src, dst, coef=coef, divisor=divisor, box=box)

    if divisor:
        raise MatchError("divided wave form")
    if dims != 3:
        raise MatchError("2-D degree-2 form")
    # WAVE: deg-2 terms are vel[0] * u[o]
    vel_cands = None
    for k in deg2:
        pair = {k[0], k[1]}
        zero_reads = {rd for rd in pair if not any(rd[1])}
        cands = set()
        for z in zero_reads:
            other = (pair - {z}) or {z}
            (o,) = other
            if o[0] != z[0]:
                cands.add(z[0])
        vel_cands = cands if vel_cands is None else (vel_cands & cands)
    if not vel_cands or len(vel_cands) != 1:
        raise MatchError("degree-2 terms are not velocity * grid reads")
    vel_param = vel_cands.pop()
    u_grids = set()
    lap = {}
    for k, v in deg2.items():
        a, b = k
        rd = b if (a[0] == vel_param and not any(a[1])) else a
        u_grids.add(rd[0])
        lap[rd[1]] = lap.get(rd[1], 0.0) + v
    if len(u_grids) != 1:
        raise MatchError("the velocity multiplies reads of several grids")
    u_param = u_grids.pop()
    offs = list(lap)
    if not _is_star(offs, 3):
        raise MatchError("not star-shaped")
    r = max(max(abs(c) for c in o) for o in offs)
    if r < 1 or r > MAX_FAST_RADIUS:
        raise MatchError(f"radius {r} outside 1..{MAX_FAST_RADIUS}")
    a_coef, b_coef, prev_param = 0.0, 0.0, None
    for k, v in deg1.items():
        (g, o), = k
        if any(o):
            raise MatchError("linear term away from the centre")
        if g == u_param:
            a_coef += v
        elif prev_param in (None, g):
            prev_param, b_coef = g, b_coef + v
        else:
            raise MatchError("linear terms over more than two grids")
    src, vel = params[u_param], params[vel_param]
    prev = params[prev_param] if prev_param else src
    if dst in (src, vel):
        raise MatchError("wave update writes a grid it reads at a non-centre offset")
    coef = [0.0] * (6 * r + 1)
    for o, v in lap.items():
        coef[coef_index(o, r)] = v
    return MapPlan("wave", r, src, dst, prev=prev, vel=vel, coef=coef, wave_a=a_coef, wave_b=b_coef, box=box)


def _const_value(n):
    """A literal constant (negation of a literal folds exactly)."""
    k = node_kind(n)
    if k == "Const":
        return float(n.value)
    if k == "Unary" and node_kind(n.operand) == "Const":
        return -float(n.operand.value)
    return None


def _exact_sum(bmap, params: dict):
    """The update as (divisor, [(coefficient, offset)], src, dst) when it is a left-associated
    sum of `literal * read` terms of one grid, optionally `/ literal`; else MatchError."""
    kern = bmap.kernel
    if len(kern.updates) != 1 or kern.locals:
        raise MatchError("not a single update without locals")
    upd = kern.updates[0]
    if len(upd.offset) not in (2, 3):
        raise MatchError("the exact streaming kernels are 2-D and 3-D")
    if any(upd.offset):
        raise MatchError("destination offset is not the centre")
    expr = upd.expr
    divisor = 0.0
    if node_kind(expr) == "Binary" and expr.op == "/":
        d = _const_value(expr.right)
        if d is None or d == 0.0:
            raise MatchError("division by something other than a non-zero literal")
        divisor, expr = d, expr.left
    terms = []
    while node_kind(expr) == "Binary" and expr.op == "+":
        terms.append(expr.right)
        expr = expr.left
    terms.append(expr)
    terms.reverse()
    out, grids = [], set()
    for t in terms:
        if node_kind(t) != "Binary" or t.op != "*":
            raise MatchError("a term is not coefficient * read")
        c, rd = _const_value(t.left), t.right
        if c is None:
            c, rd = _const_value(t.right), t.left
        if c is None or node_kind(rd) != "Read":
            raise MatchError("a term is not coefficient * read")
        out.append((c, tuple(rd.offset)))
        grids.add(rd.grid)
    if len(grids) != 1:
        raise MatchError("terms read several grids")
    src, dst = params[grids.pop()], params[upd.dest]
    if src == dst:
        raise MatchError("in-place update (reads and writes the same grid)")
    return divisor, out, src, dst


XBOX_MAX_RADIUS = {2: 4, 3: 4}  # by dimension


def match_exact_box(bmap, params: Optional[dict] = None, box: tuple = ()) -> MapPlan:
    """XBOX: the canonical dense box (corpus box3d1r..box3d4r, j3d27pt; box2d*, j2d9pt_gol) —
    every offset of the (2R+1)^3 cube (square in 2-D), centre first and the rest in sorted
    (lexicographic) order, left-associated, optionally `/ D` — evaluated with the same
    float64 operations in the same order (executor.py:81-106) on the exact box kernel
    (radius 1..4)."""
    params = params if params is not None else dict(bmap.grid_args)
    divisor, terms, src, dst = _exact_sum(bmap, params)
    offs = [o for _, o in terms]
    dims = len(offs[0])
    r = max(max(abs(v) for v in o) for o in offs)
    if r < 1 or r > XBOX_MAX_RADIUS[dims]:
        raise MatchError(f"{dims}-D box radius {r} outside 1..{XBOX_MAX_RADIUS[dims]}")
    cube = sorted(o for o in itertools.product(range(-r, r + 1), repeat=dims) if any(o))
    if offs != [(0,) * dims] + cube:
        raise MatchError("terms are not the full box in corpus order (centre, then sorted offsets)")
    n = 2 * r + 1
    coef = [0.0] * n ** dims
    for c, o in terms:
        k = 0
        for v in o:
            k = k * n + (v + r)
        coef[k] = c
    return MapPlan("xbox", r, src, dst, coef=coef, divisor=divisor, box=box)


def match_exact_star(bmap, params: Optional[dict] = None, box: tuple = ()) -> MapPlan:
    """XSTAR: the update is the canonical weighted star sum, term by term (executor.py's
    evaluation: each ``c * u`` one float64 multiply, each ``+`` one float64 add, the
    optional ``/ D`` one float64 division, then one rounding)."""
    params = params if params is not None else dict(bmap.grid_args)
    divisor, terms, src, dst = _exact_sum(bmap, params)
    coefs = [c for c, _ in terms]
    offs = [o for _, o in terms]
    dims = len(offs[0])
    r = max(max(abs(v) for v in o) for o in offs)
    if r < 1 or r > MAX_FAST_RADIUS:
        raise MatchError(f"radius {r} outside 1..{MAX_FAST_RADIUS}")
    star = [(0,) * dims]
    for axis in range(dims):
        for m in range(1, r + 1):
            for sgn in (-1, 1):
                o = [0] * dims
                o[axis] = sgn * m
                star.append(tuple(o))
    if offs != [star[0]] + sorted(star[1:]):
        raise MatchError("terms are not the full star in corpus order (centre, then sorted offsets)")
    coef = [0.0] * (6 * r + 1)
    for o, c in zip(offs, coefs):
        coef[coef_index(o, r)] = c
    return MapPlan("xstar", r, src, dst, coef=coef, divisor=divisor, box=box)


def _chain(expr, op: str) -> list:
    """Operands of a left-associated chain ((a op b) op c) ... in source order."""
    out = []
    while node_kind(expr) == "Binary" and expr.op == op:
        out.append(expr.right)
        expr = expr.left
    out.append(expr)
    return out[::-1]


def _read_at(n, offset=None):
    """(grid param, offset) of a Read node (optionally required at ``offset``), else None."""
    if node_kind(n) != "Read":
        return None
    o = tuple(n.offset)
    return None if offset is not None and o != tuple(offset) else (n.grid, o)


def _const_times(n):
    """(constant, other operand) of ``c * x`` or ``x * c``, else None."""
    if node_kind(n) != "Binary" or n.op != "*":
        return None
    c = _const_value(n.left)
    if c is not None:
        return c, n.right
    c = _const_value(n.right)
    return (c, n.left) if c is not None else None


def match_exact_wave(bmap, params: Optional[dict] = None, box: tuple = ()) -> MapPlan:
    """XWAVE: the acoustic wave exactly as SURVEY.md §8(d) writes it (corpus.kernel_source
    "wave"): ``A*u0 - p0 + k0 * (C0*u0 + L1*(S_1) + ... + LR*(S_R))`` with each S_m the six
    axis taps in the order (-m,0,0), (m,0,0), (0,-m,0), (0,m,0), (0,0,-m), (0,0,m)."""
    params = params if params is not None else dict(bmap.grid_args)
    kern = bmap.kernel
    if len(kern.updates) != 1 or kern.locals:
        raise MatchError("not a single update without locals")
    upd = kern.updates[0]
    if len(upd.offset) != 3 or any(upd.offset):
        raise MatchError("not a 3-D update at the centre")
    e = upd.expr
    zero = (0, 0, 0)
    if node_kind(e) != "Binary" or e.op != "+":
        raise MatchError("not head + kappa * laplacian")
    head, tail = e.left, e.right
    if node_kind(head) != "Binary" or head.op != "-":
        raise MatchError("head is not A*u - p")
    ct = _const_times(head.left)
    p_rd = _read_at(head.right, zero)
    if ct is None or p_rd is None or _read_at(ct[1], zero) is None:
        raise MatchError("head is not A*u - p")
    wave_a, u = ct[0], _read_at(ct[1], zero)[0]
    p = p_rd[0]
    if node_kind(tail) != "Binary" or tail.op != "*" or _read_at(tail.left, zero) is None:
        raise MatchError("tail is not kappa * laplacian")
    k = _read_at(tail.left, zero)[0]
    terms = _chain(tail.right, "+")
    first = _const_times(terms[0])
    if first is None or _read_at(first[1], zero) != (u, zero):
        raise MatchError("the laplacian does not start with C0 * u")
    coef = [first[0]]
    r = len(terms) - 1
    if r < 1 or r > MAX_FAST_RADIUS:
        raise MatchError(f"radius {r} outside 1..{MAX_FAST_RADIUS}")
    for m, t in enumerate(terms[1:], start=1):
        ct = _const_times(t)
        if ct is None:
            raise MatchError("a ring term is not L_m * (sum)")
        taps = _chain(ct[1], "+")
        want = [(-m, 0, 0), (m, 0, 0), (0, -m, 0), (0, m, 0), (0, 0, -m), (0, 0, m)]
        if len(taps) != 6 or [_read_at(x) for x in taps] != [(u, o) for o in want]:
            raise MatchError(f"ring {m} is not the six axis taps of u in order")
        coef.append(ct[0])
    if len({u, p, k}) != 3:
        raise MatchError("u, u_prev and kappa must be three grids")
    src, dst, prev, vel = params[u], params[upd.dest], params[p], params[k]
    if dst in (src, vel):
        raise MatchError("wave update writes a grid it reads at a non-centre offset")
    return MapPlan("xwave", r, src, dst, prev=prev, vel=vel, coef=coef, wave_a=wave_a, box=box)


# ---------------------------------------------------------------------------
# EXPR bytecode


def compile_expr(bmap) -> MapPlan:
    from . import _lib as L

    kern = bmap.kernel
    gparams = [p for p, _ in bmap.grid_args]
    index = {p: i for i, p in enumerate(gparams)}
    if len(gparams) > L.EXPR_MAX_ARGS:
        raise MatchError(f"kernel has more than {L.EXPR_MAX_ARGS} grid parameters")
    scalars = {n: float(v) for n, v in bmap.scalar_args}
    local_ids = {name: i for i, (name, _) in enumerate(kern.locals)}
    if len(local_ids) > L.EXPR_MAX_LOCALS:
        raise MatchError("too many kernel locals")
    code: list = []
    consts: list = []
    depth = [0, 0]

    def push(n=1):
        depth[0] += n
        depth[1] = max(depth[1], depth[0])

    def const(v: float) -> None:
        consts.append(float(v))
        code.append([L.OP_CONST, len(consts) - 1, 0, 0, 0])
        push()

    def off3(o) -> list:
        o = list(o)
        return o + [0] * (3 - len(o))

    def emit(e) -> None:
        stack = [(e, False)]
        while stack:  # iterative post-order: deep left-associated sums
            n, done = stack.pop()
            k = node_kind(n)
            if k == "Const":
                const(n.value)
            elif k == "Read":
                if n.grid not in index:
                    raise MatchError(f"'{n.grid}' is not a grid parameter")
                code.append([L.OP_READ, index[n.grid], *off3(n.offset)])
                push()
            elif k == "Var":
                if n.name in local_ids:
                    code.append([L.OP_LOCAL, local_ids[n.name], 0, 0, 0])
                    push()
                elif n.name in scalars:
                    const(scalars[n.name])
                else:
                    raise MatchError(f"unbound name '{n.name}' in kernel expression")
            elif k == "Unary":
                if done:
                    code.append([L.OP_NEG, 0, 0, 0, 0])
                else:
                    stack.append((n, True))
                    stack.append((n.operand, False))
            elif k == "Binary":
                if done:
                    op = {"+": L.OP_ADD, "-": L.OP_SUB, "*": L.OP_MUL, "/": L.OP_DIV}[n.op]
                    code.append([op, 0, 0, 0, 0])
                    depth[0] -= 1
                else:
                    stack.append((n, True))
                    stack.append((n.right, False))
                    stack.append((n.left, False))
            else:
                raise MatchError(f"unsupported expression node {k}")

    for name, e in kern.locals:
        emit(e)
        code.append([L.OP_SETLOCAL, local_ids[name], 0, 0, 0])
        depth[0] -= 1
    for upd in kern.updates:
        emit(upd.expr)
        code.append([L.OP_STORE, index[upd.dest], *off3(upd.offset)])
        depth[0] -= 1
    if depth[1] > L.EXPR_MAX_STACK:
        raise MatchError("expression nests deeper than the device evaluator's stack")
    args = [dict(bmap.grid_args)[p] for p in gparams]
    return MapPlan("expr", args=args, code=code, consts=consts)
