"""Minimal ``.stpy`` loader for the GPU box, where the reference front end is absent.

Reads the restricted-Python stencil DSL (the language of the reference's
pkg/README.md "The DSL" section: ``@st.kernel`` / ``@st.target`` functions,
``st.grid`` declarations, one ``st.launch``) straight into this package's
bound program model (program.py), so existing programs run unchanged with
``python -m paper_2309_04671_b200 run prog.stpy``.  Expression trees are
built exactly as the reference parser builds them (left-associated BinOps,
negated literals folded — parser.py:279-321), which the tests check by
comparing canonical dumps with the reference's ``bind_target`` output.

This is a loader, not the reference's validator: programs are expected to
be valid (the reference's ``validate`` is out of scope); malformed input
raises :class:`~paper_2309_04671_b200.program.AnalysisError`.
"""

from __future__ import annotations

import ast
from dataclasses import dataclass, field
from typing import Optional

from .program import (
    AnalysisError,
    Binary,
    BoundFor,
    BoundMap,
    BoundSwap,
    BoundTarget,
    Const,
    GridDecl,
    KernelDecl,
    Read,
    Unary,
    Update,
    Var,
    analyze_kernel,
    decompose_regions,
)

BACKEND_ALIASES = {"seq": "seq", "omp": "omp", "gpu": "gpu", "cuda": "gpu", "hip": "gpu", "sycl": "gpu",
                   "dataflow": "dataflow", "csl": "dataflow"}
PARAM_TYPES = ("grid", "f32", "f64", "i32")


@dataclass
class Program:
    grids: dict  # name -> GridDecl (declaration order)
    kernels: dict  # name -> KernelDecl
    targets: dict  # name -> (params, body ast)
    backend: str = "seq"
    params: dict = field(default_factory=dict)  # launch backend parameters
    target: Optional[str] = None
    args: tuple = ()


def _fail(node, msg: str):
    raise AnalysisError(f"line {getattr(node, 'lineno', 0)}: {msg}")


def _st_attr(node) -> Optional[str]:
    if isinstance(node, ast.Attribute) and isinstance(node.value, ast.Name):
        return node.attr
    return None


def _literal(node):
    """Python literal (ints, floats, strings, bools, tuples, st.<Enum>.<name> tails)."""
    if isinstance(node, ast.Constant):
        return node.value
    if isinstance(node, ast.UnaryOp) and isinstance(node.op, ast.USub):
        v = _literal(node.operand)
        return -v
    if isinstance(node, ast.Tuple):
        return tuple(_literal(e) for e in node.elts)
    if isinstance(node, ast.Attribute):  # st.CUDABackend.Template.gmem -> "gmem"
        return node.attr
    _fail(node, "unsupported literal")


def _expr(node, grids: set, names: set):
    if isinstance(node, ast.Constant) and type(node.value) in (int, float):
        return Const(float(node.value))
    if isinstance(node, ast.UnaryOp) and isinstance(node.op, ast.USub):
        inner = _expr(node.operand, grids, names)
        return Const(-inner.value) if isinstance(inner, Const) else Unary("neg", inner)
    if isinstance(node, ast.BinOp):
        ops = {ast.Add: "+", ast.Sub: "-", ast.Mult: "*", ast.Div: "/"}
        op = ops.get(type(node.op))
        if op is None:
            _fail(node, "unsupported operator")
        return Binary(op, _expr(node.left, grids, names), _expr(node.right, grids, names))
    if isinstance(node, ast.Call) and isinstance(node.func, ast.Attribute) and node.func.attr == "at":
        g = node.func.value
        if not isinstance(g, ast.Name) or g.id not in grids:
            _fail(node, "reads must be <grid param>.at(...)")
        return Read(g.id, tuple(int(_literal(a)) for a in node.args))
    if isinstance(node, ast.Name) and node.id in names:
        return Var(node.id)
    _fail(node, "unsupported expression")


def _params(fn: ast.FunctionDef) -> tuple:
    out = []
    for a in fn.args.args:
        t = _st_attr(a.annotation) if a.annotation is not None else None
        if t not in PARAM_TYPES:
            _fail(a, f"parameter '{a.arg}' needs an st.grid / st.f32 / st.f64 / st.i32 annotation")
        out.append((a.arg, t))
    return tuple(out)


def _kernel(fn: ast.FunctionDef) -> KernelDecl:
    params = _params(fn)
    grids = {n for n, t in params if t == "grid"}
    names = {n for n, t in params if t != "grid"}
    locals_, updates = [], []
    for st in fn.body:
        if isinstance(st, ast.Expr) and isinstance(st.value, ast.Constant):
            continue  # docstring
        if isinstance(st, ast.Assign) and len(st.targets) == 1 and isinstance(st.targets[0], ast.Name):
            name = st.targets[0].id
            locals_.append((name, _expr(st.value, grids, names)))
            names.add(name)
            continue
        if (isinstance(st, ast.Expr) and isinstance(st.value, ast.Call) and isinstance(st.value.func, ast.Attribute)
                and st.value.func.attr == "set"):
            at = st.value.func.value
            if not (isinstance(at, ast.Call) and isinstance(at.func, ast.Attribute) and at.func.attr == "at"
                    and isinstance(at.func.value, ast.Name) and at.func.value.id in grids):
                _fail(st, "updates are <grid>.at(...).set(expr)")
            off = tuple(int(_literal(a)) for a in at.args)
            updates.append(Update(at.func.value.id, off, _expr(st.value.args[0], grids, names)))
            continue
        _fail(st, "unsupported kernel statement")
    return KernelDecl(fn.name, params, tuple(locals_), tuple(updates))


def load(text: str, file: str = "<input>") -> Program:
    tree = ast.parse(text, file)
    prog = Program({}, {}, {})
    for node in tree.body:
        if isinstance(node, (ast.Import, ast.ImportFrom)):
            continue
        if isinstance(node, ast.FunctionDef):
            deco = [_st_attr(d) for d in node.decorator_list]
            if "kernel" in deco:
                k = _kernel(node)
                prog.kernels[k.name] = k
            elif "target" in deco:
                prog.targets[node.name] = (_params(node), node.body)
            else:
                _fail(node, "functions must be @st.kernel or @st.target")
            continue
        if (isinstance(node, ast.Assign) and isinstance(node.value, ast.Call)
                and _st_attr(node.value.func) == "grid"):
            kw = {k.arg: k.value for k in node.value.keywords}
            name = node.targets[0].id
            dtype = _st_attr(kw["dtype"])
            shape = tuple(int(v) for v in _literal(kw["shape"]))
            order = int(_literal(kw.get("order", ast.Constant(0))))
            prog.grids[name] = GridDecl(name, dtype, shape, order)
            continue
        if isinstance(node, ast.Expr) and isinstance(node.value, ast.Call):
            call = node.value  # st.launch(backend=st.X(...))(target)(args...)
            inner = call.func
            if isinstance(inner, ast.Call) and isinstance(inner.func, ast.Call) and _st_attr(inner.func.func) == "launch":
                be = next(k.value for k in inner.func.keywords if k.arg == "backend")
                kind = _st_attr(be.func)
                prog.backend = BACKEND_ALIASES.get(kind, kind)
                prog.params = {k.arg: _literal(k.value) for k in be.keywords}
                prog.target = inner.args[0].id
                prog.args = tuple(a.id if isinstance(a, ast.Name) else _literal(a) for a in call.args)
                continue
        _fail(node, "unsupported top-level statement")
    return prog


def _spec_value(node, grids: dict, scal: dict):
    """Map argument: int, scalar param, <grid>.shape, or a tuple of those."""
    if isinstance(node, ast.Attribute) and node.attr == "shape" and isinstance(node.value, ast.Name):
        g = grids.get(node.value.id)
        if g is None:
            _fail(node, f"unknown grid '{node.value.id}'")
        return tuple(g.shape)
    if isinstance(node, ast.Name):
        if node.id not in scal:
            _fail(node, f"unbound map bound '{node.id}'")
        return int(scal[node.id])
    if isinstance(node, ast.Tuple):
        return tuple(_spec_value(e, grids, scal) for e in node.elts)
    if isinstance(node, ast.BinOp) and isinstance(node.op, (ast.Add, ast.Sub)):
        a, b = _spec_value(node.left, grids, scal), _spec_value(node.right, grids, scal)
        return a + b if isinstance(node.op, ast.Add) else a - b
    return int(_literal(node))


def _desugar(kw: dict) -> tuple:
    """Map shorthand -> per-dim (a0, a1, a2, a3) (pkg/README.md "Map shorthand")."""
    dims = [k for k in ("i", "j", "k") if k in kw]
    if not dims:
        ext, w = kw["e"], kw.get("w", 0)
        return tuple((0, w, e - w, e) for e in ext)
    vals = [kw[d] for d in dims]
    if all(isinstance(v, int) for v in vals):
        w = kw.get("w", 0)
        return tuple((0, w, v - w, v) for v in vals)
    if all(isinstance(v, tuple) and len(v) == 2 for v in vals):
        e = kw.get("e", 0)
        return tuple((lo, lo + e, hi - e, hi) for lo, hi in vals)
    if all(isinstance(v, tuple) and len(v) == 4 for v in vals):
        return tuple(tuple(v) for v in vals)
    raise AnalysisError("inconsistent map arguments")


def bind(prog: Program, target: Optional[str] = None, args=None, scheme: Optional[str] = None,
         iters: Optional[int] = None) -> BoundTarget:
    """Resolve the launched target into a BoundTarget (analysis.py:419-548 semantics)."""
    target = target or prog.target
    params, body = prog.targets[target]
    args = list(args if args is not None else prog.args)
    if iters is not None:
        slots = [i for i, (_, t) in enumerate(params) if t != "grid"]
        if len(slots) != 1:
            raise AnalysisError("--iters needs a target with exactly one scalar parameter")
        args[slots[0]] = iters
    scheme = scheme or str(prog.params.get("scheme", "cross_product"))
    gmap, scal = {}, {}
    for (p, t), a in zip(params, args):
        if t == "grid":
            gmap[p] = a
        else:
            scal[p] = a
    visible = dict(prog.grids)
    visible.update({p: prog.grids[g] for p, g in gmap.items()})

    def stmts(nodes):
        out = []
        for st in nodes:
            if isinstance(st, ast.For):
                cnt = st.iter.args[0]
                count = int(scal[cnt.id]) if isinstance(cnt, ast.Name) else int(_literal(cnt))
                out.append(BoundFor(st.target.id, count, stmts(st.body)))
            elif isinstance(st, ast.Assign) and isinstance(st.targets[0], ast.Tuple):
                a, b = (e.id for e in st.targets[0].elts)
                out.append(BoundSwap(gmap.get(a, a), gmap.get(b, b)))
            elif isinstance(st, ast.Expr) and isinstance(st.value, ast.Call):
                call = st.value  # st.map(spec)(kernel)(args)
                kern = prog.kernels[call.func.args[0].id]
                spec_kw = {k.arg: _spec_value(k.value, visible, scal) for k in call.func.func.keywords}
                spec = _desugar(spec_kw)
                margs = [a.id if isinstance(a, ast.Name) else _literal(a) for a in call.args]
                garg, sarg = [], []
                for (kp, kt), a in zip(kern.params, margs):
                    if kt == "grid":
                        garg.append((kp, gmap.get(a, a)))
                    else:
                        sarg.append((kp, float(scal[a]) if isinstance(a, str) else float(a)))
                info = analyze_kernel(kern, {kp: prog.grids[g] for kp, g in garg})
                out.append(BoundMap(kern, info, tuple(garg), tuple(sarg), spec,
                                    tuple(decompose_regions(spec, scheme))))
            elif isinstance(st, ast.Expr) and isinstance(st.value, ast.Constant):
                continue
            else:
                _fail(st, "unsupported target statement")
        return tuple(out)

    grid_params = tuple((p, g) for p, g in gmap.items())
    scalar_params = tuple((p, float(v)) for p, v in scal.items())
    return BoundTarget(target, stmts(body), grid_params, scalar_params, scheme)
