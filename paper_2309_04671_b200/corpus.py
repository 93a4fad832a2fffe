"""The BASELINE.json configurations as ``.stpy`` programs, bound by the reference.

Every program here is SOURCE TEXT in the reference DSL, parsed, validated
and bound by the reference front end (``stencilkit.parser`` /
``stencilkit.analysis``, via :mod:`.front`), so the device path and the
reference executor see the very same ``BoundTarget``.  The canonical corpus
kernels come straight from ``stencilkit.corpus`` (coefficients
corpus.py:93-103, ``source_text`` :127-171); this module only adds the
configuration programs of SURVEY.md §8(d) in the same target shape
(``map(e=u.shape)`` then a swap):

  c1  star3d4r, 128^3, 10 steps (corpus coefficients)
  c2  7-point radius-1 normalised Jacobi, 512^3, 100 steps
  c3  acoustic wave ``up = 2u - up + kap*Lap8(u)``, 1024^3, swap (up, u)
  c4  star3d4r normalised (corpus coefficients / their sum), 1024^3
  c5  fp64 radius-2 13-point and radius-4 25-point normalised, 2048x2048x1024
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import front  # noqa: F401  (corpus.front is used by tests)

_ref = front.module("corpus")

KERNELS = {k.name: k for k in _ref.TABLE_KERNELS}  # the reference's kernel table, by name
offsets_of = _ref.offsets_of
coefficients = _ref.coefficients
divisor_of = _ref.divisor_of

# Lap8: 8th-order centred second derivative, per axis c0 and c_m (m = 1..4)
LAP8 = (-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0)


def _num(c: float) -> str:
    return f"({c!r})" if c < 0 else repr(c)


def _at(off) -> str:
    return ", ".join(str(c) for c in off)


def _weighted(terms) -> str:
    return " + ".join(f"{_num(c)} * u.at({_at(o)})" for o, c in terms)


def kernel_source(builder: str) -> tuple:
    """(kernel name, grid params, dest grid, update expression text) of a config kernel."""
    if builder == "wave":
        rings = []
        for m in range(1, 5):
            taps = []
            for axis in range(3):
                for sign in (-1, 1):
                    o = [0, 0, 0]
                    o[axis] = sign * m
                    taps.append(f"u.at({_at(o)})")
            rings.append(f"{_num(LAP8[m])} * ({' + '.join(taps)})")
        lap = f"{_num(3.0 * LAP8[0])} * u.at(0, 0, 0) + " + " + ".join(rings)
        expr = f"2.0 * u.at(0, 0, 0) - up.at(0, 0, 0) + kap.at(0, 0, 0) * ({lap})"
        return "kernel_acoustic_iso", ("u", "up", "kap"), "up", expr
    if builder == "jacobi7":  # c2: 0.4*centre + 0.1*each face neighbour (weights sum to 1)
        terms = [(o, 0.4 if not any(o) else 0.1) for o in offsets_of(KERNELS["star3d1r"])]
        return "kernel_jacobi7", ("u", "v"), "v", _weighted(terms)
    if builder.endswith("_norm"):  # the corpus star divided by its coefficient sum
        base = KERNELS[builder.removesuffix("_norm")]
        terms = coefficients(base)
        total = round(sum(c for _, c in terms), 5)
        return f"kernel_{builder}", ("u", "v"), "v", f"({_weighted(terms)}) / {total!r}"
    k = KERNELS[builder]
    return f"kernel_{k.name}", ("u", "v"), "v", _ref.update_expr_text(k)


def radius_of(builder: str) -> int:
    if builder in ("wave",):
        return 4
    if builder == "jacobi7":
        return 1
    return KERNELS[builder.removesuffix("_norm")].radius


def program_text(builder: str, shape: Sequence[int], iters=1, dtype: str = "f32", map_width: int = 0,
                 order: Optional[int] = None, backend: str = "st.seq()") -> str:
    """A complete ``.stpy`` program for a configuration kernel (the corpus target
    shape, corpus.py:155-171): map over the first grid's extent, then swap the
    destination with the first grid.  ``iters`` may be a name (runtime bound)."""
    name, gparams, dest, expr = kernel_source(builder)
    order = radius_of(builder) if order is None else order
    zeros = ", ".join(["0"] * len(shape))
    sig = ", ".join(f"{p}: st.grid" for p in gparams)
    spec = f"e={gparams[0]}.shape" + (f", w={map_width}" if map_width else "")
    target = "target_acoustic_iso" if builder == "wave" else f"target_{name.removeprefix('kernel_')}"
    first = gparams[0]
    decls = "".join(f"{p} = st.grid(dtype=st.{dtype}, shape=({', '.join(str(e) for e in shape)}), order={order})\n"
                    for p in gparams)
    launch_iters = iters if isinstance(iters, int) else 1
    return (
        "import stencilpy as st\n\n"
        f"@st.kernel\ndef {name}({sig}):\n"
        f"    {dest}.at({zeros}).set({expr})\n\n"
        f"@st.target\ndef {target}({sig}, iter: st.i32):\n"
        f"    for _t in range(iter):\n"
        f"        st.map({spec})({name})({', '.join(gparams)})\n"
        f"        ({dest}, {first}) = ({first}, {dest})\n\n"
        f"{decls}"
        f"st.launch(\n    backend={backend}\n)({target})({', '.join(gparams)}, {launch_iters})\n"
    )


def bind_text(text: str, iters=None, scheme: Optional[str] = None, file: str = "<corpus>") -> tuple:
    """(BoundTarget, {grid name: GridDecl}) of a program, bound by the reference.
    A non-integer ``iters`` keeps the loop bound a runtime argument (``iter``)."""
    frozen = iters is None or isinstance(iters, int)
    unit, bound = front.parse_bind(text, file, scheme=scheme, freeze_loop_bounds=frozen)
    return bound, {g.name: g for g in unit.grids}


def config_target(builder: str, shape: Sequence[int], iters, dtype: str = "f32", map_width: int = 0,
                  scheme: Optional[str] = None, order: Optional[int] = None) -> tuple:
    """(BoundTarget, decls) for a named kernel: a reference corpus kernel
    (``star3d4r``, ``j3d27pt``, ...; the reference's own ``source_text``), its
    ``_norm`` variant, ``jacobi7`` or ``wave``.  ``iters`` = "iter" leaves the
    loop bound to ``bindings={"iter": n}``."""
    if builder in KERNELS and (order is None or order == KERNELS[builder].radius):
        text = _ref.source_text(builder, shape=tuple(shape), iters=iters if isinstance(iters, int) else 1,
                                dtype=dtype, map_width=map_width)
    else:
        text = program_text(builder, shape, iters, dtype, map_width, order)
    return bind_text(text, iters, scheme)


def corpus_target(name: str, shape: Sequence[int], iters, dtype: str = "f32", order: Optional[int] = None,
                  map_width: int = 0, scheme: Optional[str] = None) -> tuple:
    return config_target(name, shape, iters, dtype, map_width, scheme, order)


def wave_target(shape: Sequence[int], iters, dtype: str = "f32", order: int = 4, map_width: int = 0,
                scheme: Optional[str] = None) -> tuple:
    return config_target("wave", shape, iters, dtype, map_width, scheme, order)


def grids_for(decls: dict, grid_cls=None) -> dict:
    """Zero-initialised ``GridBuffer`` per declared grid (the reference's class)."""
    cls = grid_cls or front.module("grids").GridBuffer
    return {n: cls.zeros(tuple(d.shape), d.order, d.dtype) for n, d in decls.items()}


def wave_inputs(grids: dict, seed: int = 3, courant: float = 0.2) -> None:
    """c3 inputs: kap = (v*dt/h)^2, v ~ U[1500, 4500] (seed), v_max*dt/h = courant;
    u0 = centred Gaussian pulse + 1e-3 N(0,1) noise; up = u0."""
    rng = np.random.default_rng(seed)
    shape = tuple(grids["u"].shape)
    kap = grids["kap"].interior
    dt_h = courant / 4500.0
    for z in range(shape[0]):
        v = rng.uniform(1500.0, 4500.0, size=shape[1:])
        kap[z] = ((v * dt_h) ** 2).astype(kap.dtype)
    axes = [np.arange(n, dtype=np.float64) - (n - 1) / 2.0 for n in shape]
    sig = max(shape) / 16.0
    u = grids["u"].interior
    for z in range(shape[0]):
        r2 = axes[0][z] ** 2 + axes[1][:, None] ** 2 + axes[2][None, :] ** 2
        u[z] = (np.exp(-r2 / (2 * sig * sig)) + 1e-3 * rng.standard_normal(shape[1:])).astype(u.dtype)
    grids["up"].interior[...] = u


CONFIGS = {
    "c1": dict(kernel="star3d4r", shape=(128, 128, 128), steps=10, dtype="f32"),
    "c2": dict(kernel="jacobi7", shape=(512, 512, 512), steps=100, dtype="f32"),
    "c3": dict(kernel="wave", shape=(1024, 1024, 1024), steps=100, dtype="f32"),
    "c4": dict(kernel="star3d4r_norm", shape=(1024, 1024, 1024), steps=100, dtype="f32"),
    "c5a": dict(kernel="star3d2r_norm", shape=(2048, 2048, 1024), steps=20, dtype="f64"),
    "c5b": dict(kernel="star3d4r_norm", shape=(2048, 2048, 1024), steps=20, dtype="f64"),
}

__all__ = ["CONFIGS", "KERNELS", "LAP8", "bind_text", "coefficients", "config_target",
           "corpus_target", "divisor_of", "grids_for", "kernel_source", "offsets_of", "program_text",
           "radius_of", "wave_inputs", "wave_target"]
