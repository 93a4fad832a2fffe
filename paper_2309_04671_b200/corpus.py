"""Canonical star kernels and the BASELINE.json configurations as bound programs.

Restates the reference corpus (pkg/src/stencilkit/corpus.py): offsets centre
first then sorted (corpus.py:77-90), per-offset coefficients
``round(U(0.05, 0.95), 5)`` from ``default_rng([20240817, *name.encode()])``
(corpus.py:93-103), Jacobi divisors (:106-108) and the ``v.at(0..).set(<sum>)``
/ swap target shape of ``source_text`` (:127-171).  Expressions are built
with the same left-associated tree the reference parser produces for that
source text, so the reference oracle and this backend see identical programs.

Configuration programs:
  c1  star3d4r, 128^3, 10 steps (corpus coefficients)
  c2  7-point radius-1 normalised Jacobi, 512^3, 100 steps
  c3  acoustic wave, 25-point Lap8 with variable velocity, 1024^3
  c4  star3d4r normalised (corpus coefficients / their sum), 1024^3
  c5  fp64 radius-2 13-point and radius-4 25-point normalised, 2048x2048x1024
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .program import (
    BoundTarget,
    GridDecl,
    GridRef,
    KernelDecl,
    Update,
    bind_map,
    time_loop,
)

COEFF_SEED = 20240817

_STAR2D4R_CENTER = 0.25005
_STAR2D4R_PAIRS = (
    ((-4, 0), 0.11111), ((-3, 0), 0.06251), ((-2, 0), 0.06255), ((-1, 0), 0.06245),
    ((0, -1), 0.06248), ((0, -2), 0.06243), ((0, -3), 0.06253), ((0, -4), -0.22220),
)


@dataclass(frozen=True)
class CorpusKernel:
    name: str
    shape: str  # star | box
    dims: int
    radius: int
    jacobi: bool = False


def _table() -> dict:
    rows = {}
    for kind in ("star", "box"):
        for dims in (2, 3):
            for r in (1, 2, 3, 4):
                rows[f"{kind}{dims}d{r}r"] = CorpusKernel(f"{kind}{dims}d{r}r", kind, dims, r)
    rows["j2d5pt"] = CorpusKernel("j2d5pt", "star", 2, 1, True)
    rows["j2d9pt_gol"] = CorpusKernel("j2d9pt_gol", "box", 2, 1, True)
    rows["j2d9pt"] = CorpusKernel("j2d9pt", "star", 2, 2, True)
    rows["j3d27pt"] = CorpusKernel("j3d27pt", "box", 3, 1, True)
    return rows


KERNELS = _table()


def offsets_of(k: CorpusKernel) -> tuple:
    if k.shape == "star":
        rest = []
        for axis in range(k.dims):
            for m in range(1, k.radius + 1):
                for sign in (-1, 1):
                    o = [0] * k.dims
                    o[axis] = sign * m
                    rest.append(tuple(o))
        return ((0,) * k.dims, *sorted(rest))
    cube = itertools.product(range(-k.radius, k.radius + 1), repeat=k.dims)
    return ((0,) * k.dims, *sorted(o for o in cube if any(o)))


def coefficients(k: CorpusKernel) -> tuple:
    offs = offsets_of(k)
    if k.name == "star2d4r":
        table = {(0, 0): _STAR2D4R_CENTER}
        for (a, b), c in _STAR2D4R_PAIRS:
            table[(a, b)] = c
            table[(-a, -b)] = c
        return tuple((o, table[o]) for o in offs)
    # the coefficient stream reads the name's characters as seed words
    rng = np.random.default_rng([COEFF_SEED, *k.name.encode()])
    return tuple((o, round(float(rng.uniform(0.05, 0.95)), 5)) for o in offs)


def divisor_of(k: CorpusKernel) -> float:
    rng = np.random.default_rng([COEFF_SEED + 1, *k.name.encode()])
    return round(float(rng.uniform(2.0, 9.0)), 5)


def weighted_sum(src: str, terms: Sequence[tuple]):
    """``c0 * u.at(o0) + c1 * u.at(o1) + ...`` (left associated)."""
    u = GridRef(src)
    expr = None
    for off, c in terms:
        t = float(c) * u.at(*off)
        expr = t if expr is None else expr + t
    return expr


def corpus_kernel(name: str, divisor: Optional[float] = None) -> KernelDecl:
    """The corpus kernel ``kernel_<name>(u, v)``; ``divisor`` overrides the
    Jacobi divisor (or adds one, for the normalised long-run variants)."""
    k = KERNELS[name]
    expr = weighted_sum("u", coefficients(k))
    if divisor is not None:
        expr = expr / float(divisor)
    elif k.jacobi:
        expr = expr / divisor_of(k)
    zero = (0,) * k.dims
    return KernelDecl(f"kernel_{name}", (("u", "grid"), ("v", "grid")), (), (Update("v", zero, expr),))


def jacobi_target(kernel: KernelDecl, shape: Sequence[int], order: int, iters, dtype: str = "f32",
                  map_width: int = 0, scheme: str = "cross_product", name: str = "") -> tuple:
    """``target(u, v, iter): for _t in range(iter): map(e=u.shape)(k)(u, v); (v, u) = (u, v)``.

    Returns (BoundTarget, {grid name: GridDecl})."""
    decls = {g: GridDecl(g, dtype, tuple(shape), order) for g in ("u", "v")}
    bmap = bind_map(kernel, (("u", "u"), ("v", "v")), decls, width=map_width, scheme=scheme)
    tgt = time_loop(name or "target_" + kernel.name.removeprefix("kernel_"), [bmap], [("v", "u")], iters,
                    (("u", "u"), ("v", "v")), scheme)
    return tgt, decls


def corpus_target(name: str, shape: Sequence[int], iters, dtype: str = "f32", order: Optional[int] = None,
                  map_width: int = 0, scheme: str = "cross_product") -> tuple:
    k = KERNELS[name]
    return jacobi_target(corpus_kernel(name), shape, k.radius if order is None else order, iters, dtype,
                         map_width, scheme, name=f"target_{name}")


def normalised_star_kernel(name: str) -> KernelDecl:
    """Corpus star kernel divided by its coefficient sum (bounded for long runs)."""
    total = round(sum(c for _, c in coefficients(KERNELS[name])), 5)
    kern = corpus_kernel(name, divisor=total)
    return KernelDecl(f"kernel_{name}_norm", kern.params, kern.locals, kern.updates)


def jacobi7_kernel() -> KernelDecl:
    """c2: 0.4*centre + 0.1*each of the 6 face neighbours (weights sum to 1)."""
    k = KERNELS["star3d1r"]
    terms = [(o, 0.4 if not any(o) else 0.1) for o in offsets_of(k)]
    return KernelDecl("kernel_jacobi7", (("u", "grid"), ("v", "grid")), (),
                      (Update("v", (0, 0, 0), weighted_sum("u", terms)),))


# Lap8: 8th-order centred second derivative, per axis c0 and c_m (m = 1..4)
LAP8 = (-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0)


def wave_kernel(radius: int = 4) -> KernelDecl:
    """c3: up.at(0,0,0).set(2.0*u.at(0,0,0) - up.at(0,0,0) + kap.at(0,0,0) * (Lap(u)))."""
    if radius != 4:
        raise ValueError("the acoustic ISO kernel is radius 4")
    u, up, kap = GridRef("u"), GridRef("up"), GridRef("kap")
    lap = (3.0 * LAP8[0]) * u.at(0, 0, 0)
    for m in range(1, 5):
        ring = None
        for axis in range(3):
            for sign in (-1, 1):
                o = [0, 0, 0]
                o[axis] = sign * m
                r = u.at(*o)
                ring = r if ring is None else ring + r
        lap = lap + LAP8[m] * ring
    expr = 2.0 * u.at(0, 0, 0) - up.at(0, 0, 0) + kap.at(0, 0, 0) * lap
    return KernelDecl("kernel_acoustic_iso", (("u", "grid"), ("up", "grid"), ("kap", "grid")), (),
                      (Update("up", (0, 0, 0), expr),))


def wave_target(shape: Sequence[int], iters, dtype: str = "f32", order: int = 4, map_width: int = 0,
                scheme: str = "cross_product") -> tuple:
    names = ("u", "up", "kap")
    decls = {g: GridDecl(g, dtype, tuple(shape), order) for g in names}
    bmap = bind_map(wave_kernel(), tuple((g, g) for g in names), decls, width=map_width, scheme=scheme)
    tgt = time_loop("target_acoustic_iso", [bmap], [("up", "u")], iters, tuple((g, g) for g in names), scheme)
    return tgt, decls


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


def config_target(kernel: str, shape: Sequence[int], iters, dtype: str = "f32", map_width: int = 0,
                  scheme: str = "cross_product") -> tuple:
    """(BoundTarget, decls) for a named kernel of the configuration table."""
    if kernel == "wave":
        return wave_target(shape, iters, dtype, 4, map_width, scheme)
    if kernel == "jacobi7":
        return jacobi_target(jacobi7_kernel(), shape, 1, iters, dtype, map_width, scheme, "target_jacobi7")
    if kernel.endswith("_norm"):
        base = kernel.removesuffix("_norm")
        return jacobi_target(normalised_star_kernel(base), shape, KERNELS[base].radius, iters, dtype,
                             map_width, scheme, f"target_{kernel}")
    return corpus_target(kernel, shape, iters, dtype, map_width=map_width, scheme=scheme)


def source_text(kernel: KernelDecl, shape: Sequence[int], order: int, iters: int, dtype: str = "f32",
                swap: tuple = ("v", "u"), map_width: int = 0, target: str = "",
                backend: str = "st.seq()") -> str:
    """A ``.stpy`` program for ``kernel`` in the corpus target shape
    (corpus.py:127-171): map over the first grid's extent, then swap."""
    from .program import expr_source

    gparams = [p for p, t in kernel.params if t == "grid"]
    (upd,) = kernel.updates
    sig = ", ".join(f"{p}: st.grid" for p in gparams)
    spec = f"e={gparams[0]}.shape" + (f", w={map_width}" if map_width else "")
    target = target or "target_" + kernel.name.removeprefix("kernel_")
    offs = ", ".join(str(c) for c in upd.offset)
    decls = "".join(
        f"{p} = st.grid(dtype=st.{dtype}, shape=({', '.join(str(e) for e in shape)}), order={order})\n"
        for p in gparams)
    return (
        "import stencilpy as st\n\n"
        f"@st.kernel\ndef {kernel.name}({sig}):\n"
        f"    {upd.dest}.at({offs}).set({expr_source(upd.expr)})\n\n"
        f"@st.target\ndef {target}({sig}, iter: st.i32):\n"
        f"    for _t in range(iter):\n"
        f"        st.map({spec})({kernel.name})({', '.join(gparams)})\n"
        f"        ({swap[0]}, {swap[1]}) = ({swap[1]}, {swap[0]})\n\n"
        f"{decls}"
        f"st.launch(\n    backend={backend}\n)({target})({', '.join(gparams)}, {iters})\n"
    )
