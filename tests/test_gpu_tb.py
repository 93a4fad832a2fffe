"""Two time steps per sweep (csrc/star_tb.cuh) — B200 only.

The fused sweep keeps each step's FMA order, so every grid must hold exactly the
single-step kernel's values (bit for bit) after any step count, for any region
box and any halo contents; against the oracle it keeps the fast-path tolerance
(fp32 max relative error <= 1e-5, fp64 <= 1e-12).
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import oracle
from paper_2309_04671_b200 import DeviceTarget, compare, corpus, fill_loguniform, run_gpu
from paper_2309_04671_b200 import _lib as L
from paper_2309_04671_b200 import GridBuffer
from paper_2309_04671_b200 import plan_gpu

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "f64": 1e-12}


def _inputs(builder, shape, dtype, steps, seed=5, halo=0.0):
    bound, decls = corpus.config_target(builder, shape, steps, dtype)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    for i, n in enumerate(("u", "v")):
        g = grids[n]
        g.data[...] = halo * (i + 1)
        fill_loguniform(g, seed + i)
    return bound, grids


def _device_run(bound, grids, steps, fused, box=None):
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    with DeviceTarget(grids, ["u", "v"]) as dt:
        for n in ("u", "v"):
            dt.upload(n, grids[n].data)
        dt.set_fused_steps(fused)
        dt.set_multi_steps(False)  # small grids would take the multi-step launch instead
        if box is None:
            dt.set_program(body)
        else:  # one map over a sub-box of the interior, then the swap
            bmap = next(s for s in body if type(s).__name__ == "BoundMap")
            d = dt.compile_map(bmap, 0, box=box)
            L.call("stkb_program_reset", dt.h)
            L.call("stkb_program_add_map", dt.h, ctypes.byref(d))
            L.call("stkb_program_add_swap", dt.h, dt.index["v"], dt.index["u"])
        dt.run(steps)
        dt.sync()
        launches = dt.launches()
        return {n: dt.download(n) for n in ("u", "v")}, launches


def _fused_launches(steps, builder="star3d1r", whole=True):
    """Kernel launches of one fresh fused run: sweeps, single steps, the frozen-ring
    check and (map over the whole interior) the scratch's halo copy."""
    if "1r" not in builder and builder != "jacobi7":
        return steps  # radius 2+: single steps (stkb200.cu tb_map)
    n_tb = (steps - 2) // 2
    return n_tb + steps - 2 * n_tb + 1 + (1 if whole else 0)


@pytest.mark.parametrize("builder,dtype", [("star3d1r", "f32"), ("jacobi7", "f32"), ("star3d1r_norm", "f32"),
                                           ("star3d2r", "f32"), ("star3d1r", "f64"), ("star3d1r_norm", "f64")])
@pytest.mark.parametrize("shape", [(37, 45, 133), (9, 70, 250), (64, 64, 64), (5, 7, 9)])
@pytest.mark.parametrize("steps", [4, 7, 10])
def test_fused_sweeps_bitwise_equal_single_steps(builder, dtype, shape, steps):
    bound, grids = _inputs(builder, shape, dtype, steps)
    one, n1 = _device_run(bound, grids, steps, fused=False)
    two, n2 = _device_run(bound, grids, steps, fused=True)
    assert n1 == steps and n2 == _fused_launches(steps, builder), (n1, n2)
    for n in one:
        assert np.array_equal(one[n], two[n]), (builder, dtype, shape, steps, n)


@pytest.mark.parametrize("builder,dtype", [("star3d1r", "f32"), ("jacobi7", "f32"), ("star3d1r_norm", "f64")])
@pytest.mark.parametrize("box", [((3, 30), (5, 40), (9, 120)), ((0, 37), (0, 45), (1, 132)), ((10, 11), (0, 45), (0, 133))])
def test_fused_sweeps_sub_box_and_halo_bitwise(builder, dtype, box):
    """A region smaller than the interior and non-zero halos: outside the box v keeps
    the v buffer's content, and u(t+2) lands in a scratch that took over u's halo."""
    steps = 9
    bound, grids = _inputs(builder, (37, 45, 133), dtype, steps, halo=0.25)
    one, _ = _device_run(bound, grids, steps, fused=False, box=box)
    two, n2 = _device_run(bound, grids, steps, fused=True, box=box)
    whole = box == ((0, 37), (0, 45), (0, 133))
    assert n2 == _fused_launches(steps, whole=whole)
    for n in one:
        assert np.array_equal(one[n], two[n]), (builder, dtype, box, n)


@pytest.mark.parametrize("halo", [0.0, -0.0, 1e-30])
def test_fused_sweeps_zero_and_nonzero_halo_bitwise(halo):
    """Zero halo: the sweeps skip staging v's frozen values (ring check); -0.0 and a tiny
    non-zero halo must take the staged path and still match single steps bit for bit."""
    steps = 8
    bound, grids = _inputs("star3d1r", (33, 70, 250), "f32", steps)
    for n in ("u", "v"):
        g = grids[n]
        inner = g.interior.copy()
        g.data[...] = halo
        g.interior[...] = inner
    one, _ = _device_run(bound, grids, steps, fused=False)
    two, _ = _device_run(bound, grids, steps, fused=True)
    for n in one:
        assert np.array_equal(one[n].view(np.uint32), two[n].view(np.uint32)), (halo, n)


@pytest.mark.parametrize("builder,dtype,shape", [("jacobi7", "f32", (96, 80, 200)), ("star3d1r", "f64", (33, 40, 70)),
                                                 ("star3d1r_norm", "f32", (40, 50, 300))])
def test_fused_run_gpu_within_tolerance_vs_c_oracle(builder, dtype, shape, monkeypatch):
    from paper_2309_04671_b200 import release_device_cache

    monkeypatch.setenv("STKB_MULTI", "0")  # these grids are small enough for multi-step launches
    release_device_cache()
    steps = 12
    bound, decls = corpus.config_target(builder, shape, steps, dtype)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    fill_loguniform(grids["u"], 3)
    bmap = next(s for s in next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
                if type(s).__name__ == "BoundMap")
    plan = plan_gpu(bmap.info, {"template": "unroll", "computeCapability": "10.0"})
    from paper_2309_04671_b200.backend import LAST_RUN

    got = run_gpu(bound, plan, grids)
    assert LAST_RUN["launches"] == _fused_launches(steps)
    ref = oracle.run_target_c(bound, grids)
    for n in ref:
        rep = compare(ref[n], got[n])
        assert rep.max_relative <= TOL[dtype], (builder, n, rep.render())
        assert np.array_equal(ref[n].data[0], got[n].data[0])  # halo plane untouched


def test_fused_sweep_reports_nonfinite():
    bound, grids = _inputs("star3d1r", (20, 24, 40), "f32", 6)
    grids["u"].interior[7, 3, 11] = np.inf
    bmap = next(s for s in next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
                if type(s).__name__ == "BoundMap")
    plan = plan_gpu(bmap.info, {"template": "unroll", "computeCapability": "10.0"})
    with pytest.warns(RuntimeWarning, match="non-finite"):
        run_gpu(bound, plan, grids)


def test_fused_repeated_runs_and_scratch_reuse():
    """Runs back to back on one domain (the scratch pairing is reused without a copy),
    then an upload in between (the pairing must be re-established)."""
    bound, grids = _inputs("star3d1r", (21, 30, 90), "f32", 6)
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    res = {}
    for fused in (False, True):
        with DeviceTarget(grids, ["u", "v"]) as dt:
            for n in ("u", "v"):
                dt.upload(n, grids[n].data)
            dt.set_fused_steps(fused)
            dt.set_multi_steps(False)  # small grids would take the multi-step launch instead
            dt.set_program(body)
            dt.run(6)
            dt.run(8)
            mid = {n: dt.download(n) for n in ("u", "v")}
            fresh = grids["u"].data * np.float32(0.5)
            dt.upload("u", fresh)
            dt.run(5)
            dt.sync()
            res[fused] = (mid, {n: dt.download(n) for n in ("u", "v")})
    for k in range(2):
        for n in ("u", "v"):
            assert np.array_equal(res[False][k][n], res[True][k][n]), (k, n)


BC_TEXT = """import stencilpy as st

@st.kernel
def kernel_bc(u: st.grid, v: st.grid):
    u.at(0, 0, 0).set(0.5 * v.at(0, 0, 0) + 0.25)

@st.target
def target_bc(u: st.grid, v: st.grid):
    st.map(e=u.shape)(kernel_bc)(u, v)

u = st.grid(dtype=st.f32, shape=({shape}), order=1)
v = st.grid(dtype=st.f32, shape=({shape}), order=1)
st.launch(
    backend=st.seq()
)(target_bc)(u, v)
"""


@pytest.mark.parametrize("steps", [6, 7])
def test_fused_pair_invalidated_by_writes_outside_the_box(steps):
    """`for k: { loop(v = S(u) on a sub-box; swap); bc(u) over the whole interior }`:
    the map between the loops rewrites u outside the fused map's box, so the fused
    sweeps' scratch must take u over again (a stale scratch would feed old values
    outside the box to the second sweep as neighbours).  Fused == single steps."""
    shape = (20, 24, 70)
    box = ((3, 17), (4, 20), (9, 60))
    bound, grids = _inputs("star3d1r", shape, "f32", steps)
    bc_bound, _ = corpus.bind_text(BC_TEXT.format(shape=", ".join(map(str, shape))))
    bc = bc_bound.stmts[0]
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    bmap = next(s for s in body if type(s).__name__ == "BoundMap")
    res = {}
    for fused in (False, True):
        with DeviceTarget(grids, ["u", "v"]) as dt:
            for n in ("u", "v"):
                dt.upload(n, grids[n].data)
            dt.set_fused_steps(fused)
            dt.set_multi_steps(False)  # small grids would take the multi-step launch instead
            for _ in range(3):
                d = dt.compile_map(bmap, 0, box=box)
                L.call("stkb_program_reset", dt.h)
                L.call("stkb_program_add_map", dt.h, ctypes.byref(d))
                L.call("stkb_program_add_swap", dt.h, dt.index["v"], dt.index["u"])
                dt._program_key = None
                dt.run(steps)
                dt.set_program((bc,))
                dt.run(1)
            dt.sync()
            res[fused] = {n: dt.download(n) for n in ("u", "v")}
    for n in ("u", "v"):
        assert np.array_equal(res[False][n], res[True][n]), n
