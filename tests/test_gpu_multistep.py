"""Several time steps per launch on small grids (StarArgs::n_steps) — B200 only.

A multi-step launch runs the ping-pong `v = S(u); swap(u, v)` for up to 64 steps
with a grid barrier between steps; per point it is the single-step kernel's
arithmetic, so every grid must hold exactly the single-step values (bit for bit)
after any step count, for any region box and any halo contents; against the
reference oracle the fast-path tolerance holds (fp32 1e-5, fp64 1e-12).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest

from oracle import oracle
from paper_2309_04671_b200 import DeviceTarget, GridBuffer, compare, corpus, fill_loguniform, plan_gpu, run_gpu
from paper_2309_04671_b200 import _lib as L

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


def _run(bound, grids, steps, multi, box=None, runs=(None,)):
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    with DeviceTarget(grids, ["u", "v"]) as dt:
        for n in ("u", "v"):
            dt.upload(n, grids[n].data)
        dt.set_multi_steps(multi)
        dt.set_fused_steps(False)
        if box is None:
            dt.set_program(body)
        else:
            bmap = next(s for s in body if type(s).__name__ == "BoundMap")
            d = dt.compile_map(bmap, 0, box=box)
            L.call("stkb_program_reset", dt.h)
            L.call("stkb_program_add_map", dt.h, ctypes.byref(d))
            L.call("stkb_program_add_swap", dt.h, dt.index["v"], dt.index["u"])
        launches = []
        for n in runs:
            dt.run(steps if n is None else n)
            launches.append(dt.launches())
        dt.sync()
        return {n: dt.download(n) for n in ("u", "v")}, launches


@pytest.mark.parametrize("builder,dtype", [("star3d4r", "f32"), ("star3d4r_norm", "f32"), ("star3d1r", "f32"),
                                           ("star3d2r", "f64"), ("star3d3r", "f32"), ("star3d4r_norm", "f64"),
                                           ("j3d27pt", "f32"), ("box3d2r", "f64")])
@pytest.mark.parametrize("shape", [(37, 45, 133), (128, 128, 128), (9, 20, 40)])
@pytest.mark.parametrize("steps", [2, 3, 10])
def test_multi_step_bitwise_equal_single_steps(builder, dtype, shape, steps):
    bound, grids = _inputs(builder, shape, dtype, steps)
    one, n1 = _run(bound, grids, steps, multi=False)
    many, n2 = _run(bound, grids, steps, multi=True)
    assert n1 == [steps] and n2 == [math.ceil(steps / 64)], (n1, n2)
    for n in one:
        assert np.array_equal(one[n], many[n]), (builder, dtype, shape, steps, n)


def test_multi_step_longer_than_one_launch():
    """150 steps = launches of 64, 64 and 22 steps; repeated runs on one domain."""
    bound, grids = _inputs("star3d4r_norm", (40, 50, 70), "f32", 150)
    one, _ = _run(bound, grids, None, multi=False, runs=(150, 7))
    many, launches = _run(bound, grids, None, multi=True, runs=(150, 7))
    assert launches == [3, 1]
    for n in one:
        assert np.array_equal(one[n], many[n]), n


@pytest.mark.parametrize("box", [((3, 30), (5, 40), (9, 120)), ((0, 37), (0, 45), (1, 132))])
@pytest.mark.parametrize("halo", [0.0, 0.25])
def test_multi_step_sub_box_and_halo(box, halo):
    """A region smaller than the interior and non-zero halos: the values outside the box
    stay each buffer's own, exactly as with single steps."""
    bound, grids = _inputs("star3d4r", (37, 45, 133), "f32", 9, halo=halo)
    one, _ = _run(bound, grids, 9, multi=False, box=box)
    many, n2 = _run(bound, grids, 9, multi=True, box=box)
    assert n2 == [1]
    for n in one:
        assert np.array_equal(one[n], many[n]), (box, halo, n)


@pytest.mark.parametrize("builder,dtype,shape,steps", [("star3d4r", "f32", (128, 128, 128), 10),
                                                       ("jacobi7", "f32", (64, 72, 96), 12),
                                                       ("star3d2r_norm", "f64", (48, 40, 64), 7),
                                                       ("j3d27pt", "f32", (64, 48, 80), 9)])
def test_multi_step_run_gpu_vs_oracle(builder, dtype, shape, steps):
    """The public path (run_gpu) on BASELINE config c1's program and shape: one launch for
    all steps, within the fast-path tolerance of the reference oracle."""
    from paper_2309_04671_b200.backend import LAST_RUN

    bound, decls = corpus.config_target(builder, shape, steps, dtype)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    fill_loguniform(grids["u"], 7)
    plan = plan_gpu(bound.stmts[0].body[0].info, {"template": "unroll", "computeCapability": "10.0"})
    got = run_gpu(bound, plan, grids)
    assert LAST_RUN["launches"] == 1
    ref = oracle.run_target_c(bound, grids)
    for n in ref:
        rep = compare(ref[n], got[n])
        assert rep.max_relative <= TOL[dtype], (builder, n, rep.render())


def test_multi_step_reports_nonfinite():
    bound, grids = _inputs("star3d4r", (20, 24, 40), "f32", 5)
    grids["u"].interior[7, 3, 11] = np.inf
    plan = plan_gpu(bound.stmts[0].body[0].info, {"template": "unroll", "computeCapability": "10.0"})
    with pytest.warns(RuntimeWarning, match="non-finite"):
        run_gpu(bound, plan, grids)


@pytest.mark.parametrize("builder,dtype,shape", [("star3d4r", "f32", (128, 128, 128)), ("star3d1r", "f64", (37, 45, 133)),
                                                 ("wave", "f32", (40, 48, 136))])
def test_small_grid_tile_bitwise_equal_default_tile(monkeypatch, builder, dtype, shape):
    """Small grids take the 16-row tile (StarLaunch::small_tile); the tile only changes which
    thread computes a point, so the grids match the default tile's bit for bit."""
    bound, decls = corpus.config_target(builder, shape, 4, dtype)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    for i, n in enumerate(grids):
        fill_loguniform(grids[n], 11 + i)
    if "kap" in grids:
        grids["kap"].interior[...] = 0.01
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    names = list(grids)
    outs = []
    for points in ("4194304", "0"):  # the default threshold, then the small tile disabled
        monkeypatch.setenv("STKB_SMALL_TILE_POINTS", points)
        with DeviceTarget(grids, names) as dt:
            for n in names:
                dt.upload(n, grids[n].data)
            dt.set_multi_steps(False)
            dt.set_fused_steps(False)
            dt.set_program(body)
            dt.run(4)
            dt.sync()
            outs.append({n: dt.download(n) for n in names})
    for n in names:
        assert np.array_equal(outs[0][n], outs[1][n]), n


@pytest.mark.parametrize("builder,dtype,shape,steps", [("star3d4r", "f32", (128, 128, 128), 10),
                                                       ("star3d4r_norm", "f32", (37, 45, 133), 7),
                                                       ("jacobi7", "f32", (64, 72, 96), 12),
                                                       ("star3d2r_norm", "f64", (48, 40, 64), 5),
                                                       ("star3d1r", "f32", (9, 20, 40), 70),
                                                       ("j3d27pt", "f32", (40, 48, 70), 9),
                                                       ("box3d2r", "f64", (30, 26, 40), 4),
                                                       ("box3d4r", "f32", (20, 24, 30), 3),
                                                       ("star2d4r", "f32", (1000, 1000), 9),
                                                       ("star2d1r", "f64", (37, 300), 70),
                                                       ("box2d2r", "f32", (90, 130), 6),
                                                       ("j2d9pt_gol", "f32", (64, 200), 5)])
def test_exact_multi_step_bitwise_vs_oracle(builder, dtype, shape, steps):
    """precision='exact' small-grid ping-pongs run their steps in multi-step launches of the
    exact star and box kernels (one launch per 64 steps): bit for bit the reference's evaluation."""
    from paper_2309_04671_b200.backend import LAST_RUN

    bound, decls = corpus.config_target(builder, shape, steps, dtype)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    fill_loguniform(grids["u"], 11)
    plan = plan_gpu(bound.stmts[0].body[0].info, {"template": "unroll", "computeCapability": "10.0"})
    got = run_gpu(bound, plan, grids, precision="exact")
    assert LAST_RUN["launches"] == math.ceil(steps / 64)
    ref = oracle.run_target_c(bound, grids)
    for n in ref:
        assert np.array_equal(ref[n].data, got[n].data), (builder, n, compare(ref[n], got[n]).render())


@pytest.mark.parametrize("shape,dtype,steps", [((40, 48, 136), "f32", 6), ((128, 128, 128), "f32", 9),
                                               ((33, 20, 70), "f64", 5)])
def test_wave_multi_step_bitwise_equal_single_steps(shape, dtype, steps):
    """The in-place acoustic-wave ping-pong (`up = 2u - up + k L(u); swap(u, up)`) also runs its
    steps in multi-step launches (odd steps swap the u / u_prev centre maps): bit for bit the
    single steps, within tolerance of the oracle."""
    bound, decls = corpus.wave_target(shape, steps, dtype)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    corpus.wave_inputs(grids)
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    names = list(grids)
    outs, launches = [], []
    for multi in (False, True):
        with DeviceTarget(grids, names) as dt:
            for n in names:
                dt.upload(n, grids[n].data)
            dt.set_multi_steps(multi)
            dt.set_fused_steps(False)
            dt.set_program(body)
            dt.run(steps)
            dt.sync()
            launches.append(dt.launches())
            outs.append({n: dt.download(n) for n in names})
    assert launches == [steps, 1], launches
    for n in names:
        assert np.array_equal(outs[0][n], outs[1][n]), n
    ref = oracle.run_target_c(bound, grids)
    for n in ref:
        got = GridBuffer(ref[n].dtype, ref[n].shape, ref[n].order, outs[1][n])
        assert compare(ref[n], got).max_relative <= TOL[dtype], n


@pytest.mark.parametrize("shape,dtype,steps", [((40, 48, 136), "f32", 6), ((64, 64, 64), "f32", 70),
                                               ((33, 20, 70), "f64", 5)])
def test_exact_wave_multi_step_bitwise_vs_oracle(shape, dtype, steps):
    """precision='exact' small-grid acoustic waves run their steps in multi-step launches of the
    exact wave kernel: bit for bit the reference's evaluation."""
    from paper_2309_04671_b200.backend import LAST_RUN

    bound, decls = corpus.wave_target(shape, steps, dtype)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    corpus.wave_inputs(grids)
    plan = plan_gpu(bound.stmts[0].body[0].info, {"template": "unroll", "computeCapability": "10.0"})
    got = run_gpu(bound, plan, grids, precision="exact")
    assert LAST_RUN["launches"] == math.ceil(steps / 64)
    ref = oracle.run_target_c(bound, grids)
    for n in ref:
        assert np.array_equal(ref[n].data, got[n].data), (n, compare(ref[n], got[n]).render())
