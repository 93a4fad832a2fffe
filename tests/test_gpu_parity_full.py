"""N-step parity at every BASELINE configuration's FULL size, against the reference's
own CPU path — B200 only.

The oracle here is the reference's CPU implementation itself: the OpenMP C it
emits for each configuration program (``codegen.generate(..., "omp", plan_omp(
{"template": "loop"}))``, openmp.py:14-53; float64 per point, one rounding, like
``run_target``, executor.py:267-286), built by oracle/build_ref.py at the
configuration's own shape and driven through its own C-ABI ``run_<target>(T*...,
int64_t iter)`` (serial.py:126-208) on all host cores (oracle/ref_runner.call).

* c2 (jacobi7 512^3 x 100 steps: fused two-step sweeps), c3 (wave 1024^3 x 10),
  c4 (star3d4r/S 1024^3 x 10): the whole grid, every grid, against the C run on the
  same inputs (downloaded from the device after the on-device fill).
* c5a / c5b (fp64 r2 / r4 stars, 2048 x 2048 x 1024, 34.9 GB per grid; the host
  could not hold the C oracle's two grids plus its internal copies plus ours): the
  device runs the FULL grid; the C oracle runs d0 windows of 104 planes (low end,
  middle, high end — the high end puts offsets past 2^32 elements) cut from the same
  input.  After N steps a window's outputs more than N*R planes from a cut are exact
  (the dependency cone of N radius-R steps), and at the grid's own ends the window's
  zero halo IS the grid's halo, so those planes are checked too.

Tolerances (north star): fp32 max relative error (grids.compare: max |a-b| / max
|ref|, grids.py:138-174) <= 1e-5, fp64 <= 1e-12.  Every case also records the
reference's own verdict (1e-7 max / 1e-8 RMSD, cli.py:37-38) to
gpurun_out/parity_full.json (summarised in profiles/parity_r2.json).
"""

from __future__ import annotations

import json
import math
import time

import numpy as np
import pytest

from conftest import ROOT
from oracle import build_ref, ref_runner
from paper_2309_04671_b200 import DeviceTarget, corpus, front

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "f64": 1e-12}
OUT = ROOT / "gpurun_out" / "parity_full.json"


def _record(case: str, **kw) -> None:
    OUT.parent.mkdir(exist_ok=True)
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    data[case] = kw
    OUT.write_text(json.dumps(data, indent=1, sort_keys=True))


def _torch():
    import torch

    return torch


def _interior(dt, name):
    """Torch view of the interior of the buffer ``name`` is bound to (pitched layout)."""
    torch = _torch()
    lay = dt.layout()
    tdt = torch.float32 if dt.dtype == "f32" else torch.float64

    class _A:
        __cuda_array_interface__ = {"shape": (lay["elems"],), "typestr": "<f4" if dt.dtype == "f32" else "<f8",
                                    "data": (dt.device_ptr(name), False), "version": 3}

    flat = torch.as_tensor(_A(), device="cuda")
    assert flat.dtype == tdt
    o = dt.order
    return flat.as_strided(dt.shape, (lay["plane"], lay["pitch"], 1), o * lay["plane"] + o * lay["pitch"] + lay["lead"])


def _fill_loguniform(view, seed: int) -> None:
    torch = _torch()
    g = torch.Generator(device="cuda").manual_seed(seed)
    for z in range(0, view.shape[0], 64):
        sl = view[z:z + 64]
        r = torch.rand(sl.shape, device="cuda", generator=g, dtype=torch.float64)
        sl.copy_(torch.pow(10.0, r * 9.0 - 4.0))


def _fill_wave(dt, seed: int = 3, courant: float = 0.2) -> None:
    """The c3 inputs of SURVEY.md §8(d) drawn on the device: kap = (v dt/h)^2 with
    v ~ U[1500, 4500] and v_max dt/h = courant; u0 = centred Gaussian pulse + 1e-3 N(0,1);
    up = u0."""
    torch = _torch()
    g = torch.Generator(device="cuda").manual_seed(seed)
    u, up, kap = _interior(dt, "u"), _interior(dt, "up"), _interior(dt, "kap")
    n0, n1, n2 = dt.shape
    dt_h = courant / 4500.0
    sig = max(dt.shape) / 16.0
    y = (torch.arange(n1, device="cuda", dtype=torch.float64) - (n1 - 1) / 2.0) ** 2
    x = (torch.arange(n2, device="cuda", dtype=torch.float64) - (n2 - 1) / 2.0) ** 2
    for z0 in range(0, n0, 32):
        z1 = min(n0, z0 + 32)
        z = (torch.arange(z0, z1, device="cuda", dtype=torch.float64) - (n0 - 1) / 2.0) ** 2
        r2 = z[:, None, None] + y[None, :, None] + x[None, None, :]
        noise = torch.randn((z1 - z0, n1, n2), device="cuda", generator=g, dtype=torch.float64)
        u[z0:z1].copy_(torch.exp(-r2 / (2 * sig * sig)) + 1e-3 * noise)
        v = torch.rand((z1 - z0, n1, n2), device="cuda", generator=g, dtype=torch.float64) * 3000.0 + 1500.0
        kap[z0:z1].copy_((v * dt_h) ** 2)
    up.copy_(u)
    torch.cuda.synchronize()


def _domain(decls, names):
    GridBuffer = front.module("grids").GridBuffer
    dummies = {n: GridBuffer(decls[n].dtype, tuple(decls[n].shape), decls[n].order, np.zeros((1,) * len(decls[n].shape)))
               for n in names}
    return DeviceTarget(dummies, names)


def _verdict(max_rel: float, rmsd_rel: float) -> dict:
    return {"max_relative": max_rel, "rmsd_relative": rmsd_rel,
            "reference_default_verdict": "pass" if max_rel <= 1e-7 and rmsd_rel <= 1e-8 else "fail",
            "reference_default_tolerance": "max 1e-7, rmsd 1e-8 (cli.py:37-38)"}


FULL = [
    ("c4", "star3d4r_norm", (1024, 1024, 1024), "f32", 10, "p_c4_star3d4r_norm"),
    ("c3", "wave", (1024, 1024, 1024), "f32", 10, "p_c3_wave"),
    ("c2", "jacobi7", (512, 512, 512), "f32", 100, "p_c2_jacobi7"),
]


@pytest.mark.parametrize("case,builder,shape,dtype,steps,ref_name", FULL, ids=[c[0] for c in FULL])
def test_full_size_n_steps_vs_reference_cpu(case, builder, shape, dtype, steps, ref_name):
    compare = front.module("grids").compare
    GridBuffer = front.module("grids").GridBuffer
    bound, decls = corpus.config_target(builder, shape, steps, dtype)
    names = [g for _, g in bound.grid_params]
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    with _domain(decls, names) as dt:
        if builder == "wave":
            _fill_wave(dt)
        else:
            for n in names:
                _interior(dt, n).zero_()
            _fill_loguniform(_interior(dt, names[0]), 7)
        _torch().cuda.synchronize()
        host = {n: dt.download(n) for n in names}  # the inputs, in GridBuffer.data layout
        dt.set_program(body)
        t0 = time.perf_counter()
        dt.run(steps)
        dt.sync()
        gpu_s = time.perf_counter() - t0
        launches = dt.launches()
        got = {n: dt.download(n) for n in names}
    order = decls[names[0]].order
    cpu_s = ref_runner.call(ref_name, [host[n] for n in names], steps)  # in place: final grids under their names
    result = {"shape": list(shape), "dtype": dtype, "steps": steps, "gpu_launches": launches,
              "gpu_seconds": gpu_s, "cpu_seconds": cpu_s, "cpu_threads": ref_runner.host_cores(),
              "oracle": f"oracle/_ref/{ref_name}.c (reference-emitted OpenMP C, template loop)", "grids": {}}
    for n in names:
        ref = GridBuffer(dtype, shape, order, host[n])
        mine = GridBuffer(dtype, shape, order, got[n])
        rep = compare(ref, mine)
        halo_same = bool(np.array_equal(host[n][:order], got[n][:order]) and
                         np.array_equal(host[n][-order:], got[n][-order:]))
        result["grids"][n] = {**_verdict(rep.max_relative, rep.rmsd_relative), "halo_planes_equal": halo_same}
        assert math.isfinite(rep.max_relative) and rep.scale > 0, n
        assert rep.max_relative <= TOL[dtype], (case, n, rep.render())
        assert halo_same, (case, n)
    _record(case, **result)


WINDOWED = [("c5a", "star3d2r_norm", 2, "p_c5a_star3d2r_norm_win"),
            ("c5b", "star3d4r_norm", 4, "p_c5b_star3d4r_norm_win")]


@pytest.mark.parametrize("case,builder,radius,ref_name", WINDOWED, ids=[c[0] for c in WINDOWED])
def test_c5_full_grid_n_steps_vs_reference_cpu_windows(case, builder, radius, ref_name):
    shape, dtype, steps = (2048, 2048, 1024), "f64", 5
    W = build_ref.PARITY_WINDOW
    reach = steps * radius
    bound, decls = corpus.config_target(builder, shape, steps, dtype)
    names = [g for _, g in bound.grid_params]
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    starts = (0, shape[0] // 2 - W // 2, shape[0] - W)
    R = radius
    padded_win = (W + 2 * R, shape[1] + 2 * R, shape[2] + 2 * R)
    wins_in, wins_out = {}, {}
    with _domain(decls, names) as dt:
        for n in names:
            _interior(dt, n).zero_()
        _fill_loguniform(_interior(dt, "u"), 11)
        for z0 in starts:
            a = np.zeros(padded_win, np.float64)
            a[R:-R, R:-R, R:-R] = _interior(dt, "u")[z0:z0 + W].cpu().numpy()
            wins_in[z0] = a
        dt.set_program(body)
        dt.run(steps)
        dt.sync()
        launches = dt.launches()
        for z0 in starts:
            wins_out[z0] = {n: _interior(dt, n)[z0:z0 + W].cpu().numpy() for n in names}
    result = {"shape": list(shape), "dtype": dtype, "steps": steps, "gpu_launches": launches,
              "oracle": f"oracle/_ref/{ref_name}.c on d0 windows of {W} planes", "windows": {}}
    for z0 in starts:
        arrays = {"u": wins_in[z0], "v": np.zeros(padded_win, np.float64)}
        cpu_s = ref_runner.call(ref_name, [arrays[n] for n in names], steps)
        lo = 0 if z0 == 0 else reach
        hi = W if z0 + W == shape[0] else W - reach
        rec = {"planes": [z0 + lo, z0 + hi], "cpu_seconds": cpu_s}
        for n in names:
            ref = arrays[n][R:-R, R:-R, R:-R][lo:hi]
            mine = wins_out[z0][n][lo:hi]
            diff = np.abs(ref - mine)
            scale = float(np.abs(ref).max())
            max_rel = float(diff.max()) / scale
            rmsd_rel = float(np.sqrt(np.mean(diff * diff))) / scale
            rec[n] = _verdict(max_rel, rmsd_rel)
            assert scale > 0 and max_rel <= TOL[dtype], (case, z0, n, max_rel)
        result["windows"][str(z0)] = rec
    _record(case, **result)


EXACT = [
    ("c4", "star3d4r_norm", (1024, 1024, 1024), "f32", 10, "p_c4_star3d4r_norm"),
    ("c3", "wave", (1024, 1024, 1024), "f32", 3, None),
    ("c2", "jacobi7", (512, 512, 512), "f32", 20, "p_c2_jacobi7"),
]


@pytest.mark.parametrize("case,builder,shape,dtype,steps,ref_name", EXACT, ids=[c[0] for c in EXACT])
def test_full_size_exact_path_bitwise_vs_reference_cpu(case, builder, shape, dtype, steps, ref_name):
    """precision='exact' at the BASELINE sizes (the exact streaming kernels), bit for bit.

    Stars: against the reference-emitted C built without FMA contraction (every term is
    ``double * float`` and every sum is in float64, as in run_target).  The wave: against the
    pinned C restatement of run_target (oracle/stkoracle.c) — the reference's own emitted C is
    NOT bit-identical to its oracle there: ``u[a] + u[b]`` of two ``float`` taps is a
    single-precision addition in C, while run_target sums in float64 (executor.py:1-10)."""
    bound, decls = corpus.config_target(builder, shape, steps, dtype)
    names = [g for _, g in bound.grid_params]
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    GridBuffer = front.module("grids").GridBuffer
    dummies = {n: GridBuffer(decls[n].dtype, tuple(decls[n].shape), decls[n].order, np.zeros((1, 1, 1)))
               for n in names}
    with DeviceTarget(dummies, names, precision="exact") as dt:
        if builder == "wave":
            _fill_wave(dt)
        else:
            for n in names:
                _interior(dt, n).zero_()
            _fill_loguniform(_interior(dt, names[0]), 9)
        _torch().cuda.synchronize()
        host = {n: dt.download(n) for n in names}
        dt.set_program(body)
        dt.run(steps)
        dt.sync()
        kinds = sorted({p.kind for p in dt.plans})
        got = {n: dt.download(n) for n in names}
    assert kinds in (["xstar"], ["xwave"]), kinds
    if ref_name is None:
        from oracle import oracle

        order = decls[names[0]].order
        ins = {n: GridBuffer(dtype, shape, order, host[n]) for n in names}
        outs = oracle.run_target_c(bound, ins)
        host = {n: outs[n].data for n in names}
        what = "oracle/stkoracle.c (run_target's float64 evaluation, pinned to the reference goldens)"
    else:
        ref_runner.call(ref_name, [host[n] for n in names], steps, strict=True)
        what = f"oracle/_ref/{ref_name}.c built with -ffp-contract=off"
    result = {"shape": list(shape), "dtype": dtype, "steps": steps, "device_kernel": kinds[0],
              "oracle": what, "bitwise_equal": {}}
    for n in names:
        same = bool(np.array_equal(host[n].view(np.uint32), got[n].view(np.uint32)))
        result["bitwise_equal"][n] = same
        assert same, (case, n, float(np.abs(host[n].astype(np.float64) - got[n]).max()))
    _record(f"{case}_exact", **result)
