"""The drop-in's wiring into the reference, checked without a GPU.

`integrate.install()` rebinds the reference's own `stencilkit.executor.run_tile_plan` (and the
CLI's reference to it): GPU plans go to `run_gpu`, every other plan to the original emulation,
unchanged; `uninstall()` restores it.  `python -m paper_2309_04671_b200` is the reference CLI
with the drop-in installed (commands that do not execute a GPU plan run as they always did).
"""

from __future__ import annotations

import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2309_04671_b200 import backend, front, integrate

sk_corpus = front.module("corpus")
sk_executor = front.module("executor")
sk_parser = front.module("parser")
sk_planning = front.module("planning")
sk_grids = front.module("grids")
sk_analysis = front.module("analysis")


def _unit(name="star3d2r", shape=(8, 8, 8), iters=2):
    unit = sk_parser.parse_source(sk_corpus.source_text(name, shape=shape, iters=iters), "t.stpy")
    assert not sk_parser.validate(unit)
    return unit


def _info(unit):
    k = unit.kernels[0]
    gp = [n for n, t in k.params if t == "grid"]
    return sk_analysis.analyze_kernel(k, dict(zip(gp, unit.grids)))


def test_install_patches_and_uninstall_restores():
    original = sk_executor.run_tile_plan
    try:
        patched = integrate.install("fast")
        assert sk_executor.run_tile_plan is patched and front.module("cli").run_tile_plan is patched
        assert integrate.installed() and patched.__wrapped__ is original
        again = integrate.install("exact")  # re-installing wraps the original, not the wrapper
        assert again.__wrapped__ is original
    finally:
        integrate.uninstall()
    assert sk_executor.run_tile_plan is original and not integrate.installed()


def test_non_gpu_plans_keep_the_reference_emulation():
    unit = _unit()
    grids = {g.name: sk_grids.GridBuffer.zeros(g.shape, g.order, g.dtype) for g in unit.grids}
    sk_grids.fill_loguniform(grids["u"], 3)
    ref = sk_executor.run_target(unit, grids)
    try:
        integrate.install()
        out = sk_executor.run_tile_plan(unit, sk_planning.plan_omp(_info(unit), {"template": "loop"}), grids)
    finally:
        integrate.uninstall()
    assert np.array_equal(out["u"].data, ref["u"].data)


def test_gpu_plans_reach_run_gpu(monkeypatch):
    seen = {}

    def fake_run_gpu(unit, plan, grids, bindings=None, target=None, args=None, scheme=None, *, precision="fast",
                     **kw):
        seen.update(plan=plan, precision=precision)
        return {n: b.copy() for n, b in grids.items()}

    monkeypatch.setattr(integrate, "run_gpu", fake_run_gpu)
    unit = _unit()
    grids = {g.name: sk_grids.GridBuffer.zeros(g.shape, g.order, g.dtype) for g in unit.grids}
    plan = sk_planning.plan_gpu(_info(unit), {"template": "unroll", "computeCapability": "10.0"})
    try:
        integrate.install()
        sk_executor.run_tile_plan(unit, plan, grids)
        assert seen["plan"] is plan and seen["precision"] == "exact"  # the patch's default
        monkeypatch.setenv("STKB_PRECISION", "fast")
        sk_executor.run_tile_plan(unit, plan, grids)
        assert seen["precision"] == "fast"
    finally:
        integrate.uninstall()


def test_without_the_library_the_gpu_path_raises_not_falls_back(monkeypatch):
    """No silent CPU fallback: a missing libstkb200.so is an error on the GPU path."""
    from paper_2309_04671_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setenv("STKB_LIB", str(ROOT / "does_not_exist.so"))
    unit = _unit()
    grids = {g.name: sk_grids.GridBuffer.zeros(g.shape, g.order, g.dtype) for g in unit.grids}
    plan = sk_planning.plan_gpu(_info(unit), {"template": "unroll"})
    with pytest.raises(ImportError, match="no CPU fallback"):
        backend.run_gpu(unit, plan, grids)


@pytest.mark.parametrize("args", [["inspect", "--plan"], ["run", "--backend", "seq", "--random-init", "3"],
                                  ["run", "--backend", "omp", "--template", "loop", "--random-init", "3", "--oracle"]])
def test_cli_wrapper_runs_the_reference_commands(tmp_path, args):
    """Commands without a GPU plan: the reference's own behaviour, through the wrapper."""
    prog = tmp_path / "p.stpy"
    prog.write_text(sk_corpus.source_text("star3d1r", shape=(8, 8, 8), iters=2))
    cmd = [sys.executable, "-m", "paper_2309_04671_b200", args[0], str(prog), *args[1:]]
    if args[0] == "run":
        cmd += ["-o", str(tmp_path / "out")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr


def test_cli_wrapper_rejects_a_bad_precision(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_2309_04671_b200", "run", "x.stpy", "--precision", "half"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 1 and "fast or exact" in r.stderr
