"""`python -m paper_2309_04671_b200 run prog.stpy` end to end on the B200."""

from __future__ import annotations

import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, build_case, load_golden
from oracle import oracle
from paper_2309_04671_b200 import compare
from paper_2309_04671_b200 import load_grid, save_grid

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case,precision", [("star3d4r_16", "exact"), ("wave_16", "fast"), ("j3d27pt_12", "fast")])
def test_cli_run_writes_stg1_grids(tmp_path, case, precision):
    meta, source, _, ins, outs = load_golden(case)
    prog = tmp_path / f"{case}.stpy"
    prog.write_text(source.replace("backend=st.seq()", 'backend=st.cuda(computeCapability="10.0", template=st.CUDABackend.Template.unroll)'))
    args = []
    for name, g in ins.items():
        save_grid(tmp_path / f"in_{name}.grid", g)
        args += ["--grid", f"{name}={tmp_path / f'in_{name}.grid'}"]
    r = subprocess.run([sys.executable, "-m", "paper_2309_04671_b200", "run", str(prog), "-o", str(tmp_path / "out"),
                        "--precision", precision, "--profile", *args], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "wrote" in r.stderr and "execution=" in r.stdout
    for name, ref in outs.items():
        got = load_grid(tmp_path / "out" / f"{name}.grid")
        if precision == "exact":
            assert np.array_equal(got.data, ref.data), name
        else:
            assert compare(ref, got).max_relative <= 1e-5, name


def test_cli_reports_bad_plan_as_exit_1(tmp_path):
    _, source, _, _, _ = load_golden("star3d4r_16")
    prog = tmp_path / "p.stpy"
    prog.write_text(source)
    r = subprocess.run([sys.executable, "-m", "paper_2309_04671_b200", "run", str(prog), "--backend", "gpu",
                        "--template", "tma",
                        "-o", str(tmp_path / "o")], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 1 and "unknown GPU template" in r.stderr
