"""Build oracle/_ref: the REFERENCE's own CPU path for the bench workloads.

The reference's CPU implementation of the hot path is the OpenMP C it emits
(codegen/openmp.py:14-53, template ``loop``: ``#pragma omp parallel for``
over d0, float64 per point, one rounding) with the C-ABI of
codegen/serial.py:126-208 (``void run_<target>(T *u, T *v, ..., int64_t
iter)``).  This script — run only where /root/reference exists — parses
each bench program with the reference front end, lets the reference emit
that C (``codegen.generate(unit, bound, "omp", plan_omp(info, {"template":
"loop"}))``), and compiles it with gcc into oracle/_ref/<name>.so.  Only the
generated .c/.so land in oracle/_ref/ (git-ignored; they travel to the GPU
box with the snapshot).  No reference source is copied.

    python oracle/build_ref.py
"""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
OUT = HERE / "_ref"
REF_SRC = Path("/root/reference/pkg/src")

# name -> (program builder, sample shape, dtype); samples bound the CPU time
SAMPLES = {
    "c1_star3d4r": ("star3d4r", (128, 128, 128), "f32"),
    "c2_jacobi7": ("jacobi7", (128, 512, 512), "f32"),
    "c3_wave": ("wave", (64, 1024, 1024), "f32"),
    "c4_star3d4r_norm": ("star3d4r_norm", (64, 1024, 1024), "f32"),
    "c5_star3d2r_norm_f64": ("star3d2r_norm", (32, 2048, 1024), "f64"),
    "c5_star3d4r_norm_f64": ("star3d4r_norm", (32, 2048, 1024), "f64"),
}
# full-size parity programs (tests/test_gpu_parity_full.py): the BASELINE configs at their
# own shapes; c5 (2048 x 2048 x 1024 fp64) as d0 windows of PARITY_WINDOW planes of the
# full grid (outputs more than steps x radius planes from a cut are exact, see the test)
PARITY_WINDOW = 104
PARITY = {
    "p_c2_jacobi7": ("jacobi7", (512, 512, 512), "f32"),
    "p_c3_wave": ("wave", (1024, 1024, 1024), "f32"),
    "p_c4_star3d4r_norm": ("star3d4r_norm", (1024, 1024, 1024), "f32"),
    "p_c5a_star3d2r_norm_win": ("star3d2r_norm", (PARITY_WINDOW, 2048, 1024), "f64"),
    "p_c5b_star3d4r_norm_win": ("star3d4r_norm", (PARITY_WINDOW, 2048, 1024), "f64"),
}
CFLAGS = ["-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared"]


def available() -> bool:
    return REF_SRC.exists()


def program_text(builder: str, shape, dtype: str) -> str:
    sys.path.insert(0, str(ROOT))
    from paper_2309_04671_b200 import corpus

    return corpus.program_text(builder, shape, 1, dtype, backend="st.omp()")


def build(force: bool = False) -> dict:
    if not available():
        raise RuntimeError("the reference is not present here; oracle/_ref is built in the build container")
    sys.path.insert(0, str(REF_SRC))
    from stencilkit.analysis import bind_target
    from stencilkit.codegen import generate
    from stencilkit.parser import parse_source, validate
    from stencilkit.planning import plan_omp

    OUT.mkdir(exist_ok=True)
    manifest = {}
    for name, (builder, shape, dtype) in {**SAMPLES, **PARITY}.items():
        text = program_text(builder, shape, dtype)
        unit = parse_source(text, f"{name}.stpy")
        assert not validate(unit)
        bound = bind_target(unit, freeze_loop_bounds=False)  # keep `iter` a runtime argument
        first = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body[0]
        plan = plan_omp(first.info, {"template": "loop"})
        art = generate(unit, bound, "omp", plan)
        (rel, src), = art.files
        c_path = OUT / f"{name}.c"
        so_path = OUT / f"{name}.so"
        if force or not c_path.exists() or c_path.read_text() != src or not so_path.exists():
            c_path.write_text(src)
            subprocess.run(["gcc", *CFLAGS, str(c_path), "-o", str(so_path)], check=True)
        manifest[name] = dict(builder=builder, shape=list(shape), dtype=dtype, entry=art.entry,
                              grids=[g for _, g in bound.grid_params], source=c_path.name, lib=so_path.name,
                              emitted_as=rel, template="loop", cflags=CFLAGS)
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1))
    return manifest


if __name__ == "__main__":
    m = build(force="--force" in sys.argv)
    print("\n".join(f"{k}: {v['entry']} {v['shape']}" for k, v in m.items()))
