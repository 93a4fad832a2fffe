"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

For every case it writes tests/golden/<case>.npz holding
  * ``source``: the .stpy program text, parsed by the reference front end
    (parser.parse_source + validate) and bound by analysis.bind_target;
  * ``dump``: the reference's own analysis dump of the bound program
    (stencilkit.analysis.dump_analysis), for inspection;
  * ``in_<grid>`` / ``out_<grid>``: padded inputs (reference
    grids.fill_loguniform, or the c3 wave initialiser) and the reference
    executor.run_target outputs (float64 accumulate, one rounding).
Nothing here runs on the GPU box; the fixtures travel with the repo.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(REF))

from stencilkit import corpus as ref_corpus  # noqa: E402
from stencilkit.analysis import bind_target, dump_analysis  # noqa: E402
from stencilkit.executor import run_target  # noqa: E402
from stencilkit.grids import GridBuffer, fill_loguniform  # noqa: E402
from stencilkit.parser import parse_source, validate  # noqa: E402

from paper_2309_04671_b200 import corpus  # noqa: E402

# (case, builder, shape, iters, dtype, map_width, scheme, seed)
CASES = [
    ("star3d1r_12", "star3d1r", (12, 12, 12), 3, "f32", 0, None, 7),
    ("star3d2r_12", "star3d2r", (12, 12, 12), 3, "f32", 0, None, 31),
    ("star3d3r_10x12x14", "star3d3r", (10, 12, 14), 2, "f32", 0, None, 5),
    ("star3d4r_16", "star3d4r", (16, 16, 16), 3, "f32", 0, None, 7),
    ("star3d4r_w2_cross", "star3d4r", (14, 13, 18), 2, "f32", 2, "cross_product", 11),
    ("star3d4r_w3_slab7", "star3d4r", (12, 12, 12), 2, "f32", 3, "slab7", 12),
    ("star3d4r_f64", "star3d4r", (12, 12, 12), 3, "f64", 0, None, 19),
    ("star3d4r_norm_16", "star3d4r_norm", (16, 16, 16), 6, "f32", 0, None, 7),
    ("jacobi7_16", "jacobi7", (16, 16, 16), 6, "f32", 0, None, 7),
    ("j3d27pt_12", "j3d27pt", (12, 12, 12), 3, "f32", 0, None, 1),
    ("box3d2r_10", "box3d2r", (10, 10, 10), 2, "f32", 0, None, 2),
    ("star2d4r_24", "star2d4r", (24, 24), 3, "f32", 0, None, 11),
    ("wave_16", "wave", (16, 16, 16), 5, "f32", 0, None, 3),
    ("wave_f64_12", "wave", (12, 12, 12), 4, "f64", 0, None, 3),
]


def source_for(builder, shape, iters, dtype, width):
    if builder in corpus.KERNELS:  # the corpus kernels: the reference's own source_text
        return ref_corpus.source_text(builder, shape=shape, iters=iters, dtype=dtype, map_width=width)
    return corpus.program_text(builder, shape, iters, dtype, width)


def main() -> None:
    import stencilkit

    for case, builder, shape, iters, dtype, width, scheme, seed in CASES:
        text = source_for(builder, shape, iters, dtype, width)
        unit = parse_source(text, f"{case}.stpy")
        diags = validate(unit)
        assert not diags, diags
        bound = bind_target(unit, scheme=scheme)
        grids = {g.name: GridBuffer.zeros(g.shape, g.order, g.dtype) for g in unit.grids}
        if builder == "wave":
            corpus.wave_inputs(grids, seed=seed)
        else:
            fill_loguniform(grids[unit.launch.args[0]], seed)
        out = run_target(bound, grids)
        arrays = {f"in_{n}": b.data for n, b in grids.items()}
        arrays.update({f"out_{n}": b.data for n, b in out.items()})
        meta = dict(case=case, builder=builder, shape=list(shape), iters=iters, dtype=dtype, map_width=width,
                    scheme=scheme or "cross_product", seed=seed, numpy=np.__version__,
                    reference=f"stencilkit {stencilkit.__version__}")
        np.savez_compressed(HERE / f"{case}.npz", meta=json.dumps(meta), source=text, dump=dump_analysis(unit, bound),
                            **arrays)
        print(case, "ok")


if __name__ == "__main__":
    main()
