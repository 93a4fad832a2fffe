"""The criterion-10 shim (shim.py), without a GPU: `emit` gives the reference's own C entry
`run_<target>(T*..., int64_t iter)` over libstkb200.so for every map kind it routes to (fast and
exact star / box / wave, box coefficient tables beyond 125 values, 2-D grids), and the artifact
compiles and loads like the reference's ctypes harness does it (test_acceptance.py:325-343)."""

from __future__ import annotations

import ctypes
import shutil

import pytest

from paper_2309_04671_b200 import front, shim

sk_corpus = front.module("corpus")
sk_parser = front.module("parser")


@pytest.mark.skipif(shutil.which("cc") is None, reason="needs a C compiler")
@pytest.mark.parametrize("name,shape", [("star3d4r", (12, 12, 12)), ("box3d4r", (10, 10, 10)), ("j3d27pt", (8, 9, 10)),
                                        ("box2d4r", (16, 16)), ("star2d1r", (10, 12))])
@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_emit_compiles_and_loads(tmp_path, name, shape, precision):
    unit = sk_parser.parse_source(sk_corpus.source_text(name, shape=shape, iters=2), f"{name}.stpy")
    art = shim.emit(unit, precision=precision)
    assert art.entry == f"run_target_{name}"
    text = art.files[0][1]
    assert f"void {art.entry}(" in text and "int64_t" in text
    if name == "box3d4r":
        assert "cube_0[]" in text  # 729 coefficients through box_coef_ext
    so = shim.build(art, tmp_path)
    assert hasattr(ctypes.CDLL(str(so)), art.entry)
