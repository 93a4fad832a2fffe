"""The .stpy loader reproduces the reference front end's bound programs.

Against the golden fixtures' sources (parsed+bound by the reference when the
fixtures were made) and, where /root/reference is present, every corpus
program and the README listing parsed live by the reference parser."""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

from conftest import golden_cases, load_golden
from paper_2309_04671_b200 import stpy
from paper_2309_04671_b200.program import dump

REF = Path("/root/reference/pkg")


@pytest.mark.parametrize("case", golden_cases())
def test_loader_matches_reference_binding(case):
    meta, source, ref_dump, _, _ = load_golden(case)
    prog = stpy.load(source, f"{case}.stpy")
    scheme = None if meta["scheme"] == "cross_product" else meta["scheme"]
    assert dump(stpy.bind(prog, scheme=scheme)) == ref_dump


def _ref_corpus():
    if not REF.exists():
        return []
    return sorted(p.name for p in (REF / "corpus").glob("*.stpy") if "dataflow" not in p.name)


@pytest.mark.skipif(not REF.exists(), reason="reference not present (GPU box)")
@pytest.mark.parametrize("name", _ref_corpus())
def test_loader_matches_reference_parser_on_corpus(name):
    sys.path.insert(0, str(REF / "src"))
    from stencilkit.analysis import bind_target
    from stencilkit.parser import parse_source

    text = (REF / "corpus" / name).read_text()
    ref = bind_target(parse_source(text, name))
    mine = stpy.bind(stpy.load(text, name))
    assert dump(mine) == dump(ref)


def test_launch_parameters_and_iters_override():
    meta, source, _, _, _ = load_golden("star3d4r_16")
    text = source.replace("backend=st.seq()", "backend=st.cuda(computeCapability=\"10.0\", "
                                              "threadsPerBlock=(32, 4, 4), template=st.CUDABackend.Template.unroll)")
    prog = stpy.load(text)
    assert prog.backend == "gpu"
    assert prog.params == {"computeCapability": "10.0", "threadsPerBlock": (32, 4, 4), "template": "unroll"}
    bound = stpy.bind(prog, iters=7)
    assert bound.stmts[0].count == 7
