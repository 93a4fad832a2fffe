"""The oracle is pinned against the reference's own outputs (tests/golden/).

Fixtures were produced by running the reference (parse_source -> bind_target
-> run_target, pkg/src/stencilkit) on the programs in each file; see
tests/golden/make_golden.py.  Bit-for-bit equality is required: the oracle
restates the reference's float64-accumulate / round-once arithmetic.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import build_case, golden_cases, load_golden
from oracle import oracle
from paper_2309_04671_b200 import GridBuffer, corpus, fill_loguniform

CASES = golden_cases()


def test_fixture_set_present():
    assert len(CASES) >= 12


@pytest.mark.parametrize("case", CASES)
def test_config_programs_are_the_golden_sources(case):
    """corpus.config_target emits exactly the program text the reference ran for
    the fixture, so every test and bench program is a reference-checked one."""
    meta, source, _, _, _ = load_golden(case)
    b, shape = meta["builder"], tuple(meta["shape"])
    if b in corpus.KERNELS:
        text = corpus.front.module("corpus").source_text(b, shape=shape, iters=meta["iters"], dtype=meta["dtype"],
                                                          map_width=meta["map_width"])
    else:
        text = corpus.program_text(b, shape, meta["iters"], meta["dtype"], meta["map_width"])
    assert text == source


@pytest.mark.parametrize("case", CASES)
def test_numpy_oracle_bitwise(case):
    meta, _, _, ins, outs = load_golden(case)
    got = oracle.run_target(build_case(meta), ins)
    for name, ref in outs.items():
        assert np.array_equal(got[name].data, ref.data), name


@pytest.mark.parametrize("case", CASES)
def test_c_oracle_bitwise(case):
    meta, _, _, ins, outs = load_golden(case)
    got = oracle.run_target_c(build_case(meta), ins, threads=2)
    for name, ref in outs.items():
        assert np.array_equal(got[name].data, ref.data), name


@pytest.mark.parametrize("case", [c for c in CASES if not c.startswith("wave")])
def test_loguniform_inputs_reproduced(case):
    meta, _, _, ins, _ = load_golden(case)
    g = GridBuffer.zeros(tuple(meta["shape"]), ins["u"].order, meta["dtype"])
    fill_loguniform(g, meta["seed"])
    assert np.array_equal(g.data, ins["u"].data)


def test_oracle_halo_never_written():
    meta, _, _, ins, _ = load_golden("star3d4r_16")
    before = {n: b.halo_bytes() for n, b in ins.items()}
    out = oracle.run_target_c(build_case(meta), ins, threads=2)
    for n, b in out.items():
        assert b.halo_bytes() == before[n]


def test_oracle_nonfinite_warned():
    meta, _, _, ins, _ = load_golden("star3d4r_16")
    ins["u"].interior[3, 4, 5] = np.inf
    with pytest.warns(RuntimeWarning, match="non-finite"):
        oracle.run_target(build_case(meta), ins)
