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
from paper_2309_04671_b200.grids import GridBuffer, fill_loguniform
from paper_2309_04671_b200.program import dump

CASES = golden_cases()


def test_fixture_set_present():
    assert len(CASES) >= 12


@pytest.mark.parametrize("case", CASES)
def test_program_builder_matches_reference_binding(case):
    meta, _, ref_dump, _, _ = load_golden(case)
    assert dump(build_case(meta)) == ref_dump


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


def test_loguniform_chunked_stream_identical():
    a = GridBuffer.zeros((9, 7, 5), 2)
    b = GridBuffer.zeros((9, 7, 5), 2)
    fill_loguniform(a, 42)
    fill_loguniform(b, 42, chunk_rows=40)  # forces plane-by-plane draws
    assert np.array_equal(a.data, b.data)


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
