"""Randomised parity on the B200 (tools/fuzz_parity.py): random corpus kernel, shape, step
count, dtype, precision, template and region width against the C oracle — exact bitwise,
fast within 1e-5 (fp32) / 1e-12 (fp64)."""

from __future__ import annotations

import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [101, 202])
def test_random_programs_match_the_oracle(seed):
    sys.path.insert(0, str(ROOT / "tools"))
    import fuzz_parity

    assert fuzz_parity.main(150, seed) == 0
