"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

from paper_2309_04671_b200 import corpus  # noqa: E402
from paper_2309_04671_b200 import GridBuffer  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built CUDA library")


def golden_cases():
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load_golden(case: str):
    """(meta, source, dump, inputs {name: GridBuffer}, outputs {name: GridBuffer})."""
    z = np.load(GOLDEN / f"{case}.npz")
    meta = json.loads(str(z["meta"]))
    order = _order(meta)
    shape = tuple(meta["shape"])
    ins, outs = {}, {}
    for k in z.files:
        if k.startswith("in_"):
            ins[k[3:]] = GridBuffer(meta["dtype"], shape, order, z[k].copy())
        elif k.startswith("out_"):
            outs[k[4:]] = GridBuffer(meta["dtype"], shape, order, z[k].copy())
    return meta, str(z["source"]), str(z["dump"]), ins, outs


def _order(meta) -> int:
    b = meta["builder"]
    if b == "wave":
        return 4
    if b == "jacobi7":
        return 1
    return corpus.KERNELS[b.removesuffix("_norm")].radius


def build_case(meta):
    """The reference-bound BoundTarget of a golden case: the very program text the
    reference ran to make the fixture, parsed and bound by the reference front end."""
    z = np.load(GOLDEN / f"{meta['case']}.npz")
    return corpus.bind_text(str(z["source"]), meta["iters"], meta["scheme"], f"{meta['case']}.stpy")[0]


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
