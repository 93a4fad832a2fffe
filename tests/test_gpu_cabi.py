"""The raw C-ABI driven with ctypes exactly as INTEGRATION.md shows (the
reference's criterion-10 style), checked against the oracle."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import oracle
from paper_2309_04671_b200 import _lib as L
from paper_2309_04671_b200 import compare, corpus
from paper_2309_04671_b200 import GridBuffer, fill_loguniform
from paper_2309_04671_b200.matcher import coef_index

pytestmark = pytest.mark.gpu


def test_stkb_run_target_ctypes_stub():
    shape, iters = (40, 36, 68), 7
    bound, decls = corpus.corpus_target("star3d4r", shape, iters)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    fill_loguniform(grids["u"], 2)
    ref = oracle.run_target(bound, grids)

    lib = L.load()
    desc = L.DomainDesc(dtype=L.STKB_F32, ndim=3, order=4, n_grids=2, device=0)
    desc.shape[:] = shape
    dom = ctypes.c_void_p()
    L.check("create", lib.stkb_domain_create(ctypes.byref(desc), ctypes.byref(dom)))
    try:
        coefs = [0.0] * 25
        for off, c in corpus.coefficients(corpus.KERNELS["star3d4r"]):
            coefs[coef_index(off, 4)] = c
        m = L.MapDesc(kind=L.STKB_MAP_STAR, radius=4, src=0, dst=1, prev=-1, vel=-1)
        m.coef[:25] = coefs
        m.lo[:], m.hi[:] = (0, 0, 0), shape
        L.check("map", lib.stkb_program_add_map(dom, ctypes.byref(m)))
        L.check("swap", lib.stkb_program_add_swap(dom, 1, 0))
        u = grids["u"].data.copy()
        v = grids["v"].data.copy()
        bufs = (ctypes.c_void_p * 2)(u.ctypes.data, v.ctypes.data)
        L.check("run", lib.stkb_run_target(dom, bufs, ctypes.c_int64(iters)))
    finally:
        lib.stkb_domain_destroy(dom)
    for name, arr in (("u", u), ("v", v)):
        got = GridBuffer("f32", shape, 4, arr)
        assert compare(ref[name], got).max_relative <= 1e-5, name


def test_bad_map_is_reported_not_run():
    lib = L.load()
    desc = L.DomainDesc(dtype=L.STKB_F32, ndim=3, order=2, n_grids=2, device=0)
    desc.shape[:] = (8, 8, 8)
    dom = ctypes.c_void_p()
    L.check("create", lib.stkb_domain_create(ctypes.byref(desc), ctypes.byref(dom)))
    try:
        m = L.MapDesc(kind=L.STKB_MAP_STAR, radius=4, src=0, dst=1, prev=-1, vel=-1)
        m.hi[:] = (8, 8, 8)
        assert lib.stkb_program_add_map(dom, ctypes.byref(m)) == L.STKB_ERR_ARG
        assert b"radius exceeds" in lib.stkb_last_error()
        m.radius, m.dst = 2, 0
        assert lib.stkb_program_add_map(dom, ctypes.byref(m)) == L.STKB_ERR_ARG
        assert b"same grid" in lib.stkb_last_error()
    finally:
        lib.stkb_domain_destroy(dom)


def test_device_out_of_memory_is_an_execution_error():
    """A target larger than the GPU's memory fails as the reference's ExecutionError (the CLI's
    exit 1), not a crash; the device stays usable.  Host grids are lazily allocated zeros."""
    from paper_2309_04671_b200 import GridBuffer, corpus, plan_gpu, run_gpu
    from paper_2309_04671_b200.backend import ExecutionError, release_device_cache

    release_device_cache()
    bound, decls = corpus.config_target("star3d1r", (2048, 2048, 3000), 2, "f64")  # 2 x 101 GB
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    bmap = next(s for s in bound.stmts[0].body if type(s).__name__ == "BoundMap")
    plan = plan_gpu(bmap.info, {"template": "unroll", "computeCapability": "10.0"})
    with pytest.raises(ExecutionError, match="out of memory"):
        run_gpu(bound, plan, grids)
    del grids
    small, sdecls = corpus.config_target("star3d1r", (16, 16, 16), 2, "f32")
    g2 = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in sdecls.items()}
    g2["u"].interior[...] = 1.0
    out = run_gpu(small, plan_gpu(next(s for s in small.stmts[0].body if type(s).__name__ == "BoundMap").info,
                                  {"template": "unroll"}), g2)
    assert np.isfinite(out["u"].data).all()
