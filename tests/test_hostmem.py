"""The exact-size page-locked host pool behind run_gpu(pinned=True) (hostmem.py), on CPU:
registration is faked, lifetimes and reuse are real."""

from __future__ import annotations

import gc

import numpy as np
import pytest

from paper_2309_04671_b200 import hostmem


@pytest.fixture
def pool(monkeypatch):
    log = []
    monkeypatch.setattr(hostmem, "_register", lambda b: log.append(("reg", b.nbytes)))
    monkeypatch.setattr(hostmem, "_unregister", lambda b: (log.append(("unreg", b.nbytes)), b.close()))
    p = hostmem.PinnedPool()
    p.log = log
    yield p
    p.release()


def test_exact_size_and_reuse_after_the_last_view_dies(pool):
    a = pool.array((3, 5, 7), np.float64)
    assert a.shape == (3, 5, 7) and a.dtype == np.float64 and a.flags.writeable
    assert pool.log == [("reg", 3 * 5 * 7 * 8)]  # exact bytes, not a power of two
    a[...] = 2.5
    view = a[1:, 2:4]  # a GridBuffer.interior-like view outlives the array
    del a
    gc.collect()
    assert pool.free_bytes() == 0  # still viewed: not back in the pool
    assert np.all(view == 2.5)
    del view
    gc.collect()
    assert pool.free_bytes() == 3 * 5 * 7 * 8
    b = pool.array((3, 5, 7), np.float64)  # same size: reused, no new registration
    assert pool.registered == 1 and len(pool.log) == 1
    del b


def test_a_miss_releases_other_sizes(pool):
    a = pool.array((64,), np.float32)
    del a
    gc.collect()
    b = pool.array((32,), np.float64)  # 256 B again: a hit
    assert pool.registered == 1
    del b
    gc.collect()
    c = pool.array((100,), np.float32)  # a miss frees the 256-B block first
    assert ("unreg", 256) in pool.log and pool.registered == 2
    assert pool.free_bytes() == 0
    del c


def test_live_blocks_are_never_handed_out_twice(pool):
    a = pool.array((16,), np.float32)
    b = pool.array((16,), np.float32)
    a[...] = 1
    b[...] = 2
    assert np.all(a == 1) and np.all(b == 2) and pool.registered == 2


def test_empty_arrays_need_no_block(pool):
    assert pool.array((0, 4), np.float32).shape == (0, 4) and pool.registered == 0
