"""Page-locked host memory for ``run_gpu(..., pinned=True)`` results.

The arrays ``run_gpu`` returns are fresh host buffers (the reference's ``run_tile_plan``
returns new ``GridBuffer``s, executor.py:491-557).  Device→host copies into pageable
memory run at a fraction of PCIe speed and fault every page in on first touch, so the
pinned variant hands out arrays over page-locked blocks instead, from a caching pool:

* blocks are exactly the array's size (anonymous ``mmap`` + ``cudaHostRegister``) —
  torch's caching host allocator rounds every block up to a power of two, which a 35 GB
  c5 grid cannot afford on a 196 GB host;
* a block goes back to the pool when the last numpy view of it dies (a ``weakref``
  finaliser on the buffer owner, which every view keeps alive), and the next call of the
  same size reuses it without registering again;
* a miss first releases the free blocks of other sizes, so the pool holds at most the
  blocks in use plus one size class.

``release()`` (also at exit) unregisters and unmaps the free blocks.
"""

from __future__ import annotations

import atexit
import ctypes
import mmap
import threading
import weakref

import numpy as np


class _Block:
    __slots__ = ("mm", "anchor", "ptr", "nbytes")

    def __init__(self, nbytes: int):
        self.nbytes = nbytes
        self.mm = mmap.mmap(-1, nbytes)
        self.anchor = ctypes.c_char.from_buffer(self.mm)  # an export: keeps the mapping in place
        self.ptr = ctypes.addressof(self.anchor)

    def close(self) -> None:
        self.anchor = None
        self.mm.close()


class _Lease:
    """Owner of one block while arrays view it (numpy keeps it as the views' base)."""

    __slots__ = ("_mv", "__weakref__")

    def __init__(self, mv: memoryview):
        self._mv = mv

    def __buffer__(self, flags):
        return self._mv


class PinnedPool:
    def __init__(self):
        self._free: dict = {}  # nbytes -> [_Block]
        self._lock = threading.Lock()
        self.registered = 0  # blocks registered so far (a hit does not register)

    def array(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        count = int(np.prod(shape))
        nbytes = count * dtype.itemsize
        if nbytes == 0:
            return np.empty(shape, dtype=dtype)
        blk = None
        stale = []
        with self._lock:
            lst = self._free.get(nbytes)
            if lst:
                blk = lst.pop()
            else:
                for k in [k for k in self._free if k != nbytes]:
                    stale += self._free.pop(k)
        for b in stale:
            _unregister(b)
        if blk is None:
            blk = _Block(nbytes)
            try:
                _register(blk)
            except BaseException:
                blk.close()
                raise
            self.registered += 1
        lease = _Lease(memoryview(blk.mm))
        weakref.finalize(lease, self._give_back, blk)
        return np.frombuffer(lease, dtype=dtype, count=count).reshape(shape)

    def _give_back(self, blk: _Block) -> None:
        with self._lock:
            self._free.setdefault(blk.nbytes, []).append(blk)

    def free_bytes(self) -> int:
        with self._lock:
            return sum(b.nbytes for lst in self._free.values() for b in lst)

    def release(self) -> None:
        with self._lock:
            blocks = [b for lst in self._free.values() for b in lst]
            self._free.clear()
        for b in blocks:
            _unregister(b)


def _register(blk: _Block) -> None:
    import torch

    rc = torch.cuda.cudart().cudaHostRegister(blk.ptr, blk.nbytes, 0)
    if int(rc) != 0:
        raise MemoryError(f"cudaHostRegister of {blk.nbytes} B failed ({rc})")


def _unregister(blk: _Block) -> None:
    try:
        import torch

        torch.cuda.cudart().cudaHostUnregister(blk.ptr)
    except Exception:  # interpreter shutdown / no CUDA: the mapping goes anyway
        pass
    blk.close()


POOL = PinnedPool()
atexit.register(POOL.release)
