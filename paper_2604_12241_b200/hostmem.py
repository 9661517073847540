"""Page-locked host buffers for mined feature blocks.

The reference's `mine` allocates `FeatureMatrix.values` with a pageable
`np.zeros` (engine.py:693).  A device-to-host copy into pageable memory
blocks the host thread and goes through the driver's staging buffers, so the
8-piece D2H overlap of tm_mine (tempmine_b200.h) would be lost.  Here the
block comes from `tm_host_alloc` (cudaHostAlloc) instead; when the last
array viewing a block is garbage collected the block returns to a small
pool, so a `mine` called in a loop re-uses its pinned pages instead of
pinning (and zero-filling) tens of GB again every call.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _lib

KEEP_BLOCKS = 2  # freed blocks kept for re-use

_pool: list[tuple[int, int]] = []  # (capacity bytes, pointer)
stats = {"fresh": 0, "reused": 0, "returned": 0}  # block counters (diagnostics)
_lock = threading.Lock()


class _Block:
    """Owner of one pinned allocation; numpy arrays keep it alive via .base."""

    __slots__ = ("ptr", "nbytes", "__weakref__")

    def __init__(self, ptr: int, nbytes: int):
        self.ptr = ptr
        self.nbytes = nbytes

    @property
    def __array_interface__(self):
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False), "version": 3}


def _release(ptr: int, nbytes: int) -> None:
    with _lock:
        stats["returned"] += 1
        _pool.append((nbytes, ptr))
        _pool.sort()
        while len(_pool) > KEEP_BLOCKS:
            _, p = _pool.pop(0)  # the smallest block goes back to the driver
            _lib.load().tm_host_free(ctypes.c_void_p(p))


def _take(nbytes: int) -> tuple[int, int] | None:
    with _lock:
        for i, (cap, p) in enumerate(_pool):  # sorted: best fit first
            if nbytes <= cap <= 2 * nbytes + (64 << 20):
                return _pool.pop(i)
    return None


def pinned_empty(shape: tuple, dtype=np.int64) -> np.ndarray:
    """Uninitialised C-ordered array in page-locked host memory (pageable
    np.empty if the driver refuses to pin that much)."""
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) * dtype.itemsize
    if n == 0:
        return np.empty(shape, dtype=dtype)
    got = _take(n)
    if got is None:
        p = ctypes.c_void_p()
        lib = _lib.load()
        if lib.tm_host_alloc(n, ctypes.byref(p)) != _lib.TM_OK or not p.value:
            return np.empty(shape, dtype=dtype)
        got = (n, p.value)
        stats["fresh"] += 1
    else:
        stats["reused"] += 1
    cap, ptr = got
    blk = _Block(ptr, cap)
    fin = weakref.finalize(blk, _release, ptr, cap)
    fin.atexit = False  # the process exit returns pinned pages anyway
    return np.asarray(blk)[:n].view(dtype).reshape(shape)


def is_pinned(a: np.ndarray) -> bool:
    base = a
    while isinstance(base, np.ndarray) and base.base is not None:
        base = base.base
    return isinstance(base, _Block)
