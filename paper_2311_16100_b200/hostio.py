"""Host-side staging of the numpy (reference-signature) calls: pinned buffers and threaded casts.

The reference's callers hand ``loss_and_grad`` a numpy complex128 volume and expect a numpy
complex128 gradient (optim.py:165-190).  The device works in complex64, so each call casts v into a
page-locked complex64 buffer (the copy engines then stream it at full PCIe rate) and casts the
pinned complex64 gradient back into a fresh complex128 array.  numpy's casting loops release the
GIL, so the casts are split over a thread pool (one chunk per core).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_POOL = None
_WORKERS = max(1, min(16, os.cpu_count() or 1))
_MIN_CHUNK = 1 << 16  # elements per task (smaller arrays cast on the calling thread)


def _pool() -> ThreadPoolExecutor:
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=_WORKERS, thread_name_prefix="fsld-cast")
    return _POOL


def cast_into(dst: np.ndarray, src: np.ndarray) -> np.ndarray:
    """dst[...] = src (any numeric cast), flat, in parallel chunks."""
    d = dst.reshape(-1)
    s = np.asarray(src).reshape(-1)
    if d.size != s.size:
        raise ValueError(f"size mismatch {s.size} -> {d.size}")
    n = d.size
    k = min(_WORKERS, max(1, n // _MIN_CHUNK))
    if k == 1:
        np.copyto(d, s, casting="unsafe")
        return dst
    step = -(-n // k)
    futs = [_pool().submit(np.copyto, d[i:i + step], s[i:i + step], casting="unsafe") for i in range(0, n, step)]
    for f in futs:
        f.result()
    return dst


def cast_native(fn, src_ptr: int, dst_ptr: int, n: int, src_item: int, dst_item: int) -> None:
    """Run a fsld_host_cast_* over n reals split into 16-byte-aligned chunks on the thread pool
    (ctypes releases the GIL for the foreign call, so the chunks run in parallel)."""
    k = min(_WORKERS, max(1, n // (4 * _MIN_CHUNK)))
    step = (-(-n // k) + 3) & ~3  # multiple of 4 reals: each chunk start stays 16-byte aligned
    jobs = [(i, min(step, n - i)) for i in range(0, n, step)]
    if len(jobs) == 1:
        if fn(src_ptr, dst_ptr, n) != 0:
            raise ValueError("host cast failed")
        return
    futs = [_pool().submit(fn, src_ptr + i * src_item, dst_ptr + i * dst_item, m) for i, m in jobs]
    for f in futs:
        if f.result() != 0:
            raise ValueError("host cast failed")


class PinnedArrays:
    """Recycled page-locked numpy arrays for results handed to the caller (the numpy call path's
    complex128 gradients).  The copy engine writes them directly (no host cast, no first-touch page
    faults of a fresh array); an array goes back to the pool when the caller drops it."""

    def __init__(self, n: int, dtype, keep: int = 8):
        self.n, self.dtype, self.keep = int(n), dtype, keep
        self.free: list = []
        self.live = 0

    def get(self):
        """(numpy array, backing pinned tensor) -- None when `keep` arrays are already out."""
        import weakref

        import torch
        from . import _capi as C
        if self.free:
            t = self.free.pop()
        elif self.live < self.keep:
            t = C.host_empty(self.n, self.dtype)
            self.live += 1
        else:
            return None
        arr = t.numpy()
        weakref.finalize(arr, self.free.append, t)
        return arr, t
