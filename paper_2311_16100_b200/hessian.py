"""Normal-operator utilities on the B200 path (drop-in for fsld.hessian.hvp / exact_diag).

/root/reference/pkg/src/fsld/hessian.py:62-118.  ``exact_diag`` scatters
C^2 w^2 (tri) or C^2 (nn) for every image in one kernel pass, accumulating
in int64 fixed point (order-independent, so bitwise repeatable).
"""
from __future__ import annotations

import numpy as np

from .engine import SliceEngine, records_for


def hvp(op, z, batch, lam: float, n_total: int | None = None):
    """Unbiased mini-batch Hessian-vector product (hessian.py:110-118)."""
    return op.hvp(z, batch, lam, n_total)


def exact_diag(poses, ctfs, lam: float, mode: str, spec, mask, dedupe: bool = False) -> np.ndarray:
    """Exact diagonal of H = sum_i P_i^* C_i^2 P_i + lam I (hessian.py:62-107)."""
    if lam < 0:
        raise ValueError("lam must be non-negative")
    if dedupe and mode != "nn":
        raise ValueError("dedupe is only defined for nn mode")
    if dedupe:
        raise NotImplementedError("dedupe (hit-count analysis path) is outside the B200 hot path")
    quats = np.array([p.q for p in poses], dtype=np.float64)
    recs = records_for(spec.M, quats, None, ctfs)
    e = SliceEngine(spec.M, mode, mask, recs, None, deterministic=True)
    acc, fx = e.exact_diag_acc(e.all_indices())
    return e.finalize_r(acc, fx, 1.0, 0.0).cpu().numpy().astype(np.float64) + lam
