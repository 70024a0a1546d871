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
    if dedupe:  # the idealised analysis path: one (lowest-pixel-index) hit per image and voxel
        return _exact_diag_nn_dedupe(poses, ctfs, spec, mask) + lam
    quats = np.array([p.q for p in poses], dtype=np.float64)
    recs = records_for(spec.M, quats, None, ctfs)
    e = SliceEngine(spec.M, mode, mask, recs, None, deterministic=True)
    acc, fx = e.exact_diag_acc(e.all_indices())
    return e.finalize_r(acc, fx, 1.0, 0.0).cpu().numpy().astype(np.float64) + lam


def hit_counts(poses, spec, mask) -> np.ndarray:
    """Per-voxel number of images whose nearest-neighbour slice reaches the voxel, each image counted
    once per voxel (hessian.py:45-59).  The bit-exact nn voxel indices come from the fsld_assign_nn
    kernel; the per-image de-duplication and the count are host bincounts."""
    quats = np.array([p.q for p in poses], dtype=np.float64)
    e = SliceEngine(spec.M, "nn", mask, records_for(spec.M, quats), None)
    counts = np.zeros(spec.n_voxels, dtype=np.int64)
    for lo in range(0, len(poses), 4096):
        idx = e.assign_nn(np.arange(lo, min(lo + 4096, len(poses)))).cpu().numpy().astype(np.int64)
        idx.sort(axis=1)
        first = np.ones_like(idx, dtype=bool)
        first[:, 1:] = idx[:, 1:] != idx[:, :-1]
        counts += np.bincount(idx[first], minlength=spec.n_voxels)
    return counts


def condition_number(diag, spec=None, restrict_radius: int | None = None) -> float:
    """max / min of a diagonal Hessian, optionally over voxels of rounded radius <= restrict_radius
    (hessian.py:121-145)."""
    d = np.asarray(diag, dtype=np.float64)
    if restrict_radius is not None:
        if spec is None:
            raise ValueError("restrict_radius requires the grid spec")
        d = d[np.round(spec.voxel_radii()) <= restrict_radius]
    if d.size == 0:
        raise ValueError("no entries selected")
    lo = d.min()
    if lo <= 0:
        raise ValueError("non-positive diagonal entry: lam = 0 with an unhit voxel makes the condition "
                         "number undefined")
    return float(d.max() / lo)


def cond_bound_is_exact(n_images: int, p_of_r: float) -> bool:
    """1/p(R) > N: some voxel is certainly unhit and kappa = (N + lam) / lam (hessian.py:148-150)."""
    return 1.0 / p_of_r > n_images


def cond_lower_bound(n_images: int, lam: float, p_of_r: float) -> float:
    """Pigeonhole lower bound on kappa(H) from the pixel / voxel ratio p(R) (hessian.py:153-167)."""
    if not 0.0 < p_of_r <= 1.0:
        raise ValueError("p_of_r must lie in (0, 1]")
    if lam < 0:
        raise ValueError("lam must be non-negative")
    if cond_bound_is_exact(n_images, p_of_r):
        return float(np.inf) if lam == 0 else (n_images + lam) / lam
    return (n_images + lam) / (p_of_r * n_images + lam)


def condition_report(poses, ctfs, lam: float, spec, mask, radii) -> dict:
    """Per-radius measured condition numbers (nn diagonal: hit counts without CTF, the CTF-weighted
    exact diagonal with it) and the lower bound (hessian.py:170-210)."""
    from .grid import shell_table

    counts = hit_counts(poses, spec, mask)
    diag_noctf = counts.astype(np.float64) + lam
    diag_ctf = exact_diag(poses, ctfs, lam, "nn", spec, mask) if ctfs is not None else None
    shells = shell_table(spec, spec.max_mask_radius)
    radii = np.asarray(radii, dtype=np.int64)
    out = {"radius": radii, "kappa_measured_noctf": np.empty(len(radii)),
           "kappa_measured_ctf": np.full(len(radii), np.nan), "lower_bound": np.empty(len(radii)),
           "one_over_lambda": np.full(len(radii), np.inf if lam == 0 else 1.0 / lam)}
    for i, r in enumerate(radii):
        out["kappa_measured_noctf"][i] = condition_number(diag_noctf, spec, int(r))
        if diag_ctf is not None:
            out["kappa_measured_ctf"][i] = condition_number(diag_ctf, spec, int(r))
        out["lower_bound"][i] = cond_lower_bound(len(poses), lam, shells.pixel_voxel_ratio(int(r)))
    return out


def assignment_table(poses, spec, mask) -> np.ndarray:
    """Nearest-neighbour voxel index per (image, masked pixel), (N, n_mask) int64 (hessian.py:28-35),
    from the bit-exact fsld_assign_nn kernel."""
    quats = np.array([p.q for p in poses], dtype=np.float64)
    e = SliceEngine(spec.M, "nn", mask, records_for(spec.M, quats), None)
    return e.assign_nn(np.arange(len(poses))).cpu().numpy().astype(np.int64)


def _exact_diag_nn_dedupe(poses, ctfs, spec, mask) -> np.ndarray:
    """hessian.py:95-101: per image, C^2 of the lowest-index pixel among those sharing a voxel."""
    from .forward import Projector

    proj = Projector(spec, mask, "nn")
    diag = np.zeros(spec.n_voxels, dtype=np.float64)
    for lo in range(0, len(poses), 4096):
        batch = poses[lo:lo + 4096]
        idx = assignment_table(batch, spec, mask)
        w = proj.ctf_batch(ctfs[lo:lo + len(batch)] if ctfs is not None else None, len(batch)) ** 2
        order = np.argsort(idx, axis=1, kind="stable")
        si = np.take_along_axis(idx, order, axis=1)
        sw = np.take_along_axis(w, order, axis=1)
        keep = np.ones_like(si, dtype=bool)
        keep[:, 1:] = si[:, 1:] != si[:, :-1]
        diag += np.bincount(si[keep], weights=sw[keep], minlength=spec.n_voxels)
    return diag
