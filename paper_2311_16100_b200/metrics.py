"""Reconstruction metrics (drop-in for fsld.metrics, /root/reference/pkg/src/fsld/metrics.py).

``fsc`` runs the fsld_fsc kernel (per-shell Re(u conj v), |u|^2, |v|^2 in fp64, per-CTA partial
rows added in a fixed order; metrics.py:38-63); the host forms the per-shell ratio.  It accepts
the reference's arguments (FourierVolume pair + ShellTable) or device volumes with a ShellIndex
(the per-epoch call inside optim.run).  Volumes are read as complex64 (the path's precision).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _capi as C
from .grid import ShellTable, voxel_coords


@dataclass
class FscCurve:
    """Per-shell Re(sum u conj(v)) / sqrt(sum|u|^2 sum|v|^2); NaN where undefined (metrics.py:21-36)."""

    radii: np.ndarray
    values: np.ndarray
    counts: np.ndarray
    defined: np.ndarray

    def __len__(self) -> int:
        return self.values.size


def shell_of_voxel(M: int, max_radius: int) -> np.ndarray:
    """Rounded voxel radius, -1 beyond max_radius (grid.py:241-257)."""
    r = np.round(np.sqrt((voxel_coords(M).astype(np.float64) ** 2).sum(axis=1))).astype(np.int64)
    return np.where(r <= max_radius, r, -1).astype(np.int32)


class ShellIndex:
    """Device-side FSC context for one grid: shell populations and the kernel's scratch rows."""

    def __init__(self, M: int, max_radius: int, device):
        self.M = int(M)
        self.max_radius = int(max_radius)
        self.device = torch.device(device)
        s = shell_of_voxel(M, max_radius)
        self.counts = np.bincount(s[s >= 0], minlength=max_radius + 1)
        nbytes = int(C.load().fsld_fsc_scratch_bytes(self.M, self.max_radius))
        self.scratch = torch.empty((nbytes + 7) // 8, dtype=torch.float64, device=self.device)
        self.out = torch.empty(3 * (max_radius + 1), dtype=torch.float64, device=self.device)


def _volume_c64(u, dev) -> torch.Tensor:
    vals = u if isinstance(u, (torch.Tensor, np.ndarray)) else getattr(u, "values", u)
    if isinstance(vals, torch.Tensor):
        return vals.to(dev, torch.complex64).contiguous().reshape(-1)
    return torch.from_numpy(np.ascontiguousarray(vals, dtype=np.complex64)).to(dev).reshape(-1)


def fsc(u, v, shells) -> FscCurve:
    """Fourier shell correlation of u against v (metrics.py:38-63) on the device."""
    from .engine import _stream, ctypes_ptr, require_device

    if isinstance(shells, ShellTable):
        if getattr(u, "spec", shells.spec) != shells.spec or getattr(v, "spec", shells.spec) != shells.spec:
            raise ValueError("volumes and shell table must share one grid spec")
        ctx = _shell_index(shells.spec.M, shells.max_radius, require_device())
    else:
        ctx = shells
    a = _volume_c64(u, ctx.device)
    b = _volume_c64(v, ctx.device)
    if a.numel() != ctx.M ** 3 or b.numel() != ctx.M ** 3:
        raise ValueError("volumes must have M^3 entries")
    C.check(C.load().fsld_fsc(ctx.M, ctx.max_radius, ctypes_ptr(a), ctypes_ptr(b), ctypes_ptr(ctx.out),
                              ctypes_ptr(ctx.scratch), ctx.scratch.numel() * 8, _stream()), "fsld_fsc")
    sums = ctx.out.cpu().numpy().reshape(3, ctx.max_radius + 1)
    num, pu, pv = sums
    defined = (pu > 0) & (pv > 0)
    values = np.full(ctx.max_radius + 1, np.nan)
    values[defined] = num[defined] / np.sqrt(pu[defined] * pv[defined])
    return FscCurve(radii=np.arange(ctx.max_radius + 1), values=values, counts=ctx.counts.copy(),
                    defined=defined)


_SHELL_CACHE: dict = {}


def _shell_index(M: int, R: int, dev) -> ShellIndex:
    key = (M, R, str(dev))
    if key not in _SHELL_CACHE:
        _SHELL_CACHE[key] = ShellIndex(M, R, dev)
    return _SHELL_CACHE[key]


def relative_l2(estimate, truth) -> float:
    """||estimate - truth|| / ||truth|| (metrics.py:66-73)."""
    if isinstance(estimate, torch.Tensor):
        estimate = estimate.cpu().numpy()
    if isinstance(truth, torch.Tensor):
        truth = truth.cpu().numpy()
    truth = np.asarray(truth)
    estimate = np.asarray(estimate)
    denom = np.linalg.norm(truth)
    if denom == 0:
        raise ValueError("truth vector has zero norm")
    return float(np.linalg.norm(estimate - truth) / denom)


def epochs_to_threshold(fsc_history: np.ndarray, theta: float) -> np.ndarray:
    """Per shell, the first epoch whose FSC reaches theta; -1 if none does (metrics.py:76-91)."""
    hist = np.asarray(fsc_history, dtype=np.float64)
    if hist.ndim != 2 or hist.shape[0] == 0:
        raise ValueError("fsc_history must be a nonempty (epochs, shells) array")
    with np.errstate(invalid="ignore"):
        hit = hist >= theta
    first = np.where(hit.any(axis=0), hit.argmax(axis=0), -1)
    return first.astype(np.int64)


def grad_variance_shells(op, v, shells: ShellTable, config, precond=None):
    """Per-shell variance of the mini-batch gradient at a fixed iterate (metrics.py:94-124): every
    batch gradient of epoch 0 through the fused loss+grad kernel, the per-voxel sample variance
    (real + imaginary) and its shell means; plus the shell means of 1/precond when given."""
    from .optim import epoch_batches, loss_and_grad

    batches = epoch_batches(op.n_images, config.batch_size, config.seed, epoch=0)
    if len(batches) < 2:
        raise ValueError("gradient variance needs at least 2 batches per epoch")
    grads = np.stack([loss_and_grad(op, v, b, config.lam)[1] for b in batches])
    var = (np.abs(grads - grads.mean(axis=0)) ** 2).sum(axis=0) / (len(batches) - 1)
    sel = shells.shell_of_voxel >= 0
    s = shells.shell_of_voxel[sel].astype(np.int64)
    nsh = shells.max_radius + 1
    counts = np.bincount(s, minlength=nsh).astype(np.float64)
    var_shells = np.bincount(s, weights=var[sel], minlength=nsh) / counts
    dinv = None
    if precond is not None:
        dinv = np.bincount(s, weights=1.0 / np.asarray(precond)[sel], minlength=nsh) / counts
    return var_shells, dinv
