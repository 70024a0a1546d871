"""Per-epoch reconstruction metrics used by optim.run (metrics.py:38-74 of the reference).

Fourier shell correlation on the device: per-voxel shell index (rounded
radius, grid.py:241-257) and three weighted bincounts in fp64.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .grid import voxel_coords


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
    """Device copy of the voxel shell table for repeated FSC evaluations."""

    def __init__(self, M: int, max_radius: int, device):
        s = shell_of_voxel(M, max_radius)
        self.max_radius = int(max_radius)
        sel = np.flatnonzero(s >= 0)
        self.sel = torch.from_numpy(sel).to(device)
        self.shell = torch.from_numpy(s[sel].astype(np.int64)).to(device)
        self.counts = np.bincount(s[sel], minlength=max_radius + 1)


def fsc(u, v, shells: ShellIndex) -> FscCurve:
    """FSC of u against v (metrics.py:38-63); u, v complex (M^3,) numpy or CUDA tensors."""
    dev = shells.sel.device
    a = torch.as_tensor(u, device=dev).reshape(-1)[shells.sel].to(torch.complex128)
    b = torch.as_tensor(v, device=dev).reshape(-1)[shells.sel].to(torch.complex128)
    nsh = shells.max_radius + 1
    num = torch.bincount(shells.shell, weights=(a * b.conj()).real, minlength=nsh)
    pu = torch.bincount(shells.shell, weights=a.abs() ** 2, minlength=nsh)
    pv = torch.bincount(shells.shell, weights=b.abs() ** 2, minlength=nsh)
    num, pu, pv = num.cpu().numpy(), pu.cpu().numpy(), pv.cpu().numpy()
    defined = (pu > 0) & (pv > 0)
    values = np.full(nsh, np.nan)
    values[defined] = num[defined] / np.sqrt(pu[defined] * pv[defined])
    return FscCurve(radii=np.arange(nsh), values=values, counts=shells.counts.copy(), defined=defined)


def relative_l2(estimate, truth) -> float:
    """||estimate - truth|| / ||truth|| (metrics.py:66-74)."""
    if isinstance(estimate, torch.Tensor):
        estimate = estimate.double().cpu().numpy()
    truth = np.asarray(truth, dtype=np.float64 if not np.iscomplexobj(truth) else np.complex128)
    estimate = np.asarray(estimate)
    denom = np.linalg.norm(truth)
    if denom == 0:
        raise ValueError("truth vector has zero norm")
    return float(np.linalg.norm(estimate - truth) / denom)
