"""Grid layout contract of the reference (grid.py:9-31), restated for the B200 path.

Volumes are M^3 vectors: x/y axes centred (index = k + ceil(M/2)), z axis in
FFT order (kz < 0 -> kz + M), linear index j = (z*M + y)*M + x; the first M^2
entries are the kz = 0 slice, which is also the image (pixel) layout.
Masks keep points whose rounded radius is <= the cutoff (grid.py:185-196).
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np


@dataclass(frozen=True)
class GridSpec:
    """Cubic Fourier grid of side M (grid.py:50-94)."""

    M: int

    def __post_init__(self):
        if self.M < 2:
            raise ValueError(f"grid side length must be >= 2, got {self.M}")

    @property
    def n_pixels(self) -> int:
        return self.M * self.M

    @property
    def n_voxels(self) -> int:
        return self.M ** 3

    @property
    def half(self) -> int:
        return self.M // 2

    @property
    def centre(self) -> int:
        return (self.M + 1) // 2

    @property
    def max_mask_radius(self) -> int:
        return self.half - 1

    @property
    def dc_index(self) -> int:
        return self.centre * (self.M + 1)

    def pixel_coords(self) -> np.ndarray:
        return pixel_coords(self.M)

    def voxel_coords(self) -> np.ndarray:
        return voxel_coords(self.M)

    def pixel_radii(self) -> np.ndarray:
        """|k| per pixel in linear-index order (grid.py:136-141)."""
        return np.sqrt((pixel_coords(self.M).astype(np.float64) ** 2).sum(axis=1))

    def voxel_radii(self) -> np.ndarray:
        """|k| per voxel in linear-index order (grid.py:143-148)."""
        return np.sqrt((voxel_coords(self.M).astype(np.float64) ** 2).sum(axis=1))


@lru_cache(maxsize=16)
def _pix(M: int) -> np.ndarray:
    k = np.arange(M, dtype=np.int64) - (M + 1) // 2
    ky, kx = np.meshgrid(k, k, indexing="ij")
    out = np.stack([kx.ravel(), ky.ravel()], axis=1)
    out.setflags(write=False)
    return out


def pixel_coords(M: int) -> np.ndarray:
    """(M^2, 2) int64 (kx, ky) per ascending pixel index."""
    return _pix(int(M))


def voxel_coords(M: int) -> np.ndarray:
    """(M^3, 3) int64 (kx, ky, kz) per ascending voxel index."""
    c = (M + 1) // 2
    k = np.arange(M, dtype=np.int64) - c
    zi = np.arange(M, dtype=np.int64)
    kz_axis = np.where(zi < M - c, zi, zi - M)
    kz, ky, kx = np.meshgrid(kz_axis, k, k, indexing="ij")
    return np.stack([kx.ravel(), ky.ravel(), kz.ravel()], axis=1)


def _as_M(spec_or_M) -> int:
    return int(spec_or_M.M) if hasattr(spec_or_M, "M") else int(spec_or_M)


def disk_mask(spec_or_M, mask_radius: int) -> np.ndarray:
    """Pixel indices with rounded radius <= mask_radius, ascending (grid.py:185-189)."""
    M = _as_M(spec_or_M)
    if not 0 <= mask_radius <= M // 2 - 1:
        raise ValueError(f"mask_radius must be in [0, {M // 2 - 1}] for M={M}, got {mask_radius}")
    c = pixel_coords(M)
    r = np.round(np.sqrt((c.astype(np.float64) ** 2).sum(axis=1))).astype(np.int64)
    return np.flatnonzero(r <= mask_radius)


def ball_mask(spec_or_M, mask_radius: int) -> np.ndarray:
    """Voxel indices with rounded radius <= mask_radius, ascending (grid.py:192-196)."""
    M = _as_M(spec_or_M)
    if not 0 <= mask_radius <= M // 2 - 1:
        raise ValueError(f"mask_radius must be in [0, {M // 2 - 1}] for M={M}, got {mask_radius}")
    c = voxel_coords(M)
    r = np.round(np.sqrt((c.astype(np.float64) ** 2).sum(axis=1))).astype(np.int64)
    return np.flatnonzero(r <= mask_radius)


def shell_counts(M: int, mask_radius: int) -> tuple[np.ndarray, np.ndarray]:
    """Per-integer-radius pixel and voxel populations P_x(r), P_v(r) (grid.py:228-257)."""
    pr = np.round(np.sqrt((pixel_coords(M).astype(np.float64) ** 2).sum(axis=1))).astype(np.int64)
    vr = np.round(np.sqrt((voxel_coords(M).astype(np.float64) ** 2).sum(axis=1))).astype(np.int64)
    px = np.bincount(pr[pr <= mask_radius], minlength=mask_radius + 1)
    vx = np.bincount(vr[vr <= mask_radius], minlength=mask_radius + 1)
    return px, vx


def touched_ball(M: int, mask_radius: int) -> np.ndarray:
    """Voxel indices (ascending, int32) a scatter can reach: radius < R + 1/2 + sqrt(3).

    A masked pixel has |k| < R + 1/2 (round(|k|) <= R, grid.py:185-189); rotation keeps the
    radius, the clamp only shortens it (kernels.py:42-60), and the trilinear footprint stays
    within sqrt(3) of the rotated point.  The data-parallel all-reduce
    moves only these voxels.
    """
    r = np.sqrt((voxel_coords(M).astype(np.float64) ** 2).sum(axis=1))
    return np.flatnonzero(r < mask_radius + 0.5 + np.sqrt(3.0)).astype(np.int32)


@dataclass
class ShellTable:
    """Shell (rounded-radius) membership and populations of one grid (grid.py:200-238).

    ``shell_of_pixel`` / ``shell_of_voxel``: shell index per grid point in linear-index order, -1
    beyond ``max_radius``; ``px_count[r]`` / ``vx_count[r]``: 2D / 3D shell populations.
    """

    spec: GridSpec
    max_radius: int
    px_count: np.ndarray
    vx_count: np.ndarray
    shell_of_pixel: np.ndarray
    shell_of_voxel: np.ndarray

    @property
    def radii(self) -> np.ndarray:
        return np.arange(self.max_radius + 1)

    def n_masked_pixels(self) -> int:
        return int(self.px_count.sum())

    def n_masked_voxels(self) -> int:
        return int(self.vx_count.sum())

    def _check(self, r: int) -> None:
        if not 0 <= r <= self.max_radius:
            raise ValueError(f"radius {r} outside table range {self.max_radius}")

    def shell_ratio(self, r: int) -> float:
        """P_x(r) / P_v(r)."""
        self._check(r)
        if self.vx_count[r] == 0:
            raise ValueError(f"empty 3D shell at radius {r}")
        return float(self.px_count[r]) / float(self.vx_count[r])

    def pixel_voxel_ratio(self, r: int) -> float:
        """|disk(r)| / |ball(r)| (the condition-number bound's p(r))."""
        self._check(r)
        return float(self.px_count[: r + 1].sum()) / float(self.vx_count[: r + 1].sum())


def shell_table(spec: GridSpec, mask_radius: int) -> ShellTable:
    """ShellTable of the points with rounded radius <= mask_radius (grid.py:241-257)."""
    if not 1 <= mask_radius <= spec.max_mask_radius:
        raise ValueError(f"mask_radius must be in [1, {spec.max_mask_radius}] for M={spec.M}, got {mask_radius}")
    ps = np.round(spec.pixel_radii()).astype(np.int64)
    vs = np.round(spec.voxel_radii()).astype(np.int64)
    sp = np.where(ps <= mask_radius, ps, -1).astype(np.int32)
    sv = np.where(vs <= mask_radius, vs, -1).astype(np.int32)
    return ShellTable(spec=spec, max_radius=int(mask_radius),
                      px_count=np.bincount(sp[sp >= 0], minlength=mask_radius + 1),
                      vx_count=np.bincount(sv[sv >= 0], minlength=mask_radius + 1),
                      shell_of_pixel=sp, shell_of_voxel=sv)
