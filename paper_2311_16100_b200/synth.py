"""Seeded synthetic workloads of BASELINE.json configs 1-5.

There is no public benchmark data for this path (the paper's EMPIAR-10076
images are not available); these generators stand in with the shapes, sizes
and value distributions BASELINE.json names:

  volume : real M^3 sum of 20 isotropic Gaussians (sigma U[1.5,3] vox,
           centres uniform in a ball of radius 0.3 M, amplitudes U[0.5,1]),
           ifftshift -> fftn -> centre x/y (z stays in FFT order) = the
           reference layout (grid.py:9-31);
  poses  : Haar-uniform unit quaternions (normalised Gaussians, as
           forward.sample_uniform_poses), shifts N(0, 2 px) per axis;
  CTF    : defocus U[1,3] um, astigmatism U[0,0.1] um at a uniform angle,
           300 kV, Cs 2.7 mm, amplitude contrast 0.1, 1 A/px (PhysicalCtf);
  noise  : sigma = sqrt(mean_masked |clean|^2 / SNR), complex Gaussian with
           sigma/sqrt(2) per part (cli.py:108-114, forward.py:411-424).

The dataset itself is projected on the GPU by the product kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .engine import SliceEngine, records_for
from .forward import PhysicalCtf
from .grid import disk_mask


@dataclass(frozen=True)
class Config:
    name: str
    M: int
    n_images: int
    mode: str
    ctf: bool
    shifts: bool
    snr: float
    batch: int
    probes: int = 1


CONFIGS = {
    "cfg1": Config("cfg1_M32_nn", 32, 1000, "nn", False, False, 0.1, 1000, 8),
    "cfg2": Config("cfg2_M64_tri", 64, 10000, "tri", True, True, 0.05, 10000, 32),
    "cfg3": Config("cfg3_M128_tri_B512", 128, 50000, "tri", True, True, 0.05, 512, 64),
    "cfg4": Config("cfg4_M256_tri_B1024", 256, 200000, "tri", True, True, 0.05, 1024, 1),
    "cfg5": Config("cfg5_M128_hutch_sweep", 128, 4096, "tri", True, True, 0.05, 4096, 256),
}


def gaussian_blob_volume(M: int, seed: int = 0, n_blobs: int = 20) -> np.ndarray:
    """Fourier volume (M^3 complex128, reference layout) of a real Gaussian-blob density."""
    rng = np.random.default_rng(seed)
    sig = rng.uniform(1.5, 3.0, n_blobs)
    d = rng.standard_normal((n_blobs, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rad = 0.3 * M * rng.uniform(0.0, 1.0, n_blobs) ** (1.0 / 3.0)
    centres = M / 2.0 + d * rad[:, None]
    amp = rng.uniform(0.5, 1.0, n_blobs)
    ax = np.arange(M, dtype=np.float64)
    vol = np.zeros((M, M, M))  # [z][y][x]
    for s, c, a in zip(sig, centres, amp):
        gx = np.exp(-0.5 * ((ax - c[0]) / s) ** 2)
        gy = np.exp(-0.5 * ((ax - c[1]) / s) ** 2)
        gz = np.exp(-0.5 * ((ax - c[2]) / s) ** 2)
        vol += a * gz[:, None, None] * gy[None, :, None] * gx[None, None, :]
    F = np.fft.fftn(np.fft.ifftshift(vol.astype(np.float32).astype(np.float64)))
    c = (M + 1) // 2
    F = np.roll(F, c, axis=2)  # x: index = kx + ceil(M/2)
    F = np.roll(F, c, axis=1)  # y
    return np.ascontiguousarray(F.reshape(-1))


def haar_quaternions(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def normal_shifts(n: int, seed: int, sd: float = 2.0) -> np.ndarray:
    return np.random.default_rng(seed).normal(0.0, sd, (n, 2))


def physical_ctfs(n: int, seed: int) -> list:
    rng = np.random.default_rng(seed)
    df = rng.uniform(1.0e4, 3.0e4, n)
    ast = rng.uniform(0.0, 1.0e3, n)
    ang = rng.uniform(0.0, np.pi, n)
    return [PhysicalCtf(defocus=float(df[i]), astig=float(ast[i]), astig_angle=float(ang[i]),
                        voltage_kv=300.0, cs_mm=2.7, amp_contrast=0.1, apix=1.0) for i in range(n)]


def ctf_param_array(ctfs) -> np.ndarray:
    """(N, 7) rows (defocus, astig, angle, kV, Cs mm, amp, apix), the oracle's table input."""
    return np.array([[c.defocus, c.astig, c.astig_angle, c.voltage_kv, c.cs_mm, c.amp_contrast, c.apix]
                     for c in ctfs], dtype=np.float64)


@dataclass
class Workload:
    cfg: Config
    M: int
    mask: np.ndarray
    v_true: np.ndarray          # host complex128
    quats: np.ndarray
    shifts: np.ndarray | None
    ctfs: list | None
    engine: SliceEngine         # device-resident dataset (x filled)
    sigma: float
    n_total: int = 0            # images of the whole (unsharded) dataset


def build_workload(cfg: Config, seed: int = 0, n_images: int | None = None, deterministic: bool = False,
                   chunk: int = 4096, shard: tuple[int, int] = (0, 1)) -> Workload:
    """Generate the config's dataset directly in HBM with the product projection kernel.

    shard=(r, W): only images [r N/W, (r+1) N/W) of the N-image dataset (same poses / shifts /
    CTFs as the unsharded one; the noise stream is per shard)."""
    M = cfg.M
    N_all = n_images or cfg.n_images
    r, W = shard
    lo, hi = (r * N_all) // W, ((r + 1) * N_all) // W
    mask = disk_mask(M, M // 2 - 1)
    v = gaussian_blob_volume(M, seed)
    quats = haar_quaternions(N_all, seed + 1)[lo:hi]
    shifts = normal_shifts(N_all, seed + 2)[lo:hi] if cfg.shifts else None
    ctfs = physical_ctfs(N_all, seed + 3)[lo:hi] if cfg.ctf else None
    N = hi - lo
    recs = records_for(M, quats, shifts, ctfs)
    eng = SliceEngine(M, cfg.mode, mask, recs, None, deterministic=deterministic)
    vd = torch.from_numpy(v.astype(np.complex64)).to(eng.dev)
    x = torch.empty((N, mask.size), dtype=torch.complex64, device=eng.dev)
    power = 0.0
    for lo in range(0, N, chunk):
        idx = torch.arange(lo, min(lo + chunk, N), dtype=torch.int32, device=eng.dev)
        # project straight into the engine's dataset layout (brick-sorted for tri)
        if eng.layout == "sorted":
            eng.project_sorted(vd, idx, out=x[lo:lo + idx.numel()])
        else:
            x[lo:lo + idx.numel()] = eng.project(vd, idx)
        power += float(torch.view_as_real(x[lo:lo + idx.numel()]).pow(2).sum().item())
    sigma = float(np.sqrt(power / (N * mask.size) / cfg.snr))
    g = torch.Generator(device=eng.dev)
    g.manual_seed(seed + 100 + 7919 * r)
    for lo in range(0, N, chunk):
        hi = min(lo + chunk, N)
        nz = torch.randn((hi - lo, mask.size, 2), generator=g, device=eng.dev, dtype=torch.float32)
        x[lo:hi] += torch.view_as_complex(nz * (sigma / np.sqrt(2.0)))
    eng.set_images(x, sorted_order=True)
    return Workload(cfg, M, mask, v, quats, shifts, ctfs, eng, sigma, N_all)
