"""Seeded BASELINE-config datasets built on the HOST with the oracle (test infrastructure).

The parity tests at the named configurations need the SAME seeded inputs on both
sides: the volume, poses, shifts, CTF table and noisy images are generated here in
fp64 with the oracle's restated kernels (oracle/oracle.py, pinned to the reference),
then the images are uploaded into the B200 engine.  Generators are those of
SURVEY.md §8d (paper_2311_16100_b200.synth restates them): Gaussian-blob volume,
Haar poses, N(0, 2 px) shifts, physical astigmatic CTF, and the reference's noise
definition sigma = sqrt(mean_masked |clean|^2 / SNR) (cli.py:108-114) with one
complex Gaussian per pixel (sigma / sqrt(2) per part).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle import oracle as O


@dataclass
class CfgData:
    M: int
    mode: str
    mask: np.ndarray
    pix: np.ndarray
    v_true: np.ndarray          # complex128, reference layout
    quats: np.ndarray
    shifts: np.ndarray | None
    ctfs: list | None           # PhysicalCtf objects (GPU records)
    ctab: np.ndarray | None     # (N, n) fp64 CTF table (oracle)
    x: np.ndarray               # (N, n) complex128 noisy masked images
    oop: O.OracleOperator


def make(M: int, n_images: int, mode: str, ctf: bool, shifts: bool, snr: float, seed: int = 0) -> CfgData:
    from paper_2311_16100_b200 import synth

    mask = O.disk_mask(M, M // 2 - 1)
    pix = O.mask_pix(M, mask)
    v = synth.gaussian_blob_volume(M, seed)
    q = synth.haar_quaternions(n_images, seed + 1)
    sh = synth.normal_shifts(n_images, seed + 2) if shifts else None
    ctfs = synth.physical_ctfs(n_images, seed + 3) if ctf else None
    ctab = O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M) if ctf else None
    sh0 = sh if sh is not None else np.zeros((n_images, 2))
    oop = O.OracleOperator(M, mode, mask, q, sh0, ctab, None)
    clean = oop.project(v, np.arange(n_images))
    sigma = np.sqrt(np.mean(clean.real ** 2 + clean.imag ** 2) / snr)
    rng = np.random.default_rng(seed + 100)
    noise = rng.standard_normal(clean.shape) + 1j * rng.standard_normal(clean.shape)
    x = clean + noise * (sigma / np.sqrt(2.0))
    oop.x = np.ascontiguousarray(x)
    return CfgData(M, mode, mask, pix, v, q, sh, ctfs, ctab, oop.x, oop)


def gpu_operator(d: CfgData):
    from paper_2311_16100_b200.engine import SliceEngine, records_for
    from paper_2311_16100_b200.forward import DatasetOperator

    recs = records_for(d.M, d.quats, d.shifts, d.ctfs)
    eng = SliceEngine(d.M, d.mode, d.mask, recs, d.x)
    return DatasetOperator.from_engine(eng)
