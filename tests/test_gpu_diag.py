"""The exact Hessian diagonal on the table-driven brick kernel (DIAG pass, fsld_exact_diag_sorted_tab).

hessian.exact_diag (hessian.py:62-107) scatters C^2 w^2 per (image, pixel, corner) with
kernels.scatter_sq_tri (kernels.py:251-294).  On a table-built sorted dataset the brick kernel does it
from the per-pixel tables (|f|^2 = C^2, the stored footprint): checked against the oracle, against the
compute-path tile kernel, bitwise across launch grids and batch orders in deterministic mode, and
across the 1024-image chunks the deterministic call takes.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

import cfg_data
import paper_2311_16100_b200 as F
from paper_2311_16100_b200.engine import SliceEngine, records_for

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def data():
    d = cfg_data.make(64, 2500, "tri", ctf=True, shifts=True, snr=0.05, seed=21)
    recs = records_for(d.M, d.quats, d.shifts, d.ctfs)
    return d, recs


def _diag(e, idx):
    acc, fx = e.exact_diag_acc(idx)
    return e.finalize_r(acc, fx, 1.0, 0.0).cpu().numpy().astype(np.float64)


def _kernel_names(fn):
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return {e.name for e in prof.events()}


def test_brick_diag_vs_oracle_tile_and_det(data):
    d, recs = data
    det = SliceEngine(d.M, "tri", d.mask, recs, None, deterministic=True)
    plain = SliceEngine(d.M, "tri", d.mask, recs, None)
    tile = SliceEngine(d.M, "tri", d.mask, recs, None, tile_path=True)
    assert det.ptab is not None and plain.ptab is not None
    ref = O.exact_diag(d.oop, 0.0)
    idx = np.arange(2500)  # three deterministic chunks (1024, 1024, 452)
    dd, dp, dt = _diag(det, idx), _diag(plain, idx), _diag(tile, idx)
    assert O.relative_l2(dd, ref) < TOL
    assert O.relative_l2(dp, ref) < TOL
    assert O.relative_l2(dt, ref) < TOL
    assert O.relative_l2(dd, dt) < 2e-6
    assert np.all(dd >= 0) and np.all((ref > 0) | (dd == 0))


def test_brick_diag_runs_the_brick_kernel(data):
    d, recs = data
    e = SliceEngine(d.M, "tri", d.mask, recs, None, deterministic=True)
    names = _kernel_names(lambda: e.exact_diag_acc(np.arange(512)))
    assert any("brick_loss_grad_kernel" in n for n in names), names
    assert not any("slice_kernel" in n for n in names), names


def test_brick_diag_det_bitwise_any_grid_and_order(data):
    d, recs = data
    e = SliceEngine(d.M, "tri", d.mask, recs, None, deterministic=True)
    idx = np.random.default_rng(2).permutation(2500)[:1000]
    a1, fx = e.exact_diag_acc(idx)
    a2, _ = e.exact_diag_acc(idx[::-1].copy(), fx=fx)
    os.environ["FSLD_DET_GRID"] = "29"
    try:
        a3, _ = e.exact_diag_acc(np.random.default_rng(3).permutation(idx), fx=fx)
    finally:
        del os.environ["FSLD_DET_GRID"]
    assert a1.dtype == torch.int64 and int(a1.max()) > 0
    assert torch.equal(a1, a2) and torch.equal(a1, a3)


def test_hessian_exact_diag_public_api(data):
    """F.exact_diag (the reference's signature) lands on the brick path and equals the oracle + lam."""
    d, _ = data
    lam = 0.25
    poses = [F.Pose(q, t) for q, t in zip(d.quats, d.shifts)]
    got = F.exact_diag(poses, d.ctfs, lam, "tri", F.GridSpec(d.M), d.mask)
    ref = O.exact_diag(d.oop, lam)
    assert O.relative_l2(got, ref) < TOL
    again = F.exact_diag(poses, d.ctfs, lam, "tri", F.GridSpec(d.M), d.mask)
    assert np.array_equal(got.view(np.uint64), again.view(np.uint64))


@pytest.mark.parametrize("M", [17, 33])
def test_brick_diag_odd_sizes_vs_oracle(M):
    """Odd M (the half-open z range, bricks cut by the grid edge) and a ragged last chunk."""
    d = cfg_data.make(M, 1100, "tri", ctf=True, shifts=False, snr=0.05, seed=M)
    recs = records_for(d.M, d.quats, None, d.ctfs)
    for det in (True, False):
        e = SliceEngine(d.M, "tri", d.mask, recs, None, deterministic=det)
        assert e.ptab is not None
        got = _diag(e, np.arange(1100))
        assert O.relative_l2(got, O.exact_diag(d.oop, 0.0)) < TOL
