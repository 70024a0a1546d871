"""Deterministic mode on the table-driven brick kernel (FSLD_DETERMINISTIC).

The reference's contract (kernels.py:15-18, 297-302): results do not depend on the number of
threads.  Here the brick kernel's per-item int32 sums are order-free already; in deterministic
mode the work items are formed in brick order with their segments sorted by dataset offset, each
item is flushed into the int64 fixed-point accumulator at the caller's power-of-two scale (exact
shifts, order-free 64-bit integer adds), and the loss is summed per item in item order.  So the
gradient accumulator and the loss are bitwise the same for any launch grid, any claim order and
any order of the batch -- and still within the fp32 tolerance of the oracle.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

import cfg_data
import paper_2311_16100_b200 as F
from paper_2311_16100_b200.engine import SliceEngine, records_for
from paper_2311_16100_b200.forward import DatasetOperator

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def data():
    d = cfg_data.make(64, 1024, "tri", ctf=True, shifts=True, snr=0.05, seed=11)
    recs = records_for(d.M, d.quats, d.shifts, d.ctfs)
    det = SliceEngine(d.M, "tri", d.mask, recs, d.x, deterministic=True)
    plain = SliceEngine(d.M, "tri", d.mask, recs, d.x)
    assert det.ptab is not None and det.layout == "sorted"
    return d, det, plain


def _kernel_names(fn):
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return {e.name for e in prof.events()}


def test_det_brick_bitwise_any_grid_and_batch_order(data):
    d, det, _ = data
    v = torch.from_numpy((0.9 * d.v_true).astype(np.complex64)).cuda()
    batch = np.random.default_rng(3).permutation(1024)[:512]
    sq1, acc1, fx = det.loss_grad(v, batch)
    sq2, acc2, _ = det.loss_grad(v, batch, fx=fx)
    sq3, acc3, _ = det.loss_grad(v, batch[::-1].copy(), fx=fx)  # another batch order
    os.environ["FSLD_DET_GRID"] = "37"  # another launch grid (37 persistent CTAs instead of 740)
    try:
        sq4, acc4, _ = det.loss_grad(v, np.random.default_rng(4).permutation(batch), fx=fx)
    finally:
        del os.environ["FSLD_DET_GRID"]
    for sq, acc in ((sq2, acc2), (sq3, acc3), (sq4, acc4)):
        assert float(sq) == float(sq1)
        assert torch.equal(acc, acc1)
    assert acc1.dtype == torch.int64 and int(acc1.abs().max()) > 0


def test_det_brick_runs_the_brick_kernel(data):
    d, det, _ = data
    v = torch.from_numpy(d.v_true.astype(np.complex64)).cuda()
    names = _kernel_names(lambda: det.loss_grad(v, np.arange(256)))
    assert any("brick_loss_grad_kernel" in n for n in names), names
    assert any("sort_pairs_kernel" in n for n in names), names
    assert not any("slice_kernel" in n for n in names), names


def test_det_brick_vs_oracle_and_plain(data):
    d, det, plain = data
    lam = 1e-3
    batch = np.random.default_rng(5).permutation(1024)[:512]
    v1 = (0.9 * d.v_true).astype(np.complex64).astype(np.complex128)
    opd, op = DatasetOperator.from_engine(det), DatasetOperator.from_engine(plain)
    ld, gd = F.loss_and_grad(opd, v1, batch, lam)
    lp, gp = F.loss_and_grad(op, v1, batch, lam)
    lr, gr = O.loss_and_grad(d.oop, v1, batch, lam)
    assert abs(ld - lr) / lr < TOL
    assert O.relative_l2(gd, gr) < TOL
    assert O.relative_l2(gd, gp) < TOL
    # and the numpy-level result is bitwise repeatable
    ld2, gd2 = F.loss_and_grad(opd, v1, batch[::-1].copy(), lam)
    assert ld2 == ld and np.array_equal(gd2.view(np.uint64), gd.view(np.uint64))


def test_numpy_signature_call_pinned_and_pageable_outputs(data):
    """optim.loss_and_grad(op, numpy complex128 v, ...) -> fsld_loss_grad_host_np: the recycled page-locked
    output arrays (device-side complex128 cast) and, once more than the pool's arrays are held, plain
    numpy arrays (complex64 gradient cast back on the host threads) -- both equal the device step."""
    from paper_2311_16100_b200 import optim as Opt
    d, _, plain = data
    op = DatasetOperator.from_engine(plain)
    lam = 1e-3
    v = (0.9 * d.v_true).astype(np.complex128)
    batch = np.random.default_rng(8).permutation(1024)[:512]
    ref_l, ref_g = O.loss_and_grad(d.oop, v.astype(np.complex64).astype(np.complex128), batch, lam)
    held = []
    for i in range(10):  # the pool keeps 8 page-locked arrays: calls 9 and 10 return pageable ones
        l, g = Opt.loss_and_grad(op, v, batch, lam)
        assert g.dtype == np.complex128 and g.shape == (d.M ** 3,)
        assert abs(l - ref_l) / ref_l < TOL
        assert O.relative_l2(g, ref_g) < TOL
        held.append(g)
    assert O.relative_l2(held[-1], held[0]) < 1e-6
