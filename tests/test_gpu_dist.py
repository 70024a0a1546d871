"""GPU: the data-parallel step's default per-rank compute (B200 engine) at world size 1."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

import paper_2311_16100_b200 as F
from paper_2311_16100_b200 import dist as D
from paper_2311_16100_b200 import synth
from paper_2311_16100_b200.forward import DatasetOperator

pytestmark = pytest.mark.gpu


def test_sharded_step_world1_matches_loss_and_grad_and_probe_fold():
    wl = synth.build_workload(synth.CONFIGS["cfg2"], seed=0, n_images=256)
    op = DatasetOperator.from_engine(wl.engine)
    e = wl.engine
    batch = np.arange(0, 256, 3)
    lam = 1e-3
    v = torch.from_numpy((wl.v_true * 0.95).astype(np.complex64)).cuda()
    z = np.random.default_rng(0).integers(0, 2, size=(4, e.n_voxels)).astype(np.float64) * 2 - 1
    zbits, k = e.pack_probes(z)
    loss, grad, hs = D.sharded_step(op, v, batch, lam, zbits=zbits, k=k)
    loss_ref, grad_ref = F.loss_and_grad(op, v, torch.from_numpy(batch).cuda(), lam)
    assert abs(float(loss) - float(loss_ref)) / float(loss_ref) < 1e-6
    assert O.relative_l2(grad.cpu().numpy(), grad_ref.cpu().numpy()) < 1e-5  # two runs of fp32 atomics: order differs
    from paper_2311_16100_b200.optim import hutchinson_sample
    hs_ref, _ = hutchinson_sample(op, z, batch, lam)
    assert O.relative_l2(hs.cpu().numpy(), hs_ref) < 1e-6


def test_sharded_step_with_ball_compaction_matches_full_buffer():
    """The touched-ball compacted all-reduce buffer gives the same step as the full one (world 1)."""
    from paper_2311_16100_b200.grid import touched_ball
    wl = synth.build_workload(synth.CONFIGS["cfg2"], seed=1, n_images=256)
    op = DatasetOperator.from_engine(wl.engine)
    e = wl.engine
    batch = np.arange(1, 256, 3)
    lam = 1e-3
    v = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).cuda()
    zbits = e.gen_probes(1, 3)
    ball = touched_ball(e.M, e.M // 2 - 1)
    assert ball.size < e.n_voxels
    buf = D.PackedBuffer.new(e.n_voxels, True, torch.device("cuda"), ball=ball)
    assert buf.flat.numel() == 3 * ball.size + 2
    l1, g1, h1 = D.sharded_step(op, v, batch, lam, buf=buf, zbits=zbits, k=1)
    l2, g2, h2 = D.sharded_step(op, v, batch, lam, zbits=zbits, k=1)
    assert abs(float(l1) - float(l2)) / float(l2) < 1e-6
    assert O.relative_l2(g1.cpu().numpy(), g2.cpu().numpy()) < 1e-5
    assert O.relative_l2(h1.cpu().numpy(), h2.cpu().numpy()) < 1e-5
