"""The NVLS data-parallel exchange (dist.NvlsGroup, fsld_loss_grad_planned_mc, fsld_nvls_barrier).

On a 1-GPU box the multicast team has one member: the brick pass flushes through the multicast
address (multimem.red) into the one bound copy, the barriers arrive and pass, and the epilogue reads
the copy back.  That step must equal the fused single-GPU step (fsld_loss_grad_step_planned) and the
oracle, leave the copy zeroed for the next step, and replay from a CUDA graph.  The N > 1 exchange
is the same code with more team members (the fd hand-over is covered on CPU in test_dist_gloo.py).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O

import cfg_data
from paper_2311_16100_b200 import dist as D
from paper_2311_16100_b200.engine import SliceEngine, records_for

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def setup():
    if not D.nvls_available(0):
        pytest.skip("no NVSwitch multicast on this box (fsld_nvls_supported: cuMulticastCreate refused)")
    d = cfg_data.make(64, 2048, "tri", ctf=True, shifts=True, snr=0.05, seed=31)
    recs = records_for(d.M, d.quats, d.shifts, d.ctfs)
    e = SliceEngine(d.M, "tri", d.mask, recs, d.x)
    assert e.table_path
    rng = np.random.default_rng(5)
    batches = np.stack([rng.permutation(2048)[:512] for _ in range(3)]).astype(np.int32)
    plan = e.make_plan(batches)
    g = D.NvlsGroup(d.M ** 3)
    yield d, e, plan, batches, g
    g.close()


def _nvls(e, g, plan, k, v, scale, lam):
    dev = e.dev
    grad = torch.empty(e.n_voxels, dtype=torch.complex64, device=dev)
    sq, sqt, loss = (torch.empty(1, dtype=torch.float64, device=dev) for _ in range(3))
    D.nvls_planned_step(e, g, plan, k, v, scale, lam, grad, sq, sqt, loss, e._norm_scratch())
    return grad, sq, sqt, loss


def test_nvls_step_equals_fused_step_and_oracle(setup):
    d, e, plan, batches, g = setup
    lam, scale = 1e-3, 2048 / 512
    v = torch.from_numpy((0.9 * d.v_true).astype(np.complex64)).cuda()
    grad, sq, sqt, loss = _nvls(e, g, plan, 1, v, scale, lam)
    ref_grad = torch.empty_like(grad)
    ref_loss, ref_sq = e.loss_grad_step_planned(v, plan, 1, scale, lam, ref_grad)
    torch.cuda.synchronize()
    g.check()
    assert float(sqt) == float(sq)  # one team member: the rank-ordered sum is its own
    assert abs(float(sq) - float(ref_sq)) / float(ref_sq) < 1e-12
    assert abs(float(loss) - float(ref_loss)) / float(ref_loss) < 1e-9
    assert O.relative_l2(grad.cpu().numpy(), ref_grad.cpu().numpy()) < 1e-6
    lr, gr = O.loss_and_grad(d.oop, (0.9 * d.v_true).astype(np.complex64).astype(np.complex128),
                             batches[1].astype(np.int64), lam)
    assert abs(float(loss) - lr) / lr < TOL
    assert O.relative_l2(grad.cpu().numpy().astype(np.complex128), gr) < TOL


def test_nvls_copy_is_rezeroed_between_steps(setup):
    d, e, plan, _, g = setup
    v = torch.from_numpy((0.8 * d.v_true).astype(np.complex64)).cuda()
    g1, _, _, l1 = _nvls(e, g, plan, 0, v, 4.0, 1e-3)
    g2, _, _, l2 = _nvls(e, g, plan, 2, v, 4.0, 1e-3)
    g3, _, _, l3 = _nvls(e, g, plan, 0, v, 4.0, 1e-3)  # batch 0 again: nothing left over from batch 2
    torch.cuda.synchronize()
    g.check()
    assert O.relative_l2(g3.cpu().numpy(), g1.cpu().numpy()) < 1e-6
    assert abs(float(l3) - float(l1)) / float(l1) < 1e-9
    assert O.relative_l2(g2.cpu().numpy(), g1.cpu().numpy()) > 1e-3  # (a different batch)


def test_nvls_step_replays_from_a_cuda_graph(setup):
    d, e, plan, _, g = setup
    v = torch.from_numpy((0.9 * d.v_true).astype(np.complex64)).cuda()
    dev = e.dev
    grad = torch.empty(e.n_voxels, dtype=torch.complex64, device=dev)
    sq, sqt, loss = (torch.empty(1, dtype=torch.float64, device=dev) for _ in range(3))
    nscr = e._norm_scratch()
    e.scratch(plan.B)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        D.nvls_planned_step(e, g, plan, 1, v, 4.0, 1e-3, grad, sq, sqt, loss, nscr)  # warm (grids, attributes)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        D.nvls_planned_step(e, g, plan, 1, v, 4.0, 1e-3, grad, sq, sqt, loss, nscr)
    outs = []
    for _ in range(3):
        graph.replay()
        torch.cuda.synchronize()
        outs.append((grad.clone(), float(loss)))
    g.check()
    ref_grad = torch.empty_like(grad)
    ref_loss, _ = e.loss_grad_step_planned(v, plan, 1, 4.0, 1e-3, ref_grad)
    for gg, ll in outs:
        assert O.relative_l2(gg.cpu().numpy(), ref_grad.cpu().numpy()) < 1e-6
        assert abs(ll - float(ref_loss)) / float(ref_loss) < 1e-9
