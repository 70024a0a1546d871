"""GPU parity at the NAMED BASELINE configurations, on the same seeded inputs as the oracle.

north_star: "Correctness is checked against the reference's CPU implementation on the
same seeded inputs": nn voxel indices bit-exact; projections, gradients and Hutchinson
diagonals within relative L2 1e-5 (fp32); preconditioned-SGD loss trajectories within
1e-4 relative over 10 steps.  The datasets are generated on the host in fp64 by the
oracle (tests/cfg_data.py) and uploaded, so both sides see identical images.

* cfg1  M=32, 1,000 images, nn, no CTF / shifts, SNR 0.1: full-batch loss + gradient,
        all 1,000 x 749 nn voxel indices bit-exact, 8-probe Hutchinson.
* cfg2  M=64, 10,000 images, tri, physical CTF, shifts, SNR 0.05: full-dataset loss +
        gradient and the 32-probe Hutchinson diagonal.
* cfg3  M=128, tri, physical CTF, shifts, SNR 0.05 (a 2,048-image subset of the 50,000):
        the EXACT timed bench step -- fsld_loss_grad_step_planned at B=512 with
        n_total = 50,000 (scale = 50,000 / 512), v = 0.9 v_true, full 64-segment work
        items -- plus the fused probe fold and the line-search energy of the same plan;
        and a 10-step Algorithm-1 trajectory (optim.run on the device) against the
        oracle's loop (optim.py:362-382).

Reference lines: loss_and_grad / hutchinson_update optim.py:165-229; run optim.py:309-393;
project_nn / backproject_nn kernels.py:180-190, 233-248; _nn_index kernels.py:69-120.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O

import cfg_data
from harness import sgd_harness
import paper_2311_16100_b200 as F
from paper_2311_16100_b200 import kernels as K
from paper_2311_16100_b200 import optim as Opt

pytestmark = pytest.mark.gpu

TOL = 1e-5


def rel(a, b):
    return O.relative_l2(np.asarray(a), np.asarray(b))


@pytest.fixture(scope="module")
def cfg1():
    d = cfg_data.make(32, 1000, "nn", ctf=False, shifts=False, snr=0.1)
    return d, cfg_data.gpu_operator(d)


@pytest.fixture(scope="module")
def cfg2():
    d = cfg_data.make(64, 10000, "tri", ctf=True, shifts=True, snr=0.05)
    return d, cfg_data.gpu_operator(d)


@pytest.fixture(scope="module")
def cfg3():
    d = cfg_data.make(128, 2048, "tri", ctf=True, shifts=True, snr=0.05)
    return d, cfg_data.gpu_operator(d)


def _probes(k, n, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 2, size=(k, n)).astype(np.float64) * 2.0 - 1.0


def _oracle_hutch(oop, Z, batch, lam, n_total=None):
    return np.mean([z * oop.hvp(z, batch, lam, n_total).real for z in Z], axis=0)


# ---------------------------------------------------------------- cfg1 (M=32, nn)

def test_cfg1_nn_indices_bitexact_all_images(cfg1):
    d, op = cfg1
    got = K.assign_nn(d.oop.rots, d.pix, d.M)
    ref = O.assign_nn(d.oop.rots, d.pix, d.M)
    assert got.shape == (1000, 749)
    assert np.array_equal(got, ref)
    dev = op.engine.assign_nn(np.arange(1000)).cpu().numpy().astype(np.int64)
    assert np.array_equal(dev, ref)


def test_cfg1_nn_loss_grad_full_batch(cfg1):
    d, op = cfg1
    idx = np.arange(1000)
    v = 0.9 * d.v_true
    lam = 1e-3
    lr, gr = O.loss_and_grad(d.oop, v, idx, lam)
    lg, gg = F.loss_and_grad(op, v, idx, lam)
    assert abs(lg - lr) / lr < TOL
    assert rel(gg, gr) < TOL
    assert rel(op.project(v, idx[:100]), d.oop.project(v, idx[:100])) < TOL


def test_cfg1_nn_hutchinson_8_probes(cfg1):
    d, op = cfg1
    idx = np.arange(1000)
    Z = _probes(8, d.M ** 3, 11)
    lam = 1e-3
    got, k = Opt.hutchinson_sample(op, Z, idx, lam)
    assert k == 8
    assert rel(got, _oracle_hutch(d.oop, Z, idx, lam)) < TOL
    # nn: z (.) (A*A z) with one image's mask is exact per probe (SPEC "NN Hutchinson exact")
    st = F.PreconditionerState.initial(d.M ** 3, 1.0)
    F.hutchinson_update(st, op, Z, idx, lam)
    assert rel(st.d_avg, O.exact_diag(d.oop, lam)) < 1e-6


# ---------------------------------------------------------------- cfg2 (M=64, tri, 10,000 images)

def test_cfg2_full_loss_grad(cfg2):
    d, op = cfg2
    idx = np.arange(10000)
    v = 0.9 * d.v_true
    lam = 1e-3
    lr, gr = O.loss_and_grad(d.oop, v, idx, lam)
    lg, gg = F.loss_and_grad(op, v, idx, lam)
    assert abs(lg - lr) / lr < TOL
    assert rel(gg, gr) < TOL


def test_cfg2_hutchinson_32_probes(cfg2):
    d, op = cfg2
    idx = np.arange(10000)
    Z = _probes(32, d.M ** 3, 12)
    lam = 1e-3
    got, k = Opt.hutchinson_sample(op, Z, idx, lam)
    assert k == 32
    assert rel(got, _oracle_hutch(d.oop, Z, idx, lam)) < TOL


# ---------------------------------------------------------------- cfg3 (M=128, the timed step)

N_TOTAL_CFG3 = 50000


def test_cfg3_exact_timed_step_vs_oracle(cfg3):
    """The bench's timed call (fsld_loss_grad_step_planned, batch k of a binning plan, grad
    overwritten with scale * sum P^* conj(f) r + lam v) at B=512 against the oracle."""
    d, op = cfg3
    e = op.engine
    assert e.brick_path
    perm = np.random.default_rng(7).permutation(2048)
    batches = perm.reshape(4, 512)
    plan = e.make_plan(batches)
    v_h = 0.9 * d.v_true
    v = torch.from_numpy(v_h.astype(np.complex64)).cuda()
    lam = 1e-3
    scale = N_TOTAL_CFG3 / 512
    grad = torch.empty(d.M ** 3, dtype=torch.complex64, device="cuda")
    for k in (0, 3):
        loss, sq = e.loss_grad_step_planned(v, plan, k, scale, lam, grad)
        lr, gr = O.loss_and_grad(d.oop, v_h.astype(np.complex64).astype(np.complex128), batches[k], lam,
                                 n_total=N_TOTAL_CFG3)
        assert abs(float(loss) - lr) / lr < TOL, k
        assert rel(grad.cpu().numpy(), gr) < TOL, k
    # the batches really fill work items of 64 segments (the fixed-point budget's worst case):
    # segments per brick over batch 0, from the dataset's (brick, start | count << 16) list
    so = e.seg_off.cpu().numpy()
    sg = e.segs.cpu().numpy()
    bricks = np.concatenate([sg[so[r]:so[r + 1], 0] for r in batches[0]])
    assert np.bincount(bricks).max() >= 64


def test_cfg3_fused_probe_and_line_search_energy(cfg3):
    """The Algorithm-1 step's other two brick passes on the same plan: the loss+grad pass carrying
    the k=1 probe (fold = z (.) sum P^*C^2P z) and the gather-only ||A d||^2."""
    d, op = cfg3
    e = op.engine
    batches = np.random.default_rng(8).permutation(2048).reshape(4, 512)
    plan = e.make_plan(batches)
    v_h = (0.9 * d.v_true).astype(np.complex64)
    v = torch.from_numpy(v_h).cuda()
    z = _probes(1, d.M ** 3, 13)[0]
    zbits, _ = e.pack_probes(z)
    acc = torch.zeros(d.M ** 3, dtype=torch.complex64, device="cuda")
    fold = torch.zeros(d.M ** 3, dtype=torch.float32, device="cuda")
    sq = e.loss_grad_planned(v, plan, 1, acc, zbits=zbits, fold=fold)
    b = batches[1]
    hz = d.oop.hvp(z, b, 0.0, n_total=len(b)).real
    assert rel(fold.cpu().numpy(), z * hz) < TOL
    sq_r, acc_r = O._resid_pass(d.oop, v_h.astype(np.complex128), b, True)
    assert abs(float(sq) - sq_r) / sq_r < TOL
    assert rel(acc.cpu().numpy(), acc_r) < TOL
    dvec = d.v_true - v_h.astype(np.complex128)
    en = float(e.proj_energy_planned(torch.from_numpy(dvec.astype(np.complex64)).cuda(), plan, 1).item())
    ad = d.oop.project(dvec.astype(np.complex64).astype(np.complex128), b)
    en_r = float((ad.real ** 2 + ad.imag ** 2).sum())
    assert abs(en - en_r) / en_r < TOL


def test_cfg3_algorithm1_10_steps_vs_oracle_loop(cfg3):
    """optim.run on the device (estimated variant, reference z stream, B=512) against the oracle's
    loop (optim.py:362-382): identical Armijo step sizes and backtracks, f0 / accepted loss within
    1e-4 relative over the first 10 steps."""
    d, op = cfg3
    lam = 1e-3
    seed = 0
    spec = F.GridSpec(d.M)
    # alpha from the oracle's CTF table: P_x(R)/P_v(R) * sum_i mean_{|k|~R} C_i^2 + lam
    R = d.M // 2 - 1
    radii = np.round(np.sqrt((d.pix ** 2).sum(axis=1))).astype(int)
    ring = radii == R
    from paper_2311_16100_b200.grid import shell_counts
    px, vx = shell_counts(d.M, R)
    alpha = float(px[R]) / float(vx[R]) * float(np.sum(np.mean(d.ctab[:, ring] ** 2, axis=1))) + lam
    rec, v_ref, _ = sgd_harness(O, d.oop, d.M ** 3, 2048, lam, alpha, 512, seed, 10)
    images = np.zeros((2048, d.M * d.M), dtype=np.complex128)
    images[:, d.mask] = d.x
    poses = [F.Pose(q, t) for q, t in zip(d.quats, d.shifts)]
    stack = F.ImageStack(spec, images, poses, d.ctfs, sigma=0.05, seed=seed, mask_radius=R, mode="tri")
    assert abs(Opt.threshold_alpha(stack, None, lam) - alpha) <= 1e-7 * alpha
    cfg = Opt.OptimConfig(lam=lam, batch_size=512, epochs=3, seed=seed, mode="tri")
    vol, tr = Opt.run(cfg, stack, op=op, alpha=alpha)
    etas = np.array(tr.accepted_etas[:10])
    assert np.array_equal(etas, rec[:, 1])
    assert np.array_equal(np.array(tr.step_backtracks[:10]), rec[:, 3].astype(int))
    assert np.max(np.abs(np.array(tr.step_f0[:10]) - rec[:, 0]) / np.abs(rec[:, 0])) < 1e-4
    assert np.max(np.abs(np.array(tr.step_f_next[:10]) - rec[:, 2]) / np.abs(rec[:, 2])) < 1e-4


def test_cfg1_nn_brick_kernel_vs_tile_path(cfg1):
    """nn mode on the table-driven brick kernel (FSLD_NN_BRICK: one gather, one complex shared add per
    pixel) equals the per-pixel tile kernel (one global RED per pixel, the nn default: faster at every
    measured M) in loss and gradient, and its Hessian product matches the oracle's."""
    d, _ = cfg1
    from paper_2311_16100_b200.engine import SliceEngine, records_for
    from paper_2311_16100_b200.forward import DatasetOperator
    e = SliceEngine(d.M, "nn", d.mask, records_for(d.M, d.quats), d.x, nn_brick=True)
    op = DatasetOperator.from_engine(e)
    assert e.table_path and e.mode == "nn"
    idx = np.arange(1000)
    v = torch.from_numpy((0.9 * d.v_true).astype(np.complex64)).cuda()
    sq1, a1, _ = e.loss_grad(v, idx)
    tile = SliceEngine(d.M, "nn", d.mask, records_for(d.M, d.quats), d.x, tile_path=True)
    sq2, a2, _ = tile.loss_grad(v, idx)
    assert abs(float(sq1) - float(sq2)) <= 1e-6 * float(sq2)
    assert rel(a1.cpu().numpy(), a2.cpu().numpy()) < 1e-5
    z = _probes(1, d.M ** 3, 21)[0]
    assert rel(op.hvp(z, idx, 0.0), d.oop.hvp(z, idx, 0.0)) < TOL
