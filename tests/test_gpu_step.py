"""GPU: the device-resident Algorithm-1 step against the reference.

* fsld_armijo_terms + fsld_precond_step give batch_loss(v - eta d) in closed form;
  checked against explicit batch_loss passes at several eta;
* fsld_precond_step's grad / dhat / direction against the reference formulas
  (optim.py:186-189, 210-247, 292-293) evaluated by the oracle;
* optim.run (device loop) reproduces the reference's 10-step Algorithm-1
  trajectory of the golden fixtures (made by the reference itself,
  tests/golden/make_golden.py): identical Armijo step sizes and backtracks,
  f0 / accepted loss within 1e-4;
* the plain and precomputed variants against an oracle loop.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O

import paper_2311_16100_b200 as F
from paper_2311_16100_b200 import _capi as C
from paper_2311_16100_b200 import optim as Opt
from paper_2311_16100_b200.engine import SliceEngine, records_for
from paper_2311_16100_b200.forward import CtfParams, DatasetOperator

pytestmark = pytest.mark.gpu


def rel(a, b):
    return O.relative_l2(np.asarray(a), np.asarray(b))


def radial_ctfs(params):
    return [CtfParams(float(d), float(w), float(b)) for d, w, b in params] if len(params) else None


def golden_stack(g, seed):
    M = int(g["M"])
    spec = F.GridSpec(M)
    mask = g["mask"]
    images = np.zeros((g["x"].shape[0], M * M), dtype=np.complex128)
    images[:, mask] = g["x"]
    poses = [F.Pose(q, t) for q, t in zip(g["quats"], g["shifts"])]
    return F.ImageStack(spec, images, poses, radial_ctfs(g["ctf_params"]), sigma=0.05, seed=seed,
                        mask_radius=M // 2 - 1, mode=str(g["mode"]))


def golden_op(g, layout=None, deterministic=False):
    M = int(g["M"])
    recs = records_for(M, g["quats"], g["shifts"], radial_ctfs(g["ctf_params"]))
    eng = SliceEngine(M, str(g["mode"]), g["mask"], recs, g["x"], deterministic=deterministic, layout=layout)
    return DatasetOperator.from_engine(eng, F.GridSpec(M))


@pytest.mark.parametrize("name", ["dataset_m16_nn.npz", "dataset_m16_tri.npz"])
@pytest.mark.parametrize("layout", ["sorted", "mask"])
def test_closed_form_line_search_matches_batch_loss(golden, name, layout):
    g = golden(name)
    op = golden_op(g, layout=layout)
    e = op.engine
    lam = float(g["lam"])
    batch = g["batch"]
    n = op.n_images
    scale = n / batch.size
    v = torch.from_numpy(g["v1"].astype(np.complex64)).cuda()
    sq, acc, _ = e.loss_grad(v, batch)
    dirv = torch.empty_like(v)
    dh = torch.from_numpy((1.0 + np.random.default_rng(0).random(v.numel())).astype(np.float32)).cuda()
    p = C.StepParams(scale=scale, lam=lam, beta=0.9, floor=1.0, w_old=0.0, w_new=1.0, hutch_scale=scale,
                     estimating=0)
    vol4 = e.precond_step(acc, v, p, dirv, dhat_fixed=dh).cpu().numpy()
    t3 = e.armijo_terms(v, dirv, batch).cpu().numpy()
    qq = float(e.proj_energy(dirv, batch).item())
    if e.brick_path:  # reusing the loss+grad call's work items gives the same energy
        bt = e.idx_tensor(batch)
        e.loss_grad(v, bt)
        qq2 = float(e.proj_energy(dirv, bt, reuse_bins=True).item())
        assert abs(qq2 - qq) / qq < 1e-6
        with pytest.raises(ValueError):  # a different batch tensor was never binned on this scratch
            e.proj_energy(dirv, e.idx_tensor(batch[::-1].copy()), reuse_bins=True)
    sq = float(sq.item())
    assert abs(t3[0] - sq) / sq < 1e-6
    assert abs(t3[1] - vol4[4]) / abs(t3[1]) < 1e-5  # Re<r, A d> from the pixels == Re<A^* r, d> from acc
    assert abs(t3[2] - qq) / t3[2] < 1e-5            # brick gather-only energy == tile projection
    f0 = 0.5 * scale * sq + 0.5 * lam * vol4[1]
    d_h = dirv.cpu().numpy().astype(np.complex128)
    v_h = g["v1"]
    for eta in (1.0, 0.25, 1e-3):
        f_cf = f0 + 0.5 * scale * (eta * eta * t3[2] - 2 * eta * t3[1]) + 0.5 * lam * (eta * eta * vol4[3]
                                                                                     - 2 * eta * vol4[2])
        f_ex = F.batch_loss(op, v_h - eta * d_h, batch, lam)
        assert abs(f_cf - f_ex) / abs(f_ex) < 1e-5, (eta, f_cf, f_ex)


@pytest.mark.parametrize("name", ["dataset_m16_nn.npz", "dataset_m16_tri.npz"])
def test_precond_step_matches_reference_formulas(golden, name):
    g = golden(name)
    op = golden_op(g)
    e = op.engine
    lam = float(g["lam"])
    batch = g["batch"]
    n = op.n_images
    scale = n / batch.size
    M3 = int(g["M"]) ** 3
    rng = np.random.default_rng(5)
    v_h = g["v1"]
    v = torch.from_numpy(v_h.astype(np.complex64)).cuda()
    z = O.rademacher(rng, M3)
    d_avg0 = rng.random(M3) * 3
    d0 = rng.random(M3) * 3
    k_old, beta, alpha = 3, 0.9, 0.7
    # device step
    zbits, k = e.pack_probes(z)
    fold = torch.zeros(M3, dtype=torch.float32, device="cuda")
    e.hutch_fold(zbits, k, batch, acc=fold)
    sq, acc, _ = e.loss_grad(v, batch)
    d_avg = torch.from_numpy(d_avg0.astype(np.float32)).cuda()
    d = torch.from_numpy(d0.astype(np.float32)).cuda()
    dirv = torch.empty_like(v)
    grad = torch.empty_like(v)
    dhat = torch.empty(M3, dtype=torch.float32, device="cuda")
    p = C.StepParams(scale=scale, lam=lam, beta=beta, floor=alpha, w_old=k_old / (k_old + 1),
                     w_new=1.0 / (k_old + 1), hutch_scale=scale, estimating=1)
    vol4 = e.precond_step(acc, v, p, dirv, fold=fold, d_avg=d_avg, d=d, grad_out=grad, dhat_out=dhat)
    # reference formulas on the oracle
    _, oop = _oracle_op(g)
    st = O.OracleState(M3, alpha)
    st.d_avg, st.d, st.k = d_avg0.copy(), d0.copy(), k_old
    O.hutchinson_update(st, oop, z, batch, lam)
    dh_ref = O.ema_and_threshold(st, beta, alpha, True)
    _, g_ref = O.loss_and_grad(oop, v_h, batch, lam)
    dir_ref = g_ref / dh_ref
    assert rel(grad.cpu().numpy(), g_ref) < 1e-5
    assert rel(d_avg.cpu().numpy(), st.d_avg) < 1e-5
    assert rel(dhat.cpu().numpy(), dh_ref) < 1e-5
    assert rel(dirv.cpu().numpy(), dir_ref) < 1e-5
    o = vol4.cpu().numpy()
    dec_ref = float(((g_ref.real ** 2 + g_ref.imag ** 2) / dh_ref).sum())
    assert abs(o[0] - dec_ref) / dec_ref < 1e-5
    assert abs(o[1] - float((np.abs(v_h) ** 2).sum())) / float((np.abs(v_h) ** 2).sum()) < 1e-5
    assert abs(o[2] - float((v_h.conj() * dir_ref).real.sum())) / abs(float((v_h.conj() * dir_ref).real.sum())) < 1e-4
    assert abs(o[3] - float((np.abs(dir_ref) ** 2).sum())) / float((np.abs(dir_ref) ** 2).sum()) < 1e-5
    ad_ref = float(((g_ref - lam * v_h) / scale * dir_ref.conj()).real.sum())
    assert abs(o[4] - ad_ref) / abs(ad_ref) < 1e-4
    # accumulators were consumed
    assert float(acc.abs().max()) == 0.0 and float(fold.abs().max()) == 0.0


def _oracle_op(g):
    M = int(g["M"])
    mode = str(g["mode"])
    ctfs = radial_ctfs(g["ctf_params"])
    ctab = None if ctfs is None else O.ctf_table_radial(g["ctf_params"], O.mask_pix(M, g["mask"]), M)
    return None, O.OracleOperator(M, mode, g["mask"], g["quats"], g["shifts"], ctab, g["x"])


@pytest.mark.parametrize("name,seed", [("dataset_m16_nn.npz", 3), ("dataset_m16_tri.npz", 4)])
def test_device_run_reproduces_reference_trajectory(golden, name, seed):
    g = golden(name)
    stack = golden_stack(g, seed)
    lam = float(g["lam"])
    assert abs(Opt.threshold_alpha(stack, None, lam) - float(g["alpha"])) <= 1e-12 * float(g["alpha"])
    cfg = Opt.OptimConfig(lam=lam, batch_size=int(g["batch"].size), epochs=3, seed=seed, mode=str(g["mode"]))
    vol, tr = Opt.run(cfg, stack)
    ref = g["sgd_rec"]
    etas = np.array(tr.accepted_etas[:10])
    assert np.array_equal(etas, ref[:, 1])  # identical Armijo decisions
    assert np.array_equal(np.array(tr.step_backtracks[:10]), ref[:, 3].astype(int))
    f0 = np.array(tr.step_f0[:10])
    fn = np.array(tr.step_f_next[:10])
    assert np.max(np.abs(f0 - ref[:, 0]) / np.abs(ref[:, 0])) < 1e-4
    assert np.max(np.abs(fn - ref[:, 2]) / np.abs(ref[:, 2])) < 1e-4
    assert tr.armijo_violations == 0 and tr.armijo_steps == 12
    assert np.all(np.isfinite(tr.loss)) and tr.loss[-1] < tr.loss[0]
    assert tr.final_dhat.shape == (int(g["M"]) ** 3,) and np.all(tr.final_dhat >= float(g["alpha"]) * (1 - 1e-6))


def _oracle_fixed_dhat_loop(oop, n, lam, batch_size, seed, dhat, n_epochs, c=0.5, eta0=1.0):
    v = np.zeros(oop.M ** 3, dtype=np.complex128)
    eta = eta0
    rec = []
    for epoch in range(n_epochs):
        for batch in O.epoch_batches(n, batch_size, seed, epoch):
            f0, grad = O.loss_and_grad(oop, v, batch, lam)
            eta, v, f_next, nbt = O.armijo_search(v, grad, dhat, lambda w: O.batch_loss(oop, w, batch, lam),
                                                  eta, c, f0)
            rec.append((f0, eta, f_next, nbt))
    return np.array(rec), v


@pytest.mark.parametrize("variant", ["plain", "precomputed"])
def test_device_run_fixed_preconditioner_variants(golden, variant):
    g = golden("dataset_m16_tri.npz")
    seed = 4
    stack = golden_stack(g, seed)
    lam = float(g["lam"])
    _, oop = _oracle_op(g)
    n = oop.n_images
    alpha = float(g["alpha"])
    dhat = np.ones(int(g["M"]) ** 3) if variant == "plain" else np.maximum(g["exact_diag"], alpha)
    rec, v_ref = _oracle_fixed_dhat_loop(oop, n, lam, 24, seed, dhat, 2)
    cfg = Opt.OptimConfig(lam=lam, batch_size=24, epochs=2, seed=seed, mode="tri", variant=variant)
    vol, tr = Opt.run(cfg, stack, exact_diag_vec=g["exact_diag"] if variant == "precomputed" else None)
    assert np.array_equal(np.array(tr.accepted_etas), rec[:, 1])
    assert np.max(np.abs(np.array(tr.step_f_next) - rec[:, 2]) / np.abs(rec[:, 2])) < 1e-4
    assert rel(vol.values, v_ref) < 1e-4


def test_device_run_deterministic_engine_and_fsc(golden):
    g = golden("dataset_m16_tri.npz")
    seed = 4
    stack = golden_stack(g, seed)
    lam = float(g["lam"])
    cfg = Opt.OptimConfig(lam=lam, batch_size=24, epochs=2, seed=seed, mode="tri")
    _, tr = Opt.run(cfg, stack)
    opd = golden_op(g, deterministic=True)
    vol_d, trd = Opt.run(cfg, stack, op=opd, reference=F.FourierVolume(g["v_true"], F.GridSpec(16)))
    assert trd.accepted_etas == tr.accepted_etas
    assert np.max(np.abs(trd.loss - tr.loss) / tr.loss) < 1e-4
    # deterministic engine: bitwise repeatable trajectory
    vol_d2, trd2 = Opt.run(cfg, stack, op=golden_op(g, deterministic=True))
    assert np.array_equal(vol_d.values, vol_d2.values)
    assert trd.fsc_history.shape == (2, 8) and np.all(np.isfinite(trd.fsc_history[:, 1:]))


@pytest.mark.parametrize("cfgname", ["m32", "m64"])
def test_fused_loss_grad_hutch_matches_separate_passes_and_oracle(cfgname):
    from paper_2311_16100_b200 import synth
    M = 32 if cfgname == "m32" else 64
    N = 96
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(N, 21)
    sh = synth.normal_shifts(N, 22)
    ctfs = synth.physical_ctfs(N, 23)
    pix = O.mask_pix(M, mask)
    rng = np.random.default_rng(24)
    x = (rng.standard_normal((N, mask.size)) + 1j * rng.standard_normal((N, mask.size))).astype(np.complex64)
    recs = records_for(M, q, sh, ctfs)
    e = SliceEngine(M, "tri", mask, recs, x)
    assert e.layout == "sorted"
    v = torch.from_numpy((rng.standard_normal(M ** 3) + 1j * rng.standard_normal(M ** 3)).astype(np.complex64)).cuda()
    z = O.rademacher(rng, M ** 3)
    zbits, _ = e.pack_probes(z)
    batch = rng.permutation(N)[:64]
    acc1 = torch.zeros(M ** 3, dtype=torch.complex64, device="cuda")
    fold1 = torch.zeros(M ** 3, dtype=torch.float32, device="cuda")
    sq1 = e.loss_grad_hutch(v, batch, zbits, acc1, fold1)
    sq2, acc2, _ = e.loss_grad(v, batch)
    fold2 = torch.zeros(M ** 3, dtype=torch.float32, device="cuda")
    e.hutch_fold(zbits, 1, batch, acc=fold2)
    assert abs(float(sq1) - float(sq2)) / float(sq2) < 1e-6
    assert rel(acc1.cpu().numpy(), acc2.cpu().numpy()) < 1e-5
    assert rel(fold1.cpu().numpy(), fold2.cpu().numpy()) < 1e-5
    # oracle: fold = z * Re(sum_b P^* C^2 P z)  (hvp with lam = 0, scale 1)
    oop = O.OracleOperator(M, "tri", mask, q, sh, O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M), None)
    hz = oop.hvp(z, batch, 0.0, n_total=len(batch))
    assert rel(fold1.cpu().numpy(), z * hz.real) < 1e-5


@pytest.mark.parametrize("k", [1, 5, 37, 64, 256])
def test_brick_probe_batcher_matches_tile_batcher(k):
    from paper_2311_16100_b200 import synth
    M, N = 64, 128
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(N, 31)
    sh = synth.normal_shifts(N, 32)
    ctfs = synth.physical_ctfs(N, 33)
    recs = records_for(M, q, sh, ctfs)
    brick = SliceEngine(M, "tri", mask, recs)
    tile = SliceEngine(M, "tri", mask, recs, tile_path=True)
    assert brick.layout == "sorted"
    zb = brick.gen_probes(k, 7 + k)
    batch = np.random.default_rng(k).permutation(N)[:100]
    f1, _ = brick.hutch_fold(zb, k, batch)
    f2, _ = tile.hutch_fold(zb, k, batch)
    assert rel(f1.cpu().numpy(), f2.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("M,N,nb", [(32, 96, 64), (64, 300, 300)])
def test_brick_hessian_product_matches_tile_and_oracle(M, N, nb):
    """fsld_hvp_sorted (brick loss+grad kernel with zero images) vs fsld_hvp (tile) and the oracle;
    its sq_out is ||A z||^2 = the line-search energy of z.  HVP_CHUNK is lowered to 128 so that
    several launches accumulate into one accumulator."""
    from paper_2311_16100_b200 import synth
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(N, 41)
    sh = synth.normal_shifts(N, 42)
    ctfs = synth.physical_ctfs(N, 43)
    pix = O.mask_pix(M, mask)
    recs = records_for(M, q, sh, ctfs)
    brick = SliceEngine(M, "tri", mask, recs)
    tile = SliceEngine(M, "tri", mask, recs, tile_path=True)
    assert brick.brick_path and not tile.brick_path
    rng = np.random.default_rng(44)
    z = torch.from_numpy((rng.standard_normal(M ** 3) + 1j * rng.standard_normal(M ** 3)).astype(np.complex64)).cuda()
    batch = rng.permutation(N)[:nb]
    brick.HVP_CHUNK = 128  # several launches accumulate into one acc
    h1, _ = brick.hvp_acc(z, batch)
    h2, _ = tile.hvp_acc(z, batch)
    assert rel(h1.cpu().numpy(), h2.cpu().numpy()) < 1e-5
    oop = O.OracleOperator(M, "tri", mask, q, sh, O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M), None)
    hz = oop.hvp(z.cpu().numpy().astype(np.complex128), batch, 0.0, n_total=len(batch))
    assert rel(h1.cpu().numpy(), hz) < 1e-5
    # ||A z||^2 through the ABI (one launch) against the gather-only energy pass
    idx = brick.idx_tensor(batch)
    acc = torch.zeros(M ** 3, dtype=torch.complex64, device="cuda")
    sq = torch.zeros(1, dtype=torch.float64, device="cuda")
    scr = brick.scratch(nb)
    from paper_2311_16100_b200.engine import ctypes_ptr, _stream
    C.check(C.load().fsld_hvp_sorted(M, brick.mode_id, brick.n_mask, ctypes_ptr(brick.recs), ctypes_ptr(idx), nb,
                                     ctypes_ptr(z), ctypes_ptr(brick.pc), ctypes_ptr(brick.ptab), ctypes_ptr(brick.seg_off),
                                     ctypes_ptr(brick.segs), ctypes_ptr(acc), ctypes_ptr(sq), 0, ctypes_ptr(scr),
                                     scr.numel() * 8, _stream()), "fsld_hvp_sorted")
    en = brick.proj_energy(z, batch)
    assert abs(float(sq) - float(en)) / float(en) < 1e-5
    assert rel(acc.cpu().numpy(), hz) < 1e-5
    assert C.load().fsld_hvp_sorted(M, brick.mode_id, brick.n_mask, ctypes_ptr(brick.recs), ctypes_ptr(idx), nb,
                                    ctypes_ptr(z), ctypes_ptr(brick.pc), ctypes_ptr(brick.ptab), ctypes_ptr(brick.seg_off),
                                    ctypes_ptr(brick.segs), ctypes_ptr(acc), None, 0, ctypes_ptr(scr),
                                    scr.numel() * 8, _stream()) == C.FSLD_EINVAL


@pytest.mark.parametrize("name,seed", [("dataset_m16_nn.npz", 3), ("dataset_m16_tri.npz", 4)])
def test_device_run_ragged_last_batch_vs_oracle(golden, name, seed):
    """N = 96 with batch_size 28: every epoch ends with a 12-image batch (scale N/12, optim.py:183)."""
    from harness import sgd_harness
    g = golden(name)
    stack = golden_stack(g, seed)
    lam = float(g["lam"])
    _, oop = _oracle_op(g)
    rec, v_ref, _ = sgd_harness(O, oop, int(g["M"]) ** 3, oop.n_images, lam, float(g["alpha"]), 28, seed, 8)
    cfg = Opt.OptimConfig(lam=lam, batch_size=28, epochs=2, seed=seed, mode=str(g["mode"]))
    vol, tr = Opt.run(cfg, stack)
    assert tr.armijo_steps == 8
    assert np.array_equal(np.array(tr.accepted_etas), rec[:, 1])
    assert np.array_equal(np.array(tr.step_backtracks), rec[:, 3].astype(int))
    assert np.max(np.abs(np.array(tr.step_f0) - rec[:, 0]) / np.abs(rec[:, 0])) < 1e-4
    assert rel(vol.values, v_ref) < 1e-4


def test_binning_plan_matches_per_step_binning():
    """fsld_plan_build bins K batches at once; each planned step equals the per-step binned call."""
    from paper_2311_16100_b200 import synth
    wl = synth.build_workload(synth.CONFIGS["cfg2"], seed=3, n_images=512)
    e = wl.engine
    rng = np.random.default_rng(0)
    batches = np.stack([rng.choice(e.n_images, 96, replace=False) for _ in range(5)])
    plan = e.make_plan(batches)
    v = torch.from_numpy((wl.v_true * 0.8).astype(np.complex64)).cuda()
    zb = e.gen_probes(1, 9)
    for k in (0, 3, 4, 3):  # any order, repeated
        acc1 = torch.zeros(e.n_voxels, dtype=torch.complex64, device="cuda")
        fold1 = torch.zeros(e.n_voxels, dtype=torch.float32, device="cuda")
        sq1 = e.loss_grad_planned(v, plan, k, acc1, zbits=zb, fold=fold1)
        acc2 = torch.zeros_like(acc1)
        fold2 = torch.zeros_like(fold1)
        sq2 = e.loss_grad_hutch(v, batches[k], zb, acc2, fold2)
        assert abs(float(sq1) - float(sq2)) / float(sq2) < 1e-6
        assert rel(acc1.cpu().numpy(), acc2.cpu().numpy()) < 1e-5
        assert rel(fold1.cpu().numpy(), fold2.cpu().numpy()) < 1e-5
        q1 = float(e.proj_energy_planned(v, plan, k).item())
        q2 = float(e.proj_energy(v, batches[k]).item())
        assert abs(q1 - q2) / q2 < 1e-6
    with pytest.raises(ValueError):
        e.loss_grad_planned(v, plan, 5, acc1)  # k out of range


def test_fused_epilogue_step_matches_accumulator_path_and_oracle():
    """fsld_loss_grad_step_planned (grad = lam v, brick pass adding scale * sums into grad, loss
    finalize) against the accumulator path (planned loss+grad + epilogue) and the oracle's
    loss_and_grad (optim.py:165-190)."""
    from paper_2311_16100_b200 import synth
    M, N, B = 32, 200, 64
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(N, 51)
    sh = synth.normal_shifts(N, 52)
    ctfs = synth.physical_ctfs(N, 53)
    pix = O.mask_pix(M, mask)
    rng = np.random.default_rng(54)
    x = (rng.standard_normal((N, mask.size)) + 1j * rng.standard_normal((N, mask.size))).astype(np.complex64)
    e = SliceEngine(M, "tri", mask, records_for(M, q, sh, ctfs), x)
    assert e.brick_path
    batches = np.stack([rng.choice(N, B, replace=False) for _ in range(3)])
    plan = e.make_plan(batches)
    v_h = synth.gaussian_blob_volume(M, 5).astype(np.complex64)
    v = torch.from_numpy(v_h).cuda()
    lam = 0.37
    oop = O.OracleOperator(M, "tri", mask, q, sh, O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M),
                           x.astype(np.complex128))
    for k in (2, 0):
        scale = N / B
        grad = torch.full((M ** 3,), 7.0, dtype=torch.complex64, device="cuda")  # overwritten, not accumulated
        loss, sq = e.loss_grad_step_planned(v, plan, k, scale, lam, grad)
        acc = torch.zeros(M ** 3, dtype=torch.complex64, device="cuda")
        sq2 = e.loss_grad_planned(v, plan, k, acc)
        loss2, grad2 = e.epilogue(acc, v, scale, lam, sq2)
        assert abs(float(sq) - float(sq2)) <= 1e-12 * abs(float(sq2))
        assert abs(float(loss) - float(loss2[0])) <= 1e-7 * abs(float(loss2[0]))
        assert rel(grad.cpu().numpy(), grad2.cpu().numpy()) < 1e-6
        l_ref, g_ref = O.loss_and_grad(oop, v_h.astype(np.complex128), batches[k], lam)
        assert abs(float(loss) - l_ref) / abs(l_ref) < 1e-5
        assert rel(grad.cpu().numpy(), g_ref) < 1e-5
    with pytest.raises(ValueError):
        e.loss_grad_step_planned(v, plan, 0, 1.0, lam, v)  # grad must not alias v


@pytest.mark.parametrize("name,seed", [("dataset_m16_nn.npz", 3), ("dataset_m16_tri.npz", 4)])
def test_reference_solve_residual_vs_oracle(golden, name, seed):
    """Device CG (optim.reference_solve, optim.py:396-450): the returned volume solves H v = b to the
    fp32 floor, checked with the oracle's fp64 operator (H from oracle hvp, b from oracle b_vector)."""
    g = golden(name)
    stack = golden_stack(g, seed)
    lam = float(g["lam"])
    vol = Opt.reference_solve(stack, lam, str(g["mode"]))
    _, oop = _oracle_op(g)
    idx = np.arange(oop.n_images)
    b = oop.b_vector()
    res = oop.hvp(vol.values, idx, lam) - b
    assert np.linalg.norm(res) / np.linalg.norm(b) < 1e-5
    with pytest.raises(ValueError):
        Opt.reference_solve(stack, 0.0, str(g["mode"]))


def test_streaming_fsd1_loader_matches_host_reader():
    """io.load_operator streams the complex128 payload chunk-wise into HBM (masked, complex64 on the
    device) and gives the same operator as DatasetOperator(read_dataset(path))."""
    import os
    from conftest import ROOT
    from paper_2311_16100_b200 import io as fio
    path = os.path.join(ROOT, "tests", "golden", "tiny_m8.fsd1")
    op1, hs = fio.load_operator(path, chunk_images=2)
    st = fio.read_dataset(path)
    op2 = DatasetOperator(st)
    assert np.array_equal(op1.x, op2.x)
    assert np.array_equal(op1.x, st.images[:, op2.mask].astype(np.complex64).astype(np.complex128))
    v = np.random.default_rng(0).standard_normal(512) + 0j
    l1, g1 = F.loss_and_grad(op1, v, np.arange(5), 0.1)
    l2, g2 = F.loss_and_grad(op2, v, np.arange(5), 0.1)
    assert abs(l1 - l2) <= 1e-6 * abs(l2) and rel(g1, g2) < 1e-6


@pytest.mark.parametrize("M,N,B,K", [(33, 40, 1, 3), (16, 24, 24, 1), (64, 64, 17, 4), (256, 20, 6, 2)])
def test_binning_plan_edge_shapes(M, N, B, K):
    """Plans at odd M, single-image batches, whole-dataset batches and M=256 equal per-step binning."""
    from paper_2311_16100_b200 import synth
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(N, M + 11)
    recs = records_for(M, q, synth.normal_shifts(N, M + 12), synth.physical_ctfs(N, M + 13))
    rng = np.random.default_rng(M)
    x = (rng.standard_normal((N, mask.size)) + 1j * rng.standard_normal((N, mask.size))).astype(np.complex64)
    e = SliceEngine(M, "tri", mask, recs, x)
    assert e.brick_path
    batches = np.stack([rng.choice(N, B, replace=False) for _ in range(K)])
    plan = e.make_plan(batches)
    v = torch.from_numpy(synth.gaussian_blob_volume(M, 2).astype(np.complex64)).cuda()
    for k in range(K):
        acc1 = torch.zeros(M ** 3, dtype=torch.complex64, device="cuda")
        sq1 = e.loss_grad_planned(v, plan, k, acc1)
        sq2, acc2, _ = e.loss_grad(v, batches[k])
        assert abs(float(sq1) - float(sq2)) <= 1e-6 * abs(float(sq2))
        assert rel(acc1.cpu().numpy(), acc2.cpu().numpy()) < 1e-5


def test_reuse_bins_rebins_when_rows_were_rewritten_in_place(golden):
    """FSLD_REUSE_BINS is checked by content on the device: the same idx tensor rewritten in place
    after the loss+grad call must give the new batch's energy, not the stale work items'."""
    g = golden("dataset_m16_tri.npz")
    op = golden_op(g)
    e = op.engine
    assert e.brick_path
    rng = np.random.default_rng(3)
    b1 = rng.permutation(e.n_images)[:24]
    b2 = rng.permutation(e.n_images)[:24]
    d = torch.from_numpy((g["v1"] * 0.3).astype(np.complex64)).cuda()
    bt = e.idx_tensor(b1)
    e.loss_grad(d, bt)
    q_same = float(e.proj_energy(d, bt, reuse_bins=True).item())
    assert abs(q_same - float(e.proj_energy(d, b1).item())) <= 1e-6 * q_same
    e.loss_grad(d, bt)
    bt.copy_(torch.from_numpy(b2.astype(np.int32)).cuda())  # same pointer, new rows
    q_new = float(e.proj_energy(d, bt, reuse_bins=True).item())
    q_ref = float(e.proj_energy(d, b2).item())
    assert abs(q_new - q_ref) <= 1e-6 * q_ref
