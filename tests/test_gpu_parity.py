"""GPU parity: the sm_100a path vs the CPU oracle (pinned to the reference) on identical inputs.

Bars (BASELINE.json north_star): nn voxel indices bit-exact; projections,
gradients, Hessian products and Hutchinson diagonals within relative L2
1e-5 (fp32 path vs fp64 reference); SGD loss trajectory within 1e-4
relative over 10 steps.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O

from harness import sgd_harness
import paper_2311_16100_b200 as F
from paper_2311_16100_b200 import kernels as K
from paper_2311_16100_b200 import optim as Opt
from paper_2311_16100_b200 import synth
from paper_2311_16100_b200.engine import SliceEngine, records_for
from paper_2311_16100_b200.forward import CtfParams, DatasetOperator, PhysicalCtf

pytestmark = pytest.mark.gpu

TOL = 1e-5  # relative L2, fp32 path (north_star)


def rel(a, b):
    return O.relative_l2(np.asarray(a), np.asarray(b))


def radial_ctfs(params):
    return [CtfParams(float(d), float(w), float(b)) for d, w, b in params] if len(params) else None


def gpu_op(M, mode, mask, quats, shifts, ctfs, x, deterministic=False):
    recs = records_for(M, quats, shifts, ctfs)
    eng = SliceEngine(M, mode, mask, recs, x, deterministic=deterministic)
    return DatasetOperator.from_engine(eng)


def golden_ops(g, deterministic=False):
    M = int(g["M"])
    mode = str(g["mode"])
    ctfs = radial_ctfs(g["ctf_params"])
    op = gpu_op(M, mode, g["mask"], g["quats"], g["shifts"], ctfs, g["x"], deterministic)
    ctab = None if ctfs is None else O.ctf_table_radial(g["ctf_params"], O.mask_pix(M, g["mask"]), M)
    oop = O.OracleOperator(M, mode, g["mask"], g["quats"], g["shifts"], ctab, g["x"])
    return op, oop


# ---------------------------------------------------------------- kernels.* (table-driven)

@pytest.mark.parametrize("name", ["kernels_m8.npz", "kernels_m16.npz"])
def test_assign_nn_bitexact_golden(golden, name):
    g = golden(name)
    out = K.assign_nn(g["rt"], g["pix"], int(g["M"]))
    assert np.array_equal(out, g["assign_nn"])


@pytest.mark.parametrize("name", ["kernels_m8.npz", "kernels_m16.npz"])
@pytest.mark.parametrize("mode", ["tri", "nn"])
def test_numba_signature_kernels_golden(golden, name, mode):
    g = golden(name)
    M = int(g["M"])
    B, n = g["phase"].shape
    out = np.empty((B, n), dtype=np.complex128)
    (K.project_tri if mode == "tri" else K.project_nn)(g["v"], g["rt"], g["pix"], g["phase"], g["ctf"], M, out)
    assert rel(out, g[f"project_{mode}"]) < TOL
    vols = np.zeros((K.n_chunks(B), M ** 3), dtype=np.complex128)
    (K.backproject_tri if mode == "tri" else K.backproject_nn)(g["img"], g["rt"], g["pix"], g["phase"], g["ctf"],
                                                                 M, vols)
    assert rel(K.fold_chunks(vols), g[f"backproject_{mode}"]) < TOL


def test_scatter_sq_tri_golden(golden):
    g = golden("kernels_m16.npz")
    M = int(g["M"])
    vols = np.zeros((1, M ** 3))
    K.scatter_sq_tri(np.ascontiguousarray(g["ctf"] ** 2), g["rt"], g["pix"], M, vols)
    assert rel(vols[0], g["scatter_sq_tri"]) < TOL


# ---------------------------------------------------------------- in-kernel CTF / shift model

@pytest.mark.parametrize("name", ["kernels_m8.npz", "kernels_m16.npz"])
def test_inkernel_radial_ctf_and_shift_project(golden, name):
    g = golden(name)
    M = int(g["M"])
    ctfs = radial_ctfs(g["ctf_params"])
    recs = records_for(M, g["quats"], g["shifts"], ctfs)
    eng = SliceEngine(M, "tri", g["mask"], recs)
    B = len(g["quats"])
    out = eng.project(torch.from_numpy(g["v"].astype(np.complex64)).cuda(), np.arange(B))
    assert rel(out.cpu().numpy(), g["project_tri"]) < TOL
    acc, fx = eng.backproject(torch.from_numpy(g["img"].astype(np.complex64)).cuda(), np.arange(B))
    assert rel(eng.finalize_c(acc, fx, 1.0, 0.0).cpu().numpy(), g["backproject_tri"]) < TOL


def test_inkernel_physical_ctf_matches_reference_kernels_with_table(golden):
    g = golden("kernels_m16.npz")
    M = int(g["M"])
    ctfs = [PhysicalCtf(*p) for p in g["phys_params"]]
    recs = records_for(M, g["quats"], g["shifts"], ctfs)
    eng = SliceEngine(M, "tri", g["mask"], recs)
    B = len(g["quats"])
    out = eng.project(torch.from_numpy(g["v"].astype(np.complex64)).cuda(), np.arange(B))
    assert rel(out.cpu().numpy(), g["project_tri_phys"]) < TOL
    acc, fx = eng.backproject(torch.from_numpy(g["img"].astype(np.complex64)).cuda(), np.arange(B))
    assert rel(eng.finalize_c(acc, fx, 1.0, 0.0).cpu().numpy(), g["backproject_tri_phys"]) < TOL


@pytest.mark.parametrize("M", [32, 64, 128])
def test_assign_nn_bitexact_vs_oracle_large(M):
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(64, M)
    eng = SliceEngine(M, "nn", mask, records_for(M, q))
    out = eng.assign_nn(np.arange(64)).cpu().numpy().astype(np.int64)
    ref = O.assign_nn(O.rot_table(q), O.mask_pix(M, mask), M)
    assert np.array_equal(out, ref)


# ---------------------------------------------------------------- DatasetOperator / optim

@pytest.mark.parametrize("name", ["dataset_m16_nn.npz", "dataset_m16_tri.npz"])
def test_dataset_operator_golden(golden, name):
    g = golden(name)
    op, _ = golden_ops(g)
    M = int(g["M"])
    lam = float(g["lam"])
    idx = np.arange(op.n_images)
    loss, grad = F.loss_and_grad(op, np.zeros(M ** 3, complex), idx, lam)
    assert abs(loss - float(g["loss0_full"])) / float(g["loss0_full"]) < TOL
    assert rel(grad, g["grad0_full"]) < TOL
    loss, grad = F.loss_and_grad(op, g["v1"], g["batch"], lam)
    assert abs(loss - float(g["loss1_batch"])) / float(g["loss1_batch"]) < TOL
    assert rel(grad, g["grad1_batch"]) < TOL
    bl = F.batch_loss(op, g["v1"], g["batch"], lam)
    assert abs(bl - float(g["bloss1_batch"])) / float(g["bloss1_batch"]) < TOL
    assert rel(op.hvp(g["z"], g["batch"], lam), g["hvp_batch"]) < TOL
    assert rel(op.hvp(g["v1"], idx, lam), g["hvp_full_complex"]) < TOL
    assert rel(op.b_vector(), g["b_vector"]) < TOL


@pytest.mark.parametrize("name,seed", [("dataset_m16_nn.npz", 3), ("dataset_m16_tri.npz", 4)])
def test_hutchinson_epoch_golden(golden, name, seed):
    g = golden(name)
    op, _ = golden_ops(g)
    M = int(g["M"])
    st = F.PreconditionerState.initial(M ** 3, 1.0)
    zr = Opt.z_stream(seed)
    for b in F.epoch_batches(op.n_images, op.n_images // 4, seed, 0):
        F.hutchinson_update(st, op, F.rademacher(zr, M ** 3), b, float(g["lam"]))
    assert rel(st.d_avg, g["d_avg_epoch"]) < TOL


def test_nn_hutchinson_is_exact_diag(golden):
    g = golden("dataset_m16_nn.npz")
    op, _ = golden_ops(g)
    M = int(g["M"])
    lam = float(g["lam"])
    st = F.PreconditionerState.initial(M ** 3, 1.0)
    zr = Opt.z_stream(3)
    for b in F.epoch_batches(op.n_images, op.n_images // 4, 3, 0):
        F.hutchinson_update(st, op, F.rademacher(zr, M ** 3), b, lam)
    exact = F.exact_diag([F.Pose(q, t) for q, t in zip(g["quats"], g["shifts"])], None, lam, "nn",
                         F.GridSpec(M), g["mask"])
    assert rel(exact, g["exact_diag"]) < 1e-6
    assert rel(st.d_avg, exact) < 1e-6


@pytest.mark.parametrize("name", ["dataset_m16_nn.npz", "dataset_m16_tri.npz"])
def test_exact_diag_golden(golden, name):
    g = golden(name)
    M = int(g["M"])
    poses = [F.Pose(q, t) for q, t in zip(g["quats"], g["shifts"])]
    d = F.exact_diag(poses, radial_ctfs(g["ctf_params"]), float(g["lam"]), str(g["mode"]), F.GridSpec(M),
                     g["mask"])
    assert rel(d, g["exact_diag"]) < TOL


class _GpuNS:
    """The harness namespace bound to the B200 facade (numpy in/out, reference semantics)."""
    new_state = staticmethod(lambda n, a: F.PreconditionerState.initial(n, a))
    z_stream = staticmethod(Opt.z_stream)
    rademacher = staticmethod(F.rademacher)
    epoch_batches = staticmethod(F.epoch_batches)
    hutchinson_update = staticmethod(F.hutchinson_update)
    ema_and_threshold = staticmethod(F.ema_and_threshold)
    loss_and_grad = staticmethod(F.loss_and_grad)
    batch_loss = staticmethod(F.batch_loss)

    @staticmethod
    def armijo_search(v, grad, dhat, loss_fn, eta, c, f0):
        return F.armijo_search(v, grad, dhat, loss_fn, eta, c, f0=f0)


@pytest.mark.parametrize("name,seed", [("dataset_m16_nn.npz", 3), ("dataset_m16_tri.npz", 4)])
def test_sgd_trajectory_10_steps(golden, name, seed):
    g = golden(name)
    op, _ = golden_ops(g)
    rec, v, st = sgd_harness(_GpuNS, op, op.spec.M ** 3, op.n_images, float(g["lam"]), float(g["alpha"]),
                             int(g["batch"].size), seed, 10)
    ref = g["sgd_rec"]
    assert np.max(np.abs(rec[:, 0] - ref[:, 0]) / np.abs(ref[:, 0])) < 1e-4  # f0 per step
    assert np.max(np.abs(rec[:, 2] - ref[:, 2]) / np.abs(ref[:, 2])) < 1e-4  # accepted loss
    assert np.array_equal(rec[:, 1], ref[:, 1])  # identical step sizes (Armijo decisions)
    assert rel(v, g["sgd_v_end"]) < 1e-4


# ---------------------------------------------------------------- deterministic mode

def test_deterministic_mode_bitwise_repeatable_and_close(golden):
    g = golden("dataset_m16_tri.npz")
    opd, _ = golden_ops(g, deterministic=True)
    op, _ = golden_ops(g)
    lam = float(g["lam"])
    l1, g1 = F.loss_and_grad(opd, g["v1"], g["batch"], lam)
    l2, g2 = F.loss_and_grad(opd, g["v1"], g["batch"], lam)
    assert l1 == l2 and np.array_equal(g1.view(np.uint64), g2.view(np.uint64))
    l3, g3 = F.loss_and_grad(op, g["v1"], g["batch"], lam)
    assert rel(g1, g3) < TOL
    assert rel(g1, g["grad1_batch"]) < TOL
    # batch order does not matter bitwise (integer accumulation)
    l4, g4 = F.loss_and_grad(opd, g["v1"], g["batch"][::-1].copy(), lam)
    assert np.array_equal(g1.view(np.uint64), g4.view(np.uint64))


# ---------------------------------------------------------------- probe batcher

@pytest.mark.parametrize("k", [1, 5, 37, 64])
def test_probe_batcher_matches_k_single_probe_samples(k):
    M = 32
    mask = O.disk_mask(M, M // 2 - 1)
    N = 40
    q = synth.haar_quaternions(N, 7)
    sh = synth.normal_shifts(N, 8)
    ctfs = synth.physical_ctfs(N, 9)
    pix = O.mask_pix(M, mask)
    oop = O.OracleOperator(M, "tri", mask, q, sh, O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M), None)
    op = gpu_op(M, "tri", mask, q, sh, ctfs, np.zeros((N, mask.size), np.complex64))
    rng = np.random.default_rng(k)
    Z = rng.integers(0, 2, size=(k, M ** 3)).astype(np.float64) * 2 - 1
    batch = np.arange(N)
    lam = 0.5
    ref = np.mean([z * oop.hvp(z, batch, lam).real for z in Z], axis=0)
    got, kk = Opt.hutchinson_sample(op, Z, batch, lam)
    assert kk == k
    assert rel(got, ref) < TOL


# ---------------------------------------------------------------- SPEC known-answer tests on GPU

def test_kat_90deg_permutation_m4_gpu():
    M = 4
    mask = O.disk_mask(M, 1)
    s = np.sqrt(0.5)
    eng = SliceEngine(M, "nn", mask, records_for(M, [[s, 0, 0, s]]))
    v = torch.arange(M ** 3, dtype=torch.float32).to(torch.complex64).cuda()
    out = eng.project(v, [0]).cpu().numpy()
    assert list(out[0].real.astype(int)) == [13, 9, 5, 14, 10, 6, 15, 11, 7]


@pytest.mark.parametrize("mode", ["nn", "tri"])
def test_kat_identity_pose_is_z0_slice_gpu(mode):
    M = 32
    mask = O.disk_mask(M, M // 2 - 1)
    v = np.random.default_rng(0).standard_normal(M ** 3).astype(np.complex64)
    eng = SliceEngine(M, mode, mask, records_for(M, [[1.0, 0, 0, 0]]))
    out = eng.project(torch.from_numpy(v).cuda(), [0]).cpu().numpy()
    assert np.array_equal(out[0], v[mask])


def test_kat_shift_phase_gpu():
    M = 8
    mask = O.disk_mask(M, M // 2 - 1)
    eng = SliceEngine(M, "nn", mask, records_for(M, [[1.0, 0, 0, 0]], [[1.0, 0.0]]))
    v = torch.ones(M ** 3, dtype=torch.complex64).cuda()
    out = eng.project(v, [0]).cpu().numpy()[0]
    pix = O.mask_pix(M, mask)
    k1 = np.flatnonzero((pix[:, 0] == 1) & (pix[:, 1] == 0))[0]
    assert abs(out[k1] - np.exp(-2j * np.pi / M)) < 1e-6


def test_empty_batch_raises_value_error(golden):
    g = golden("dataset_m16_nn.npz")
    op, _ = golden_ops(g)
    with pytest.raises(ValueError):
        F.loss_and_grad(op, np.zeros(16 ** 3, complex), np.array([], dtype=int), 0.1)
    with pytest.raises(ValueError):
        op.hvp(np.zeros(16 ** 3), np.array([], dtype=int), 0.1)


# ---------------------------------------------------------------- full-size, size-independent properties

@pytest.mark.parametrize("M,mode", [(128, "tri"), (128, "nn"), (256, "tri")])
def test_adjointness_full_size(M, mode):
    """<P v, y> = <v, P^* y> at BASELINE sizes with the physical CTF and shifts."""
    B = 64
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(B, 11)
    recs = records_for(M, q, synth.normal_shifts(B, 12), synth.physical_ctfs(B, 13))
    eng = SliceEngine(M, mode, mask, recs)
    gen = torch.Generator(device="cuda").manual_seed(0)
    v = torch.randn(M ** 3, dtype=torch.complex64, device="cuda", generator=gen)
    y = torch.randn((B, mask.size), dtype=torch.complex64, device="cuda", generator=gen)
    idx = np.arange(B)
    pv = eng.project(v, idx)
    acc, fx = eng.backproject(y, idx)
    pty = eng.finalize_c(acc, fx, 1.0, 0.0)
    lhs = torch.vdot(y.reshape(-1).to(torch.complex128), pv.reshape(-1).to(torch.complex128))
    rhs = torch.vdot(pty.to(torch.complex128), v.to(torch.complex128))
    assert abs(complex(lhs - rhs)) / abs(complex(lhs)) < 1e-5


def test_loss_grad_vs_oracle_cfg3_subset():
    """cfg3 shapes (M=128, physical CTF, shifts, tri) on a 64-image batch vs the fp64 oracle."""
    M = 128
    B = 64
    mask = O.disk_mask(M, M // 2 - 1)
    pix = O.mask_pix(M, mask)
    v = synth.gaussian_blob_volume(M, 0)
    q = synth.haar_quaternions(B, 1)
    sh = synth.normal_shifts(B, 2)
    ctfs = synth.physical_ctfs(B, 3)
    ctab = O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M)
    rng = np.random.default_rng(5)
    clean = O.project("tri", v, O.rot_table(q), pix, O.phase_table(sh, pix, M), ctab, M)
    x = clean + 0.5 * np.sqrt(np.mean(np.abs(clean) ** 2)) * (rng.standard_normal(clean.shape)
                                                               + 1j * rng.standard_normal(clean.shape))
    oop = O.OracleOperator(M, "tri", mask, q, sh, ctab, x)
    op = gpu_op(M, "tri", mask, q, sh, ctfs, x)
    v1 = v * (1 + 0.05 * rng.standard_normal(v.size))
    batch = np.arange(B)
    lam = 1e-3
    lr, gr = O.loss_and_grad(oop, v1, batch, lam, n_total=50000)
    lg, gg = F.loss_and_grad(op, v1, batch, lam, n_total=50000)
    assert abs(lg - lr) / lr < TOL
    assert rel(gg, gr) < TOL
    assert rel(op.project(v1, batch), oop.project(v1, batch)) < TOL


def test_device_resident_loss_grad_matches_numpy_api():
    wl = synth.build_workload(synth.CONFIGS["cfg2"], seed=0, n_images=512)
    op = DatasetOperator.from_engine(wl.engine)
    batch = np.arange(0, 512, 2)
    v = wl.v_true * 0.9
    l_np, g_np = F.loss_and_grad(op, v, batch, 1e-3)
    vd = torch.from_numpy(v.astype(np.complex64)).cuda()
    l_d, g_d = F.loss_and_grad(op, vd, torch.from_numpy(batch).cuda(), 1e-3)
    assert abs(float(l_d) - l_np) / l_np < 1e-6
    assert rel(g_d.cpu().numpy(), g_np) < 1e-5


@pytest.mark.parametrize("M,B", [(8, 50), (16, 300), (33, 64), (36, 200), (64, 512), (65, 100), (128, 512),
                                 (256, 128)])
def test_brick_path_processes_every_pixel_exactly_once(M, B):
    """Exact coverage: with v = 0 and x = 1 every processed pixel adds exactly 1 to sum |r|^2."""
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(B, 7 * M)
    # include exact-axis poses (w == 0 on whole rows, clamped rim pixels)
    q[:3] = [[1, 0, 0, 0], [np.sqrt(0.5), 0, 0, np.sqrt(0.5)], [0.5, 0.5, 0.5, 0.5]]
    eng = SliceEngine(M, "tri", mask, records_for(M, q), np.ones((B, mask.size), np.complex64))
    v = torch.zeros(M ** 3, dtype=torch.complex64, device="cuda")
    sq, acc, _ = eng.loss_grad(v, np.arange(B))
    assert float(sq) == float(B * mask.size)


@pytest.mark.parametrize("M,B", [(16, 40), (33, 64), (36, 64), (64, 256), (65, 96), (128, 512), (256, 64)])
def test_brick_path_matches_tile_path(M, B):
    """The brick-binned fused loss+grad (default, tri) equals the per-pixel tile kernel: every pixel
    is owned by exactly one brick (incl. clamped rim pixels, M not a multiple of the brick edge)."""
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(B, M + 1)
    sh = synth.normal_shifts(B, M + 2)
    ctfs = synth.physical_ctfs(B, M + 3)
    recs = records_for(M, q, sh, ctfs)
    gen = torch.Generator(device="cuda").manual_seed(M)
    x = torch.randn((B, mask.size), dtype=torch.complex64, device="cuda", generator=gen)
    v = torch.from_numpy(synth.gaussian_blob_volume(M, 1).astype(np.complex64)).cuda()
    fast = SliceEngine(M, "tri", mask, recs, x)
    tile = SliceEngine(M, "tri", mask, recs, x, tile_path=True)
    idx = np.arange(B)
    sq1, acc1, _ = fast.loss_grad(v, idx)
    sq2, acc2, _ = tile.loss_grad(v, idx)
    assert abs(float(sq1) - float(sq2)) / float(sq2) < 1e-6
    a1 = acc1.cpu().numpy()
    a2 = acc2.cpu().numpy()
    assert rel(a1, a2) < 5e-6


@pytest.mark.parametrize("M,radius", [(33, 15), (32, 8), (48, 23)])
def test_odd_sizes_and_small_masks_vs_oracle(M, radius):
    """Odd M (centre ceil(M/2), grid.py:9-31) and mask radii below M/2-1 on the default (brick) path."""
    B = 24
    mask = O.disk_mask(M, radius)
    pix = O.mask_pix(M, mask)
    q = synth.haar_quaternions(B, M)
    sh = synth.normal_shifts(B, M + 1)
    ctfs = synth.physical_ctfs(B, M + 2)
    ctab = O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M)
    rng = np.random.default_rng(M)
    v = rng.standard_normal(M ** 3) + 1j * rng.standard_normal(M ** 3)
    x = rng.standard_normal((B, mask.size)) + 1j * rng.standard_normal((B, mask.size))
    oop = O.OracleOperator(M, "tri", mask, q, sh, ctab, x)
    op = gpu_op(M, "tri", mask, q, sh, ctfs, x)
    assert op.engine.layout == "sorted"
    batch = rng.permutation(B)[:17]
    lr, gr = O.loss_and_grad(oop, v, batch, 0.01)
    lg, gg = F.loss_and_grad(op, v, batch, 0.01)
    assert abs(lg - lr) / lr < TOL
    assert rel(gg, gr) < TOL
    assert rel(op.project(v, batch), oop.project(v, batch)) < TOL
    # nn indices stay bit-exact at odd M
    assert np.array_equal(K.assign_nn(oop.rots[batch], pix, M), O.assign_nn(oop.rots[batch], pix, M))


@pytest.mark.parametrize("M,radius,slabs", [(33, 9, 12), (32, 15, 5), (64, 20, 12), (64, 31, 16), (40, 6, 1)])
def test_numpy_call_touched_ball_copies_vs_whole_planes_and_oracle(M, radius, slabs, monkeypatch):
    """fsld_loss_grad_host_np_ball: the z-slab copies restricted to the boxes around the touched ball
    (grid.touched_ball; outside, grad = lam v and ||v||^2 on the host threads in fp64) against the same
    call with whole-plane copies and against the oracle -- v is dense noise, so any voxel the boxes
    miss, or any stale voxel they pick up, shows."""
    from paper_2311_16100_b200.engine import SliceEngine
    B = 40
    mask = O.disk_mask(M, radius)
    pix = O.mask_pix(M, mask)
    q = synth.haar_quaternions(B, M + 5)
    sh = synth.normal_shifts(B, M + 6)
    ctfs = synth.physical_ctfs(B, M + 7)
    ctab = O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M)
    rng = np.random.default_rng(M + radius)
    x = rng.standard_normal((B, mask.size)) + 1j * rng.standard_normal((B, mask.size))
    oop = O.OracleOperator(M, "tri", mask, q, sh, ctab, x)
    op = gpu_op(M, "tri", mask, q, sh, ctfs, x)
    monkeypatch.setattr(SliceEngine, "HOST_SLABS", slabs)
    monkeypatch.setattr(SliceEngine, "NP_SLABS", slabs)
    batch = rng.permutation(B)[:33]
    lam = 0.02
    for trial in range(3):  # new v every call: the device copy outside the boxes goes stale
        v = rng.standard_normal(M ** 3) + 1j * rng.standard_normal(M ** 3)
        monkeypatch.setattr(SliceEngine, "HOST_BALL", True)
        lb, gb = op.loss_and_grad_numpy(v, batch, lam)
        gb = gb.copy()
        monkeypatch.setattr(SliceEngine, "HOST_BALL", False)
        lw, gw = op.loss_and_grad_numpy(v, batch, lam)
        lr, gr = O.loss_and_grad(oop, v, batch, lam)
        assert abs(lb - lw) / lw < 1e-6 and abs(lb - lr) / lr < TOL
        assert rel(gb, gw) < 1e-6 and rel(gb, gr) < TOL
        # outside the ball the gradient is lam v in fp64, exactly
        from paper_2311_16100_b200.grid import touched_ball
        out = np.ones(M ** 3, bool)
        out[touched_ball(M, radius)] = False
        assert np.allclose(gb[out], lam * v[out], rtol=1e-6, atol=0)


@pytest.mark.parametrize("M", [128, 256])
def test_large_defocus_phase_brick_vs_oracle(M):
    """Stress the fixed-point CTF / shift phases of the brick path: 5 um defocus, 0.5 um astigmatism,
    10 px shifts (gamma ~ 10^3 - 10^4 rad at the mask edge), checked against the fp64 oracle."""
    B = 12
    mask = O.disk_mask(M, M // 2 - 1)
    pix = O.mask_pix(M, mask)
    q = synth.haar_quaternions(B, M + 5)
    rng = np.random.default_rng(M)
    sh = rng.normal(0.0, 10.0, (B, 2))
    ctfs = [PhysicalCtf(defocus=float(d), astig=5.0e3, astig_angle=float(a), voltage_kv=300.0, cs_mm=2.7,
                        amp_contrast=0.07, apix=0.8)
            for d, a in zip(rng.uniform(3.0e4, 5.0e4, B), rng.uniform(0, np.pi, B))]
    ctab = O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M)
    v = synth.gaussian_blob_volume(M, 3)
    x = (rng.standard_normal((B, mask.size)) + 1j * rng.standard_normal((B, mask.size)))
    oop = O.OracleOperator(M, "tri", mask, q, sh, ctab, x)
    op = gpu_op(M, "tri", mask, q, sh, ctfs, x)
    assert op.engine.brick_path
    batch = np.arange(B)
    lr, gr = O.loss_and_grad(oop, v, batch, 1e-3)
    lg, gg = F.loss_and_grad(op, v, batch, 1e-3)
    assert abs(lg - lr) / lr < TOL
    assert rel(gg, gr) < TOL


from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=15, deadline=None)
@given(M=st.integers(8, 72), B=st.integers(1, 40), seed=st.integers(0, 10 ** 6),
       radius_frac=st.floats(0.3, 1.0))
def test_brick_path_randomised_vs_tile_and_coverage(M, B, seed, radius_frac):
    """Randomised shapes (odd / even M, any mask radius, any batch size): the brick path covers every
    pixel exactly once and its loss+grad equals the per-pixel tile kernel's."""
    R = max(1, int(radius_frac * (M // 2 - 1)))
    mask = O.disk_mask(M, R)
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sh = rng.normal(0, 2, (B, 2))
    ctfs = synth.physical_ctfs(B, seed % 1000)
    recs = records_for(M, q, sh, ctfs)
    ones = np.ones((B, mask.size), np.complex64)
    cov = SliceEngine(M, "tri", mask, records_for(M, q), ones)
    sq, _, _ = cov.loss_grad(torch.zeros(M ** 3, dtype=torch.complex64, device="cuda"), np.arange(B))
    assert float(sq) == float(B * mask.size)
    x = torch.from_numpy((rng.standard_normal((B, mask.size)) + 1j * rng.standard_normal((B, mask.size)))
                         .astype(np.complex64)).cuda()
    v = torch.from_numpy((rng.standard_normal(M ** 3) + 1j * rng.standard_normal(M ** 3))
                         .astype(np.complex64)).cuda()
    brick = SliceEngine(M, "tri", mask, recs, x)
    tile = SliceEngine(M, "tri", mask, recs, x, tile_path=True)
    idx = rng.permutation(B)
    sq1, a1, _ = brick.loss_grad(v, idx)
    sq2, a2, _ = tile.loss_grad(v, idx)
    assert abs(float(sq1) - float(sq2)) <= 1e-6 * float(sq2)
    assert rel(a1.cpu().numpy(), a2.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("M,B,slabs", [(16, 40, 1), (33, 64, 3), (40, 64, 2), (64, 256, 8), (65, 96, 16),
                                       (128, 512, 8), (128, 300, 5), (128, 64, 16)])
def test_host_step_pipelined_matches_device_step(M, B, slabs):
    """fsld_loss_grad_host (z-slab pipelined copies, per-slab work items) equals the device-resident
    loss_and_grad for any slab count, including M whose brick layers straddle kz = 0 (M=40, 65),
    and agrees with the fp64 oracle (loss_and_grad, optim.py:165-190) within the fp32 tolerance."""
    mask = O.disk_mask(M, M // 2 - 1)
    pix = O.mask_pix(M, mask)
    n_img = 2 * B
    q = synth.haar_quaternions(n_img, 11 * M)
    sh = synth.normal_shifts(n_img, 11 * M + 1)
    ctfs = synth.physical_ctfs(n_img, 11 * M + 2)
    rng = np.random.default_rng(M)
    x = (rng.standard_normal((n_img, mask.size)) + 1j * rng.standard_normal((n_img, mask.size))) * 1e-3
    op = gpu_op(M, "tri", mask, q, sh, ctfs, x)
    v = synth.gaussian_blob_volume(M, 2) * (1 + 0.1 * rng.standard_normal(M ** 3))
    batch = np.sort(rng.choice(n_img, B, replace=False)).astype(np.int32)
    lam = 2e-3
    l_ref, g_ref = F.loss_and_grad(op, v, batch, lam)
    v_h = torch.from_numpy(v.astype(np.complex64)).pin_memory()
    g_h = torch.zeros(M ** 3, dtype=torch.complex64).pin_memory()
    idx_h = torch.from_numpy(batch).pin_memory()
    op.engine.HOST_SLABS = slabs
    for _ in range(2):  # re-entrant: the second call reuses the staging buffers and events
        g_h.zero_()
        l_h = op.loss_and_grad_host(v_h, idx_h, lam, g_h)
    assert abs(l_h - l_ref) / l_ref < 1e-6
    assert rel(g_h.numpy(), g_ref) < 5e-6  # fp32 epilogue on the device vs fp64 on the host
    if M <= 65:
        ctab = O.ctf_table_physical(synth.ctf_param_array(ctfs), pix, M)
        oop = O.OracleOperator(M, "tri", mask, q, sh, ctab, x)
        lr, gr = O.loss_and_grad(oop, v, batch, lam)
        assert abs(l_h - lr) / lr < TOL
        assert rel(g_h.numpy(), gr) < TOL


def test_host_step_rejects_bad_buffers():
    M, B = 16, 8
    mask = O.disk_mask(M, M // 2 - 1)
    q = synth.haar_quaternions(B, 5)
    op = gpu_op(M, "tri", mask, q, None, None, np.ones((B, mask.size), np.complex64))
    v_h = torch.zeros(M ** 3, dtype=torch.complex64).pin_memory()
    g_h = torch.zeros(M ** 3, dtype=torch.complex64).pin_memory()
    with pytest.raises(ValueError):
        op.loss_and_grad_host(v_h, torch.zeros(0, dtype=torch.int32).pin_memory(), 0.0, g_h)
    with pytest.raises(ValueError):
        op.loss_and_grad_host(v_h, torch.tensor([0, B], dtype=torch.int32).pin_memory(), 0.0, g_h)
    with pytest.raises(ValueError):
        op.loss_and_grad_host(v_h, torch.tensor([0, 1], dtype=torch.int32).pin_memory(), 0.0,
                              torch.zeros(M ** 3, dtype=torch.complex64))


def test_host_step_graph_cache_across_shapes_and_scalars():
    """The host step caches one CUDA graph per call shape: alternating batch sizes, lam values and
    host buffers must each give the device path's result (no stale graph, rows re-staged per call)."""
    from paper_2311_16100_b200 import _capi as C
    M = 48
    mask = O.disk_mask(M, M // 2 - 1)
    n_img = 300
    q = synth.haar_quaternions(n_img, 91)
    sh = synth.normal_shifts(n_img, 92)
    ctfs = synth.physical_ctfs(n_img, 93)
    rng = np.random.default_rng(94)
    x = (rng.standard_normal((n_img, mask.size)) + 1j * rng.standard_normal((n_img, mask.size))) * 1e-2
    op = gpu_op(M, "tri", mask, q, sh, ctfs, x)
    v = synth.gaussian_blob_volume(M, 5)
    v_h = [C.host_empty(M ** 3, torch.complex64), torch.zeros(M ** 3, dtype=torch.complex64).pin_memory()]
    for t in v_h:
        t.copy_(torch.from_numpy(v.astype(np.complex64)))
    g_h = C.host_empty(M ** 3, torch.complex64)
    for it, (B, lam) in enumerate([(64, 1e-3), (100, 1e-3), (64, 5e-2), (100, 1e-3), (64, 1e-3)]):
        batch = np.sort(rng.choice(n_img, B, replace=False)).astype(np.int32)
        l_ref, g_ref = F.loss_and_grad(op, v, batch, lam, n_total=n_img)
        l_h = op.loss_and_grad_host(v_h[it % 2], torch.from_numpy(batch).pin_memory(), lam, g_h, n_total=n_img)
        assert abs(l_h - l_ref) / l_ref < 1e-6, it
        assert rel(g_h.numpy(), g_ref) < 5e-6, it  # fp32 epilogue on the device vs fp64 on the host


def test_host_step_graph_cache_survives_freed_and_reused_buffers(golden):
    """The numpy call path stages through pinned buffers (fsld_host_alloc) that die with their
    operator; a later operator can get the same addresses.  Cached host-step graphs that captured
    a freed buffer must be dropped (fsld_host_free), never replayed."""
    import gc
    g = golden("dataset_m16_tri.npz")
    lam = float(g["lam"])
    for _ in range(4):
        op, _ = golden_ops(g)
        loss, grad = F.loss_and_grad(op, g["v1"], g["batch"], lam)
        assert abs(loss - float(g["loss1_batch"])) / float(g["loss1_batch"]) < TOL
        assert rel(grad, g["grad1_batch"]) < TOL
        del op
        gc.collect()


@pytest.mark.parametrize("mode,nn_brick", [("tri", False), ("nn", True)])
def test_fixed_point_budget_identical_planes(mode, nn_brick):
    """Worst case of the brick kernel's int32 budget (fixed_lim): 256 images with ONE pose, so every
    brick's work items hold 64 segments of the same plane and every voxel collects 64 copies of the
    largest per-image weight sum, with large-amplitude images.  No int32 overflow: the loss and the
    gradient still match the oracle."""
    from paper_2311_16100_b200.engine import SliceEngine
    M, N = 32, 256
    mask = O.disk_mask(M, M // 2 - 1)
    pix = O.mask_pix(M, mask)
    q = np.tile(synth.haar_quaternions(1, 5), (N, 1))
    sh = np.zeros((N, 2))
    v = synth.gaussian_blob_volume(M, 6) * 1e3
    oop = O.OracleOperator(M, mode, mask, q, sh, None, None)
    rng = np.random.default_rng(7)
    x = oop.project(v, np.arange(N)) * 3.0 + 50.0 * (rng.standard_normal((N, pix.shape[0])) +
                                                     1j * rng.standard_normal((N, pix.shape[0])))
    oop.x = np.ascontiguousarray(x)
    eng = SliceEngine(M, mode, mask, records_for(M, q, None, None), x, nn_brick=nn_brick)
    assert eng.table_path
    op = DatasetOperator.from_engine(eng)
    batch = np.arange(N)
    lg, gg = F.loss_and_grad(op, v, batch, 1e-3)
    lr, gr = O.loss_and_grad(oop, v, batch, 1e-3)
    assert abs(lg - lr) / lr < TOL
    assert rel(gg, gr) < TOL
