"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The fixtures (``tests/golden/*.npz``) pin the CPU oracle (``oracle/``)
bit-exactly and give the GPU parity tests reference-produced vectors.
Everything is seeded; re-running reproduces the same bytes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import fsld  # noqa: E402  (the reference package)
from fsld import forward as F  # noqa: E402
from fsld import kernels as K  # noqa: E402
from fsld import optim as Op  # noqa: E402
from fsld import hessian as H  # noqa: E402

from oracle import oracle as O  # noqa: E402  (only for the builder-defined physical CTF table)


def special_quats():
    """Poses with exact grid alignment and exact 0.5 nn ties."""
    s = np.sqrt(0.5)
    c30, s30 = np.sqrt(0.75), 0.5
    return np.array([
        [1.0, 0.0, 0.0, 0.0],        # identity
        [s, 0.0, 0.0, s],            # 90 deg about z
        [0.0, 0.0, 1.0, 0.0],        # 180 deg about y
        [c30, 0.0, 0.0, s30],        # 60 deg about z  -> R00 = 0.5: x ties
        [c30, s30, 0.0, 0.0],        # 60 deg about x  -> R11 = 0.5: y ties
        [c30, 0.0, s30, 0.0],        # 60 deg about y  -> z/x ties
        [0.5, 0.5, 0.5, 0.5],        # 120 deg about (1,1,1): permutation
    ])


def kernels_fixture(M, n_random, seed):
    rng = np.random.default_rng(seed)
    spec = fsld.GridSpec(M)
    mask = fsld.disk_mask(spec, M // 2 - 1)
    poses = [fsld.Pose(q=q, t=rng.normal(0, 2, 2)) for q in special_quats()]
    poses += fsld.sample_uniform_poses(n_random, 2.0, seed + 1)
    proj = F.Projector(spec, mask, "tri")
    rt = proj.rot_batch(poses)
    pix = proj.pix
    ph = proj.phase_batch(poses)
    ctfs = [fsld.CtfParams(defocus=rng.uniform(0.5, 3.0), amp_contrast=0.1,
                           b_factor=rng.uniform(0, 1)) for _ in poses]
    cv = np.ascontiguousarray(proj.ctf_batch(ctfs, len(poses)))
    v = rng.standard_normal(M ** 3) + 1j * rng.standard_normal(M ** 3)
    img = rng.standard_normal((len(poses), len(mask))) + 1j * rng.standard_normal((len(poses), len(mask)))
    out = {"M": M, "mask": mask, "quats": np.array([p.q for p in poses]),
           "shifts": np.array([p.t for p in poses]),
           "ctf_params": np.array([[c.defocus, c.amp_contrast, c.b_factor] for c in ctfs]),
           "rt": rt, "pix": pix, "phase": ph, "ctf": cv, "v": v, "img": img}
    for mode in ("tri", "nn"):
        o = np.empty((len(poses), len(mask)), dtype=np.complex128)
        (K.project_tri if mode == "tri" else K.project_nn)(v, rt, pix, ph, cv, M, o)
        vols = np.zeros((K.n_chunks(len(poses)), M ** 3), dtype=np.complex128)
        (K.backproject_tri if mode == "tri" else K.backproject_nn)(img, rt, pix, ph, cv, M, vols)
        out[f"project_{mode}"] = o
        out[f"backproject_{mode}"] = K.fold_chunks(vols)
    out["assign_nn"] = K.assign_nn(rt, pix, M)
    w = np.ascontiguousarray(cv ** 2)
    vols = np.zeros((K.n_chunks(len(poses)), M ** 3))
    K.scatter_sq_tri(w, rt, pix, M, vols)
    out["scatter_sq_tri"] = K.fold_chunks(vols)
    # builder-defined physical CTF table run through the reference kernels
    phys = np.column_stack([rng.uniform(1e4, 3e4, len(poses)), rng.uniform(0, 1e3, len(poses)),
                            rng.uniform(0, np.pi, len(poses)), np.full(len(poses), 300.0),
                            np.full(len(poses), 2.7), np.full(len(poses), 0.1),
                            np.full(len(poses), 1.0)])
    pc = np.ascontiguousarray(O.ctf_table_physical(phys, pix, M))
    o = np.empty((len(poses), len(mask)), dtype=np.complex128)
    K.project_tri(v, rt, pix, ph, pc, M, o)
    vols = np.zeros((K.n_chunks(len(poses)), M ** 3), dtype=np.complex128)
    K.backproject_tri(img, rt, pix, ph, pc, M, vols)
    out.update(phys_params=phys, phys_ctf=pc, project_tri_phys=o,
               backproject_tri_phys=K.fold_chunks(vols))
    return out


def sgd_harness_ref(op, v, lam, alpha, batch_size, seed, n_steps, beta=0.9, c=0.5, eta0=1.0):
    """Algorithm 1 steps exactly as optim.run (optim.py:362-382), recording per-step loss."""
    n = op.n_images
    state = Op.PreconditionerState.initial(op.spec.n_voxels, alpha)
    z_rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(2,)))
    eta = eta0
    rec = []
    step = 0
    epoch = 0
    while step < n_steps:
        for batch in Op.epoch_batches(n, batch_size, seed, epoch):
            if step == n_steps:
                break
            z = Op.rademacher(z_rng, op.spec.n_voxels)
            Op.hutchinson_update(state, op, z, batch, lam)
            dhat = Op.ema_and_threshold(state, beta, alpha, True)
            f0, grad = Op.loss_and_grad(op, v, batch, lam)
            eta, v, f_next, nbt = Op.armijo_search(
                v, grad, dhat, lambda w: Op.batch_loss(op, w, batch, lam), eta, c, f0=f0)
            rec.append((f0, eta, f_next, nbt))
            step += 1
        epoch += 1
    return np.array(rec), v, state.d_avg


def dataset_fixture(M, N, mode, with_ctf, seed, batch):
    spec = fsld.GridSpec(M)
    v_true = fsld.gaussian_blob_phantom(spec, seed=seed)
    shift = 1.5 if with_ctf else 0.0
    poses = fsld.sample_uniform_poses(N, shift, seed + 7)
    rng = np.random.default_rng(seed + 11)
    ctfs = ([fsld.CtfParams(defocus=rng.uniform(0.5, 3.0), amp_contrast=0.1,
                            b_factor=rng.uniform(0.0, 1.0)) for _ in range(N)]
            if with_ctf else None)
    stack = fsld.synthesize_dataset(v_true, poses, ctfs, sigma=0.05, mode=mode,
                                     mask_radius=M // 2 - 1, seed=seed)
    op = F.DatasetOperator(stack)
    lam = 1e-2
    idx = np.arange(N)
    bidx = np.random.default_rng(seed + 3).permutation(N)[:batch]
    out = {"M": M, "mode": mode, "quats": np.array([p.q for p in poses]),
           "shifts": np.array([p.t for p in poses]),
           "ctf_params": (np.array([[c.defocus, c.amp_contrast, c.b_factor] for c in ctfs])
                          if ctfs is not None else np.zeros((0, 3))),
           "mask": op.mask, "x": op.x, "v_true": v_true.values, "lam": lam, "batch": bidx}
    rng2 = np.random.default_rng(seed + 5)
    v1 = v_true.values * (1.0 + 0.1 * rng2.standard_normal(M ** 3))
    out["v1"] = v1
    out["loss0_full"], out["grad0_full"] = Op.loss_and_grad(op, np.zeros(M ** 3, complex), idx, lam)
    out["loss1_batch"], out["grad1_batch"] = Op.loss_and_grad(op, v1, bidx, lam)
    out["bloss1_batch"] = Op.batch_loss(op, v1, bidx, lam)
    z = Op.rademacher(np.random.default_rng(seed + 9), M ** 3)
    out["z"] = z
    out["hvp_batch"] = H.hvp(op, z, bidx, lam)
    out["hvp_full_complex"] = op.hvp(v1, idx, lam)
    out["b_vector"] = op.b_vector()
    out["exact_diag"] = H.exact_diag(stack.poses, stack.ctfs, lam, mode, spec, op.mask)
    # Hutchinson over one epoch of equal batches
    st = Op.PreconditionerState.initial(M ** 3, 1.0)
    zr = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(2,)))
    for b in Op.epoch_batches(N, N // 4, seed, 0):
        Op.hutchinson_update(st, op, Op.rademacher(zr, M ** 3), b, lam)
    out["d_avg_epoch"] = st.d_avg
    shells = fsld.shell_table(spec, stack.mask_radius)
    alpha = Op.threshold_alpha(stack, shells, lam)
    out["alpha"] = alpha
    rec, v_end, d_avg = sgd_harness_ref(op, np.zeros(M ** 3, complex), lam, alpha, batch, seed, 10)
    out["sgd_rec"] = rec
    out["sgd_v_end"] = v_end
    out["sgd_d_avg"] = d_avg
    return out


def io_fixture():
    """A tiny FSD1 dataset and FSV1 volume written by the reference's own io module (io.py)."""
    import fsld.io as fio
    spec = fsld.GridSpec(8)
    v = fsld.gaussian_blob_phantom(spec, seed=1)
    poses = fsld.sample_uniform_poses(5, 1.0, 2)
    ctfs = [fsld.CtfParams(defocus=1.0 + 0.3 * i, amp_contrast=0.1, b_factor=0.2) for i in range(5)]
    stack = fsld.synthesize_dataset(v, poses, ctfs, sigma=0.05, mode="tri", mask_radius=3, seed=2)
    fio.write_dataset(stack, os.path.join(HERE, "tiny_m8.fsd1"))
    fio.write_volume(v, os.path.join(HERE, "tiny_m8.fsv1"))


def main():
    np.savez_compressed(os.path.join(HERE, "kernels_m16.npz"), **kernels_fixture(16, 24, 100))
    np.savez_compressed(os.path.join(HERE, "kernels_m8.npz"), **kernels_fixture(8, 12, 200))
    np.savez_compressed(os.path.join(HERE, "dataset_m16_nn.npz"),
                        **dataset_fixture(16, 96, "nn", False, 3, 24))
    np.savez_compressed(os.path.join(HERE, "dataset_m16_tri.npz"),
                        **dataset_fixture(16, 96, "tri", True, 4, 24))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    if "--io-only" in sys.argv:
        io_fixture()
    else:
        main()
        io_fixture()
