"""GPU: the drop-in surface of the reference package.

* `pkg/src/fsld` (the reference's import name) resolves to the B200 path and reproduces the
  reference's golden loss / gradient;
* the reference's OWN optim.run (the unmodified install in baseline/_ref), with the primitives it
  calls swapped for the B200 ones exactly as INTEGRATION.md §1 shows, reproduces the reference's
  golden 10-step Armijo decisions and matches the B200 device run (optim.py:309-393);
* DatasetOperator.projector / phases / ctf_vals equal the reference's tables (forward.py:523-526);
  assigning a different table raises instead of being ignored;
* synthesize_dataset (GPU projection + the reference's per-image noise streams, forward.py:427-470);
* the fsld_fsc kernel against the oracle's FSC (metrics.py:38-63).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import GOLDEN, ROOT
from oracle import oracle as O

import paper_2311_16100_b200 as F
from paper_2311_16100_b200.forward import CtfParams

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")


def _py(code, pythonpath):
    env = dict(os.environ, PYTHONPATH=pythonpath, NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/numba_cache"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_fsld_shim_is_the_b200_path():
    code = f"""
import json, numpy as np
import fsld, fsld.optim, fsld.forward, fsld.kernels
import paper_2311_16100_b200 as P
g = dict(np.load({os.path.join(GOLDEN, 'dataset_m16_tri.npz')!r}))
M = int(g['M'])
ctfs = [fsld.CtfParams(float(d), float(w), float(b)) for d, w, b in g['ctf_params']]
poses = [fsld.Pose(q, t) for q, t in zip(g['quats'], g['shifts'])]
images = np.zeros((len(poses), M * M), complex); images[:, g['mask']] = g['x']
stack = fsld.ImageStack(fsld.GridSpec(M), images, poses, ctfs, 0.05, 4, M // 2 - 1, 'tri')
op = fsld.DatasetOperator(stack)
loss, grad = fsld.optim.loss_and_grad(op, g['v1'], g['batch'], float(g['lam']))
print(json.dumps({{"same": fsld.DatasetOperator is P.DatasetOperator and fsld.kernels is P.kernels,
                  "loss_rel": abs(loss - float(g['loss1_batch'])) / float(g['loss1_batch']),
                  "grad_rel": float(np.linalg.norm(grad - g['grad1_batch']) / np.linalg.norm(g['grad1_batch']))}}))
"""
    out = _py(code, os.path.join(ROOT, "pkg", "src"))
    assert out["same"]
    assert out["loss_rel"] < 1e-5 and out["grad_rel"] < 1e-5


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "fsld")), reason="reference install (baseline/_ref) absent")
def test_reference_run_with_b200_primitives():
    code = f"""
import json, sys, numpy as np
sys.path.append({ROOT!r})
import fsld                      # the unmodified reference (baseline/_ref)
import fsld.optim as ref_optim
import paper_2311_16100_b200 as b200
assert 'baseline' in fsld.__file__
g = dict(np.load({os.path.join(GOLDEN, 'dataset_m16_tri.npz')!r}))
M = int(g['M'])
ctfs = [fsld.CtfParams(float(d), float(w), float(b)) for d, w, b in g['ctf_params']]
poses = [fsld.Pose(q, t) for q, t in zip(g['quats'], g['shifts'])]
images = np.zeros((len(poses), M * M), complex); images[:, g['mask']] = g['x']
stack = fsld.ImageStack(fsld.GridSpec(M), images, poses, ctfs, 0.05, 4, M // 2 - 1, 'tri')
cfg = ref_optim.OptimConfig(lam=float(g['lam']), batch_size=int(g['batch'].size), epochs=3, seed=4, mode='tri')
for name in ("DatasetOperator", "loss_and_grad", "batch_loss", "hutchinson_update"):   # INTEGRATION.md 1
    setattr(ref_optim, name, getattr(b200, name))
vol, tr = ref_optim.run(cfg, stack)
print(json.dumps({{"etas": [float(e) for e in tr.accepted_etas], "loss": [float(x) for x in tr.loss],
                  "v": [float(np.linalg.norm(vol.values))]}}))
"""
    out = _py(code, REF)
    g = np.load(os.path.join(GOLDEN, "dataset_m16_tri.npz"))
    assert np.array_equal(np.array(out["etas"][:10]), g["sgd_rec"][:, 1])  # the reference's own decisions
    # the B200 device loop (optim.run) on the same stack
    M = int(g["M"])
    stack = F.ImageStack(F.GridSpec(M), _images(g), [F.Pose(q, t) for q, t in zip(g["quats"], g["shifts"])],
                         [CtfParams(float(d), float(w), float(b)) for d, w, b in g["ctf_params"]], 0.05, 4, M // 2 - 1,
                         "tri")
    cfg = F.OptimConfig(lam=float(g["lam"]), batch_size=int(g["batch"].size), epochs=3, seed=4, mode="tri")
    vol, tr = F.run(cfg, stack)
    assert np.array_equal(np.array(tr.accepted_etas), np.array(out["etas"]))
    assert np.max(np.abs(np.array(tr.loss) - out["loss"]) / np.abs(out["loss"])) < 1e-4


def _images(g):
    M = int(g["M"])
    images = np.zeros((g["x"].shape[0], M * M), dtype=np.complex128)
    images[:, g["mask"]] = g["x"]
    return images


def test_dataset_operator_tables_match_reference_and_refuse_edits(golden):
    g = golden("dataset_m16_tri.npz")
    M = int(g["M"])
    poses = [F.Pose(q, t) for q, t in zip(g["quats"], g["shifts"])]
    stack = F.ImageStack(F.GridSpec(M), _images(g), poses,
                         [CtfParams(float(d), float(w), float(b)) for d, w, b in g["ctf_params"]], 0.05, 4,
                         M // 2 - 1, "tri")
    op = F.DatasetOperator(stack)
    pix = O.mask_pix(M, g["mask"])
    assert np.abs(op.phases - O.phase_table(g["shifts"], pix, M)).max() < 1e-12
    assert np.abs(op.ctf_vals - O.ctf_table_radial(g["ctf_params"], pix, M)).max() < 1e-12
    assert np.abs(op.rots - O.rot_table(g["quats"])).max() < 1e-14
    assert op.projector.n_mask == op.n_mask and np.array_equal(op.projector.mask, op.mask)
    # engine-built operators derive the same tables from the 128-byte records
    op2 = F.DatasetOperator.from_engine(op.engine, F.GridSpec(M))
    assert np.abs(op2.phases - op.phases).max() < 1e-9
    assert np.abs(op2.ctf_vals - op.ctf_vals).max() < 1e-6
    op.ctf_vals = op.ctf_vals.copy()  # the same values: accepted
    with pytest.raises(ValueError):
        op.ctf_vals = 2.0 * op.ctf_vals  # an arbitrary table cannot take effect: refused, never ignored
    with pytest.raises(ValueError):
        op.phases = np.ones_like(op.phases)


def test_synthesize_dataset_matches_reference_model():
    M = 24
    spec = F.GridSpec(M)
    v = F.gaussian_blob_phantom(spec, seed=2)
    poses = F.sample_uniform_poses(20, 2.0, 3)
    ctfs = [CtfParams(1.5 + 0.1 * i, 0.1, 0.5) for i in range(20)]
    for mode in ("tri", "nn"):
        st = F.synthesize_dataset(v, poses, ctfs, 0.3, mode=mode, seed=9)
        mask = F.disk_mask(spec, spec.max_mask_radius)
        pix = O.mask_pix(M, mask)
        q = np.array([p.q for p in poses])
        t = np.array([p.t for p in poses])
        prm = np.array([[c.defocus, c.amp_contrast, c.b_factor] for c in ctfs])
        clean = O.project(mode, v.values, O.rot_table(q), pix, O.phase_table(t, pix, M),
                          O.ctf_table_radial(prm, pix, M), M)
        ref_noise = np.stack([F.forward._noise_for_image(9, i, mask.size, 0.3) for i in range(20)])
        assert O.relative_l2(st.images[:, mask], clean + ref_noise) < 1e-5
        assert np.all(st.images[:, np.setdiff1d(np.arange(M * M), mask)] == 0)
        assert st.sigma == 0.3 and st.seed == 9 and st.mode == mode


def test_fsc_kernel_matches_oracle():
    M, R = 48, 23
    rng = np.random.default_rng(5)
    u = (rng.standard_normal(M ** 3) + 1j * rng.standard_normal(M ** 3)).astype(np.complex64)
    v = (u + 0.5 * (rng.standard_normal(M ** 3) + 1j * rng.standard_normal(M ** 3))).astype(np.complex64)
    v[np.round(F.GridSpec(M).voxel_radii()) == 7] = 0  # an undefined shell
    ref, defined = O.fsc(u.astype(np.complex128), v.astype(np.complex128), M, R)
    spec = F.GridSpec(M)
    got = F.fsc(F.FourierVolume(u, spec), F.FourierVolume(v, spec), F.shell_table(spec, R))
    assert np.array_equal(got.defined, defined) and not got.defined[7]
    assert np.max(np.abs(got.values[defined] - ref[defined])) < 1e-12
    assert np.array_equal(got.counts, F.shell_table(spec, R).vx_count)
    # device volumes through the per-epoch context of optim.run
    from paper_2311_16100_b200.metrics import ShellIndex
    got2 = F.fsc(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda(), ShellIndex(M, R, "cuda"))
    assert np.max(np.abs(got2.values[defined] - ref[defined])) < 1e-12


def test_threshold_alpha_device_ring_power_matches_host():
    """threshold_alpha's per-image ring mean of C^2 (non-radial CTF) on the device equals the host
    evaluation of the same formula (optim.py:250-266)."""
    from unittest import mock
    from paper_2311_16100_b200 import optim as Opt, synth
    M, n = 128, 3000
    spec = F.GridSpec(M)
    stack = F.ImageStack.__new__(F.ImageStack)
    stack.spec, stack.mask_radius, stack.ctfs, stack.poses = spec, M // 2 - 1, synth.physical_ctfs(n, 5), [None] * n
    a_dev = Opt.threshold_alpha(stack, F.shell_table(spec, M // 2 - 1), 1e-3)
    with mock.patch("torch.cuda.is_available", return_value=False):
        a_host = Opt.threshold_alpha(stack, F.shell_table(spec, M // 2 - 1), 1e-3)
    assert abs(a_dev - a_host) <= 1e-7 * a_host  # (records carry wsin / wcos in fp32)
