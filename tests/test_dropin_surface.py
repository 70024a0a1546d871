"""CPU: the drop-in surface -- every public name of the reference package exists here, and the
host-side pieces restated from the reference give the reference's results bit for bit
(pose samplers, phantom, shell tables, FSC epochs, condition bounds)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

import paper_2311_16100_b200 as F

_REF_SRC = next((p for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")
                 if os.path.isdir(os.path.join(p, "fsld"))), None)
needs_ref = pytest.mark.skipif(_REF_SRC is None, reason="reference package not available")


@pytest.fixture(scope="module")
def ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, _REF_SRC)
    try:
        import fsld
        yield fsld
    finally:
        sys.path.remove(_REF_SRC)


@needs_ref
def test_every_public_name_of_the_reference_exists(ref):
    assert [n for n in ref.__all__ if not hasattr(F, n)] == []
    for sub in ("forward", "optim", "grid", "hessian", "metrics", "kernels", "io", "errors"):
        r = __import__(f"fsld.{sub}", fromlist=["_"])
        m = __import__(f"paper_2311_16100_b200.{sub}", fromlist=["_"])
        public = [n for n in dir(r) if not n.startswith("_") and callable(getattr(r, n))
                  and getattr(getattr(r, n), "__module__", "") == f"fsld.{sub}"]
        assert [n for n in public if not hasattr(m, n)] == [], sub


@needs_ref
def test_host_pieces_match_reference_bit_for_bit(ref):
    a = ref.forward.sample_preferred_poses(40, 2.0, 3, 1.5)
    b = F.forward.sample_preferred_poses(40, 2.0, 3, 1.5)
    assert all(np.array_equal(x.q, y.q) and np.array_equal(x.t, y.t) for x, y in zip(a, b))
    s_ref, s = ref.GridSpec(16), F.GridSpec(16)
    assert np.array_equal(ref.gaussian_blob_phantom(s_ref, seed=4).values, F.gaussian_blob_phantom(s, seed=4).values)
    t_ref, t = ref.shell_table(s_ref, 7), F.shell_table(s, 7)
    for k in ("px_count", "vx_count", "shell_of_pixel", "shell_of_voxel"):
        assert np.array_equal(getattr(t_ref, k), getattr(t, k)), k
    assert t_ref.pixel_voxel_ratio(5) == t.pixel_voxel_ratio(5) and t_ref.shell_ratio(3) == t.shell_ratio(3)
    h = np.random.default_rng(0).random((6, 9))
    h[:, 2] = np.nan
    assert np.array_equal(ref.epochs_to_threshold(h, 0.5), F.epochs_to_threshold(h, 0.5))
    for n, lam, p in ((100, 0.1, 0.3), (5, 0.0, 0.1), (5, 0.2, 0.1)):
        assert ref.cond_lower_bound(n, lam, p) == F.cond_lower_bound(n, lam, p)
    d = np.random.default_rng(1).random(16 ** 3) + 0.1
    assert ref.condition_number(d, s_ref, 5) == F.condition_number(d, s, 5)
    with pytest.raises(ValueError):
        F.shell_table(s, 0)


def test_fsld_shim_resolves_to_this_package():
    code = ("import fsld, fsld.optim, fsld.kernels, paper_2311_16100_b200 as P; "
            "assert fsld.DatasetOperator is P.DatasetOperator and fsld.optim is P.optim and fsld.kernels is P.kernels; "
            "assert set(P.__all__) <= set(dir(fsld)); print('ok')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, PYTHONPATH=os.path.join(ROOT, "pkg", "src")), cwd="/tmp")
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr[-2000:]


@needs_ref
def test_threshold_alpha_uses_the_shell_table_like_the_reference(ref, golden):
    g = golden("dataset_m16_tri.npz")
    M = int(g["M"])
    R = M // 2 - 1
    images = np.zeros((g["x"].shape[0], M * M), complex)
    images[:, g["mask"]] = g["x"]
    rstack = ref.ImageStack(ref.GridSpec(M), images, [ref.Pose(q, t) for q, t in zip(g["quats"], g["shifts"])],
                            [ref.CtfParams(*map(float, p)) for p in g["ctf_params"]], 0.05, 4, R, "tri")
    stack = F.ImageStack(F.GridSpec(M), images, [F.Pose(q, t) for q, t in zip(g["quats"], g["shifts"])],
                         [F.CtfParams(*map(float, p)) for p in g["ctf_params"]], 0.05, 4, R, "tri")
    a_ref = ref.optim.threshold_alpha(rstack, ref.shell_table(ref.GridSpec(M), R), 0.01)
    assert abs(F.threshold_alpha(stack, F.shell_table(F.GridSpec(M), R), 0.01) - a_ref) <= 1e-14 * a_ref
    assert abs(F.threshold_alpha(stack, None, 0.01) - a_ref) <= 1e-14 * a_ref
    with pytest.raises(ValueError):
        F.threshold_alpha(stack, F.shell_table(F.GridSpec(M), R - 1), 0.01)
