"""Property-based checks (hypothesis) of host-side logic: sharding, ball compaction, ABI validation."""
import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import oracle as O

from paper_2311_16100_b200 import _capi as C
from paper_2311_16100_b200 import dist as D
from paper_2311_16100_b200 import grid as G


@settings(max_examples=60, deadline=None)
@given(n=st.integers(1, 300), ws=st.integers(1, 9), seed=st.integers(0, 10 ** 6))
def test_shard_indices_is_a_balanced_partition(n, ws, seed):
    b = np.random.default_rng(seed).permutation(10 * n)[:n]
    parts = [D.shard_indices(b, r, ws) for r in range(ws)]
    assert np.array_equal(np.concatenate(parts), b)
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1


@settings(max_examples=25, deadline=None)
@given(M=st.integers(8, 40), seed=st.integers(0, 10 ** 6))
def test_touched_ball_contains_every_trilinear_corner(M, seed):
    """Random rotations of every masked pixel (with the reference's clamp): all 8 corners lie in the ball."""
    R = M // 2 - 1
    ball = set(G.touched_ball(M, R).tolist())
    pix = O.mask_pix(M, O.disk_mask(M, R))
    q = np.random.default_rng(seed).standard_normal((3, 4))
    c2 = (M + 1) // 2
    for rot in O.rot_table(q / np.linalg.norm(q, axis=1, keepdims=True)):
        c = np.clip(pix[:, :1] * rot[0] + pix[:, 1:] * rot[1], -R, R)  # rows 0,1 of R (kernels.py:42-60)
        f = np.floor(c).astype(np.int64)
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    ix, iy, iz = f[:, 0] + dx, f[:, 1] + dy, f[:, 2] + dz
                    w = ((c[:, 0] - f[:, 0]) if dx else 1) * ((c[:, 1] - f[:, 1]) if dy else 1) * \
                        ((c[:, 2] - f[:, 2]) if dz else 1)
                    keep = np.broadcast_to(np.abs(w) > 0, ix.shape)  # zero-weight corners are never written
                    zi = np.where(iz < 0, iz + M, iz)
                    j = (zi * M + iy + c2) * M + ix + c2
                    assert set(j[keep].tolist()) <= ball


@settings(max_examples=30, deadline=None)
@given(n=st.integers(4, 200), frac=st.floats(0.1, 1.0), seed=st.integers(0, 10 ** 6))
def test_packed_buffer_ball_roundtrip_on_cpu(n, frac, seed):
    rng = np.random.default_rng(seed)
    ball = np.sort(rng.choice(n, max(1, int(frac * n)), replace=False)).astype(np.int32)
    buf = D.PackedBuffer.new(n, True, torch.device("cpu"), dtype=torch.float64, ball=ball)
    acc = buf.work_acc()
    hut = buf.work_hutch()
    vals = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    acc[torch.from_numpy(ball.astype(np.int64))] = torch.from_numpy(vals[ball])
    hut[torch.from_numpy(ball.astype(np.int64))] = torch.from_numpy(vals[ball].real)
    buf.pack()
    acc.zero_()
    hut.zero_()
    buf.unpack()
    assert np.array_equal(acc.numpy()[ball], vals[ball])
    assert np.array_equal(hut.numpy()[ball], vals[ball].real)


@settings(max_examples=80, deadline=None)
@given(M=st.integers(-4, 2048), mode=st.integers(-2, 3), n=st.integers(-5, 10 ** 6), B=st.integers(-3, 5000))
def test_abi_rejects_invalid_geometry_without_touching_memory(M, mode, n, B):
    """Invalid (M, mode, n_mask, B) never reaches a kernel: EINVAL with NULL data pointers."""
    lib = C.load()
    valid = 2 <= M <= 1024 and mode in (0, 1) and 1 <= n <= M * M and B >= 1
    st_ = lib.fsld_loss_grad(M, mode, n, 0, 0, 0, B, 0, 0, 0, 0, 0, 0, 0, 0, 0)
    assert st_ == C.FSLD_EINVAL  # NULL buffers are always rejected, valid or not
    if not valid:
        assert lib.fsld_project(M, mode, n, 1, 1, 1, B, 1, 1, 0) == C.FSLD_EINVAL
