"""Multi-rank (world_size 2, gloo, CPU) checks of the data-parallel sharding logic.

The per-rank compute is the CPU oracle (test infrastructure) injected into
paper_2311_16100_b200.dist.sharded_step; what is under test is the sharding,
the packed single all-reduce and the epilogue: the 2-rank result must equal
the single-process full-batch result of the reference algorithm.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden
from oracle import oracle as O

from paper_2311_16100_b200 import dist as D
from paper_2311_16100_b200 import grid as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_op(g):
    M = int(g["M"])
    ctab = O.ctf_table_radial(g["ctf_params"], O.mask_pix(M, g["mask"]), M) if g["ctf_params"].shape[0] else None
    return O.OracleOperator(M, str(g["mode"]), g["mask"], g["quats"], g["shifts"], ctab, g["x"])


def _oracle_compute(op, v, sub, buf, zbits=None, k=0):
    """Per-rank partial sums with the CPU oracle, written into the packed buffer (float64)."""
    sq, acc = O._resid_pass(op, np.asarray(v), sub, True)
    buf.work_acc().copy_(torch.from_numpy(acc))
    if zbits is not None:
        fold = np.zeros(op.M ** 3)
        for z in zbits:  # here: list of +-1 probe vectors
            fold += z * op.backproject(op.project(z, sub), sub).real
        buf.work_hutch().copy_(torch.from_numpy(fold))
    buf.set_loss(torch.tensor([sq], dtype=torch.float64))


def _worker(rank, world_size, port, out_path, use_ball=False):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world_size)
    g = load_golden("dataset_m16_tri.npz")
    op = _oracle_op(g)
    M = op.M
    lam = float(g["lam"])
    batch = np.asarray(g["batch"])
    v = torch.from_numpy(np.asarray(g["v1"], dtype=np.complex128))
    rng = np.random.default_rng(11)
    probes = [rng.integers(0, 2, M ** 3).astype(np.float64) * 2 - 1 for _ in range(3)]
    ball = G.touched_ball(M, M // 2 - 1) if use_ball else None
    buf = D.PackedBuffer.new(M ** 3, True, torch.device("cpu"), dtype=torch.float64, ball=ball)
    loss, grad, hs = D.sharded_step(op, v, batch, lam, buf=buf, zbits=probes, k=len(probes),
                                    compute=_oracle_compute)
    res = {"loss": float(loss), "grad": grad.numpy(), "hs": hs.numpy(), "sub": D.shard_indices(batch, rank, world_size)}
    np.savez(out_path + f".{rank}.npz", **res)
    dist.barrier()
    dist.destroy_process_group()


def _range_worker(rank, world_size, port, out_path):
    """Each rank holds only its image range of the dataset (oracle operator over those rows)."""
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world_size)
    g = load_golden("dataset_m16_tri.npz")
    M = int(g["M"])
    n = g["quats"].shape[0]
    lo, hi = D.image_range(n, rank, world_size)
    ctab = O.ctf_table_radial(g["ctf_params"], O.mask_pix(M, g["mask"]), M) if g["ctf_params"].shape[0] else None
    op = O.OracleOperator(M, str(g["mode"]), g["mask"], g["quats"][lo:hi], g["shifts"][lo:hi],
                          None if ctab is None else ctab[lo:hi], g["x"][lo:hi])
    buf = D.PackedBuffer.new(M ** 3, False, torch.device("cpu"), dtype=torch.float64)
    loss, grad, _ = D.sharded_step(op, torch.from_numpy(np.asarray(g["v1"], dtype=np.complex128)),
                                   np.asarray(g["batch"]), float(g["lam"]), n_total=n, buf=buf,
                                   compute=_oracle_compute, image_range=(lo, hi))
    np.savez(out_path + f".{rank}.npz", loss=float(loss), grad=grad.numpy(),
             sub=D.local_batch(g["batch"], lo, hi) + lo)
    dist.barrier()
    dist.destroy_process_group()


def test_image_range_partition_and_local_batch():
    b = np.random.default_rng(0).permutation(101)[:40]
    for ws in (1, 2, 3, 8):
        ranges = [D.image_range(101, r, ws) for r in range(ws)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 101
        assert all(ranges[r][1] == ranges[r + 1][0] for r in range(ws - 1))
        parts = [D.local_batch(b, lo, hi) + lo for lo, hi in ranges]
        assert np.array_equal(np.sort(np.concatenate(parts)), np.sort(b))


def test_two_rank_gloo_sharded_dataset_equals_single_process():
    """optim.run(shard_dataset=True)'s exchange: each rank holds half of the images, takes the
    batch's images of its range, one packed all-reduce -> the single-process full-batch result."""
    g = load_golden("dataset_m16_tri.npz")
    op = _oracle_op(g)
    batch = np.asarray(g["batch"])
    loss_ref, grad_ref = O.loss_and_grad(op, g["v1"], batch, float(g["lam"]))
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res")
        mp.start_processes(_range_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn")
        r0, r1 = np.load(out + ".0.npz"), np.load(out + ".1.npz")
    assert np.array_equal(np.sort(np.concatenate([r0["sub"], r1["sub"]])), np.sort(batch))
    for r in (r0, r1):
        assert abs(float(r["loss"]) - loss_ref) / loss_ref < 1e-12
        assert O.relative_l2(r["grad"], grad_ref) < 1e-12


def test_shard_indices_partition():
    b = np.arange(37)[::-1]
    for ws in (1, 2, 3, 8):
        parts = [D.shard_indices(b, r, ws) for r in range(ws)]
        assert np.array_equal(np.concatenate(parts), b)
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    with pytest.raises(ValueError):
        D.shard_indices(np.array([], dtype=int), 0, 2)


def test_packed_buffer_loss_split_roundtrip():
    buf = D.PackedBuffer.new(8, False, torch.device("cpu"))
    sq = torch.tensor([123456789.123456789], dtype=torch.float64)
    buf.set_loss(sq)
    assert abs(float(buf.loss()) - float(sq)) / float(sq) < 1e-12


@pytest.mark.parametrize("use_ball", [False, True])
def test_two_rank_gloo_step_equals_single_process(use_ball):
    g = load_golden("dataset_m16_tri.npz")
    op = _oracle_op(g)
    M = op.M
    lam = float(g["lam"])
    batch = np.asarray(g["batch"])
    loss_ref, grad_ref = O.loss_and_grad(op, g["v1"], batch, lam)
    rng = np.random.default_rng(11)
    probes = [rng.integers(0, 2, M ** 3).astype(np.float64) * 2 - 1 for _ in range(3)]
    hs_ref = np.mean([z * op.hvp(z, batch, lam).real for z in probes], axis=0)
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res")
        mp.start_processes(_worker, args=(2, _free_port(), out, use_ball), nprocs=2, start_method="spawn")
        r0 = np.load(out + ".0.npz")
        r1 = np.load(out + ".1.npz")
    assert len(r0["sub"]) + len(r1["sub"]) == batch.size
    for r in (r0, r1):
        assert abs(float(r["loss"]) - loss_ref) / loss_ref < 1e-12
        assert O.relative_l2(r["grad"], grad_ref) < 1e-12
        assert O.relative_l2(r["hs"], hs_ref) < 1e-12
    assert np.array_equal(r0["grad"], r1["grad"])  # identical on every rank


def test_touched_ball_contains_every_scatter_target(golden):
    """Every voxel the oracle's adjoint touches lies inside grid.touched_ball (incl. clamped rim pixels)."""
    g = golden("dataset_m16_tri.npz")
    op = _oracle_op(g)
    M = op.M
    ball = G.touched_ball(M, M // 2 - 1)
    ones = np.ones((op.n_images, op.pix.shape[0]), dtype=np.complex128)
    acc = op.backproject(ones, np.arange(op.n_images))
    touched = np.flatnonzero(np.abs(acc) > 0)
    assert np.isin(touched, ball).all()
    assert ball.size < M ** 3


def _fd_worker(rank, world_size, port, out_path):
    """dist.exchange_fd: rank 0's fd (here a memfd with a payload) duplicated into rank 1 over the
    library's SCM_RIGHTS socket path -- the hand-over NvlsGroup uses for the multicast handle."""
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world_size)
    fd = -1
    if rank == 0:
        fd = os.memfd_create("fsld-test")
        os.write(fd, b"fsld-nvls-handle")
    got = D.exchange_fd(fd)
    data = os.pread(got, 16, 0)
    with open(out_path + f".{rank}", "wb") as f:
        f.write(data + (b"|same" if got == fd else b"|dup"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_fd_exchange_over_unix_socket():
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "fd")
        mp.start_processes(_fd_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn")
        r0, r1 = open(out + ".0", "rb").read(), open(out + ".1", "rb").read()
    assert r0 == b"fsld-nvls-handle|same"
    assert r1 == b"fsld-nvls-handle|dup"


def test_fd_passing_rejects_bad_arguments():
    import ctypes

    from paper_2311_16100_b200 import _capi as C

    lib = C.load()
    s = ctypes.c_int(-1)
    assert lib.fsld_fd_listen(b"", ctypes.byref(s)) == C.FSLD_EINVAL
    assert lib.fsld_fd_listen(b"x" * 200, ctypes.byref(s)) == C.FSLD_EINVAL
    assert lib.fsld_fd_send(b"fsld-none", -1) == C.FSLD_EINVAL
    assert lib.fsld_fd_recv(-1, ctypes.byref(s)) == C.FSLD_EINVAL
    # NVLS entry points validate before touching a driver
    h = ctypes.c_void_p()
    sz, fd = ctypes.c_size_t(), ctypes.c_int()
    assert lib.fsld_nvls_create(0, 1024, ctypes.byref(sz), ctypes.byref(fd), ctypes.byref(h)) == C.FSLD_EINVAL
    assert lib.fsld_nvls_import(-1, 2, 1, 1024, 1 << 21, ctypes.byref(h)) == C.FSLD_EINVAL
    assert lib.fsld_nvls_barrier(None, None, None, None) == C.FSLD_EINVAL
    assert lib.fsld_nvls_supported(0) in (0, 1)
