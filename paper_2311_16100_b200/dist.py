"""Data-parallel sharding of the loss / gradient / Hutchinson step over GPUs.

The objective and the Hessian are sums over images (optim.py:186-189,
forward.py:567-570), so a global batch splits into per-rank sub-batches with
no data exchange inside the hot path.  Each rank runs the fused kernels on its
share and produces partial sums; ONE all-reduce of a packed buffer

    [ grad accumulator (2 M^3) | Hutchinson fold (M^3, optional) | sum|r|^2 (hi, lo) ]

combines them (NCCL over NVLink/NVSwitch on B200, gloo in the CPU tests), and
every rank then applies the same epilogue (scale, lam, running averages), so
all ranks hold identical gradients / preconditioners.  The global batch
composition follows the reference's per-epoch permutation (optim.py:133-139),
so results do not depend on the number of ranks beyond fp32 summation order
(and not at all in deterministic int64 mode).

The per-rank compute is injectable (``compute=``) so the sharding / packing /
reduction logic is testable on CPU with world_size 2 (tests/test_dist_gloo.py);
the product default is the B200 engine.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_indices(batch, rank: int, world_size: int):
    """Contiguous near-equal split of a global batch (ranks 0.. get the longer parts)."""
    batch = np.asarray(batch)
    if batch.size == 0:
        raise ValueError("batch must be nonempty")
    bounds = np.linspace(0, batch.size, world_size + 1).round().astype(int)
    return batch[bounds[rank]:bounds[rank + 1]]


@dataclass
class PackedBuffer:
    """One flat tensor viewed as [acc (complex) | hutch (real, optional) | loss (hi, lo)]."""

    flat: torch.Tensor
    n_voxels: int
    with_hutch: bool

    @classmethod
    def new(cls, n_voxels: int, with_hutch: bool, device, dtype=torch.float32) -> "PackedBuffer":
        size = 2 * n_voxels + (n_voxels if with_hutch else 0) + 2
        return cls(torch.zeros(size, dtype=dtype, device=device), n_voxels, with_hutch)

    @property
    def acc(self) -> torch.Tensor:
        return self.flat[:2 * self.n_voxels].view(
            torch.complex64 if self.flat.dtype == torch.float32 else torch.complex128)

    @property
    def hutch(self) -> torch.Tensor | None:
        if not self.with_hutch:
            return None
        return self.flat[2 * self.n_voxels:3 * self.n_voxels]

    def set_loss(self, sq: torch.Tensor) -> None:
        """Store a float64 device scalar as (hi, lo) in the buffer's dtype (exact-ish through a sum)."""
        hi = sq.to(self.flat.dtype)
        self.flat[-2:-1].copy_(hi)
        self.flat[-1:].copy_((sq - hi.double()).to(self.flat.dtype))

    def loss(self) -> torch.Tensor:
        return self.flat[-2:-1].double() + self.flat[-1:].double()

    def all_reduce(self, group=None) -> None:
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)


def _engine_compute(op, v, sub, buf: PackedBuffer, zbits=None, k=0):
    """Default per-rank compute: fused loss+grad (and probe fold) on this rank's GPU."""
    e = op.engine
    sq, _, _ = e.loss_grad(v, sub, acc=buf.acc)
    if zbits is not None:
        e.hutch_fold(zbits, k, sub, acc=buf.hutch)
    buf.set_loss(sq)


def sharded_step(op, v, batch, lam: float, n_total: int | None = None, buf: PackedBuffer | None = None,
                 zbits=None, k: int = 0, compute=None, group=None):
    """One data-parallel loss / gradient (/ Hutchinson fold) evaluation over a GLOBAL batch.

    Returns (loss, grad, hutch_sample) identical on every rank, where
    hutch_sample = n_total/|batch|/k * sum_p z_p * (A^*A z_p) + lam (None without probes).
    """
    rank, ws = world()
    batch = np.asarray(batch)
    n_total = op.n_images if n_total is None else n_total
    scale = n_total / batch.size
    sub = shard_indices(batch, rank, ws)
    dev = v.device if isinstance(v, torch.Tensor) else torch.device("cpu")
    if buf is None:
        buf = PackedBuffer.new(v.numel() if isinstance(v, torch.Tensor) else np.asarray(v).size,
                               zbits is not None, dev)
    else:
        buf.flat.zero_()
    (compute or _engine_compute)(op, v, sub, buf, zbits, k)
    buf.all_reduce(group)
    sq = buf.loss()
    if isinstance(v, torch.Tensor) and v.is_cuda and buf.flat.dtype == torch.float32:
        loss, grad = op.engine.epilogue(buf.acc, v, scale, lam, sq)
        loss = loss[0]
    else:
        vv = torch.as_tensor(np.asarray(v)) if not isinstance(v, torch.Tensor) else v
        vv = vv.to(buf.acc.dtype)
        grad = scale * buf.acc + lam * vv
        loss = 0.5 * scale * sq[0] + 0.5 * lam * float((vv.abs() ** 2).sum())
    hs = None
    if buf.with_hutch and k > 0:
        hs = (scale / k) * buf.hutch.double() + lam
    return loss, grad, hs
