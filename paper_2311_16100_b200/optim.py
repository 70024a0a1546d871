"""Loss / gradient / Hutchinson primitives of Algorithm 1 on the B200 path (drop-in for fsld.optim).

Same names, signatures and error behaviour as
/root/reference/pkg/src/fsld/optim.py:98-306.  ``loss_and_grad``,
``batch_loss`` and ``hutchinson_update`` run one fused sm_100a kernel pass
over the batch each (fsld_loss_grad / fsld_loss / fsld_hutch_fold); the
elementwise EMA / threshold / Armijo logic is unchanged and works on numpy
arrays (reference semantics) or torch CUDA tensors (device-resident loop).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import NumericalError
from .forward import _is_dev, _to_dev_c64, _to_host_c128
from .grid import shell_counts

NOTHRESH_FLOOR = 1e-12
MAX_HALVINGS = 60

__all__ = [
    "PreconditionerState", "epoch_batches", "rademacher", "loss_and_grad", "batch_loss",
    "hutchinson_update", "ema_and_threshold", "threshold_alpha", "armijo_search",
]


@dataclass
class PreconditionerState:
    """Running Hutchinson average and its EMA (optim.py:98-114)."""

    d_avg: np.ndarray
    d: np.ndarray
    k: int
    alpha: float

    @classmethod
    def initial(cls, n_voxels: int, alpha: float, device=None) -> "PreconditionerState":
        if device is not None:
            return cls(d_avg=torch.zeros(n_voxels, dtype=torch.float64, device=device),
                       d=torch.ones(n_voxels, dtype=torch.float64, device=device), k=0, alpha=alpha)
        return cls(d_avg=np.zeros(n_voxels), d=np.ones(n_voxels), k=0, alpha=alpha)


def epoch_batches(n_images: int, batch_size: int, seed: int, epoch: int) -> list:
    """Seeded per-epoch shuffle cut into consecutive batches (optim.py:133-139)."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(1, epoch)))
    perm = rng.permutation(n_images)
    return [perm[i:i + batch_size] for i in range(0, n_images, batch_size)]


def z_stream(seed: int) -> np.random.Generator:
    """The Rademacher stream of optim.run (optim.py:347-349)."""
    return np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(2,)))


def rademacher(rng: np.random.Generator, n: int) -> np.ndarray:
    """+-1 vector with fair signs (optim.py:142-144)."""
    return rng.integers(0, 2, size=n).astype(np.float64) * 2.0 - 1.0


def _batch_size(batch) -> int:
    return int(batch.numel()) if isinstance(batch, torch.Tensor) else int(np.asarray(batch).size)


def loss_and_grad(op, v, batch, lam: float, n_total: int | None = None):
    """Mini-batch loss and gradient in full-dataset units (optim.py:165-190).

    One fused kernel: slice -> CTF/shift -> residual -> |r|^2 -> adjoint scatter.
    numpy v -> (float, complex128 ndarray); CUDA tensor v -> (0-d float64
    tensor, complex64 tensor), no host synchronisation.
    """
    nb = _batch_size(batch)
    if nb == 0:
        raise ValueError("batch must be nonempty")
    e = op.engine
    n_total = op.n_images if n_total is None else n_total
    scale = n_total / nb
    if _is_dev(v):
        vd = e._vol(v)
        sq, acc, fx = e.loss_grad(vd, batch)
        if e.deterministic:
            loss = 0.5 * scale * sq[0] + 0.5 * lam * e.norm2(vd)[0]
            return loss, e.finalize_c(acc, fx, scale, lam, vd)
        loss, grad = e.epilogue(acc, vd, scale, lam, sq)
        return loss[0], grad
    v = np.asarray(v, dtype=np.complex128).reshape(-1)
    sq, acc, fx = e.loss_grad(_to_dev_c64(v, e.dev), batch)
    g = _to_host_c128(e.finalize_c(acc, fx, 1.0, 0.0))
    loss = 0.5 * scale * float(sq.item()) + 0.5 * lam * float((v.real ** 2 + v.imag ** 2).sum())
    return loss, scale * g + lam * v


def batch_loss(op, v, batch, lam: float, n_total: int | None = None):
    """Mini-batch loss only, for the line search (optim.py:193-207)."""
    nb = _batch_size(batch)
    if nb == 0:
        raise ValueError("batch must be nonempty")
    e = op.engine
    n_total = op.n_images if n_total is None else n_total
    scale = n_total / nb
    if _is_dev(v):
        vd = e._vol(v)
        return 0.5 * scale * e.loss(vd, batch)[0] + 0.5 * lam * e.norm2(vd)[0]
    v = np.asarray(v, dtype=np.complex128).reshape(-1)
    sq = e.loss(_to_dev_c64(v, e.dev), batch)
    return 0.5 * scale * float(sq.item()) + 0.5 * lam * float((v.real ** 2 + v.imag ** 2).sum())


def _is_rademacher(z) -> bool:
    if isinstance(z, torch.Tensor):
        return bool((z.abs() == 1).all().item())
    return bool(np.all(np.abs(np.asarray(z)) == 1.0))


def hutchinson_sample(op, z, batch, lam: float, n_total: int | None = None):
    """Mean over the supplied probes of z * Re(hvp(z)) and the probe count k.

    z: (M^3,) or (k, M^3) real.  +-1 probes go through the bit-packed probe
    batcher (one pass for all k); other real vectors through hvp.
    """
    e = op.engine
    nb = _batch_size(batch)
    if nb == 0:
        raise ValueError("batch must be nonempty")
    n_total = op.n_images if n_total is None else n_total
    scale = n_total / nb
    zz = z if isinstance(z, torch.Tensor) else np.asarray(z, dtype=np.float64)
    k = 1 if zz.ndim == 1 else zz.shape[0]
    dev_out = _is_dev(z)
    if _is_rademacher(zz):
        zbits, k = e.pack_probes(zz)
        acc, fx = e.hutch_fold(zbits, k, batch)
        fold = e.finalize_r(acc, fx, 1.0, 0.0)
        if dev_out:
            return scale / k * fold.double() + lam, k
        return scale / k * fold.cpu().numpy().astype(np.float64) + lam, k
    rows = [zz] if zz.ndim == 1 else list(zz)
    tot = None
    for zr in rows:
        hz = op.hvp(zr if dev_out else np.asarray(zr, dtype=np.complex128), batch, lam, n_total)
        s = zr * hz.real if dev_out else zr * np.asarray(hz).real
        tot = s if tot is None else tot + s
    return tot / k, k


def hutchinson_update(state, op, z, batch, lam: float, n_total: int | None = None):
    """Fold Rademacher sample(s) into the running diagonal average (optim.py:210-229).

    With one probe this is d_avg <- (k-1)/k d_avg + z*Re(Hz)/k exactly as
    the reference; with (k, M^3) probes it equals k successive updates on the
    same batch (running mean over all probes), computed in one kernel pass.
    """
    sample, kk = hutchinson_sample(op, z, batch, lam, n_total)
    k_old = state.k
    state.k += kk
    state.d_avg *= k_old / state.k
    state.d_avg += sample * (kk / state.k)
    return state


def ema_and_threshold(state, beta: float, alpha: float, thresholded: bool = True):
    """d <- beta d + (1-beta) d_avg; return max(|d|, alpha) (optim.py:232-247)."""
    state.d *= beta
    state.d += (1.0 - beta) * state.d_avg
    floor = alpha if thresholded else NOTHRESH_FLOOR
    if isinstance(state.d, torch.Tensor):
        return torch.clamp(state.d.abs(), min=floor)
    return np.maximum(np.abs(state.d), floor)


def threshold_alpha(stack, shells=None, lam: float = 0.0) -> float:
    """alpha = P_x(R)/P_v(R) * sum_i |C_i(R)|^2 + lam (optim.py:250-266).

    Radial CTFs are evaluated at R like the reference; for the astigmatic
    PhysicalCtf (not radial) |C_i(R)|^2 is the mean over the masked pixels of
    shell R (builder-defined).
    """
    M = stack.spec.M
    r = stack.mask_radius
    px, vx = shell_counts(M, r)
    if vx[r] == 0:
        raise ValueError(f"empty 3D shell at radius {r}")
    if stack.ctfs is None:
        csum = float(stack.n_images)
    else:
        from .forward import PhysicalCtf, ctf_eval
        from .grid import pixel_coords
        from .kernels import ctf_table_row
        pc = pixel_coords(M).astype(np.float64)
        ring = pc[np.round(np.sqrt((pc ** 2).sum(axis=1))) == r]
        csum = 0.0
        for c in stack.ctfs:
            if isinstance(c, PhysicalCtf) or hasattr(c, "astig"):
                csum += float(np.mean(ctf_table_row(c, ring, M) ** 2))
            else:
                csum += ctf_eval(c, r, M // 2) ** 2
    return float(px[r]) / float(vx[r]) * csum + lam


def armijo_search(v, grad, dhat, loss_fn, eta_in: float, c: float, f0=None):
    """Backtracking line search along -dhat^-1 grad (optim.py:269-306)."""
    if eta_in <= 0:
        raise ValueError("eta_in must be positive")
    if f0 is None:
        f0 = loss_fn(v)
    direction = grad / dhat
    decrease = float(((grad.real ** 2 + grad.imag ** 2) / dhat).sum())
    if decrease == 0.0:
        return eta_in, v, f0, 0
    eta = float(eta_in)
    f0 = float(f0)
    for backtracks in range(MAX_HALVINGS + 1):
        v_next = v - eta * direction
        f_next = float(loss_fn(v_next))
        if f_next <= f0 - c * eta * decrease:
            return eta, v_next, f_next, backtracks
        eta *= 0.5
    raise NumericalError(f"line search exceeded {MAX_HALVINGS} halvings (non-descent direction or numerical breakdown)")
