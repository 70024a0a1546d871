"""Algorithm 1 of the reference on the B200 path (drop-in for fsld.optim).

Same names, signatures and error behaviour as /root/reference/pkg/src/fsld/optim.py:
``loss_and_grad``, ``batch_loss`` and ``hutchinson_update`` run one fused sm_100a kernel pass over the
batch each (fsld_loss_grad(_sorted) / fsld_loss / fsld_hutch_fold(_sorted)); ``ema_and_threshold`` and
``armijo_search`` keep the reference's elementwise logic on numpy arrays (reference semantics) or
torch CUDA tensors.  ``run`` (optim.py:309-393) keeps every step on the device (fused loss+grad+probe
pass, fused preconditioner epilogue, closed-form line search, per-epoch binning plans, optional data
parallelism) and ``reference_solve`` (optim.py:396-450) runs Jacobi-preconditioned CG with the GPU
Hessian product.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import NumericalError
from .forward import _is_dev, _to_dev_c64, _to_host_c128
from .grid import shell_counts

NOTHRESH_FLOOR = 1e-12
MAX_HALVINGS = 60

VARIANTS = ("plain", "precomputed", "estimated", "estimated_nothresh")

__all__ = [
    "OptimConfig", "PreconditionerState", "RunTrace", "VARIANTS", "epoch_batches", "rademacher",
    "loss_and_grad", "batch_loss", "hutchinson_update", "ema_and_threshold", "threshold_alpha",
    "armijo_search", "run", "reference_solve",
]


@dataclass
class OptimConfig:
    """Optimizer hyper-parameters (optim.py:60-95), same validation."""

    lam: float
    batch_size: int
    epochs: int
    beta: float = 0.9
    c: float = 0.5
    eta0: float = 1.0
    variant: str = "estimated"
    seed: int = 0
    mode: str = "tri"
    eta_growth: float = 1.0

    def __post_init__(self) -> None:
        if self.lam < 0:
            raise ValueError("lam must be non-negative")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.epochs < 1:
            raise ValueError("epochs must be >= 1")
        if not 0.0 < self.beta < 1.0:
            raise ValueError("beta must lie in (0, 1)")
        if not 0.0 < self.c < 1.0:
            raise ValueError("c must lie in (0, 1)")
        if self.eta0 <= 0:
            raise ValueError("eta0 must be positive")
        if self.variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}")
        if self.mode not in ("nn", "tri"):
            raise ValueError("mode must be 'nn' or 'tri'")
        if self.eta_growth < 1.0:
            raise ValueError("eta_growth must be >= 1")


@dataclass
class RunTrace:
    """Per-epoch and per-iteration records of one optimizer run (optim.py:117-130)."""

    loss: np.ndarray
    eta_end: np.ndarray
    backtracks: np.ndarray
    precond_rel_err: np.ndarray
    fsc_history: np.ndarray | None
    shell_radii: np.ndarray | None
    accepted_etas: list = field(default_factory=list)
    armijo_steps: int = 0
    armijo_violations: int = 0
    final_dhat: np.ndarray | None = None
    step_f0: list = field(default_factory=list)      # per step (not in the reference trace)
    step_f_next: list = field(default_factory=list)
    step_backtracks: list = field(default_factory=list)


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
    if e.brick_path and hasattr(op, "loss_and_grad_numpy"):
        # the reference's call shape (numpy complex128 in / out): pinned complex64 staging with
        # threaded casts and the slab-pipelined host step (copies overlapped with the kernels)
        return op.loss_and_grad_numpy(v, batch, lam, n_total)
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

    ``shells`` (a ShellTable, as the reference passes) supplies P_x(R)/P_v(R) and must have
    max_radius == the stack's mask radius (ValueError otherwise, like the reference); None builds
    the populations from the grid.  Radial CTFs are evaluated at R like the reference; for the
    astigmatic PhysicalCtf (not radial) |C_i(R)|^2 is the mean over the masked pixels of
    shell R (builder-defined).
    """
    M = stack.spec.M
    r = stack.mask_radius
    if shells is not None:
        if shells.max_radius != r:
            raise ValueError("shell table radius must match the stack mask radius")
        if shells.vx_count[r] == 0:
            raise ValueError(f"empty 3D shell at radius {r}")
        ratio = shells.shell_ratio(r)
    else:
        px, vx = shell_counts(M, r)
        if vx[r] == 0:
            raise ValueError(f"empty 3D shell at radius {r}")
        ratio = float(px[r]) / float(vx[r])
    if stack.ctfs is None:
        csum = float(stack.n_images)
    else:
        from .forward import PhysicalCtf, ctf_eval
        from .grid import pixel_coords
        from .kernels import ctf_table_row
        pc = pixel_coords(M).astype(np.float64)
        ring = pc[np.round(np.sqrt((pc ** 2).sum(axis=1))) == r]
        csum = 0.0
        if all(isinstance(c, PhysicalCtf) or hasattr(c, "astig") for c in stack.ctfs):
            if torch.cuda.is_available():  # fsld_ctf_ring_power: one CTA per image, fp64
                csum = _ring_power_device(stack.ctfs, ring, M)
                return ratio * csum + lam
            # (no device: the same per-element formula vectorised on the host, summed in image order)
            from .forward import ctf_coefficients
            co = [ctf_coefficients(c, M) for c in stack.ctfs]
            g = np.array([t[0] for t in co], dtype=np.float64)
            env = np.array([t[1] for t in co])[:, None]
            ws = np.array([t[2] for t in co])[:, None]
            wc = np.array([t[3] for t in co])[:, None]
            kx, ky = ring[:, 0][None, :], ring[:, 1][None, :]
            k2 = kx * kx + ky * ky
            for lo in range(0, len(co), 4096):
                s = slice(lo, lo + 4096)
                gam = (g[s, 0:1] * k2 + g[s, 1:2] * (kx * kx - ky * ky) + g[s, 2:3] * (2 * kx * ky)
                       + g[s, 3:4] * k2 * k2)
                row = -(ws[s] * np.sin(gam) + wc[s] * np.cos(gam)) * np.exp(-env[s] * k2)
                for m in np.mean(row ** 2, axis=1):
                    csum += float(m)
            return ratio * csum + lam
        for c in stack.ctfs:
            if isinstance(c, PhysicalCtf) or hasattr(c, "astig"):
                csum += float(np.mean(ctf_table_row(c, ring, M) ** 2))
            else:
                csum += ctf_eval(c, r, M // 2) ** 2
    return ratio * csum + lam


def _ring_power_device(ctfs, ring: np.ndarray, M: int) -> float:
    """sum_i mean_{k in ring} C_i(k)^2 on the device (fsld_ctf_ring_power), summed in image order."""
    from . import _capi as C
    from .engine import _stream, ctypes_ptr, records_for

    n = len(ctfs)
    recs = records_for(M, np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)), None, ctfs)  # the CTF fields only
    dev = torch.device("cuda", torch.cuda.current_device())
    rd = torch.from_numpy(recs.view(np.uint8).copy()).to(dev)
    rg = torch.from_numpy(np.ascontiguousarray(ring, dtype=np.int16)).to(dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    C.check(C.load().fsld_ctf_ring_power(ctypes_ptr(rd), n, ctypes_ptr(rg), rg.shape[0], ctypes_ptr(out), _stream()),
            "fsld_ctf_ring_power")
    csum = 0.0
    for m in out.cpu().numpy():
        csum += float(m)
    return csum


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


def run(config: OptimConfig, stack, v0=None, reference=None, exact_diag_vec=None, probes: str = "reference",
        op=None, group=None, alpha: float | None = None, shard_dataset: bool = False):
    """Algorithm 1 (optim.py:309-393) with every step resident on the GPU.

    Per batch, in stream order and without host synchronisation:
      fsld_loss_grad_hutch_sorted -> acc, sum|r|^2 and (estimating) the probe's fold z*(A*A z),
                                  one fused pass (else fsld_hutch_fold + fsld_loss_grad)
      fsld_precond_step        -> grad, d_avg, d, dhat, direction, line-search volume terms
                                  (incl. Re<r, A d> = Re<A^* r, d> from the gradient accumulator)
      fsld_proj_energy_sorted  -> ||A d||^2, one gather-only pass (tile kernel for other layouts)
      fsld_armijo_select       -> closed-form backtracking (eta carried on the device)
      fsld_apply_step          -> v <- v - eta direction
    The host reads the per-step record (f0, eta, f_next, backtracks) and the
    epoch loss once per epoch.  probes="reference" draws z from the
    reference's numpy stream (parity); probes="device" generates them in-kernel
    (counter-based, no z bytes moved).  A line search that exceeds 60 halvings
    raises NumericalError at the end of that epoch (the reference raises at the step).

    Data parallel (torch.distributed initialised, one process per GPU, every rank
    holding the dataset): each rank takes its contiguous share of every global batch
    (dist.shard_indices), and per step ONE all-reduce of [gradient accumulator | probe
    fold | sum|r|^2], compacted to the touched ball, plus one scalar all-reduce of the
    line-search energy, combine the ranks; the epilogue, the line search and the update
    then run identically on every rank.  With ``shard_dataset=True`` each rank
    holds only its contiguous range of the images (1/world of the dataset in HBM) and takes
    from every global batch the images of its range; the per-epoch full-dataset loss adds one
    scalar all-reduce.  The batches, probes and the summed objective are the same, so the
    trajectory matches the replicated run up to fp32 summation order.
    """
    from .forward import DatasetOperator, FourierVolume, ImageStack
    from .hessian import exact_diag
    from .metrics import ShellIndex, fsc, relative_l2
    from . import _capi as C

    if probes not in ("reference", "device"):
        raise ValueError("probes must be 'reference' or 'device'")
    from . import dist as D
    rank, ws = D.world()
    if group is not None:
        ws = torch.distributed.get_world_size(group)
        rank = torch.distributed.get_rank(group)
    n = stack.n_images
    lo, hi = 0, n  # the images this rank holds
    if shard_dataset and ws > 1:
        if op is not None:
            raise ValueError("shard_dataset builds the rank's operator itself (op must be None)")
        lo, hi = D.image_range(n, rank, ws)
        if hi <= lo:
            raise ValueError("shard_dataset needs at least one image per rank")
        sub = ImageStack(spec=stack.spec, images=stack.images[lo:hi], poses=list(stack.poses[lo:hi]),
                         ctfs=None if stack.ctfs is None else list(stack.ctfs[lo:hi]), sigma=stack.sigma,
                         seed=stack.seed, mask_radius=stack.mask_radius, mode=stack.mode)
        op = DatasetOperator(sub, config.mode)
    sharded = hi - lo < n
    op = DatasetOperator(stack, config.mode) if op is None else op
    e = op.engine
    spec = op.spec
    nvox = spec.n_voxels
    if alpha is None:  # (callers that run several times on one dataset may pass it precomputed)
        alpha = threshold_alpha(stack, None, config.lam)
    if config.batch_size > n:
        raise ValueError("batch_size exceeds the number of images")
    dev = e.dev
    if v0 is not None:
        vals = v0.values if hasattr(v0, "values") else v0
        v = _to_dev_c64(np.asarray(vals) if not _is_dev(vals) else vals, dev).reshape(-1).clone()
    else:
        v = torch.zeros(nvox, dtype=torch.complex64, device=dev)

    estimating = config.variant in ("estimated", "estimated_nothresh")
    thresholded = config.variant != "estimated_nothresh"
    floor = alpha if thresholded else NOTHRESH_FLOOR
    d_avg = torch.zeros(nvox, dtype=torch.float32, device=dev)
    d = torch.ones(nvox, dtype=torch.float32, device=dev)
    k = 0
    dhat_fixed = None
    if config.variant == "precomputed":
        if exact_diag_vec is None:
            exact_diag_vec = exact_diag(stack.poses, stack.ctfs, config.lam, config.mode, spec, op.mask)
        dhat_fixed = torch.from_numpy(np.maximum(exact_diag_vec, alpha).astype(np.float32)).to(dev)
    z_rng = z_stream(config.seed)

    n_epochs = config.epochs
    shells = ShellIndex(spec.M, stack.mask_radius, dev) if reference is not None else None
    trace = RunTrace(
        loss=np.empty(n_epochs), eta_end=np.empty(n_epochs), backtracks=np.zeros(n_epochs, dtype=np.int64),
        precond_rel_err=np.full(n_epochs, np.nan),
        fsc_history=np.empty((n_epochs, stack.mask_radius + 1)) if reference is not None else None,
        shell_radii=np.arange(stack.mask_radius + 1) if reference is not None else None)
    ref_vals = None
    if reference is not None:
        rv = reference.values if hasattr(reference, "values") else reference
        ref_vals = torch.as_tensor(np.asarray(rv) if not _is_dev(rv) else rv, device=dev)

    from .grid import touched_ball
    if ws > 1 and e.deterministic:
        raise ValueError("the data-parallel run uses the fp32 accumulators (deterministic engines: one process)")
    pbuf = None
    if ws > 1:
        pbuf = D.PackedBuffer.new(nvox, estimating, dev, ball=touched_ball(spec.M, stack.mask_radius))
        acc = pbuf.work_acc()
        fold = pbuf.work_hutch() if estimating else torch.zeros(nvox, dtype=torch.float32, device=dev)
    else:
        acc = torch.zeros(nvox, dtype=torch.complex64, device=dev)
        fold = torch.zeros(nvox, dtype=torch.float32, device=dev)
    dirv = torch.empty(nvox, dtype=torch.complex64, device=dev)
    dhat_last = torch.empty(nvox, dtype=torch.float32, device=dev)
    st = e.new_armijo_state(config.eta0)
    st_f64 = st.view(torch.float64)
    max_steps = -(-n // config.batch_size)  # batches per epoch
    hist = torch.zeros(5 * max_steps, dtype=torch.float64, device=dev)
    lam = float(config.lam)
    all_idx = e.all_indices()
    for epoch in range(n_epochs):
        batches = epoch_batches(n, config.batch_size, config.seed, epoch)
        st.view(torch.int32)[12] = 0  # n_steps: hist rows restart each epoch
        # binning plan of this rank's share of the epoch's full-size batches (one build per epoch;
        # a short last batch is binned in its own step)
        if sharded:  # the batch's images in this rank's range, as local indices
            subs = [D.local_batch(b, lo, hi) for b in batches]
        else:
            subs = [D.shard_indices(b, rank, ws) if ws > 1 else b for b in batches]
        plan, plan_k = None, {}
        if e.brick_path:
            full = [i for i, sb in enumerate(subs) if len(sb) and len(sb) == len(subs[0])]
            if len(full) > 1:
                plan = e.make_plan([subs[i] for i in full])
                plan_k = {i: j for j, i in enumerate(full)}
        for bi, batch in enumerate(batches):
            nb = len(batch)
            scale = n / nb
            last = epoch == n_epochs - 1 and bi == len(batches) - 1
            sub = subs[bi]
            pk = plan_k.get(bi)
            # (planned steps never touch idx: no per-step host->device upload of the batch)
            idx = e.idx_tensor(sub) if len(sub) and pk is None else None
            if estimating:
                if probes == "reference":
                    zbits, kk = e.pack_probes(rademacher(z_rng, nvox))
                else:
                    zbits, kk = e.gen_probes(1, (config.seed << 32) + epoch * 1000003 + bi), 1
            if ws > 1:
                # this rank's share of the batch, then one all-reduce of [acc | fold | sum|r|^2]
                if pk is not None:
                    sq = e.loss_grad_planned(v, plan, pk, acc, zbits=zbits if estimating else None,
                                             fold=fold if estimating else None)
                elif idx is not None and estimating:
                    sq = e.loss_grad_hutch(v, idx, zbits, acc, fold)
                elif idx is not None:
                    sq, _, _ = e.loss_grad(v, idx, acc=acc)
                else:
                    sq = torch.zeros(1, dtype=torch.float64, device=dev)
                pbuf.set_loss(sq)
                pbuf.pack()
                pbuf.all_reduce(group)
                pbuf.unpack()
                sq = pbuf.loss()
                gacc = acc
            elif pk is not None:  # binned with the epoch's plan
                sq = e.loss_grad_planned(v, plan, pk, acc, zbits=zbits if estimating else None,
                                         fold=fold if estimating else None)
                gacc = acc
            elif estimating and not e.deterministic:
                # one fused pass: gradient accumulator + the probe's Hutchinson fold
                sq = e.loss_grad_hutch(v, idx, zbits, acc, fold)
                gacc = acc
            else:
                if estimating:
                    facc, ffx = e.hutch_fold(zbits, kk, idx)
                    fold = e.finalize_r(facc, ffx, 1.0, 0.0)
                sq, gacc, gfx = e.loss_grad(v, idx, acc=None if e.deterministic else acc)
                if e.deterministic:
                    gacc = e.finalize_c(gacc, gfx, 1.0, 0.0)
            params = C.StepParams(scale=scale, lam=lam, beta=float(config.beta), floor=float(floor),
                                  w_old=k / (k + 1), w_new=1.0 / (k + 1), hutch_scale=scale,
                                  estimating=1 if estimating else 0)
            vol4 = e.precond_step(gacc, v, params, dirv, fold=fold if estimating else None,
                                  d_avg=d_avg if estimating else None, d=d if estimating else None,
                                  dhat_fixed=dhat_fixed, dhat_out=dhat_last if last else None)
            if estimating:
                k += 1
            if pk is not None:
                qq = e.proj_energy_planned(dirv, plan, pk)
            elif idx is not None:
                qq = e.proj_energy(dirv, idx, reuse_bins=e.brick_path)  # same batch, same scratch
            else:
                qq = torch.zeros(1, dtype=torch.float64, device=dev)
            if ws > 1:
                torch.distributed.all_reduce(qq, group=group)
            e.armijo_select(sq, vol4[4:5], qq, vol4, scale, lam, float(config.c), st, hist, MAX_HALVINGS)
            e.apply_step(v, dirv, st)
        # ---- epoch end: the only host synchronisation of the epoch
        rows = hist[: 5 * len(batches)].view(-1, 5).cpu().numpy()
        stv = st.cpu().numpy().view(C.ARMIJO_DTYPE)[0]
        if int(stv["status"]) != 0:
            raise NumericalError(f"line search exceeded {MAX_HALVINGS} halvings "
                                 "(non-descent direction or numerical breakdown)")
        for f0, eta_s, f_next, nbt, dec in rows:
            trace.armijo_steps += 1
            if not f_next <= f0 - config.c * eta_s * dec:
                trace.armijo_violations += 1
            trace.accepted_etas.append(float(eta_s))
            trace.step_f0.append(float(f0))
            trace.step_f_next.append(float(f_next))
            trace.step_backtracks.append(int(nbt))
            trace.backtracks[epoch] += int(nbt)
        st_f64[0] *= config.eta_growth
        sq_all = e.loss(v, all_idx)
        if sharded:
            torch.distributed.all_reduce(sq_all, group=group)
        trace.loss[epoch] = 0.5 * float(sq_all.item()) + 0.5 * lam * float(e.norm2(v).item())
        trace.eta_end[epoch] = float(st_f64[0].item())
        if estimating and exact_diag_vec is not None:
            trace.precond_rel_err[epoch] = relative_l2(d_avg, exact_diag_vec)
        if reference is not None:
            trace.fsc_history[epoch] = fsc(v, ref_vals, shells).values
    if estimating or dhat_fixed is not None:
        trace.final_dhat = dhat_last.double().cpu().numpy()
    else:
        trace.final_dhat = np.ones(nvox)
    return FourierVolume(_to_host_c128(v), spec), trace


# The operator runs in fp32 (products, gathers, atomics): a relative residual below ~1e-6 is not
# reachable, so tighter requests are served at this floor.
REF_SOLVE_MIN_TOL = 1e-6


def reference_solve(stack, lam: float, mode: str, tol: float = 1e-8, max_iter: int = 500, op=None):
    """Jacobi-preconditioned CG for H v = b (optim.py:396-450) with every H application on the GPU.

    Same recursion, stopping rule (residual recomputed from scratch before accepting, restart if the
    recursion drifted) and errors as the reference; vectors are complex128 on the device, each H
    product is one pass of the fsld_hvp kernel over all images.  ``tol`` below REF_SOLVE_MIN_TOL is
    raised to it (fp32 operator).
    """
    from .forward import DatasetOperator, FourierVolume
    from .hessian import exact_diag

    if lam <= 0:
        raise ValueError("reference solve needs lam > 0 (positive definite H)")
    op = DatasetOperator(stack, mode) if op is None else op
    e = op.engine
    all_idx = e.all_indices()
    acc, fx = e.backproject_dataset(all_idx)
    b = e.finalize_c(acc, fx, 1.0, 0.0).to(torch.complex128)
    b_norm = float(torch.linalg.vector_norm(b))
    if b_norm == 0:
        return FourierVolume.zeros(op.spec)
    jacobi = torch.from_numpy(exact_diag(stack.poses, stack.ctfs, lam, mode, op.spec, op.mask)).to(e.dev)
    tol = max(float(tol), REF_SOLVE_MIN_TOL)

    def apply_h(w):
        a, f = e.hvp_acc(w.to(torch.complex64), all_idx)
        return e.finalize_c(a, f, 1.0, 0.0).to(torch.complex128) + lam * w

    def rdot(x, y) -> float:
        return float(torch.vdot(x, y).real)

    v = torch.zeros_like(b)
    r = b.clone()
    y = r / jacobi
    p = y.clone()
    rho = rdot(r, y)
    for _ in range(max_iter):
        hp = apply_h(p)
        denom = rdot(p, hp)
        if denom <= 0:
            raise NumericalError("CG breakdown: non-positive curvature")
        step = rho / denom
        v += step * p
        r -= step * hp
        if float(torch.linalg.vector_norm(r)) <= tol * b_norm:
            r = b - apply_h(v)  # certify with a residual recomputed from scratch
            if float(torch.linalg.vector_norm(r)) <= tol * b_norm:
                return FourierVolume(v.cpu().numpy(), op.spec)
            y = r / jacobi
            p = y.clone()
            rho = rdot(r, y)
            continue
        y = r / jacobi
        rho_new = rdot(r, y)
        beta = rho_new / rho
        rho = rho_new
        p = y + beta * p
    raise NumericalError(f"CG did not reach tolerance {tol} in {max_iter} iterations")
