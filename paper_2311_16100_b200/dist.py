"""Data-parallel sharding of the loss / gradient / Hutchinson step over GPUs.

The objective and the Hessian are sums over images (optim.py:186-189,
forward.py:567-570), so a global batch splits into per-rank sub-batches with
no data exchange inside the hot path.  Each rank runs the fused kernels on its
share and produces partial sums; ONE all-reduce of a packed buffer

    [ grad accumulator (2 M^3) | Hutchinson fold (M^3, optional) | sum|r|^2 (hi, lo) ]

combines them (NCCL over NVLink/NVSwitch on B200, gloo in the CPU tests) -- optionally
compacted to the voxels a scatter can reach (grid.touched_ball, ~54 % of the cube at M=128) -- and
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


def image_range(n_images: int, rank: int, world_size: int) -> tuple[int, int]:
    """The contiguous image range [lo, hi) a rank holds when the dataset itself is sharded."""
    bounds = np.linspace(0, n_images, world_size + 1).round().astype(int)
    return int(bounds[rank]), int(bounds[rank + 1])


def local_batch(batch, lo: int, hi: int):
    """The images of a global batch that fall in [lo, hi), as indices local to that range (the
    rank's share of the batch when each rank holds only its image range)."""
    b = np.asarray(batch)
    return b[(b >= lo) & (b < hi)] - lo


@dataclass
class PackedBuffer:
    """One flat tensor viewed as [acc (complex) | hutch (real, optional) | loss (hi, lo)].

    With ``ball`` (int32 voxel indices, grid.touched_ball) the accumulators in the flat buffer are
    the compacted vectors; the per-rank compute writes full-size work accumulators
    (``work_acc`` / ``work_hutch``) that ``pack`` gathers before and ``unpack`` scatters after the
    all-reduce (voxels outside the ball are zero on every rank)."""

    flat: torch.Tensor
    n_voxels: int
    with_hutch: bool
    ball: torch.Tensor | None = None
    _wacc: torch.Tensor | None = None
    _whutch: torch.Tensor | None = None

    @classmethod
    def new(cls, n_voxels: int, with_hutch: bool, device, dtype=torch.float32, ball=None) -> "PackedBuffer":
        if ball is not None:
            ball = torch.as_tensor(np.asarray(ball, dtype=np.int32) if not isinstance(ball, torch.Tensor) else ball,
                                   device=device).to(torch.int32).contiguous()
        ne = n_voxels if ball is None else int(ball.numel())
        size = 2 * ne + (ne if with_hutch else 0) + 2
        return cls(torch.zeros(size, dtype=dtype, device=device), n_voxels, with_hutch, ball)

    @property
    def n_elems(self) -> int:
        return self.n_voxels if self.ball is None else int(self.ball.numel())

    def _cdtype(self):
        return torch.complex64 if self.flat.dtype == torch.float32 else torch.complex128

    @property
    def acc(self) -> torch.Tensor:
        return self.flat[:2 * self.n_elems].view(self._cdtype())

    @property
    def hutch(self) -> torch.Tensor | None:
        if not self.with_hutch:
            return None
        return self.flat[2 * self.n_elems:3 * self.n_elems]

    def work_acc(self) -> torch.Tensor:
        """Full-size accumulator the per-rank compute adds into (the flat view without a ball)."""
        if self.ball is None:
            return self.acc
        if self._wacc is None:
            self._wacc = torch.zeros(self.n_voxels, dtype=self._cdtype(), device=self.flat.device)
        return self._wacc

    def work_hutch(self) -> torch.Tensor | None:
        if self.ball is None or not self.with_hutch:
            return self.hutch
        if self._whutch is None:
            self._whutch = torch.zeros(self.n_voxels, dtype=self.flat.dtype, device=self.flat.device)
        return self._whutch

    def zero(self) -> None:
        self.flat.zero_()
        if self._wacc is not None:
            self._wacc.zero_()
        if self._whutch is not None:
            self._whutch.zero_()

    def _move(self, gather: bool, full: torch.Tensor, compact: torch.Tensor, elem_bytes: int) -> None:
        if full.is_cuda and full.dtype in (torch.complex64, torch.float32):
            from . import _capi as C
            from .engine import _stream, ctypes_ptr
            fn = C.load().fsld_ball_gather if gather else C.load().fsld_ball_scatter
            src, dst = (full, compact) if gather else (compact, full)
            C.check(fn(self.ball.numel(), ctypes_ptr(self.ball), ctypes_ptr(src), ctypes_ptr(dst), elem_bytes,
                       _stream()), "fsld_ball_gather" if gather else "fsld_ball_scatter")
        else:  # CPU (gloo tests): plain indexing
            idx = self.ball.long()
            if gather:
                compact.copy_(full[idx])
            else:
                full[idx] = compact

    def pack(self) -> None:
        """Work accumulators -> compacted flat buffer (no-op without a ball)."""
        if self.ball is None:
            return
        self._move(True, self._wacc, self.acc, 8)
        if self.with_hutch and self._whutch is not None:
            self._move(True, self._whutch, self.hutch, 4)

    def unpack(self) -> None:
        """All-reduced compacted buffer -> work accumulators (voxels outside the ball stay zero)."""
        if self.ball is None:
            return
        self._move(False, self._wacc, self.acc, 8)
        if self.with_hutch and self._whutch is not None:
            self._move(False, self._whutch, self.hutch, 4)

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
    sq, _, _ = e.loss_grad(v, sub, acc=buf.work_acc())
    if zbits is not None:
        e.hutch_fold(zbits, k, sub, acc=buf.work_hutch())
    buf.set_loss(sq)


def sharded_step(op, v, batch, lam: float, n_total: int | None = None, buf: PackedBuffer | None = None,
                 zbits=None, k: int = 0, compute=None, group=None, image_range: tuple[int, int] | None = None):
    """One data-parallel loss / gradient (/ Hutchinson fold) evaluation over a GLOBAL batch.

    Returns (loss, grad, hutch_sample) identical on every rank, where
    hutch_sample = n_total/|batch|/k * sum_p z_p * (A^*A z_p) + lam (None without probes).
    image_range=(lo, hi): the dataset itself is sharded -- ``op`` holds only images [lo, hi) and
    the rank computes the batch's images of that range (n_total is then required).
    """
    rank, ws = world()
    batch = np.asarray(batch)
    if image_range is not None and n_total is None:
        raise ValueError("a sharded dataset needs n_total (the number of images over all ranks)")
    n_total = op.n_images if n_total is None else n_total
    scale = n_total / batch.size
    sub = shard_indices(batch, rank, ws) if image_range is None else local_batch(batch, *image_range)
    dev = v.device if isinstance(v, torch.Tensor) else torch.device("cpu")
    if buf is None:
        buf = PackedBuffer.new(v.numel() if isinstance(v, torch.Tensor) else np.asarray(v).size,
                               zbits is not None, dev)
    else:
        buf.zero()
    (compute or _engine_compute)(op, v, sub, buf, zbits, k)
    buf.pack()
    buf.all_reduce(group)
    buf.unpack()
    sq = buf.loss()
    acc = buf.work_acc()
    if isinstance(v, torch.Tensor) and v.is_cuda and buf.flat.dtype == torch.float32:
        loss, grad = op.engine.epilogue(acc, v, scale, lam, sq)
        loss = loss[0]
    else:
        vv = torch.as_tensor(np.asarray(v)) if not isinstance(v, torch.Tensor) else v
        vv = vv.to(acc.dtype)
        grad = scale * acc + lam * vv
        loss = 0.5 * scale * sq[0] + 0.5 * lam * float((vv.abs() ** 2).sum())
    hs = None
    if buf.with_hutch and k > 0:
        hs = (scale / k) * buf.work_hutch().double() + lam
    return loss, grad, hs


def exchange_fd(fd: int, group=None, tag: str = "fsld") -> int:
    """Rank 0's file descriptor, duplicated into every rank of the node (SCM_RIGHTS over abstract
    unix sockets, fsld_fd_listen / fsld_fd_send / fsld_fd_recv).  Rank 0 returns its own fd."""
    import ctypes
    import uuid

    from . import _capi as C

    lib = C.load()
    rank, ws = dist.get_rank(group), dist.get_world_size(group)
    token = [uuid.uuid4().hex[:16] if rank == 0 else None]
    dist.broadcast_object_list(token, src=0, group=group)
    name = lambda r: f"{tag}-{token[0]}-{r}".encode()  # noqa: E731
    sock = ctypes.c_int(-1)
    if rank > 0:
        C.check(lib.fsld_fd_listen(name(rank), ctypes.byref(sock)), "fd_listen")
    dist.barrier(group)
    if rank == 0:
        for r in range(1, ws):
            C.check(lib.fsld_fd_send(name(r), int(fd)), "fd_send")
        out = int(fd)
    else:
        got = ctypes.c_int(-1)
        C.check(lib.fsld_fd_recv(sock.value, ctypes.byref(got)), "fd_recv")
        out = got.value
    dist.barrier(group)
    return out


class NvlsGroup:
    """A gradient accumulator shared through NVSwitch multicast (include/fsld_b200.h, fsld_nvls_*).

    Every rank holds a local copy (``uc``, read and zeroed by its epilogue) and the multicast
    address (``mc``) its brick pass flushes into: each flush lands in every rank's copy, so after
    ``barrier(sq, sq_total)`` all copies hold the sum over ranks of the partial adjoints and
    sq_total the sum of the ranks' |r|^2 in rank order -- the exchange rides on the pass instead of
    an all-reduce after it (optim.py:186-189: the objective is a sum over images).
    With no process group (or world 1) the group has one member: the same kernels, no exchange.
    """

    def __init__(self, n_voxels: int, group=None):
        import ctypes

        from . import _capi as C

        self._C = C
        lib = C.load()
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        ws = dist.get_world_size(group) if multi else 1
        rank = dist.get_rank(group) if multi else 0
        self.n_ranks, self.rank = ws, rank
        self.data_bytes = int(n_voxels) * 8
        h = ctypes.c_void_p()
        self._h = None
        size = ctypes.c_size_t(0)
        fd = ctypes.c_int(-1)

        def agree(st: int, what: str) -> None:  # every rank learns whether every rank succeeded
            sts = [st]
            if multi:
                sts = [None] * ws
                dist.all_gather_object(sts, st, group=group)
            if any(x != 0 for x in sts):
                if h.value:
                    lib.fsld_nvls_destroy(h)
                raise C.FsldError(f"{what}: status {sts}")

        st = lib.fsld_nvls_create(ws, self.data_bytes, ctypes.byref(size), ctypes.byref(fd), ctypes.byref(h)) \
            if rank == 0 else 0
        agree(st, "fsld_nvls_create")
        if multi:
            meta = [int(size.value)]
            dist.broadcast_object_list(meta, src=0, group=group)
            got = exchange_fd(fd.value if rank == 0 else -1, group)
            st = lib.fsld_nvls_import(got, ws, rank, self.data_bytes, meta[0], ctypes.byref(h)) if rank > 0 else 0
            agree(st, "fsld_nvls_import")
            size.value = meta[0]
        self.size = int(size.value)
        # every device joins the team before any memory is bound
        agree(lib.fsld_nvls_add_device(h), "fsld_nvls_add_device")
        uc, mc = ctypes.c_void_p(), ctypes.c_void_p()
        agree(lib.fsld_nvls_bind(h, ctypes.byref(uc), ctypes.byref(mc)), "fsld_nvls_bind")
        self._h = h
        self.uc, self.mc = int(uc.value), int(mc.value)

    def barrier(self, sq_in=None, sq_out=None, stream=None) -> None:
        from .engine import _stream, ctypes_ptr

        self._C.check(self._C.load().fsld_nvls_barrier(self._h, ctypes_ptr(sq_in), ctypes_ptr(sq_out),
                                                        _stream() if stream is None else stream), "nvls_barrier")

    def check(self) -> None:
        self._C.check(self._C.load().fsld_nvls_status(self._h), "nvls barrier (a peer did not arrive)")

    def close(self) -> None:
        if self._h:
            self._C.load().fsld_nvls_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nvls_available(device: int = 0) -> bool:
    from . import _capi as C

    try:
        return bool(C.load().fsld_nvls_supported(int(device)))
    except OSError:
        return False


def nvls_planned_step(eng, g: NvlsGroup, plan, k: int, v, scale: float, lam: float, grad, sq, sq_total, loss,
                      norm_scratch, events=None) -> None:
    """One data-parallel loss+grad step over NVLS (stream-ordered, CUDA-graph capturable):
    barrier (every copy zeroed) -> the brick pass of batch k of ``plan`` flushing into the multicast
    accumulator -> barrier (all flushes landed, |r|^2 summed over ranks) -> grad = scale uc + lam v,
    uc <- 0, loss."""
    from . import _capi as C
    from .engine import _stream, ctypes_ptr

    lib = C.load()
    s = _stream()
    scr = eng.scratch(plan.B)
    g.barrier(stream=s)
    if events is not None:
        events[0].record()
    C.check(lib.fsld_loss_grad_planned_mc(eng.M, eng.mode_id, eng.n_mask, ctypes_ptr(eng.recs), ctypes_ptr(plan.buf),
                                          plan.B, int(k), ctypes_ptr(v), ctypes_ptr(eng.x), ctypes_ptr(eng.pc),
                                          ctypes_ptr(eng.ptab), g.mc, ctypes_ptr(sq), ctypes_ptr(scr),
                                          scr.numel() * 8, s), "loss_grad_planned_mc")
    if events is not None:
        events[1].record()
    g.barrier(sq, sq_total, stream=s)
    C.check(lib.fsld_grad_epilogue(eng.M ** 3, g.uc, ctypes_ptr(v), float(scale), float(lam), ctypes_ptr(grad),
                                   ctypes_ptr(sq_total), ctypes_ptr(loss), 0, ctypes_ptr(norm_scratch),
                                   norm_scratch.numel() * 8, s), "epilogue")
