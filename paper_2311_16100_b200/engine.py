"""Device-resident slice engine: the B200 dataset operator core.

Holds one dataset in HBM in the layout of include/fsld_b200.h and enqueues
the C-ABI kernels on the current torch CUDA stream:

  pix   (n_mask, 2) int16          masked pixel frequencies (grid.disk_mask order)
  recs  (N, 128 B) fsld_image_rec  rotation rows 0-1, shift, CTF coefficients
  x     (N, n_mask) complex64      compact masked observed images
  v / grad accumulators            M^3 complex64 (or int64 pairs, deterministic)

Every method takes and returns torch CUDA tensors and never synchronises the
host, except where a Python float is explicitly requested.  PyTorch is only
the allocator / stream provider here; all arithmetic of the path runs in the
sm_100a kernels of libfsld_b200.so.
"""
from __future__ import annotations

import math
import os
import ctypes

import numpy as np
import torch

from . import _capi as C
from .grid import disk_mask, pixel_coords

# per-image bound on how many pixels of one image can touch one voxel's
# 2x2x2 support (cube cross-section 4*sqrt(2) ~ 5.7 -> at most ~12 lattice points)
HITS_PER_IMAGE = 16


def ctypes_ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream() -> int:
    """The current torch stream of the current device as a raw cudaStream_t (the capture stream
    under CUDA-graph capture); the raw accessor avoids building a Stream object per launch."""
    if _raw_stream is not None:
        return int(_raw_stream(torch.cuda.current_device()))
    return int(torch.cuda.current_stream().cuda_stream)


def require_device() -> torch.device:
    """The B200 path needs a CUDA device; there is no CPU fallback."""
    C.load()
    if not torch.cuda.is_available():
        raise C.FsldError("no CUDA device visible: the fsld B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


class SliceEngine:
    """One dataset resident on one GPU (see module docstring)."""

    def __init__(self, M: int, mode: str, mask: np.ndarray, recs: np.ndarray, x=None,
                 deterministic: bool = False, device=None, tile_path: bool = False, layout: str | None = None,
                 tables: bool = True, nn_brick: bool = False):
        if mode not in ("nn", "tri"):
            raise ValueError("mode must be one of ('nn', 'tri')")
        self.dev = device or require_device()
        self.M = int(M)
        self.mode = mode
        self.mode_id = C.MODE_TRI if mode == "tri" else C.MODE_NN
        self.mask = np.asarray(mask, dtype=np.int64)
        self.n_mask = int(self.mask.size)
        self.n_voxels = self.M ** 3
        self.deterministic = bool(deterministic)
        self.flags = ((C.DETERMINISTIC if self.deterministic else 0) | (C.TILE_PATH if tile_path else 0)
                      | (C.NN_BRICK if nn_brick else 0))
        pix = pixel_coords(self.M)[self.mask].astype(np.int16)
        self.pix = torch.from_numpy(np.ascontiguousarray(pix)).to(self.dev)
        recs = np.ascontiguousarray(recs, dtype=C.REC_DTYPE)
        self.n_images = int(recs.shape[0])
        self.recs = torch.from_numpy(recs.view(np.uint8).copy()).to(self.dev)
        # dataset layout of x: "sorted" = brick-sorted (fsld_sorted_*; needs M <= 256), "mask" = mask order
        if layout is None:
            layout = "sorted" if (self.M <= 256 and self.n_mask <= 65535 and self.n_images > 0) else "mask"
        if layout not in ("sorted", "mask"):
            raise ValueError("layout must be 'sorted' or 'mask'")
        self.layout = layout
        self.pc = self.seg_off = self.segs = self.ptab = None
        # per-pixel tables (f, trilinear footprint; 24 B per pixel) of the sorted layout: the table-driven brick kernel
        self.use_tables = bool(tables) and not os.environ.get("FSLD_NO_TABLES")
        if layout == "sorted":
            self._build_sorted_index()
        self.x = None
        self.x_maxabs = 0.0
        self._scratch = None
        if x is not None:
            self.set_images(x)
        self._bad = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._all_idx = None

    # ---- data -----------------------------------------------------------
    def _build_sorted_index(self):
        """Per-image brick-sorted pixel order: pc (N, n, 2) int8 and the segment list (once per dataset)."""
        lib = C.load()
        N = self.n_images
        self.seg_off = torch.empty(N + 1, dtype=torch.int32, device=self.dev)
        C.check(lib.fsld_sorted_count(self.M, self.n_mask, ctypes_ptr(self.pix), ctypes_ptr(self.recs), N,
                                      ctypes_ptr(self.seg_off), _stream()), "fsld_sorted_count")
        nseg = int(self.seg_off[N].item())
        self.segs = torch.empty((max(nseg, 1), 2), dtype=torch.int32, device=self.dev)
        self.pc = torch.empty((N, self.n_mask, 2), dtype=torch.int8, device=self.dev)
        C.check(lib.fsld_sorted_fill(self.M, self.n_mask, ctypes_ptr(self.pix), ctypes_ptr(self.recs), N, 0, 0,
                                     ctypes_ptr(self.pc), ctypes_ptr(self.seg_off), ctypes_ptr(self.segs),
                                     _stream()), "fsld_sorted_fill")
        self._build_tables()

    def _build_tables(self):
        """fsld_sorted_tables: per-pixel f = C * phase and trilinear footprint in the sorted order
        (24 B per pixel; rebuilt whenever the sorted order pc is rewritten)."""
        if not self.use_tables or self.layout != "sorted":
            self.ptab = None
            return
        nbytes = int(C.load().fsld_sorted_tables_bytes(self.n_images, self.n_mask))
        if self.ptab is None:
            free, _ = torch.cuda.mem_get_info(self.dev)
            if nbytes > free // 2:  # large datasets (e.g. cfg4's 200k images) keep the compute path
                self.use_tables = False
                return
            self.ptab = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)  # 256-B aligned (caching allocator)
        C.check(C.load().fsld_sorted_tables(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs), self.n_images,
                                            ctypes_ptr(self.pc), ctypes_ptr(self.seg_off), ctypes_ptr(self.segs),
                                            ctypes_ptr(self.ptab), _stream()), "fsld_sorted_tables")

    def _sort_images(self, xd: torch.Tensor) -> torch.Tensor:
        """Mask-order images -> brick-sorted order (same permutation as pc; order within a segment may differ
        between builds, pc is rewritten consistently)."""
        lib = C.load()
        xs = torch.empty_like(xd)
        C.check(lib.fsld_sorted_fill(self.M, self.n_mask, ctypes_ptr(self.pix), ctypes_ptr(self.recs),
                                     self.n_images, ctypes_ptr(xd), ctypes_ptr(xs), ctypes_ptr(self.pc),
                                     ctypes_ptr(self.seg_off), ctypes_ptr(self.segs), _stream()), "fsld_sorted_fill")
        self._build_tables()  # pc was rewritten (order within a segment may differ between builds)
        return xs

    def x_masked(self) -> torch.Tensor:
        """Observed images in mask (reference) pixel order (N, n_mask) complex64."""
        if self.layout == "mask" or self.x is None:
            return self.x
        c = (self.M + 1) // 2
        lut = torch.full((self.M * self.M,), -1, dtype=torch.int64, device=self.dev)
        pix = self.pix.long()
        lut[(pix[:, 1] + c) * self.M + pix[:, 0] + c] = torch.arange(self.n_mask, device=self.dev)
        pc = self.pc.long()
        orig = lut[(pc[..., 1] + c) * self.M + pc[..., 0] + c]
        out = torch.empty_like(self.x)
        out.scatter_(1, orig, self.x)
        return out

    def set_images(self, x, sorted_order: bool = False):
        """Upload observed images (N, n_mask) as complex64 (DatasetOperator.x, forward.py:527).

        Images are given in mask order (reference layout) unless ``sorted_order`` (already in this
        engine's brick-sorted order, e.g. produced by project_sorted)."""
        if isinstance(x, torch.Tensor):
            xd = x.to(self.dev, torch.complex64).contiguous()
        else:
            xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex64)).to(self.dev)
        if tuple(xd.shape) != (self.n_images, self.n_mask):
            raise ValueError(f"images shape {tuple(xd.shape)} != ({self.n_images}, {self.n_mask})")
        if self.layout == "sorted" and not sorted_order:
            xd = self._sort_images(xd)
        self.x = xd
        if xd.numel():
            # per-image max |x| into fsld_image_rec.xmax (bounds the brick fixed-point accumulator)
            xm = xd.abs().amax(dim=1).float() * (1.0 + 1e-6)
            self.recs.view(torch.float32).view(self.n_images, 32)[:, 29] = xm
            self.x_maxabs = float(xm.max().item())
        else:
            self.x_maxabs = 0.0

    def idx_tensor(self, idx) -> torch.Tensor:
        if isinstance(idx, torch.Tensor):
            t = idx.to(self.dev, torch.int32).contiguous()
        else:
            a = np.asarray(idx)
            if a.size and (a.min() < 0 or a.max() >= self.n_images):
                raise IndexError("batch index out of range")
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(self.dev, non_blocking=True)
        if t.numel() == 0:
            raise ValueError("batch must be nonempty")
        return t

    def all_indices(self) -> torch.Tensor:
        if self._all_idx is None:
            self._all_idx = torch.arange(self.n_images, dtype=torch.int32, device=self.dev)
        return self._all_idx

    def scratch(self, B: int) -> torch.Tensor:
        """Prepared scratch (fsld_prepare) large enough for batches of B images."""
        lib = C.load()
        nbytes = int(lib.fsld_scratch_bytes(self.M, self.n_mask, int(B)))
        if self._scratch is None or self._scratch.numel() * 8 < nbytes:
            self._scratch = torch.empty((nbytes + 7) // 8, dtype=torch.float64, device=self.dev)
            C.check(lib.fsld_prepare(self.M, self.n_mask, ctypes_ptr(self.pix), ctypes_ptr(self._scratch),
                                     self._scratch.numel() * 8, _stream()), "fsld_prepare")
        return self._scratch

    # ---- accumulators -----------------------------------------------------
    def new_cacc(self) -> torch.Tensor:
        """Complex accumulator (M^3): complex64, or int64 pairs when deterministic."""
        if self.deterministic:
            return torch.zeros((self.n_voxels, 2), dtype=torch.int64, device=self.dev)
        return torch.zeros(self.n_voxels, dtype=torch.complex64, device=self.dev)

    def new_racc(self) -> torch.Tensor:
        if self.deterministic:
            return torch.zeros(self.n_voxels, dtype=torch.int64, device=self.dev)
        return torch.zeros(self.n_voxels, dtype=torch.float32, device=self.dev)

    def fixed_scale(self, data, mult: float, add: float, out=None) -> torch.Tensor:
        """Device scalar 2^k for int64 fixed-point accumulation (deterministic mode)."""
        fx = torch.empty(1, dtype=torch.float64, device=self.dev) if out is None else out
        n = 0 if data is None else data.numel()
        C.check(C.load().fsld_fixed_scale(ctypes_ptr(data), n, float(mult), float(add),
                                          ctypes_ptr(fx), _stream()), "fixed_scale")
        return fx

    def _vol(self, v) -> torch.Tensor:
        if v.dtype != torch.complex64 or v.device != self.dev or not v.is_contiguous():
            v = v.to(self.dev, torch.complex64).contiguous()
        if v.numel() != self.n_voxels:
            raise ValueError(f"volume has {v.numel()} entries, expected {self.n_voxels}")
        return v.reshape(-1)

    # ---- hot path ---------------------------------------------------------
    def loss_grad(self, v, idx, acc=None, fx=None, fx_batch=None):
        """sum|P v - x|^2 (device double) and acc += sum P^* conj(f) r (optim.py:147-162)."""
        lib = C.load()
        v = self._vol(v)
        idx = self.idx_tensor(idx)
        B = idx.numel()
        acc = self.new_cacc() if acc is None else acc
        if self.deterministic and fx is None:
            fx = self.fixed_scale(v, HITS_PER_IMAGE * (fx_batch or B), self.x_maxabs)
        sq = torch.empty(1, dtype=torch.float64, device=self.dev)
        scr = self.scratch(B)
        if self.layout == "sorted":
            C.check(lib.fsld_loss_grad_sorted(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                              ctypes_ptr(idx), B, ctypes_ptr(v), ctypes_ptr(self.x),
                                              ctypes_ptr(self.pc), ctypes_ptr(self.ptab), ctypes_ptr(self.seg_off),
                                              ctypes_ptr(self.segs), ctypes_ptr(acc), ctypes_ptr(sq), self.flags,
                                              ctypes_ptr(fx),
                                              ctypes_ptr(scr), scr.numel() * 8, _stream()), "fsld_loss_grad_sorted")
            return sq, acc, fx
        C.check(lib.fsld_loss_grad(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.pix),
                                   ctypes_ptr(self.recs), ctypes_ptr(idx), B, ctypes_ptr(v),
                                   ctypes_ptr(self.x), ctypes_ptr(acc), ctypes_ptr(sq), self.flags,
                                   ctypes_ptr(fx), ctypes_ptr(scr), scr.numel() * 8, _stream()),
                "fsld_loss_grad")
        return sq, acc, fx

    @property
    def brick_path(self) -> bool:
        """Whether loss_grad / loss_grad_hutch / proj_energy run the brick-sorted kernels."""
        return (self.layout == "sorted" and self.mode == "tri" and not self.deterministic and
                not (self.flags & C.TILE_PATH) and self.M <= 256)

    @property
    def table_path(self) -> bool:
        """Whether loss_grad / hvp run the table-driven brick kernel (tri or nn; dataset tables built)."""
        return (self.layout == "sorted" and self.ptab is not None and not self.deterministic and
                not (self.flags & C.TILE_PATH) and (self.mode == "tri" or bool(self.flags & C.NN_BRICK)))

    def loss_grad_hutch(self, v, idx, zbits, acc, fold):
        """loss_grad + the k = 1 Hutchinson fold of the same batch (acc, fold accumulate in place).

        One fused brick-path pass when available (tri, brick-sorted layout, not deterministic);
        otherwise fsld_hutch_fold + loss_grad.  Returns sq (device double)."""
        lib = C.load()
        if not self.brick_path:
            self.hutch_fold(zbits, 1, idx, acc=fold)
            sq, _, _ = self.loss_grad(v, idx, acc=acc)
            return sq
        v = self._vol(v)
        idx = self.idx_tensor(idx)
        B = idx.numel()
        sq = torch.empty(1, dtype=torch.float64, device=self.dev)
        scr = self.scratch(B)
        C.check(lib.fsld_loss_grad_hutch_sorted(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                                ctypes_ptr(idx), B, ctypes_ptr(v), ctypes_ptr(self.x),
                                                ctypes_ptr(self.pc), ctypes_ptr(self.ptab), ctypes_ptr(self.seg_off),
                                                ctypes_ptr(self.segs), ctypes_ptr(zbits), ctypes_ptr(acc), ctypes_ptr(fold), ctypes_ptr(sq),
                                                0, ctypes_ptr(scr), scr.numel() * 8, _stream()),
                "fsld_loss_grad_hutch_sorted")
        return sq

    # ---- multi-batch binning plans (fsld_plan_*) ------------------------------
    def make_plan(self, batches, build: bool = True) -> "BinPlan":
        """Bin K equal-size batches at once (e.g. the batches of an epoch): each planned step then
        runs only the work-item kernel.  batches: (K, B) array / list of K index arrays.
        build=False only sizes and allocates the plan (build it with build_plan)."""
        if not self.brick_path:
            raise ValueError("binning plans need the brick path (tri, brick-sorted layout, not deterministic)")
        lib = C.load()
        rows = (batches.cpu().numpy() if isinstance(batches, torch.Tensor)
                else np.stack([np.asarray(b) for b in batches])).astype(np.int64)
        if rows.ndim != 2 or rows.shape[1] < 1:
            raise ValueError("batches must be (K, B)")
        if rows.size and (rows.min() < 0 or rows.max() >= self.n_images):
            raise IndexError("batch index out of range")
        K, B = rows.shape
        if getattr(self, "_seg_off_host", None) is None:  # segment counts per image: host copy, once
            self._seg_off_host = self.seg_off.cpu().numpy().astype(np.int64)
        so = self._seg_off_host
        flat = rows.reshape(-1)
        total = int((so[flat + 1] - so[flat]).sum())
        nbytes = int(lib.fsld_plan_bytes(self.M, self.n_mask, B, K, total))
        buf = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        bt = torch.from_numpy(flat.astype(np.int32)).to(self.dev)
        plan = BinPlan(buf, bt.view(K, B), K, B, total)
        if build:
            self.build_plan(plan)
        return plan

    def build_plan(self, plan: "BinPlan") -> None:
        """The device part of make_plan (count -> scan -> fill for all K batches, three launches)."""
        C.check(C.load().fsld_plan_build(self.M, self.n_mask, ctypes_ptr(self.recs), ctypes_ptr(plan.batches),
                                         plan.K, plan.B, ctypes_ptr(self.seg_off), ctypes_ptr(self.segs),
                                         plan.total_pairs, ctypes_ptr(plan.buf), plan.buf.numel(), _stream()),
                "fsld_plan_build")

    def loss_grad_planned(self, v, plan: "BinPlan", k: int, acc, zbits=None, fold=None, sq=None):
        """loss_grad (zbits None) or loss_grad_hutch of batch k of a plan; returns sq (device double)."""
        lib = C.load()
        v = self._vol(v)
        sq = torch.empty(1, dtype=torch.float64, device=self.dev) if sq is None else sq
        scr = self.scratch(plan.B)
        C.check(lib.fsld_loss_grad_planned(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                           ctypes_ptr(plan.buf), plan.B, int(k), ctypes_ptr(v), ctypes_ptr(self.x),
                                           ctypes_ptr(self.pc), ctypes_ptr(self.ptab), ctypes_ptr(zbits),
                                           ctypes_ptr(acc), ctypes_ptr(fold),
                                           ctypes_ptr(sq), ctypes_ptr(scr), scr.numel() * 8, _stream()),
                "fsld_loss_grad_planned")
        return sq

    def loss_grad_step_planned(self, v, plan: "BinPlan", k: int, scale: float, lam: float, grad,
                               sq=None, loss=None):
        """The whole loss+grad step of batch k of a plan (fsld_loss_grad_step_planned): grad is
        overwritten with scale * sum P^* conj(f) r + lam v; returns (loss, sq) device doubles."""
        lib = C.load()
        v = self._vol(v)
        sq = torch.empty(1, dtype=torch.float64, device=self.dev) if sq is None else sq
        loss = torch.empty(1, dtype=torch.float64, device=self.dev) if loss is None else loss
        scr = self.scratch(plan.B)
        nscr = self._norm_scratch()
        C.check(lib.fsld_loss_grad_step_planned(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                                ctypes_ptr(plan.buf), plan.B, int(k), ctypes_ptr(v),
                                                ctypes_ptr(self.x), ctypes_ptr(self.pc), ctypes_ptr(self.ptab),
                                                float(scale), float(lam),
                                                ctypes_ptr(grad), ctypes_ptr(sq), ctypes_ptr(loss), ctypes_ptr(scr),
                                                scr.numel() * 8, ctypes_ptr(nscr), nscr.numel() * 8, _stream()),
                "fsld_loss_grad_step_planned")
        return loss, sq

    HOST_SLABS = int(os.environ.get("FSLD_HOST_SLABS", "12"))  # z-slabs of the pipelined host step

    def loss_grad_host(self, v_host, idx_host, scale: float, lam: float, grad_host, out_host,
                       stage: dict, n_slabs: int | None = None) -> None:
        """(grad_host complex128: fsld_loss_grad_host_c128, the gradient cast on the device; ``stage``
        then also holds "g128", an M^3 complex128 device staging tensor)"""
        """fsld_loss_grad_host: pinned host v / idx in, pinned host grad and out_host = [sq, loss]
        written once the current stream is synchronised.  The copies run slab by slab on the
        library's own copy streams, overlapping each other and the brick passes.  ``stage``
        holds the device staging tensors "v", "g" (M^3 complex64) and "idx" (>= B int32)."""
        lib = C.load()
        if not self.brick_path:
            raise ValueError("the host step runs the brick path (tri, sorted, non-deterministic)")
        c128 = grad_host.dtype == torch.complex128
        for t, n in ((v_host, self.n_voxels), (grad_host, self.n_voxels)):
            if t.device.type != "cpu" or not t.is_pinned() or t.numel() != n or not t.is_contiguous() or \
                    t.dtype != (torch.complex128 if (t is grad_host and c128) else torch.complex64):
                raise ValueError("v_host / grad_host must be pinned contiguous host tensors of M^3 (v complex64, "
                                 "grad complex64 or complex128)")
        if idx_host.device.type != "cpu" or not idx_host.is_pinned() or idx_host.dtype != torch.int32:
            raise ValueError("idx_host must be a pinned int32 host tensor")
        B = int(idx_host.numel())
        if B == 0:
            raise ValueError("batch must be nonempty")
        if int(idx_host.min()) < 0 or int(idx_host.max()) >= self.n_images:
            raise ValueError("batch index out of range")
        scr = self.scratch(B)
        if stage["idx"].numel() < B:
            stage["idx"] = torch.empty(B, dtype=torch.int32, device=self.dev)
        if c128:
            if stage.get("g128") is None:
                stage["g128"] = torch.empty(self.n_voxels, dtype=torch.complex128, device=self.dev)
            C.check(lib.fsld_loss_grad_host_c128(
                self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs), ctypes_ptr(idx_host), B, ctypes_ptr(v_host),
                ctypes_ptr(self.x), ctypes_ptr(self.pc), ctypes_ptr(self.ptab), ctypes_ptr(self.seg_off),
                ctypes_ptr(self.segs), float(scale), float(lam), ctypes_ptr(grad_host), ctypes_ptr(out_host),
                ctypes_ptr(stage["v"]), ctypes_ptr(stage["g"]), ctypes_ptr(stage["g128"]), ctypes_ptr(stage["idx"]),
                int(n_slabs or self.HOST_SLABS), ctypes_ptr(scr), scr.numel() * 8, _stream()),
                "fsld_loss_grad_host_c128")
            return
        C.check(lib.fsld_loss_grad_host(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                        ctypes_ptr(idx_host), B, ctypes_ptr(v_host), ctypes_ptr(self.x),
                                        ctypes_ptr(self.pc), ctypes_ptr(self.ptab), ctypes_ptr(self.seg_off),
                                        ctypes_ptr(self.segs),
                                        float(scale), float(lam), ctypes_ptr(grad_host), ctypes_ptr(out_host),
                                        ctypes_ptr(stage["v"]), ctypes_ptr(stage["g"]), ctypes_ptr(stage["idx"]),
                                        int(n_slabs or self.HOST_SLABS), ctypes_ptr(scr), scr.numel() * 8,
                                        _stream()), "fsld_loss_grad_host")

    def loss_grad_host_np(self, v128: np.ndarray, idx_host, scale: float, lam: float, grad128: np.ndarray,
                          out_host, stage: dict, n_slabs: int | None = None) -> None:
        """fsld_loss_grad_host_np_ball: numpy complex128 v in, numpy complex128 gradient out (the
        reference's call shape); only the touched ball crosses PCIe (packed complex64, one copy per
        z-slab and direction), the host threads cast each finished slab back and write lam v off the
        ball.  Blocking; out_host (pinned float64[2]) = [sum|r|^2, loss]."""
        lib = C.load()
        if not self.brick_path:
            raise ValueError("the host step runs the brick path (tri, sorted, non-deterministic)")
        for a in (v128, grad128):
            if a.dtype != np.complex128 or a.size != self.n_voxels or not a.flags.c_contiguous or a.ctypes.data % 16:
                raise ValueError("v / grad must be contiguous 16-byte-aligned complex128 arrays of M^3")
        if idx_host.device.type != "cpu" or not idx_host.is_pinned() or idx_host.dtype != torch.int32:
            raise ValueError("idx_host must be a pinned int32 host tensor")
        B = int(idx_host.numel())
        if B == 0:
            raise ValueError("batch must be nonempty")
        if int(idx_host.min()) < 0 or int(idx_host.max()) >= self.n_images:
            raise ValueError("batch index out of range")
        scr = self.scratch(B)
        if stage["idx"].numel() < B:
            stage["idx"] = torch.empty(B, dtype=torch.int32, device=self.dev)
        C.check(lib.fsld_loss_grad_host_np_ball(
            self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs), ctypes_ptr(idx_host), B, v128.ctypes.data,
            ctypes_ptr(self.x), ctypes_ptr(self.pc), ctypes_ptr(self.ptab), ctypes_ptr(self.seg_off),
            ctypes_ptr(self.segs), float(scale), float(lam), grad128.ctypes.data, ctypes_ptr(out_host),
            ctypes_ptr(stage["v"]), ctypes_ptr(stage["g"]), ctypes_ptr(stage["idx"]),
            int(n_slabs or (self.NP_SLABS if self.HOST_BALL else self.HOST_SLABS)), ctypes_ptr(scr), scr.numel() * 8,
            _stream(), self.touch_radius if self.HOST_BALL else 0.0), "fsld_loss_grad_host_np_ball")

    HOST_BALL = os.environ.get("FSLD_HOST_BALL", "1") != "0"  # (A/B: whole-plane copies)
    NP_SLABS = int(os.environ.get("FSLD_NP_SLABS", "10"))  # z-slabs of the packed-ball numpy step (6: 1.00, 8: 0.92, 10: 0.90, 12: 0.95 ms)

    @property
    def touch_radius(self) -> float:
        """Radius of the ball a scatter can reach: a rotated pixel keeps |k| (the clamp only shortens it,
        kernels.py:42-60) and its trilinear footprint stays within sqrt(3) of it (grid.touched_ball)."""
        r = getattr(self, "_touch_radius", None)
        if r is None:
            k = self.pix.to(torch.float64)
            r = self._touch_radius = float(torch.sqrt((k * k).sum(dim=1).max())) + math.sqrt(3.0) + 1e-3
        return r

    def proj_energy_planned(self, d, plan: "BinPlan", k: int, out=None) -> torch.Tensor:
        lib = C.load()
        d = self._vol(d)
        out = torch.empty(1, dtype=torch.float64, device=self.dev) if out is None else out
        scr = self.scratch(plan.B)
        C.check(lib.fsld_proj_energy_planned(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                             ctypes_ptr(plan.buf), plan.B, int(k), ctypes_ptr(d), ctypes_ptr(self.pc),
                                             ctypes_ptr(out), ctypes_ptr(scr), scr.numel() * 8, _stream()),
                "fsld_proj_energy_planned")
        return out

    def loss(self, v, idx):
        """sum|P v - x|^2 over the batch, device double (optim.py:193-207 data term)."""
        lib = C.load()
        v = self._vol(v)
        idx = self.idx_tensor(idx)
        B = idx.numel()
        sq = torch.empty(1, dtype=torch.float64, device=self.dev)
        scr = self.scratch(B)
        if self.layout == "sorted" and self.table_path and self.mode == "tri":  # brick projection pass
            C.check(lib.fsld_loss_sorted_tab(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs), ctypes_ptr(idx),
                                             B, ctypes_ptr(v), ctypes_ptr(self.x), ctypes_ptr(self.pc),
                                             ctypes_ptr(self.ptab), ctypes_ptr(self.seg_off), ctypes_ptr(self.segs),
                                             ctypes_ptr(sq), ctypes_ptr(scr), scr.numel() * 8, _stream()),
                    "fsld_loss_sorted_tab")
            return sq
        if self.layout == "sorted":
            C.check(lib.fsld_loss_sorted(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs), ctypes_ptr(idx), B,
                                         ctypes_ptr(v), ctypes_ptr(self.x), ctypes_ptr(self.pc), ctypes_ptr(sq),
                                         ctypes_ptr(scr), scr.numel() * 8, _stream()), "fsld_loss_sorted")
            return sq
        C.check(lib.fsld_loss(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.pix), ctypes_ptr(self.recs),
                              ctypes_ptr(idx), B, ctypes_ptr(v), ctypes_ptr(self.x), ctypes_ptr(sq),
                              ctypes_ptr(scr), scr.numel() * 8, _stream()), "fsld_loss")
        return sq

    def project_sorted(self, v, idx, out=None) -> torch.Tensor:
        """Projections of dataset rows idx in their brick-sorted pixel order (dataset synthesis)."""
        lib = C.load()
        v = self._vol(v)
        idx = self.idx_tensor(idx)
        if out is None:
            out = torch.empty((idx.numel(), self.n_mask), dtype=torch.complex64, device=self.dev)
        C.check(lib.fsld_project_sorted(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs), ctypes_ptr(idx),
                                        idx.numel(), ctypes_ptr(v), ctypes_ptr(self.pc), ctypes_ptr(out), _stream()),
                "fsld_project_sorted")
        return out

    def backproject_dataset(self, idx, acc=None, fx=None):
        """acc += sum_b P^* conj(f) x[idx[b]] over dataset rows (b_vector, forward.py:572-579)."""
        if self.layout == "mask":
            return self.backproject(self.x[self.idx_tensor(idx).long()], idx, acc, fx)
        lib = C.load()
        idx = self.idx_tensor(idx)
        acc = self.new_cacc() if acc is None else acc
        if self.table_path and self.mode == "tri":
            # the brick kernel with v = 0: its accumulator collects sum P^* conj(f) (0 - x) = -b
            zero = getattr(self, "_zero_vol", None)
            if zero is None:
                zero = self._zero_vol = torch.zeros(self.n_voxels, dtype=torch.complex64, device=self.dev)
            neg = torch.zeros(self.n_voxels, dtype=torch.complex64, device=self.dev)
            self.loss_grad(zero, idx, acc=neg)
            acc.sub_(neg)
            return acc, fx
        if self.deterministic and fx is None:
            fx = self.fixed_scale(self.x, HITS_PER_IMAGE * idx.numel(), 0.0)
        C.check(lib.fsld_backproject_sorted(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                            ctypes_ptr(idx), idx.numel(), ctypes_ptr(self.x), ctypes_ptr(self.pc),
                                            ctypes_ptr(acc), self.flags, ctypes_ptr(fx), _stream()),
                "fsld_backproject_sorted")
        return acc, fx

    def project(self, v, idx) -> torch.Tensor:
        lib = C.load()
        v = self._vol(v)
        idx = self.idx_tensor(idx)
        out = torch.empty((idx.numel(), self.n_mask), dtype=torch.complex64, device=self.dev)
        C.check(lib.fsld_project(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.pix), ctypes_ptr(self.recs),
                                 ctypes_ptr(idx), idx.numel(), ctypes_ptr(v), ctypes_ptr(out), _stream()),
                "fsld_project")
        return out

    def backproject(self, imgs, idx, acc=None, fx=None, fx_batch=None):
        lib = C.load()
        idx = self.idx_tensor(idx)
        B = idx.numel()
        imgs = imgs.to(self.dev, torch.complex64).contiguous()
        if tuple(imgs.shape) != (B, self.n_mask):
            raise ValueError(f"images shape {tuple(imgs.shape)} != ({B}, {self.n_mask})")
        acc = self.new_cacc() if acc is None else acc
        if self.deterministic and fx is None:
            fx = self.fixed_scale(imgs, HITS_PER_IMAGE * (fx_batch or B), 0.0)
        C.check(lib.fsld_backproject(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.pix),
                                     ctypes_ptr(self.recs), ctypes_ptr(idx), B, ctypes_ptr(imgs),
                                     ctypes_ptr(acc), self.flags, ctypes_ptr(fx), _stream()),
                "fsld_backproject")
        return acc, fx

    HVP_CHUNK = 4096  # images per brick-path Hessian launch (bounds the binning scratch)

    def hvp_acc(self, z, idx, acc=None, fx=None, fx_batch=None):
        lib = C.load()
        z = self._vol(z)
        idx = self.idx_tensor(idx)
        B = idx.numel()
        acc = self.new_cacc() if acc is None else acc
        if (self.brick_path or self.table_path) and not self.deterministic:
            # brick-sorted layout: the loss+grad work-item kernel with zero images, in chunks
            sq = torch.empty(1, dtype=torch.float64, device=self.dev)
            for lo in range(0, B, self.HVP_CHUNK):
                sub = idx[lo:lo + self.HVP_CHUNK]
                nb = sub.numel()
                scr = self.scratch(nb)
                C.check(lib.fsld_hvp_sorted(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs), ctypes_ptr(sub),
                                            nb, ctypes_ptr(z), ctypes_ptr(self.pc), ctypes_ptr(self.ptab),
                                            ctypes_ptr(self.seg_off),
                                            ctypes_ptr(self.segs), ctypes_ptr(acc), ctypes_ptr(sq), 0,
                                            ctypes_ptr(scr), scr.numel() * 8, _stream()), "fsld_hvp_sorted")
            return acc, fx
        if self.deterministic and fx is None:
            fx = self.fixed_scale(z, HITS_PER_IMAGE * (fx_batch or B), 0.0)
        C.check(lib.fsld_hvp(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.pix), ctypes_ptr(self.recs),
                             ctypes_ptr(idx), B, ctypes_ptr(z), ctypes_ptr(acc), self.flags, ctypes_ptr(fx),
                             _stream()), "fsld_hvp")
        return acc, fx

    def pack_probes(self, z) -> tuple[torch.Tensor, int]:
        """(k, M^3) or (M^3,) +-1 float64 -> bit-packed (M^3, ceil(k/32)) uint32 words."""
        lib = C.load()
        if isinstance(z, torch.Tensor):
            zd = z.to(self.dev, torch.float64).contiguous()
        else:
            zd = torch.from_numpy(np.ascontiguousarray(z, dtype=np.float64)).to(self.dev)
        if zd.dim() == 1:
            zd = zd.reshape(1, -1)
        k = zd.shape[0]
        if zd.shape[1] != self.n_voxels:
            raise ValueError("probe length must be M^3")
        words = (k + 31) // 32
        zbits = torch.empty((self.n_voxels, words), dtype=torch.int32, device=self.dev)
        self._bad.zero_()
        C.check(lib.fsld_pack_probes(self.n_voxels, k, ctypes_ptr(zd), ctypes_ptr(zbits), ctypes_ptr(self._bad),
                                     _stream()), "fsld_pack_probes")
        return zbits, k

    def probes_are_rademacher(self) -> bool:
        """Host check of the last pack_probes call (synchronises)."""
        return int(self._bad.item()) == 0

    def gen_probes(self, k: int, seed: int) -> torch.Tensor:
        lib = C.load()
        words = (k + 31) // 32
        zbits = torch.empty((self.n_voxels, words), dtype=torch.int32, device=self.dev)
        C.check(lib.fsld_gen_probes(self.n_voxels, int(k), int(seed) & 0xFFFFFFFFFFFFFFFF, ctypes_ptr(zbits),
                                    _stream()), "fsld_gen_probes")
        return zbits

    def hutch_fold(self, zbits, k: int, idx, acc=None, fx=None, fx_batch=None):
        """acc[j] += sum_p z_p[j] (sum_b P_b^* C_b^2 P_b z_p)[j] (optim.py:210-229 numerator)."""
        lib = C.load()
        idx = self.idx_tensor(idx)
        B = idx.numel()
        acc = self.new_racc() if acc is None else acc
        if (self.layout == "sorted" and self.mode == "tri" and not self.deterministic and
                not (self.flags & C.TILE_PATH) and 1 <= k <= 256):
            scr = self.scratch(B)
            C.check(lib.fsld_hutch_fold_sorted(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                               ctypes_ptr(idx), B, ctypes_ptr(self.pc), ctypes_ptr(self.seg_off),
                                               ctypes_ptr(self.segs), ctypes_ptr(zbits), int(k), ctypes_ptr(acc),
                                               ctypes_ptr(scr), scr.numel() * 8, _stream()),
                    "fsld_hutch_fold_sorted")
            return acc, fx
        if self.deterministic and fx is None:
            fx = self.fixed_scale(None, HITS_PER_IMAGE * (fx_batch or B) * k, 1.0)
        C.check(lib.fsld_hutch_fold(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.pix),
                                    ctypes_ptr(self.recs), ctypes_ptr(idx), B, ctypes_ptr(zbits), int(k),
                                    ctypes_ptr(acc), self.flags, ctypes_ptr(fx), _stream()), "fsld_hutch_fold")
        return acc, fx

    def exact_diag_acc(self, idx, acc=None, fx=None, fx_batch=None):
        lib = C.load()
        idx = self.idx_tensor(idx)
        B = idx.numel()
        acc = self.new_racc() if acc is None else acc
        if self.deterministic and fx is None:
            fx = self.fixed_scale(None, HITS_PER_IMAGE * (fx_batch or B), 1.0)
        if (self.layout == "sorted" and self.ptab is not None and self.mode == "tri" and
                not (self.flags & C.TILE_PATH)):
            # the table-driven brick kernel's DIAG pass (deterministic: <= 1024 images per call)
            chunk = 1024 if self.deterministic else self.HVP_CHUNK
            for lo in range(0, B, chunk):
                sub = idx[lo:lo + chunk]
                nb = sub.numel()
                scr = self.scratch(nb)
                C.check(lib.fsld_exact_diag_sorted_tab(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                                       ctypes_ptr(sub), nb, ctypes_ptr(self.pc), ctypes_ptr(self.ptab),
                                                       ctypes_ptr(self.seg_off), ctypes_ptr(self.segs), ctypes_ptr(acc),
                                                       self.flags, ctypes_ptr(fx), ctypes_ptr(scr), scr.numel() * 8,
                                                       _stream()), "fsld_exact_diag_sorted_tab")
            return acc, fx
        C.check(lib.fsld_exact_diag(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.pix),
                                    ctypes_ptr(self.recs), ctypes_ptr(idx), B, ctypes_ptr(acc), self.flags,
                                    ctypes_ptr(fx), _stream()), "fsld_exact_diag")
        return acc, fx

    def assign_nn(self, idx) -> torch.Tensor:
        lib = C.load()
        idx = self.idx_tensor(idx)
        out = torch.empty((idx.numel(), self.n_mask), dtype=torch.int32, device=self.dev)
        C.check(lib.fsld_assign_nn(self.M, self.n_mask, ctypes_ptr(self.pix), ctypes_ptr(self.recs),
                                   ctypes_ptr(idx), idx.numel(), ctypes_ptr(out), _stream()), "fsld_assign_nn")
        return out

    def epilogue(self, acc, v, scale: float, lam: float, sq, grad=None, loss=None):
        """Fused grad = scale*acc + lam*v, acc <- 0, loss = scale/2 sq + lam/2 ||v||^2 (optim.py:186-189).

        Complex64 accumulators only (the deterministic int64 path uses finalize_c + norm2)."""
        lib = C.load()
        v = self._vol(v)
        grad = torch.empty(self.n_voxels, dtype=torch.complex64, device=self.dev) if grad is None else grad
        loss = torch.empty(1, dtype=torch.float64, device=self.dev) if loss is None else loss
        scr = self._norm_scratch()
        C.check(lib.fsld_grad_epilogue(self.n_voxels, ctypes_ptr(acc), ctypes_ptr(v), float(scale), float(lam),
                                       ctypes_ptr(grad), ctypes_ptr(sq), ctypes_ptr(loss), 0, ctypes_ptr(scr),
                                       scr.numel() * 8, _stream()), "fsld_grad_epilogue")
        return loss, grad

    def _norm_scratch(self) -> torch.Tensor:
        if getattr(self, "_nscr", None) is None:
            self._nscr = torch.empty(148 * 8, dtype=torch.float64, device=self.dev)
        return self._nscr

    # ---- epilogues --------------------------------------------------------
    def finalize_c(self, acc, fx, scale: float, lam: float, v=None, out=None) -> torch.Tensor:
        """scale * acc + lam * v -> complex64 (optim.py:189, forward.py:570)."""
        lib = C.load()
        out = torch.empty(self.n_voxels, dtype=torch.complex64, device=self.dev) if out is None else out
        vv = self._vol(v) if v is not None else None
        C.check(lib.fsld_grad_finalize(self.n_voxels, ctypes_ptr(acc), self.flags, ctypes_ptr(fx),
                                       ctypes_ptr(vv), float(scale), float(lam), ctypes_ptr(out), _stream()),
                "fsld_grad_finalize")
        return out

    def finalize_r(self, acc, fx, scale: float, add: float, out=None) -> torch.Tensor:
        lib = C.load()
        out = torch.empty(self.n_voxels, dtype=torch.float32, device=self.dev) if out is None else out
        C.check(lib.fsld_real_finalize(self.n_voxels, ctypes_ptr(acc), self.flags, ctypes_ptr(fx), float(scale),
                                       float(add), ctypes_ptr(out), _stream()), "fsld_real_finalize")
        return out

    def norm2(self, v) -> torch.Tensor:
        """||v||^2 (device double, fixed reduction order)."""
        lib = C.load()
        v = self._vol(v)
        out = torch.empty(1, dtype=torch.float64, device=self.dev)
        scr = self._norm_scratch()
        C.check(lib.fsld_norm2(self.n_voxels, ctypes_ptr(v), ctypes_ptr(out), ctypes_ptr(scr), scr.numel() * 8,
                               _stream()), "fsld_norm2")
        return out


    # ---- Algorithm-1 step (fsld_step.cu) ------------------------------------
    def _step_scratch(self) -> torch.Tensor:
        if getattr(self, "_sscr", None) is None:
            self._sscr = torch.empty(5 * 148 * 16, dtype=torch.float64, device=self.dev)
        return self._sscr

    def precond_step(self, acc, v, params, dir_out, fold=None, d_avg=None, d=None, dhat_fixed=None,
                     grad_out=None, dhat_out=None, out4=None) -> torch.Tensor:
        """One pass: grad, Hutchinson average, EMA, threshold, direction; returns the device
        doubles {decrease, ||v||^2, Re<v, dir>, ||dir||^2, Re<acc, dir>} (fsld_precond_step)."""
        lib = C.load()
        v = self._vol(v)
        out4 = torch.empty(5, dtype=torch.float64, device=self.dev) if out4 is None else out4
        scr = self._step_scratch()
        C.check(lib.fsld_precond_step(self.n_voxels, ctypes_ptr(acc), ctypes_ptr(v), ctypes_ptr(fold),
                                      ctypes_ptr(d_avg), ctypes_ptr(d), ctypes_ptr(dhat_fixed), ctypes.byref(params),
                                      ctypes_ptr(dir_out), ctypes_ptr(grad_out), ctypes_ptr(dhat_out),
                                      ctypes_ptr(out4), ctypes_ptr(scr), scr.numel() * 8, _stream()),
                "fsld_precond_step")
        return out4

    def armijo_terms(self, v, d, idx, out3=None) -> torch.Tensor:
        """{sum|r|^2, sum Re(conj(r) q), sum|q|^2}, r = f P v - x, q = f P d over the batch (device doubles)."""
        lib = C.load()
        v = self._vol(v)
        d = self._vol(d)
        idx = self.idx_tensor(idx)
        B = idx.numel()
        out3 = torch.empty(3, dtype=torch.float64, device=self.dev) if out3 is None else out3
        scr = self.scratch(B)
        pc = self.pc if self.layout == "sorted" else None
        C.check(lib.fsld_armijo_terms(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.pix), ctypes_ptr(pc),
                                      ctypes_ptr(self.recs), ctypes_ptr(idx), B, ctypes_ptr(v), ctypes_ptr(d),
                                      ctypes_ptr(self.x), ctypes_ptr(out3), ctypes_ptr(scr), scr.numel() * 8,
                                      _stream()), "fsld_armijo_terms")
        return out3

    def new_armijo_state(self, eta0: float) -> torch.Tensor:
        st = np.zeros(1, dtype=C.ARMIJO_DTYPE)
        st["eta"] = eta0
        return torch.from_numpy(st.view(np.uint8).copy()).to(self.dev)

    def proj_energy(self, d, idx, out=None, reuse_bins: bool = False) -> torch.Tensor:
        """||A d||^2 = sum_b sum_p C^2 |P d|^2 over the batch (device double): the brick-sorted
        gather-only kernel when available, else the tile kernel's third line-search term.
        reuse_bins: idx is the same (unchanged) device tensor the preceding sorted loss+grad call of
        this step used, so its work items are reused (FSLD_REUSE_BINS)."""
        lib = C.load()
        d = self._vol(d)
        idx = self.idx_tensor(idx)
        B = idx.numel()
        if self.layout == "sorted" and self.mode == "tri":
            out = torch.empty(1, dtype=torch.float64, device=self.dev) if out is None else out
            scr = self.scratch(B)
            C.check(lib.fsld_proj_energy_sorted(self.M, self.mode_id, self.n_mask, ctypes_ptr(self.recs),
                                                ctypes_ptr(idx), B, ctypes_ptr(d), ctypes_ptr(self.pc),
                                                ctypes_ptr(self.seg_off), ctypes_ptr(self.segs), ctypes_ptr(out),
                                                C.REUSE_BINS if reuse_bins else 0, ctypes_ptr(scr),
                                                scr.numel() * 8, _stream()), "fsld_proj_energy_sorted")
            return out
        zero = getattr(self, "_zero_vol", None)
        if zero is None:
            zero = self._zero_vol = torch.zeros(self.n_voxels, dtype=torch.complex64, device=self.dev)
        return self.armijo_terms(zero, d, idx)[2:3]

    def armijo_select(self, sq, rq, qq, vol, scale: float, lam: float, c: float, st, hist=None,
                      max_halvings: int = 60) -> None:
        lib = C.load()
        cap = 0 if hist is None else hist.numel() // 5
        C.check(lib.fsld_armijo_select(ctypes_ptr(sq), ctypes_ptr(rq), ctypes_ptr(qq), ctypes_ptr(vol), float(scale),
                                       float(lam), float(c), int(max_halvings), ctypes_ptr(st), ctypes_ptr(hist),
                                       cap, _stream()), "fsld_armijo_select")

    def apply_step(self, v, dir_, st) -> None:
        """v <- v - eta_applied * dir (in place; v must be this engine's complex64 volume)."""
        C.check(C.load().fsld_apply_step(self.n_voxels, ctypes_ptr(v), ctypes_ptr(dir_), ctypes_ptr(st), _stream()),
                "fsld_apply_step")


class BinPlan:
    """Device buffer of a multi-batch binning plan (fsld_plan_build) and its batches."""

    def __init__(self, buf: torch.Tensor, batches: torch.Tensor, K: int, B: int, total_pairs: int):
        self.buf, self.batches, self.K, self.B, self.total_pairs = buf, batches, K, B, total_pairs


def _rows_contiguous(pix: np.ndarray) -> bool:
    """True if every mask row is one run of consecutive kx in ascending index order (disk masks are)."""
    ky = pix[:, 1].astype(np.int64)
    kx = pix[:, 0].astype(np.int64)
    same = ky[1:] == ky[:-1]
    return bool(np.all(np.diff(ky) >= 0) and np.all(kx[1:][same] - kx[:-1][same] == 1))


def records_for(M: int, quats, shifts=None, ctfs=None) -> np.ndarray:
    """Build fsld_image_rec records on the host (one 128-byte record per image).

    quats (N,4) unit quaternions (w,x,y,z) -> rows 0-1 of quat_to_matrix
    (forward.py:42-51, same fp64 expression order so nn indices are
    bit-exact); shifts (N,2) pixels -> shift = -2 t / M (forward.py:299-303);
    ctfs: None, or a sequence of CtfParams-like (defocus, amp_contrast,
    b_factor) / PhysicalCtf objects (see forward.ctf_coefficients).
    """
    from .forward import ctf_coefficients

    quats = np.asarray(quats, dtype=np.float64).reshape(-1, 4)
    N = quats.shape[0]
    recs = np.zeros(N, dtype=C.REC_DTYPE)
    # rows 0-1 of quat_to_matrix, vectorised with the same per-element fp64 expressions (bit-identical)
    w, x, y, z = (quats[:, i] for i in range(4))
    recs["rot"] = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                            2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], axis=1)
    if shifts is not None:
        t = np.asarray(shifts, dtype=np.float64).reshape(N, 2)
        recs["shift"] = -2.0 * t / M
        recs["flags"] |= np.where(np.any(t != 0.0, axis=1), C.REC_SHIFT, 0).astype(np.uint32)
    if ctfs is not None:
        if len(ctfs) != N:
            raise ValueError("ctfs length must match poses")
        co = [ctf_coefficients(c, M) for c in ctfs]
        recs["gamma"] = np.array([t[0] for t in co], dtype=np.float64).reshape(N, 4)
        recs["env"] = np.array([t[1] for t in co], dtype=np.float64)
        recs["wsin"] = np.array([t[2] for t in co], dtype=np.float32)
        recs["wcos"] = np.array([t[3] for t in co], dtype=np.float32)
        recs["flags"] |= np.uint32(C.REC_CTF)
    return recs
