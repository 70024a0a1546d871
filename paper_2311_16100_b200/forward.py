"""Image-formation model on the B200 path: the drop-in for fsld.forward.

Mirrors the reference's public surface (/root/reference/pkg/src/fsld/forward.py):
``Pose``, ``CtfParams``, ``FourierVolume``, ``ImageStack``, ``quat_to_matrix``,
``sample_uniform_poses``, ``ctf_eval``, ``Projector``, ``DatasetOperator``,
``project``, ``backproject`` -- same names, argument meaning and ValueError
behaviour -- but every projection / adjoint runs in the sm_100a kernels of
libfsld_b200.so (engine.SliceEngine).  Per-image phase and CTF tables are not
materialised: each image is one 128-byte record and the kernels evaluate
phase and CTF per pixel.  ``PhysicalCtf`` adds the astigmatic microscope CTF
the BASELINE configs use (not in the reference).

Inputs may be numpy (returned as numpy complex128, as the reference does) or
torch CUDA tensors (returned as torch complex64 on the device, no host sync).
Objects from the reference package itself (its Pose / CtfParams /
ImageStack) are accepted too: only their attributes are read.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .engine import SliceEngine, records_for
from .grid import GridSpec, disk_mask

MODES = ("nn", "tri")
PASS_CHUNK = 1024  # forward.py:39 (kept for API parity; the GPU path needs no chunking)

__all__ = [
    "MODES", "Pose", "CtfParams", "PhysicalCtf", "FourierVolume", "ImageStack", "quat_to_matrix",
    "sample_uniform_poses", "sample_preferred_poses", "ctf_eval", "ctf_coefficients", "Projector", "DatasetOperator",
    "project", "backproject", "synthesize_dataset", "gaussian_blob_phantom",
]


def quat_to_matrix(q) -> np.ndarray:
    """Rotation matrix of a unit quaternion (w, x, y, z) (forward.py:42-51).

    Evaluated in fp64 with the reference's expression order, so the rotation
    rows shipped to the GPU are bit-identical and nn voxel indices match.
    """
    w, x, y, z = (float(t) for t in np.asarray(q, dtype=np.float64).reshape(4))
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


@dataclass(frozen=True, eq=False)
class Pose:
    """Rotation (unit quaternion w,x,y,z) plus in-plane shift in pixels (forward.py:54-75)."""

    q: np.ndarray
    t: np.ndarray

    def __post_init__(self):
        q = np.asarray(self.q, dtype=np.float64).reshape(4)
        t = np.asarray(self.t, dtype=np.float64).reshape(2)
        if abs(np.linalg.norm(q) - 1.0) > 1e-12:
            raise ValueError("quaternion must have unit norm (within 1e-12)")
        object.__setattr__(self, "q", q)
        object.__setattr__(self, "t", t)

    def rotation_matrix(self) -> np.ndarray:
        return quat_to_matrix(self.q)


@dataclass(frozen=True)
class CtfParams:
    """The reference's radial toy CTF (forward.py:78-90)."""

    defocus: float
    amp_contrast: float
    b_factor: float

    def __post_init__(self):
        if not 0.0 < self.amp_contrast < 1.0:
            raise ValueError("amp_contrast must lie in (0, 1)")
        if self.b_factor < 0.0:
            raise ValueError("b_factor must be non-negative")


@dataclass(frozen=True)
class PhysicalCtf:
    """Astigmatic microscope CTF (BASELINE configs 2-5; builder-defined, not in the reference).

    gamma(k) = pi lam df(t) |k|^2 - (pi/2) Cs lam^3 |k|^4,
    df(t) = defocus + astig/2 cos 2(t - astig_angle), k = (kx, ky)/(M apix) [1/A],
    C = -(sqrt(1 - A^2) sin gamma + A cos gamma).
    """

    defocus: float          # Angstrom
    astig: float = 0.0      # Angstrom
    astig_angle: float = 0.0  # radians
    voltage_kv: float = 300.0
    cs_mm: float = 2.7
    amp_contrast: float = 0.1
    apix: float = 1.0

    def __post_init__(self):
        if not 0.0 <= self.amp_contrast < 1.0:
            raise ValueError("amp_contrast must lie in [0, 1)")
        if self.apix <= 0 or self.voltage_kv <= 0:
            raise ValueError("apix and voltage must be positive")


def electron_wavelength_A(kv: float) -> float:
    v = kv * 1e3
    return 12.2642598 / np.sqrt(v * (1.0 + 0.978466e-6 * v))


def ctf_coefficients(c, M: int):
    """(gamma[4], env, wsin, wcos) of the in-kernel CTF model for one image.

    Reference radial CTF (forward.py:93-111): u = r / (M//2), arg = pi d u^2,
    C = -[(1-w) sin(arg) + w cos(arg)] exp(-b u^2)  ->  gamma = (pi d/r_max^2, 0, 0, 0).
    """
    if isinstance(c, PhysicalCtf) or hasattr(c, "astig"):
        lam = electron_wavelength_A(c.voltage_kv)
        s2 = (1.0 / (M * c.apix)) ** 2
        a = np.pi * lam * 0.5 * c.astig
        g = (np.pi * lam * c.defocus * s2, a * np.cos(2 * c.astig_angle) * s2,
             a * np.sin(2 * c.astig_angle) * s2, -(0.5 * np.pi * c.cs_mm * 1e7 * lam ** 3) * s2 * s2)
        return g, 0.0, float(np.sqrt(1.0 - c.amp_contrast ** 2)), float(c.amp_contrast)
    r_max = M // 2
    return ((np.pi * float(c.defocus) / r_max ** 2, 0.0, 0.0, 0.0), float(c.b_factor) / r_max ** 2,
            1.0 - float(c.amp_contrast), float(c.amp_contrast))


def ctf_eval(params, r, r_max: int):
    """Reference radial CTF at radius r (forward.py:93-111); host-side utility."""
    r = np.asarray(r, dtype=np.float64)
    if np.any(r < 0) or np.any(r > r_max):
        raise ValueError(f"radius out of range [0, {r_max}]")
    u2 = (r / r_max) ** 2
    w = params.amp_contrast
    arg = np.pi * params.defocus * u2
    out = -((1.0 - w) * np.sin(arg) + w * np.cos(arg)) * np.exp(-params.b_factor * u2)
    return out if out.ndim else float(out)


@dataclass
class FourierVolume:
    """Complex volume vector on the grid layout (forward.py:114-136)."""

    values: np.ndarray
    spec: GridSpec

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.complex128).reshape(-1)
        if v.size != self.spec.n_voxels:
            raise ValueError(f"volume has {v.size} entries, expected {self.spec.n_voxels}")
        if not np.all(np.isfinite(v.view(np.float64))):
            raise ValueError("volume contains non-finite entries")
        self.values = v

    @classmethod
    def zeros(cls, spec):
        return cls(np.zeros(spec.n_voxels, dtype=np.complex128), spec)

    def copy(self):
        return FourierVolume(self.values.copy(), self.spec)


@dataclass
class ImageStack:
    """Images (N, M^2) complex, zero off the disk mask, with poses / CTFs (forward.py:139-173)."""

    spec: GridSpec
    images: np.ndarray
    poses: list
    ctfs: list | None
    sigma: float
    seed: int
    mask_radius: int
    mode: str

    def __post_init__(self):
        self.images = np.ascontiguousarray(self.images, dtype=np.complex128)
        n = len(self.poses)
        if n < 1:
            raise ValueError("stack needs at least one image")
        if self.images.shape != (n, self.spec.n_pixels):
            raise ValueError(f"images shape {self.images.shape} does not match (N={n}, M^2={self.spec.n_pixels})")
        if self.ctfs is not None and len(self.ctfs) != n:
            raise ValueError("ctfs length must match poses")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")

    @property
    def n_images(self) -> int:
        return len(self.poses)


def sample_uniform_poses(n: int, shift_bound: float, seed: int) -> list:
    """Haar-uniform rotations (normalised Gaussian quaternions) + uniform shifts (forward.py:176-193)."""
    if n < 1:
        raise ValueError("need n >= 1 poses")
    if shift_bound < 0:
        raise ValueError("shift_bound must be non-negative")
    rng = np.random.default_rng(seed)
    qs = rng.standard_normal((n, 4))
    qs /= np.linalg.norm(qs, axis=1, keepdims=True)
    ts = rng.uniform(-shift_bound, shift_bound, size=(n, 2)) if shift_bound > 0 else np.zeros((n, 2))
    return [Pose(q=qs[i], t=ts[i]) for i in range(n)]


def _qmul(a, b) -> np.ndarray:
    """Hamilton product of (w, x, y, z) quaternions."""
    return np.array([a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
                     a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
                     a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
                     a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]])


def sample_preferred_poses(n: int, shift_bound: float, seed: int, concentration: float) -> list:
    """Poses whose slice normals cluster around +z (forward.py:209-258): direction
    normalize(concentration z + N(0, I)), uniform in-plane spin, uniform shifts; concentration 0
    is the uniform sampler.  The pose quaternion maps z to the direction under R^T."""
    if concentration == 0:
        return sample_uniform_poses(n, shift_bound, seed)
    if n < 1:
        raise ValueError("need n >= 1 poses")
    if shift_bound < 0 or concentration < 0:
        raise ValueError("shift_bound and concentration must be non-negative")
    rng = np.random.default_rng(seed)
    dirs = rng.standard_normal((n, 3))
    dirs[:, 2] += concentration
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    psis = rng.uniform(0.0, 2.0 * np.pi, n)
    ts = rng.uniform(-shift_bound, shift_bound, size=(n, 2)) if shift_bound > 0 else np.zeros((n, 2))
    out = []
    for d, psi, t in zip(dirs, psis, ts):
        cz = float(d[2])
        if cz > 1.0 - 1e-12:
            qa = np.array([1.0, 0.0, 0.0, 0.0])
        elif cz < -1.0 + 1e-12:
            qa = np.array([0.0, 1.0, 0.0, 0.0])
        else:  # rotation about z x d by the angle between them
            ax = np.array([-d[1], d[0], 0.0])
            ax /= np.linalg.norm(ax)
            h = 0.5 * np.arccos(cz)
            qa = np.concatenate([[np.cos(h)], np.sin(h) * ax])
        q = _qmul(qa, np.array([np.cos(0.5 * psi), 0.0, 0.0, np.sin(0.5 * psi)]))
        q[1:] = -q[1:]
        out.append(Pose(q=q / np.linalg.norm(q), t=t))
    return out


# ---------------------------------------------------------------------------
# numpy <-> device helpers
# ---------------------------------------------------------------------------

def _is_dev(a) -> bool:
    return isinstance(a, torch.Tensor) and a.is_cuda


def _to_dev_c64(a, dev) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(dev, torch.complex64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex64)).to(dev)


def _to_host_c128(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.complex128)


def _mode_of(stack_mode, mode):
    m = mode or stack_mode
    if m not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    return m


class DatasetOperator:
    """Forward model bound to one stack, resident on the GPU (forward.py:509-579).

    ``project`` / ``backproject`` / ``hvp`` / ``b_vector`` keep the reference
    signatures.  ``deterministic=True`` switches every scatter to int64
    fixed-point accumulation (bitwise repeatable for any launch order and any
    number of GPUs).
    """

    def __init__(self, stack, mode: str | None = None, deterministic: bool = False):
        self.stack = stack
        self.spec = stack.spec
        self.mode = _mode_of(stack.mode, mode)
        self.mask = disk_mask(self.spec, stack.mask_radius)
        quats = np.array([p.q for p in stack.poses], dtype=np.float64)
        shifts = np.array([p.t for p in stack.poses], dtype=np.float64)
        recs = records_for(self.spec.M, quats, shifts, stack.ctfs)
        images = np.asarray(stack.images)
        x = images[:, self.mask] if images.shape[1] == self.spec.n_pixels else images
        self.engine = SliceEngine(self.spec.M, self.mode, self.mask, recs, x, deterministic=deterministic)
        self._quats = quats

    @classmethod
    def from_engine(cls, engine: SliceEngine, spec=None):
        """Wrap an already device-resident dataset (e.g. generated on the GPU)."""
        op = cls.__new__(cls)
        op.stack = None
        op.spec = spec or GridSpec(engine.M)
        op.mode = engine.mode
        op.mask = engine.mask
        op.engine = engine
        op._quats = None
        return op

    @property
    def n_images(self) -> int:
        return self.engine.n_images

    @property
    def n_mask(self) -> int:
        return self.engine.n_mask

    @property
    def deterministic(self) -> bool:
        return self.engine.deterministic

    @property
    def x(self) -> np.ndarray:
        """Masked observed images (N, n_mask), host copy (forward.py:527)."""
        return _to_host_c128(self.engine.x_masked())

    @property
    def rots(self) -> np.ndarray:
        """(N, 3, 3) rotations (forward.py:524); rows 0-1 from the records for engine-built operators."""
        if self._quats is not None:
            return np.ascontiguousarray([quat_to_matrix(q) for q in self._quats])
        r = self._host_records()["rot"].reshape(-1, 2, 3)
        return np.ascontiguousarray(np.concatenate([r, np.cross(r[:, 0], r[:, 1])[:, None, :]], axis=1))

    # -- the reference's per-(image, pixel) tables (forward.py:523-526) -----------------------
    # Here phase and CTF live in the 128-byte per-image records (and, on the brick path, in the
    # dataset's per-pixel f tables); these host views are built on first access (10 GB of
    # complex128 at cfg3, like the reference's own tables) and are read-only: the kernels never
    # read them, so an assigned table could not take effect and is refused.
    @property
    def projector(self) -> "Projector":
        if getattr(self, "_projector", None) is None:
            self._projector = Projector(self.spec, self.mask, self.mode)
        return self._projector

    def _host_records(self) -> np.ndarray:
        from . import _capi as C
        return self.engine.recs.cpu().numpy().view(C.REC_DTYPE).reshape(-1)

    @property
    def phases(self) -> np.ndarray:
        """(N, n_mask) complex128 shift phases exp(-2 pi i k.t / M) (forward.py:299-303, 525)."""
        if getattr(self, "_phases", None) is None:
            if self.stack is not None and getattr(self.stack, "poses", None) is not None:
                self._phases = self.projector.phase_batch(self.stack.poses)
            else:  # records: phase = exp(i pi (shift0 kx + shift1 ky)), shift = -2 t / M
                sh = self._host_records()["shift"]
                self._phases = np.exp(1j * np.pi * (sh @ self.projector.pix.T))
        return self._phases

    @phases.setter
    def phases(self, table):
        self._refuse("phases", table, self.phases)

    @property
    def ctf_vals(self) -> np.ndarray:
        """(N, n_mask) float64 CTF values at the unrotated pixels (forward.py:305-312, 526)."""
        if getattr(self, "_ctf_vals", None) is None:
            if self.stack is not None and getattr(self.stack, "poses", None) is not None:
                self._ctf_vals = self.projector.ctf_batch(self.stack.ctfs, self.n_images)
            else:  # records: C = -(wsin sin g + wcos cos g) exp(-env k^2) where the CTF flag is set
                from . import _capi as C
                r = self._host_records()
                kx, ky = self.projector.pix[:, 0], self.projector.pix[:, 1]
                k2 = kx * kx + ky * ky
                g = r["gamma"]
                gam = (g[:, 0:1] * k2 + g[:, 1:2] * (kx * kx - ky * ky) + g[:, 2:3] * (2 * kx * ky)
                       + g[:, 3:4] * k2 * k2)
                c = -(r["wsin"][:, None].astype(np.float64) * np.sin(gam)
                      + r["wcos"][:, None].astype(np.float64) * np.cos(gam)) * np.exp(-r["env"][:, None] * k2)
                self._ctf_vals = np.where((r["flags"] & C.REC_CTF)[:, None] != 0, c, 1.0)
        return self._ctf_vals

    @ctf_vals.setter
    def ctf_vals(self, table):
        self._refuse("ctf_vals", table, self.ctf_vals)

    def _refuse(self, name, table, current):
        t = np.asarray(table)
        if t.shape == current.shape and np.allclose(t, current, rtol=1e-12, atol=1e-12):
            return  # (the same values: nothing to change)
        raise ValueError(f"DatasetOperator.{name} is derived from the stack's poses / CTF models and evaluated "
                         "inside the kernels; an arbitrary table cannot be injected (build the ImageStack with "
                         "the CTF models, e.g. PhysicalCtf, instead)")

    def all_indices(self) -> np.ndarray:
        return np.arange(self.n_images)

    # -- core operations ------------------------------------------------------
    def project(self, values, idx):
        """Projections onto the images in ``idx``: (len(idx), n_mask) (forward.py:540-545)."""
        out = self.engine.project(_to_dev_c64(values, self.engine.dev), idx)
        return out if _is_dev(values) else _to_host_c128(out)

    def backproject(self, imgs, idx):
        """Sum of per-image adjoints over ``idx``: a volume vector (forward.py:547-552)."""
        e = self.engine
        acc, fx = e.backproject(_to_dev_c64(imgs, e.dev), idx)
        out = e.finalize_c(acc, fx, 1.0, 0.0)
        return out if _is_dev(imgs) else _to_host_c128(out)

    def hvp(self, z, idx, lam: float, n_total: int | None = None):
        """(n_total/|idx|) sum_i P_i^* C_i^2 P_i z + lam z (forward.py:554-570)."""
        e = self.engine
        if not _is_dev(idx) and np.asarray(idx).size == 0:
            raise ValueError("batch must be nonempty")
        n_total = self.n_images if n_total is None else n_total
        zd = _to_dev_c64(z, e.dev)
        idx_t = e.idx_tensor(idx)
        acc, fx = e.hvp_acc(zd, idx_t)
        out = e.finalize_c(acc, fx, n_total / idx_t.numel(), lam, zd)
        return out if _is_dev(z) else _to_host_c128(out)

    def loss_and_grad_host(self, v_host, idx_host, lam: float, grad_host, n_total: int | None = None) -> float:
        """Host-buffer loss_and_grad: pinned complex64 v (M^3) and int32 idx in, grad written to the
        pinned complex64 ``grad_host``; returns the loss.  All copies are async; one synchronisation
        at the end (for the loss value).  On the brick path the volume moves in z-slabs through
        fsld_loss_grad_host (copies overlapped with each other and with the kernels)."""
        e = self.engine
        st = getattr(self, "_host_stage", None)
        if st is None:
            st = self._host_stage = {
                "v": torch.empty(e.n_voxels, dtype=torch.complex64, device=e.dev),
                "g": torch.empty(e.n_voxels, dtype=torch.complex64, device=e.dev),
                "acc": e.new_cacc(),
                "out": torch.empty(2, dtype=torch.float64, device=e.dev),
                "out_h": torch.empty(2, dtype=torch.float64).pin_memory(),
            }
        B = int(idx_host.numel())
        if B == 0:
            raise ValueError("batch must be nonempty")
        n_total = self.n_images if n_total is None else n_total
        scale = n_total / B
        if e.brick_path:  # slab-pipelined: copies in both directions overlap the brick passes
            st.setdefault("idx", torch.empty(B, dtype=torch.int32, device=e.dev))
            e.loss_grad_host(v_host, idx_host, scale, lam, grad_host, st["out_h"], st)
            torch.cuda.current_stream().synchronize()
            return float(st["out_h"][1])
        st["v"].copy_(v_host, non_blocking=True)
        idx = idx_host.to(e.dev, non_blocking=True)
        if e.deterministic:
            st["acc"].zero_()
            sq, acc, fx = e.loss_grad(st["v"], idx, st["acc"])
            e.finalize_c(acc, fx, scale, lam, st["v"], out=st["g"])
            st["out"][0:1].copy_(0.5 * scale * sq + 0.5 * lam * e.norm2(st["v"]))
        else:  # accumulator stays zero between calls: the fused epilogue clears it
            sq, acc, fx = e.loss_grad(st["v"], idx, st["acc"])
            e.epilogue(acc, st["v"], scale, lam, sq, grad=st["g"], loss=st["out"][0:1])
        grad_host.copy_(st["g"], non_blocking=True)
        st["out_h"].copy_(st["out"], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return float(st["out_h"][0])

    def loss_and_grad_numpy(self, v, batch, lam: float, n_total: int | None = None):
        """optim.loss_and_grad with the reference's argument types (numpy complex128 v in, (float,
        complex128 gradient) out; optim.py:165-190) on the brick path, through
        fsld_loss_grad_host_np_ball: only the voxels a scatter can reach (grid.touched_ball) cross
        PCIe, cast to complex64 and packed row by row by the library's host threads, one contiguous
        copy per z-slab in each direction overlapping the brick passes; every finished gradient slab
        is cast back to complex128 into the returned array (a recycled page-locked buffer) while later
        slabs are in flight, and off the ball the host threads write grad = lam v and sum ||v||^2 in
        fp64.  Accuracy: the fp32 path on the ball (1e-7 relative), fp64 off it."""
        from .hostio import PinnedArrays

        e = self.engine
        n = e.n_voxels
        st = getattr(self, "_np_stage", None)
        if st is None:
            st = self._np_stage = {"idx": torch.empty(0, dtype=torch.int32), "out": PinnedArrays(n, torch.complex128),
                                   "out_h": torch.empty(2, dtype=torch.float64).pin_memory()}
        b = np.asarray(batch).reshape(-1)
        if b.size == 0:
            raise ValueError("batch must be nonempty")
        if st["idx"].numel() != b.size:
            st["idx"] = torch.empty(b.size, dtype=torch.int32).pin_memory()
        st["idx"].numpy()[:] = b
        vin = np.ascontiguousarray(v, dtype=np.complex128).reshape(-1)
        if vin.size != n:
            raise ValueError(f"volume has {vin.size} entries, expected {n}")
        if vin.ctypes.data % 16:
            vin = vin.copy()
        hs = getattr(self, "_host_stage", None)
        if hs is None:
            hs = self._host_stage = {"v": torch.empty(n, dtype=torch.complex64, device=e.dev),
                                     "g": torch.empty(n, dtype=torch.complex64, device=e.dev),
                                     "acc": e.new_cacc(), "out": torch.empty(2, dtype=torch.float64, device=e.dev),
                                     "out_h": torch.empty(2, dtype=torch.float64).pin_memory()}
        hs.setdefault("idx", torch.empty(b.size, dtype=torch.int32, device=e.dev))
        out = st["out"].get()
        grad = out[0] if out is not None else np.empty(n, dtype=np.complex128)  # (many results held)
        n_total = self.n_images if n_total is None else n_total
        e.loss_grad_host_np(vin, st["idx"], n_total / b.size, lam, grad, st["out_h"], hs)
        return float(st["out_h"][1]), grad

    def b_vector(self):
        """sum_i P_i^* C_i x_i over all images (forward.py:572-579)."""
        e = self.engine
        acc, fx = e.backproject_dataset(e.all_indices())
        return _to_host_c128(e.finalize_c(acc, fx, 1.0, 0.0))


# ---------------------------------------------------------------------------
# Projector (per-batch, table-driven; forward.py:276-349) and single-image API
# ---------------------------------------------------------------------------

class Projector:
    """Batched slice projector for a fixed grid, mask and mode (forward.py:276-349).

    The ``*_batch`` methods take the reference's per-(image, pixel) tables
    and run the table-driven kernels; ``rot_batch`` / ``phase_batch`` /
    ``ctf_batch`` build those tables on the host like the reference.
    """

    def __init__(self, spec, mask, mode: str):
        if mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        self.spec = spec
        self.mode = mode
        mask = np.asarray(mask, dtype=np.int64).reshape(-1)
        if mask.size == 0:
            raise ValueError("mask must not be empty")
        if np.any(np.diff(mask) <= 0):
            raise ValueError("mask must be strictly ascending pixel indices")
        if not np.isin(mask, disk_mask(spec, spec.max_mask_radius)).all():
            raise ValueError(f"mask contains pixels outside the rotation-safe disk (radius {spec.max_mask_radius})")
        self.mask = mask
        from .grid import pixel_coords
        self.pix = np.ascontiguousarray(pixel_coords(spec.M)[mask], dtype=np.float64)
        self.pix_radii = np.sqrt((self.pix ** 2).sum(axis=1))
        self._engine = None

    @property
    def n_mask(self) -> int:
        return self.mask.size

    def rot_batch(self, poses) -> np.ndarray:
        return np.ascontiguousarray([quat_to_matrix(p.q) for p in poses])

    def phase_batch(self, poses) -> np.ndarray:
        ts = np.array([p.t for p in poses], dtype=np.float64)
        return np.exp(1j * ((-2.0 * np.pi / self.spec.M) * (ts @ self.pix.T)))

    def ctf_batch(self, ctfs, n: int) -> np.ndarray:
        if ctfs is None:
            return np.ones((n, self.n_mask))
        from . import kernels as K
        return np.ascontiguousarray([K.ctf_table_row(c, self.pix, self.spec.M) for c in ctfs])

    def project_batch(self, values, rots, phases, ctf_vals) -> np.ndarray:
        from . import kernels as K
        out = np.empty((rots.shape[0], self.n_mask), dtype=np.complex128)
        (K.project_tri if self.mode == "tri" else K.project_nn)(values, rots, self.pix, phases, ctf_vals,
                                                                 self.spec.M, out)
        return out

    def backproject_batch(self, imgs, rots, phases, ctf_vals) -> np.ndarray:
        from . import kernels as K
        vols = np.zeros((1, self.spec.n_voxels), dtype=np.complex128)
        (K.backproject_tri if self.mode == "tri" else K.backproject_nn)(imgs, rots, self.pix, phases, ctf_vals,
                                                                         self.spec.M, vols)
        return vols[0]

    def assign_nn(self, rots) -> np.ndarray:
        from . import kernels as K
        return K.assign_nn(rots, self.pix, self.spec.M)

    def scatter_sq(self, rots, weights) -> np.ndarray:
        from . import kernels as K
        return K.scatter_sq(self.mode, weights, rots, self.pix, self.spec.M)


def _single_stack(spec, mask, mode, pose, ctf):
    recs = records_for(spec.M, [pose.q], [pose.t], [ctf] if ctf is not None else None)
    return SliceEngine(spec.M, mode, mask, recs)


def project(v, pose, ctf=None, mode: str = "tri", mask=None) -> np.ndarray:
    """Project one volume to one image; zeros outside the mask (forward.py:367-381)."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    if mask is None:
        mask = disk_mask(v.spec, v.spec.max_mask_radius)
    e = _single_stack(v.spec, mask, mode, pose, ctf)
    img = np.zeros(v.spec.n_pixels, dtype=np.complex128)
    img[np.asarray(mask)] = _to_host_c128(e.project(_to_dev_c64(v.values, e.dev), [0]))[0]
    return img


def backproject(img, pose, ctf=None, mode: str = "tri", mask=None, spec=None):
    """Adjoint of project for one image (forward.py:384-408)."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    img = np.asarray(img, dtype=np.complex128).reshape(-1)
    if spec is None:
        m = round(np.sqrt(img.size))
        if m * m != img.size:
            raise ValueError("image length is not a perfect square")
        spec = GridSpec(m)
    if mask is None:
        mask = disk_mask(spec, spec.max_mask_radius)
    e = _single_stack(spec, mask, mode, pose, ctf)
    acc, fx = e.backproject(_to_dev_c64(img[np.asarray(mask)][None, :], e.dev), [0])
    return FourierVolume(_to_host_c128(e.finalize_c(acc, fx, 1.0, 0.0)), spec)


# ---------------------------------------------------------------------------
# synthetic data (forward.py:411-506)
# ---------------------------------------------------------------------------

def _noise_for_image(seed: int, index: int, n: int, sigma: float) -> np.ndarray:
    """The reference's per-image noise stream (forward.py:411-424): SeedSequence(seed, (100, i)),
    complex Gaussian with sigma / sqrt(2) per part, independent of generation order."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(100, index)))
    re_im = rng.standard_normal((2, n))
    return (sigma / np.sqrt(2.0)) * (re_im[0] + 1j * re_im[1])


def synthesize_dataset(v, poses, ctfs, sigma: float, mode: str = "tri", mask_radius: int | None = None,
                       seed: int = 0, chunk: int = 4096) -> ImageStack:
    """Noisy projections of v for the given poses / CTFs (forward.py:427-470).

    The clean projections run on the GPU (the product slice kernel, mask order); the noise is the
    reference's per-image stream, so a dataset differs from the reference's only by the fp32
    projection (relative ~1e-7)."""
    if sigma < 0:
        raise ValueError("sigma must be non-negative")
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    spec = v.spec
    if mask_radius is None:
        mask_radius = spec.max_mask_radius
    mask = disk_mask(spec, mask_radius)
    n_img = len(poses)
    if ctfs is not None and len(ctfs) != n_img:
        raise ValueError("ctfs length must match poses")
    quats = np.array([p.q for p in poses], dtype=np.float64)
    shifts = np.array([p.t for p in poses], dtype=np.float64)
    eng = SliceEngine(spec.M, mode, mask, records_for(spec.M, quats, shifts, ctfs), None, layout="mask")
    vd = _to_dev_c64(v.values, eng.dev)
    images = np.zeros((n_img, spec.n_pixels), dtype=np.complex128)
    for lo in range(0, n_img, chunk):
        hi = min(lo + chunk, n_img)
        clean = _to_host_c128(eng.project(vd, np.arange(lo, hi)))
        if sigma > 0:
            for b in range(hi - lo):
                clean[b] += _noise_for_image(seed, lo + b, mask.size, sigma)
        images[lo:hi, mask] = clean
    return ImageStack(spec=spec, images=images, poses=list(poses), ctfs=list(ctfs) if ctfs is not None else None,
                      sigma=float(sigma), seed=int(seed), mask_radius=int(mask_radius), mode=mode)


def gaussian_blob_phantom(spec, n_blobs: int = 8, seed: int = 0, widths=(0.35, 1.2)) -> FourierVolume:
    """Anisotropic Gaussian blobs written analytically in the Fourier domain (forward.py:473-506):
    a exp(-2 pi^2 k^T S k / M^2) exp(-2 pi i k.mu / M) per blob, S = R diag(sig^2) R^T with a Haar
    rotation, sig ~ U[widths], mu ~ U[-M/6, M/6]^3, a ~ U[0.5, 1.5] (one seeded stream)."""
    rng = np.random.default_rng(seed)
    M = spec.M
    k = spec.voxel_coords().astype(np.float64)
    out = np.zeros(spec.n_voxels, dtype=np.complex128)
    for _ in range(n_blobs):
        q = rng.standard_normal(4)
        q /= np.linalg.norm(q)
        R = quat_to_matrix(q)
        sig = rng.uniform(widths[0], widths[1], size=3)
        S = (R * sig ** 2) @ R.T
        mu = rng.uniform(-M / 6.0, M / 6.0, size=3)
        amp = rng.uniform(0.5, 1.5)
        quad = np.einsum("vi,ij,vj->v", k, S, k)
        out += amp * np.exp(-2.0 * np.pi ** 2 * quad / M ** 2) * np.exp(-2j * np.pi * (k @ mu) / M)
    return FourierVolume(out, spec)
