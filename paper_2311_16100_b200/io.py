"""FSD1 / FSV1 containers (io.py of the reference) and a streaming loader into HBM.

Format (io.py:1-12 of the reference): 4 magic bytes, little-endian uint32 header length, UTF-8 JSON
header, then little-endian complex128 samples in grid layout order.  FSD1 header keys:
``M, N, mask_radius, sigma, seed, interp_mode, poses [{q, t}], ctfs [{defocus, amp_contrast,
b_factor}]``; payload ``N * M^2`` pixels, image-major.  FSV1: header ``{"M": M}``, ``M^3`` voxels.

``read_dataset`` / ``write_dataset`` / ``read_volume`` / ``write_volume`` keep the reference's
signatures and DataError behaviour.  ``load_operator`` is the B200 ingest path: it never holds the
complex128 dataset on the host -- the payload is streamed in chunks of images through pinned memory
into HBM, converted to complex64 and masked on the device, then laid out brick-sorted by the engine.
"""
from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np
import torch

from .errors import DataError
from .forward import CtfParams, FourierVolume, ImageStack, Pose
from .grid import GridSpec

__all__ = ["write_dataset", "read_dataset", "write_volume", "read_volume", "read_dataset_header",
           "load_operator"]

DATASET_MAGIC = b"FSD1"
VOLUME_MAGIC = b"FSV1"


def _write(path, magic: bytes, header: dict, payload: np.ndarray) -> Path:
    path = Path(path)
    blob = json.dumps(header, separators=(",", ":")).encode("utf-8")
    with open(path, "wb") as f:
        f.write(magic)
        f.write(struct.pack("<I", len(blob)))
        f.write(blob)
        f.write(np.ascontiguousarray(payload, dtype="<c16").tobytes())
    return path


def _header(f, magic: bytes, path) -> dict:
    got = f.read(4)
    if got != magic:
        raise DataError(f"{path}: bad magic {got!r}, expected {magic!r}")
    raw = f.read(4)
    if len(raw) != 4:
        raise DataError(f"{path}: truncated header length")
    (n,) = struct.unpack("<I", raw)
    blob = f.read(n)
    if len(blob) != n:
        raise DataError(f"{path}: truncated header")
    try:
        return json.loads(blob.decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise DataError(f"{path}: invalid header JSON: {exc}") from exc


def _samples(f, count: int, path) -> np.ndarray:
    raw = f.read(count * 16)
    if len(raw) != count * 16:
        raise DataError(f"{path}: truncated payload")
    return np.frombuffer(raw, dtype="<c16").astype(np.complex128)


def _stack_meta(header: dict, path):
    try:
        M = int(header["M"])
        N = int(header["N"])
        poses = [Pose(q=np.array(p["q"], dtype=np.float64), t=np.array(p["t"], dtype=np.float64))
                 for p in header["poses"]]
        ctfs = [CtfParams(defocus=float(c["defocus"]), amp_contrast=float(c["amp_contrast"]),
                          b_factor=float(c["b_factor"])) for c in header["ctfs"]]
        meta = dict(M=M, N=N, poses=poses, ctfs=ctfs or None, sigma=float(header["sigma"]),
                    seed=int(header["seed"]), mask_radius=int(header["mask_radius"]),
                    mode=str(header["interp_mode"]))
    except (KeyError, TypeError, ValueError) as exc:
        raise DataError(f"{path}: malformed dataset header: {exc}") from exc
    if len(meta["poses"]) != N:
        raise DataError(f"{path}: malformed dataset header: {len(meta['poses'])} poses for N={N}")
    return meta


def write_dataset(stack: ImageStack, path) -> Path:
    """FSD1 writer (io.py:68-88)."""
    header = {
        "M": stack.spec.M, "N": stack.n_images, "mask_radius": stack.mask_radius, "sigma": stack.sigma,
        "seed": stack.seed, "interp_mode": stack.mode,
        "poses": [{"q": np.asarray(p.q).tolist(), "t": np.asarray(p.t).tolist()} for p in stack.poses],
        "ctfs": [{"defocus": c.defocus, "amp_contrast": c.amp_contrast, "b_factor": c.b_factor}
                 for c in (stack.ctfs or [])],
    }
    return _write(path, DATASET_MAGIC, header, stack.images)


def read_dataset_header(path) -> dict:
    """The FSD1 header only (no payload read)."""
    path = Path(path)
    try:
        with open(path, "rb") as f:
            return _header(f, DATASET_MAGIC, path)
    except OSError as exc:
        raise DataError(f"{path}: {exc}") from exc


def read_dataset(path) -> ImageStack:
    """FSD1 reader into a host ImageStack (io.py:91-125)."""
    path = Path(path)
    try:
        with open(path, "rb") as f:
            meta = _stack_meta(_header(f, DATASET_MAGIC, path), path)
            M, N = meta["M"], meta["N"]
            try:
                return ImageStack(spec=GridSpec(M), images=_samples(f, N * M * M, path).reshape(N, M * M),
                                  poses=meta["poses"], ctfs=meta["ctfs"], sigma=meta["sigma"], seed=meta["seed"],
                                  mask_radius=meta["mask_radius"], mode=meta["mode"])
            except ValueError as exc:
                raise DataError(f"{path}: malformed dataset header: {exc}") from exc
    except OSError as exc:
        raise DataError(f"{path}: {exc}") from exc


def write_volume(vol: FourierVolume, path) -> Path:
    """FSV1 writer (io.py:128-135)."""
    return _write(path, VOLUME_MAGIC, {"M": vol.spec.M}, vol.values)


def read_volume(path) -> FourierVolume:
    """FSV1 reader (io.py:138-149)."""
    path = Path(path)
    try:
        with open(path, "rb") as f:
            header = _header(f, VOLUME_MAGIC, path)
            try:
                M = int(header["M"])
            except (KeyError, TypeError, ValueError) as exc:
                raise DataError(f"{path}: malformed volume header: {exc}") from exc
            values = _samples(f, M ** 3, path)
    except OSError as exc:
        raise DataError(f"{path}: {exc}") from exc
    return FourierVolume(values, GridSpec(M))


class _HeaderStack:
    """The parts of an ImageStack that DatasetOperator-building needs, without the images."""

    def __init__(self, meta):
        self.spec = GridSpec(meta["M"])
        self.poses = meta["poses"]
        self.ctfs = meta["ctfs"]
        self.sigma = meta["sigma"]
        self.seed = meta["seed"]
        self.mask_radius = meta["mask_radius"]
        self.mode = meta["mode"]
        self.images = None

    @property
    def n_images(self) -> int:
        return len(self.poses)


def file_digest(path) -> str:
    """64-bit blake2b content digest of a file as 16 hex characters (io.py:152-158)."""
    import hashlib
    h = hashlib.blake2b(digest_size=8)
    with open(path, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


def load_operator(path, mode: str | None = None, chunk_images: int = 1024, deterministic: bool = False):
    """Stream an FSD1 file into a device-resident DatasetOperator.

    The complex128 payload is read ``chunk_images`` images at a time into a pinned buffer, copied
    to the GPU, converted to complex64 and restricted to the disk mask there; the host never holds
    more than one chunk.  Returns (DatasetOperator, ImageStack-like header object).
    """
    from .engine import SliceEngine, records_for
    from .forward import DatasetOperator, _mode_of
    from .grid import disk_mask

    path = Path(path)
    if chunk_images < 1:
        raise ValueError("chunk_images must be >= 1")
    try:
        f = open(path, "rb")
    except OSError as exc:
        raise DataError(f"{path}: {exc}") from exc
    with f:
        meta = _stack_meta(_header(f, DATASET_MAGIC, path), path)
        M, N = meta["M"], meta["N"]
        hstack = _HeaderStack(meta)
        m = _mode_of(meta["mode"], mode)
        mask = disk_mask(hstack.spec, meta["mask_radius"])
        quats = np.array([p.q for p in meta["poses"]], dtype=np.float64)
        shifts = np.array([p.t for p in meta["poses"]], dtype=np.float64)
        eng = SliceEngine(M, m, mask, records_for(M, quats, shifts, meta["ctfs"]), None,
                          deterministic=deterministic)
        dev = eng.dev
        x = torch.empty((N, mask.size), dtype=torch.complex64, device=dev)
        mask_d = torch.from_numpy(mask.astype(np.int32)).to(dev)
        from . import _capi as C
        from .engine import _stream, ctypes_ptr
        lib = C.load()
        pin = torch.empty(chunk_images * M * M * 16, dtype=torch.uint8).pin_memory()
        for i0 in range(0, N, chunk_images):
            n = min(chunk_images, N - i0)
            nbytes = n * M * M * 16
            view = pin[:nbytes].numpy()
            got = f.readinto(memoryview(view))
            if got != nbytes:
                raise DataError(f"{path}: truncated payload")
            raw = pin[:nbytes].to(dev, non_blocking=True)
            # x[i0:i0+n] = (complex64) images[:, mask] (fsld_mask_images kernel)
            C.check(lib.fsld_mask_images(M, mask.size, ctypes_ptr(mask_d), n, ctypes_ptr(raw),
                                         ctypes_ptr(x[i0:i0 + n]), _stream()), "fsld_mask_images")
            torch.cuda.current_stream().synchronize()  # the pinned chunk is reused
        eng.set_images(x)
        op = DatasetOperator.from_engine(eng, hstack.spec)
        op.stack = hstack
    return op, hstack
