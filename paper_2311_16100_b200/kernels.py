"""numba-signature entry points of the reference (fsld.kernels), on the B200 kernels.

Same names and output-parameter style as /root/reference/pkg/src/fsld/kernels.py:
``assign_nn`` (123-135), ``project_tri`` / ``project_nn`` (138-190),
``backproject_tri`` / ``backproject_nn`` (193-248), ``scatter_sq_tri``
(251-294), ``fold_chunks`` / ``n_chunks`` / ``SCATTER_CHUNK`` (33-39,
297-302).  These take the reference's per-(image, pixel) ``phase`` / ``ctf``
tables and run the table-driven kernels (fsld_project_tab & co.); the
DatasetOperator path evaluates phase and CTF in-kernel instead.

Scatter outputs: the adjoint of the whole batch is ADDED to ``vols[0]``
(the GPU needs no per-chunk partials), so ``fold_chunks(vols)`` returns the
same total the reference's fold does.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _capi as C
from .engine import _stream, ctypes_ptr, require_device

SCATTER_CHUNK = 64


def n_chunks(n_images: int) -> int:
    return (n_images + SCATTER_CHUNK - 1) // SCATTER_CHUNK


def fold_chunks(vols: np.ndarray) -> np.ndarray:
    """Combine per-chunk partial volumes in chunk order (kernels.py:297-302)."""
    out = vols[0].copy()
    for c in range(1, vols.shape[0]):
        out += vols[c]
    return out


def _pix_i16(pix) -> np.ndarray:
    p = np.asarray(pix, dtype=np.float64)
    q = np.rint(p)
    if not np.array_equal(p, q):
        raise ValueError("pixel coordinates must be integer frequencies")
    return np.ascontiguousarray(q.astype(np.int16))


def _recs_from_rt(rt) -> np.ndarray:
    rt = np.asarray(rt, dtype=np.float64).reshape(-1, 3, 3)
    recs = np.zeros(rt.shape[0], dtype=C.REC_DTYPE)
    recs["rot"][:, 0:3] = rt[:, 0, :]
    recs["rot"][:, 3:6] = rt[:, 1, :]
    return recs


class _Call:
    """Device staging for one numba-style call."""

    def __init__(self, rt, pix, M):
        self.dev = require_device()
        self.M = int(M)
        recs = _recs_from_rt(rt)
        self.B = recs.shape[0]
        pix16 = _pix_i16(pix)
        self.n = pix16.shape[0]
        if self.B < 1:
            raise ValueError("batch must be nonempty")
        self.recs = torch.from_numpy(recs.view(np.uint8).copy()).to(self.dev)
        self.pix = torch.from_numpy(pix16).to(self.dev)

    def c64(self, a, shape):
        a = np.broadcast_to(np.asarray(a), shape)
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex64)).to(self.dev)


def ctf_table_row(c, pix, M: int) -> np.ndarray:
    """One image's CTF per masked pixel on the host (Projector.ctf_batch, forward.py:305-312)."""
    from .forward import ctf_coefficients
    g, env, ws, wc = ctf_coefficients(c, M)
    kx = pix[:, 0]
    ky = pix[:, 1]
    k2 = kx * kx + ky * ky
    gam = g[0] * k2 + g[1] * (kx * kx - ky * ky) + g[2] * (2 * kx * ky) + g[3] * k2 * k2
    return -(ws * np.sin(gam) + wc * np.cos(gam)) * np.exp(-env * k2)


def assign_nn(rt, pix, M) -> np.ndarray:
    """Nearest-neighbour voxel index per (image, pixel), int64 (kernels.py:123-135)."""
    call = _Call(rt, pix, M)
    out = torch.empty((call.B, call.n), dtype=torch.int32, device=call.dev)
    C.check(C.load().fsld_assign_nn(call.M, call.n, ctypes_ptr(call.pix), ctypes_ptr(call.recs), 0, call.B,
                                    ctypes_ptr(out), _stream()), "fsld_assign_nn")
    return out.cpu().numpy().astype(np.int64)


def _project(mode_id, v, rt, pix, phase, ctf, M, out):
    call = _Call(rt, pix, M)
    f = np.asarray(phase) * np.asarray(ctf)
    vd = torch.from_numpy(np.ascontiguousarray(v, dtype=np.complex64)).to(call.dev)
    fd = call.c64(f, (call.B, call.n))
    od = torch.empty((call.B, call.n), dtype=torch.complex64, device=call.dev)
    C.check(C.load().fsld_project_tab(call.M, mode_id, call.n, ctypes_ptr(call.pix), ctypes_ptr(call.recs),
                                      call.B, ctypes_ptr(vd), ctypes_ptr(fd), ctypes_ptr(od), _stream()),
            "fsld_project_tab")
    out[...] = od.cpu().numpy()


def project_tri(v, rt, pix, phase, ctf, M, out):
    _project(C.MODE_TRI, v, rt, pix, phase, ctf, M, out)


def project_nn(v, rt, pix, phase, ctf, M, out):
    _project(C.MODE_NN, v, rt, pix, phase, ctf, M, out)


def _backproject(mode_id, img, rt, pix, phase, ctf, M, vols):
    call = _Call(rt, pix, M)
    f = np.asarray(phase) * np.asarray(ctf)
    imd = call.c64(img, (call.B, call.n))
    fd = call.c64(f, (call.B, call.n))
    acc = torch.zeros(call.M ** 3, dtype=torch.complex64, device=call.dev)
    C.check(C.load().fsld_backproject_tab(call.M, mode_id, call.n, ctypes_ptr(call.pix), ctypes_ptr(call.recs),
                                          call.B, ctypes_ptr(imd), ctypes_ptr(fd), ctypes_ptr(acc), 0, 0,
                                          _stream()), "fsld_backproject_tab")
    vols[0] += acc.cpu().numpy()


def backproject_tri(img, rt, pix, phase, ctf, M, vols):
    _backproject(C.MODE_TRI, img, rt, pix, phase, ctf, M, vols)


def backproject_nn(img, rt, pix, phase, ctf, M, vols):
    _backproject(C.MODE_NN, img, rt, pix, phase, ctf, M, vols)


def scatter_sq(mode: str, weights, rt, pix, M) -> np.ndarray:
    """tri: sum w_corner^2 * weights; nn: bincount(assign_nn, weights) (forward.py:341-349)."""
    call = _Call(rt, pix, M)
    wd = call.c64(np.asarray(weights, dtype=np.float64), (call.B, call.n))
    acc = torch.zeros(call.M ** 3, dtype=torch.float32, device=call.dev)
    C.check(C.load().fsld_scatter_sq_tab(call.M, C.MODE_TRI if mode == "tri" else C.MODE_NN, call.n,
                                         ctypes_ptr(call.pix), ctypes_ptr(call.recs), call.B, ctypes_ptr(wd),
                                         ctypes_ptr(acc), 0, 0, _stream()), "fsld_scatter_sq_tab")
    return acc.cpu().numpy().astype(np.float64)


def scatter_sq_tri(weights, rt, pix, M, vols):
    vols[0] += scatter_sq("tri", weights, rt, pix, M)
