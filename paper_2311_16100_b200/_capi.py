"""ctypes binding of libfsld_b200.so (the C ABI declared in include/fsld_b200.h).

The product has exactly one compute path: the sm_100a kernels behind this
ABI.  If the shared library is missing, or no compute-capability-10 device
is visible, calls raise -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSLD_LIB_PATH") or os.path.join(_PKG, "_lib", "libfsld_b200.so")

FSLD_OK = 0
FSLD_EINVAL = -1
FSLD_ECUDA = -2
FSLD_ENODEV = -3
MODE_NN = 0
MODE_TRI = 1
DETERMINISTIC = 1
TILE_PATH = 2
NN_BRICK = 8
REUSE_BINS = 4
REC_CTF = 1
REC_SHIFT = 2
ABI_VERSION = 2

# fsld_image_rec (include/fsld_b200.h): 128 bytes
REC_DTYPE = np.dtype([
    ("rot", "<f8", (6,)),
    ("shift", "<f8", (2,)),
    ("gamma", "<f8", (4,)),
    ("env", "<f8"),
    ("wsin", "<f4"),
    ("wcos", "<f4"),
    ("flags", "<u4"),
    ("xmax", "<f4"),
    ("pad", "<u4", (2,)),
])
assert REC_DTYPE.itemsize == 128


class StepParams(ctypes.Structure):
    """fsld_step_params (include/fsld_b200.h)."""
    _fields_ = [("scale", ctypes.c_double), ("lam", ctypes.c_double), ("beta", ctypes.c_double),
                ("floor", ctypes.c_double), ("w_old", ctypes.c_double), ("w_new", ctypes.c_double),
                ("hutch_scale", ctypes.c_double), ("estimating", ctypes.c_int), ("pad", ctypes.c_int)]


# fsld_armijo_state (include/fsld_b200.h): 56 bytes, lives in device memory
ARMIJO_DTYPE = np.dtype([
    ("eta", "<f8"), ("f0", "<f8"), ("f_next", "<f8"), ("eta_applied", "<f8"), ("decrease", "<f8"),
    ("backtracks", "<i4"), ("status", "<i4"), ("n_steps", "<i4"), ("pad", "<i4"),
])
assert ARMIJO_DTYPE.itemsize == 56

P = ctypes.c_void_p
I = ctypes.c_int
I64 = ctypes.c_int64
U = ctypes.c_uint
D = ctypes.c_double
SZ = ctypes.c_size_t

# name -> (restype, argtypes); the exported surface of include/fsld_b200.h
SIGNATURES = {
    "fsld_abi_version": (I, []),
    "fsld_status_string": (ctypes.c_char_p, [I]),
    "fsld_device_count": (I, [P]),
    "fsld_host_alloc": (I, [SZ, P]),
    "fsld_host_free": (I, [P]),
    "fsld_scratch_bytes": (SZ, [I, I, I]),
    "fsld_prepare": (I, [I, I, P, P, SZ, P]),
    "fsld_loss_grad": (I, [I, I, I, P, P, P, I, P, P, P, P, U, P, P, SZ, P]),
    "fsld_loss": (I, [I, I, I, P, P, P, I, P, P, P, P, SZ, P]),
    "fsld_project": (I, [I, I, I, P, P, P, I, P, P, P]),
    "fsld_backproject": (I, [I, I, I, P, P, P, I, P, P, U, P, P]),
    "fsld_hvp": (I, [I, I, I, P, P, P, I, P, P, U, P, P]),
    "fsld_hutch_fold": (I, [I, I, I, P, P, P, I, P, I, P, U, P, P]),
    "fsld_pack_probes": (I, [I64, I, P, P, P, P]),
    "fsld_gen_probes": (I, [I64, I, ctypes.c_uint64, P, P]),
    "fsld_exact_diag": (I, [I, I, I, P, P, P, I, P, U, P, P]),
    "fsld_exact_diag_sorted_tab": (I, [I, I, I, P, P, I, P, P, P, P, P, U, P, P, SZ, P]),
    "fsld_assign_nn": (I, [I, I, P, P, P, I, P, P]),
    "fsld_project_tab": (I, [I, I, I, P, P, I, P, P, P, P]),
    "fsld_backproject_tab": (I, [I, I, I, P, P, I, P, P, P, U, P, P]),
    "fsld_scatter_sq_tab": (I, [I, I, I, P, P, I, P, P, U, P, P]),
    "fsld_sorted_count": (I, [I, I, P, P, I, P, P]),
    "fsld_sorted_fill": (I, [I, I, P, P, I, P, P, P, P, P, P]),
    "fsld_sorted_tables": (I, [I, I, I, P, I, P, P, P, P, P]),
    "fsld_sorted_tables_bytes": (SZ, [I, I]),
    "fsld_fsc_scratch_bytes": (SZ, [I, I]),
    "fsld_host_step_reset": (I, []),
    "fsld_ctf_ring_power": (I, [P, I, P, I, P, P]),
    "fsld_host_cast_f64_to_f32": (I, [P, P, I64]),
    "fsld_host_cast_f32_to_f64": (I, [P, P, I64]),
    "fsld_fsc": (I, [I, I, P, P, P, P, SZ, P]),
    "fsld_mask_images": (I, [I, I, P, I, P, P, P]),
    "fsld_loss_grad_sorted": (I, [I, I, I, P, P, I, P, P, P, P, P, P, P, P, U, P, P, SZ, P]),
    "fsld_loss_sorted": (I, [I, I, I, P, P, I, P, P, P, P, P, SZ, P]),
    "fsld_loss_sorted_tab": (I, [I, I, I, P, P, I, P, P, P, P, P, P, P, P, SZ, P]),
    "fsld_loss_grad_hutch_sorted": (I, [I, I, I, P, P, I, P, P, P, P, P, P, P, P, P, P, U, P, SZ, P]),
    "fsld_hvp_sorted": (I, [I, I, I, P, P, I, P, P, P, P, P, P, P, U, P, SZ, P]),
    "fsld_loss_grad_step_planned": (I, [I, I, I, P, P, I, I, P, P, P, P, D, D, P, P, P, P, SZ, P, SZ, P]),
    "fsld_loss_grad_host": (I, [I, I, I, P, P, I, P, P, P, P, P, P, D, D, P, P, P, P, P, I, P, SZ, P]),
    "fsld_loss_grad_host_c128": (I, [I, I, I, P, P, I, P, P, P, P, P, P, D, D, P, P, P, P, P, P, I, P, SZ, P]),
    "fsld_loss_grad_host_np": (I, [I, I, I, P, P, I, P, P, P, P, P, P, D, D, P, P, P, P, P, I, P, SZ, P]),
    "fsld_ball_voxels": (I64, [I, D]),
    "fsld_loss_grad_host_np_ball": (I, [I, I, I, P, P, I, P, P, P, P, P, P, D, D, P, P, P, P, P, I, P, SZ, P, D]),
    "fsld_project_sorted": (I, [I, I, I, P, P, I, P, P, P, P]),
    "fsld_backproject_sorted": (I, [I, I, I, P, P, I, P, P, P, U, P, P]),
    "fsld_fixed_scale": (I, [P, I64, D, D, P, P]),
    "fsld_grad_finalize": (I, [I64, P, U, P, P, D, D, P, P]),
    "fsld_real_finalize": (I, [I64, P, U, P, D, D, P, P]),
    "fsld_norm2": (I, [I64, P, P, P, SZ, P]),
    "fsld_grad_epilogue": (I, [I64, P, P, D, D, P, P, P, P, P, SZ, P]),
    "fsld_precond_step": (I, [I64, P, P, P, P, P, P, P, P, P, P, P, P, SZ, P]),
    "fsld_armijo_terms": (I, [I, I, I, P, P, P, P, I, P, P, P, P, P, SZ, P]),
    "fsld_armijo_select": (I, [P, P, P, P, D, D, D, I, P, P, I, P]),
    "fsld_proj_energy_sorted": (I, [I, I, I, P, P, I, P, P, P, P, P, U, P, SZ, P]),
    "fsld_hutch_fold_sorted": (I, [I, I, I, P, P, I, P, P, P, P, I, P, P, SZ, P]),
    "fsld_apply_step": (I, [I64, P, P, P, P]),
    "fsld_ball_gather": (I, [I64, P, P, P, I, P]),
    "fsld_plan_bytes": (SZ, [I, I, I, I, I64]),
    "fsld_plan_build": (I, [I, I, P, P, I, I, P, P, I64, P, SZ, P]),
    "fsld_loss_grad_planned": (I, [I, I, I, P, P, I, I, P, P, P, P, P, P, P, P, P, SZ, P]),
    "fsld_loss_grad_planned_mc": (I, [I, I, I, P, P, I, I, P, P, P, P, P, P, P, SZ, P]),
    "fsld_nvls_supported": (I, [I]),
    "fsld_nvls_ctl_offset": (SZ, [SZ]),
    "fsld_nvls_create": (I, [I, SZ, P, P, P]),
    "fsld_nvls_import": (I, [I, I, I, SZ, SZ, P]),
    "fsld_nvls_add_device": (I, [P]),
    "fsld_nvls_bind": (I, [P, P, P]),
    "fsld_nvls_barrier": (I, [P, P, P, P]),
    "fsld_nvls_status": (I, [P]),
    "fsld_nvls_destroy": (I, [P]),
    "fsld_fd_listen": (I, [ctypes.c_char_p, P]),
    "fsld_fd_recv": (I, [I, P]),
    "fsld_fd_send": (I, [ctypes.c_char_p, I]),
    "fsld_proj_energy_planned": (I, [I, I, I, P, P, I, I, P, P, P, P, SZ, P]),
    "fsld_ball_scatter": (I, [I64, P, P, P, I, P]),
}

_lib = None


class FsldError(RuntimeError):
    pass


def load():
    """Load libfsld_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2311_16100_b200._build` "
                "(nvcc, sm_100a). There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.fsld_abi_version() != ABI_VERSION:
            raise ImportError("libfsld_b200.so ABI version mismatch; rebuild it")
        _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    if status == FSLD_OK:
        return
    msg = load().fsld_status_string(status).decode()
    if status == FSLD_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise FsldError(f"{what}: {msg} (status {status})")


def host_empty(numel: int, dtype):
    """A page-locked host tensor backed by fsld_host_alloc (cudaHostAlloc), freed with the tensor.

    The host-buffer step streams these at full PCIe rate in both directions at once; pinned
    memory from other allocators is accepted too."""
    import weakref

    import torch

    nbytes = int(numel) * torch.empty((), dtype=dtype).element_size()
    ptr = ctypes.c_void_p()
    check(load().fsld_host_alloc(max(nbytes, 1), ctypes.byref(ptr)), "fsld_host_alloc")
    buf = (ctypes.c_char * max(nbytes, 1)).from_address(ptr.value)
    weakref.finalize(buf, load().fsld_host_free, ptr.value)
    return torch.frombuffer(buf, dtype=dtype, count=int(numel))
