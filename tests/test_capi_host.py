"""CPU-only checks of the C ABI library and the host-side logic (no kernel launches)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle as O

from paper_2311_16100_b200 import _capi as C
from paper_2311_16100_b200.engine import records_for
from paper_2311_16100_b200.forward import CtfParams, PhysicalCtf, quat_to_matrix
from paper_2311_16100_b200.grid import disk_mask, pixel_coords
from paper_2311_16100_b200.kernels import ctf_table_row
from paper_2311_16100_b200 import synth


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fsld_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(fsld_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    lib = C.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    # the ctypes signature table covers the header exactly
    assert set(syms) == set(C.SIGNATURES)


def test_abi_version_and_status_strings():
    lib = C.load()
    assert lib.fsld_abi_version() == C.ABI_VERSION
    assert lib.fsld_status_string(C.FSLD_EINVAL) == b"invalid argument"
    assert lib.fsld_status_string(0) == b"ok"


def test_record_layout_is_128_bytes():
    assert C.REC_DTYPE.itemsize == 128
    txt = open(os.path.join(ROOT, "include", "fsld_b200.h")).read()
    assert "double rot[6];" in txt and "double gamma[4];" in txt


def test_invalid_arguments_rejected_without_gpu():
    lib = C.load()
    # empty batch -> EINVAL (reference: ValueError "batch must be nonempty")
    st = lib.fsld_loss_grad(32, C.MODE_TRI, 749, 1, 1, 1, 0, 1, 1, 1, 1, 0, 0, 1, 1 << 20, 0)
    assert st == C.FSLD_EINVAL
    st = lib.fsld_project(32, 7, 749, 1, 1, 1, 4, 1, 1, 0)  # bad mode
    assert st == C.FSLD_EINVAL
    st = lib.fsld_loss_grad(32, C.MODE_TRI, 749, 1, 1, 1, 4, 1, 1, 1, 1, C.DETERMINISTIC, 0, 1, 1 << 20, 0)
    assert st == C.FSLD_EINVAL  # deterministic without a fixed-point scale
    with pytest.raises(ValueError):
        C.check(C.FSLD_EINVAL, "x")
    # numpy-signature host step: missing / misaligned host arrays are refused before any device work
    args = (128, C.MODE_TRI, 12645, 1, 1, 512)
    tail = (1, 1, 1, 1, 1, 1.0, 1e-3)
    st = lib.fsld_loss_grad_host_np(*args, 0, *tail, 16, 16, 16, 16, 16, 12, 16, 1 << 30, 0)
    assert st == C.FSLD_EINVAL  # v = NULL
    st = lib.fsld_loss_grad_host_np(*args, 24, *tail, 8, 16, 16, 16, 16, 12, 16, 1 << 30, 0)
    assert st == C.FSLD_EINVAL  # gradient not 16-byte aligned
    st = lib.fsld_loss_grad_host_np(*args, 16, *tail, 16, 16, 16, 16, 16, 99, 16, 1 << 30, 0)
    assert st == C.FSLD_EINVAL  # n_slabs out of range
    # table loss pass: an empty batch is refused
    st = lib.fsld_loss_sorted_tab(128, C.MODE_TRI, 12645, 1, 1, 0, 1, 1, 1, 1, 1, 1, 1, 1, 1 << 30, 0)
    assert st == C.FSLD_EINVAL
    # brick exact diagonal: nn mode, missing tables, deterministic without a scale or with B > 1024
    dg = lib.fsld_exact_diag_sorted_tab
    assert dg(128, C.MODE_NN, 12645, 1, 1, 8, 1, 1, 1, 1, 1, 0, 0, 1, 1 << 30, 0) == C.FSLD_EINVAL
    assert dg(128, C.MODE_TRI, 12645, 1, 1, 8, 1, 0, 1, 1, 1, 0, 0, 1, 1 << 30, 0) == C.FSLD_EINVAL
    assert dg(128, C.MODE_TRI, 12645, 1, 1, 8, 1, 1, 1, 1, 1, C.DETERMINISTIC, 0, 1, 1 << 30, 0) == C.FSLD_EINVAL
    assert dg(128, C.MODE_TRI, 12645, 1, 1, 2048, 1, 1, 1, 1, 1, C.DETERMINISTIC, 1, 1, 1 << 40, 0) == C.FSLD_EINVAL
    assert dg(128, C.MODE_TRI, 12645, 1, 1, 8, 1, 1, 1, 1, 1, 0, 0, 1, 16, 0) == C.FSLD_EINVAL  # scratch too small


def test_scratch_bytes_grows_with_batch():
    lib = C.load()
    assert lib.fsld_scratch_bytes(128, 12645, 512) >= 512 * 13 * 8
    assert lib.fsld_scratch_bytes(128, 12645, 1024) > lib.fsld_scratch_bytes(128, 12645, 512)


def test_records_rotation_rows_bitexact_with_reference_formula(golden):
    g = golden("kernels_m16.npz")
    recs = records_for(16, g["quats"], g["shifts"], None)
    rt = g["rt"]
    assert np.array_equal(recs["rot"][:, :3], rt[:, 0, :])
    assert np.array_equal(recs["rot"][:, 3:], rt[:, 1, :])
    assert np.allclose(recs["shift"], -2.0 * g["shifts"] / 16, rtol=0, atol=0)


def test_inkernel_ctf_model_matches_reference_radial_table(golden):
    g = golden("kernels_m16.npz")
    M = 16
    pix = O.mask_pix(M, g["mask"])
    for i, (d, w, b) in enumerate(g["ctf_params"]):
        row = ctf_table_row(CtfParams(d, w, b), pix, M)
        assert np.max(np.abs(row - g["ctf"][i])) < 1e-13


def test_inkernel_ctf_model_matches_oracle_physical_table(golden):
    g = golden("kernels_m16.npz")
    M = 16
    pix = O.mask_pix(M, g["mask"])
    for i, p in enumerate(g["phys_params"]):
        c = PhysicalCtf(*p)
        row = ctf_table_row(c, pix, M)
        assert np.max(np.abs(row - g["phys_ctf"][i])) < 1e-12


def test_phase_from_record_matches_reference_phase(golden):
    g = golden("kernels_m16.npz")
    M = 16
    pix = O.mask_pix(M, g["mask"])
    recs = records_for(M, g["quats"], g["shifts"], None)
    ph = np.exp(1j * np.pi * (recs["shift"] @ pix.T))
    assert np.max(np.abs(ph - g["phase"])) < 1e-13


def test_mask_and_pixel_layout_match_oracle():
    for M in (4, 8, 32, 64, 128):
        assert np.array_equal(disk_mask(M, M // 2 - 1), O.disk_mask(M, M // 2 - 1))
        assert np.array_equal(pixel_coords(M), O.pixel_coords(M))


def test_quat_to_matrix_bitexact():
    q = synth.haar_quaternions(50, 3)
    for qq in q:
        assert np.array_equal(quat_to_matrix(qq), O.quat_to_matrix(qq))


def test_blob_volume_layout_is_reference_layout():
    """The synthetic volume's DC sits at grid.dc_index and is the (real) total mass."""
    M = 16
    v = synth.gaussian_blob_volume(M, seed=0)
    dc = ((M + 1) // 2) * (M + 1)
    assert np.argmax(np.abs(v)) == dc
    assert abs(v[dc].imag) < 1e-9 * abs(v[dc].real)
    # Hermitian symmetry of the FT of a real volume: v(-k) = conj(v(k)) under the layout map
    vc = O.voxel_coords(M)
    j = 5 * M * M + 3 * M + 9
    k = vc[j]
    neg = -k
    if np.all(neg >= -((M + 1) // 2)) and np.all(neg < M // 2):
        zi = neg[2] if neg[2] >= 0 else neg[2] + M
        jn = (zi * M + neg[1] + (M + 1) // 2) * M + neg[0] + (M + 1) // 2
        assert abs(v[jn] - np.conj(v[j])) < 1e-9 * np.abs(v).max()


def test_step_abi_structs_match_header():
    txt = open(os.path.join(ROOT, "include", "fsld_b200.h")).read()
    assert "typedef struct fsld_step_params" in txt and "typedef struct fsld_armijo_state" in txt
    assert ctypes.sizeof(C.StepParams) == 7 * 8 + 2 * 4
    assert C.ARMIJO_DTYPE.itemsize == 56


def test_step_entry_points_reject_bad_arguments_without_gpu():
    lib = C.load()
    p = C.StepParams(scale=2.0, lam=0.1, beta=0.9, floor=0.0, w_old=0.0, w_new=1.0, hutch_scale=2.0, estimating=1)
    # estimating needs fold / d_avg / d and a positive floor
    assert lib.fsld_precond_step(8, 1, 1, 0, 0, 0, 0, ctypes.byref(p), 1, 0, 0, 1, 1, 1 << 16, 0) == C.FSLD_EINVAL
    p.floor = 1.0
    assert lib.fsld_precond_step(8, 16, 16, 16, 16, 16, 0, ctypes.byref(p), 16, 0, 0, 16, 16, 16, 0) == C.FSLD_EINVAL
    # misaligned vectors
    assert lib.fsld_precond_step(8, 8, 16, 16, 16, 16, 0, ctypes.byref(p), 16, 0, 0, 16, 16, 1 << 20, 0) == C.FSLD_EINVAL
    assert lib.fsld_precond_step(8, 1, 1, 1, 1, 1, 0, None, 1, 0, 0, 1, 1, 1 << 16, 0) == C.FSLD_EINVAL
    # empty batch / bad mode -> ValueError semantics
    assert lib.fsld_armijo_terms(32, C.MODE_TRI, 749, 1, 0, 1, 1, 0, 1, 1, 1, 1, 1, 1 << 20, 0) == C.FSLD_EINVAL
    assert lib.fsld_armijo_terms(32, 5, 749, 1, 0, 1, 1, 4, 1, 1, 1, 1, 1, 1 << 20, 0) == C.FSLD_EINVAL
    # c outside (0, 1), negative lam, non-positive scale
    assert lib.fsld_armijo_select(1, 1, 1, 1, 1.0, 0.1, 1.5, 60, 1, 0, 0, 0) == C.FSLD_EINVAL
    assert lib.fsld_armijo_select(1, 1, 1, 1, 1.0, -0.1, 0.5, 60, 1, 0, 0, 0) == C.FSLD_EINVAL
    assert lib.fsld_armijo_select(1, 1, 1, 1, 0.0, 0.1, 0.5, 60, 1, 0, 0, 0) == C.FSLD_EINVAL
    # brick energy pass: tri only, M <= 256
    assert lib.fsld_proj_energy_sorted(32, C.MODE_NN, 749, 1, 1, 4, 1, 1, 1, 1, 1, 0, 1, 1 << 24, 0) == C.FSLD_EINVAL
    assert lib.fsld_proj_energy_sorted(512, C.MODE_TRI, 749, 1, 1, 4, 1, 1, 1, 1, 1, 0, 1, 1 << 24, 0) == C.FSLD_EINVAL
    # reuse of a binning that was never made on this scratch / unknown flags
    assert lib.fsld_proj_energy_sorted(32, C.MODE_TRI, 749, 1, 1, 4, 1, 1, 1, 1, 1, C.REUSE_BINS, 1, 1 << 24,
                                       0) == C.FSLD_EINVAL
    assert lib.fsld_proj_energy_sorted(32, C.MODE_TRI, 749, 1, 1, 4, 1, 1, 1, 1, 1, 64, 1, 1 << 24, 0) == C.FSLD_EINVAL
    assert lib.fsld_apply_step(0, 1, 1, 1, 0) == C.FSLD_EINVAL


def test_optim_config_validation_matches_reference():
    from paper_2311_16100_b200.optim import OptimConfig, VARIANTS
    assert VARIANTS == ("plain", "precomputed", "estimated", "estimated_nothresh")
    OptimConfig(lam=0.1, batch_size=4, epochs=1)
    for bad in (dict(lam=-1.0), dict(batch_size=0), dict(epochs=0), dict(beta=1.0), dict(c=0.0),
                dict(eta0=0.0), dict(variant="x"), dict(mode="cubic"), dict(eta_growth=0.5)):
        kw = dict(lam=0.1, batch_size=4, epochs=1)
        kw.update(bad)
        with pytest.raises(ValueError):
            OptimConfig(**kw)


def test_plan_entry_points_reject_bad_arguments_without_gpu():
    lib = C.load()
    assert lib.fsld_plan_bytes(128, 12645, 512, 20, 10 ** 6) > 16 * 10 ** 6
    assert lib.fsld_plan_bytes(512, 12645, 512, 20, 10 ** 6) == 0  # brick path is M <= 256
    assert lib.fsld_plan_bytes(128, 12645, 512, 0, 10 ** 6) == 0
    assert lib.fsld_plan_build(128, 12645, 1, 1, 4, 8, 1, 1, 100, 1, 16, 0) == C.FSLD_EINVAL  # plan too small
    # a plan pointer that was never built on this process
    assert lib.fsld_loss_grad_planned(128, C.MODE_TRI, 12645, 1, 12345, 8, 0, 1, 1, 1, 0, 0, 1, 0, 1, 1, 1 << 30,
                                      0) == C.FSLD_EINVAL
    assert lib.fsld_proj_energy_planned(128, C.MODE_TRI, 12645, 1, 12345, 8, 0, 1, 1, 1, 1, 1 << 30, 0) == C.FSLD_EINVAL


def test_host_casts_are_exact_roundings_any_alignment():
    """fsld_host_cast_* (the numpy call path's staging casts) equal numpy's casts, aligned or not, and
    the thread-pool split (hostio.cast_native) covers the whole range."""
    lib = C.load()
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 1001, 1 << 16):
        a = rng.standard_normal(2 * n + 3)
        for off in (0, 1):
            src = a[off:off + 2 * n]
            dst = np.zeros(2 * n + 4, np.float32)[off:off + 2 * n]
            assert lib.fsld_host_cast_f64_to_f32(src.ctypes.data, dst.ctypes.data, 2 * n) == 0
            assert np.array_equal(dst, src.astype(np.float32))
            back = np.zeros(2 * n + 2, np.float64)[off:off + 2 * n]
            assert lib.fsld_host_cast_f32_to_f64(dst.ctypes.data, back.ctypes.data, 2 * n) == 0
            assert np.array_equal(back, dst.astype(np.float64))
    assert lib.fsld_host_cast_f64_to_f32(None, None, -1) == C.FSLD_EINVAL
    from paper_2311_16100_b200.hostio import cast_native
    big = rng.standard_normal(2 * 300001)
    out = np.zeros(2 * 300001, np.float32)
    cast_native(lib.fsld_host_cast_f64_to_f32, big.ctypes.data, out.ctypes.data, big.size, 8, 4)
    assert np.array_equal(out, big.astype(np.float32))


def test_ball_voxels_covers_the_touched_ball():
    """fsld_ball_voxels (the packed ball of fsld_loss_grad_host_np_ball; host code, no device call): at
    least the voxels grid.touched_ball lists, rows rounded out to 4 voxels, the whole cube without a radius."""
    import math
    from paper_2311_16100_b200.grid import touched_ball
    lib = C.load()
    for M, R in [(16, 7), (32, 8), (33, 15), (64, 31), (128, 63)]:
        n = lib.fsld_ball_voxels(M, R + 0.5 + math.sqrt(3.0))
        nb = len(touched_ball(M, R))
        assert nb <= n <= M ** 3
        assert n % 4 == 0 or M % 4
        if M >= 64:
            assert n < 0.75 * M ** 3 and n < 1.25 * nb
    assert lib.fsld_ball_voxels(32, 0.0) == 32 ** 3
    assert lib.fsld_ball_voxels(32, float("inf")) == 32 ** 3
