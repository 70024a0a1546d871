"""Timing of the numpy-signature call (loss_and_grad_numpy -> fsld_loss_grad_host_np) beside the pinned
complex64 C-ABI step alone (medians / minima of 30 calls after warm-up)."""
import os
import time

import numpy as np
import torch

from paper_2311_16100_b200 import synth
from paper_2311_16100_b200.forward import DatasetOperator

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=4096)
op = DatasetOperator.from_engine(wl.engine)
v = (wl.v_true * 0.9).astype(np.complex128).reshape(-1)
rng = np.random.default_rng(0)


def t_np():
    ts = []
    for i in range(35):
        rows = rng.choice(4096, 512, replace=False)
        t0 = time.perf_counter()
        loss, g = op.loss_and_grad_numpy(v, rows, 1e-3, 50000)
        ts.append((time.perf_counter() - t0) * 1e3)
        del g
    return np.median(ts[5:]), np.min(ts[5:])


from paper_2311_16100_b200 import _capi as C
vh = C.host_empty(v.size, torch.complex64)
gh = C.host_empty(v.size, torch.complex64)
vh.numpy()[:] = v
ih = torch.empty(512, dtype=torch.int32).pin_memory()


def t_cabi():
    ts = []
    for i in range(35):
        ih.numpy()[:] = rng.choice(4096, 512, replace=False)
        t0 = time.perf_counter()
        op.loss_and_grad_host(vh, ih, 1e-3, gh, 50000)
        ts.append((time.perf_counter() - t0) * 1e3)
    return np.median(ts[5:]), np.min(ts[5:])


for rep in range(2):
    print("numpy call (median, min ms):", t_np())
    print("C-ABI pinned complex64:", t_cabi())
