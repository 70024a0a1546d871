"""Split of the reference-signature e2e call (cast in, host step, allocation + cast out)."""
import time

import numpy as np
import torch

from paper_2311_16100_b200 import synth
from paper_2311_16100_b200.forward import DatasetOperator
from paper_2311_16100_b200.hostio import cast_into

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=4096)
op = DatasetOperator.from_engine(wl.engine)
e = wl.engine
v = (wl.v_true * 0.9).astype(np.complex128)
rows = np.random.default_rng(0).choice(4096, 512, replace=False)
op.loss_and_grad_numpy(v, rows, 1e-3, 50000)
st = op._np_stage
T = {"cast_in": [], "host_step": [], "alloc": [], "cast_out": [], "whole": []}
for _ in range(10):
    t0 = time.perf_counter(); cast_into(st["v"].numpy(), v); t1 = time.perf_counter()
    op.loss_and_grad_host(st["v"], st["idx"], 1e-3, st["g"], 50000); t2 = time.perf_counter()
    g = np.empty(v.size, np.complex128); t3 = time.perf_counter()
    cast_into(g, st["g"].numpy()); t4 = time.perf_counter()
    op.loss_and_grad_numpy(v, rows, 1e-3, 50000); t5 = time.perf_counter()
    for k, dt in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
        T[k].append(dt * 1e3)
print({k: round(float(np.median(x)), 3) for k, x in T.items()})

# variant: cudaHostAlloc staging (fsld_host_alloc) instead of torch pin_memory
from paper_2311_16100_b200 import _capi as C
vh = C.host_empty(v.size, torch.complex64)
gh = C.host_empty(v.size, torch.complex64)
ih = C.host_empty(512, torch.int32)
ih.copy_(torch.from_numpy(rows.astype(np.int32)))
T2 = {"cast_in": [], "host_step": [], "host_step_clean": [], "cast_out": []}
for _ in range(10):
    t0 = time.perf_counter(); cast_into(vh.numpy(), v); t1 = time.perf_counter()
    op.loss_and_grad_host(vh, ih, 1e-3, gh, 50000); t2 = time.perf_counter()
    op.loss_and_grad_host(vh, ih, 1e-3, gh, 50000); t3 = time.perf_counter()
    g = np.empty(v.size, np.complex128); cast_into(g, gh.numpy()); t4 = time.perf_counter()
    for k, dt in zip(T2, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
        T2[k].append(dt * 1e3)
print("hostalloc", {k: round(float(np.median(x)), 3) for k, x in T2.items()})
