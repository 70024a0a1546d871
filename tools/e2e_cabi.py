"""C-ABI host step (pinned complex64) per-call time under variations: dataset size, one idx buffer vs
one per call (the bench's e2e.c_abi leg uses one per call)."""
import sys
import time

import numpy as np
import torch

from paper_2311_16100_b200 import synth, _capi as C
from paper_2311_16100_b200.forward import DatasetOperator

NI = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=NI)
op = DatasetOperator.from_engine(wl.engine)
v = (wl.v_true * 0.9).astype(np.complex64).reshape(-1)
vh = C.host_empty(v.size, torch.complex64)
gh = C.host_empty(v.size, torch.complex64)
vh.numpy()[:] = v
rng = np.random.default_rng(0)
idx = []
for i in range(40):
    t = C.host_empty(512, torch.int32)
    t.numpy()[:] = rng.choice(NI, 512, replace=False)
    idx.append(t)
for mode in ("same", "distinct", "same"):
    for i in range(5):
        op.loss_and_grad_host(vh, idx[0], 1e-3, gh, 50000)
    ts = []
    for i in range(30):
        t0 = time.perf_counter()
        op.loss_and_grad_host(vh, idx[0] if mode == "same" else idx[i + 5], 1e-3, gh, 50000)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(NI, mode, "median ms", round(float(np.median(ts)), 3), "min", round(float(np.min(ts)), 3))

# the bench's sequence: the numpy-signature leg first (holding each result until the next returns)
from paper_2311_16100_b200 import optim as Opt
vn = (wl.v_true * 0.9).astype(np.complex128)
for i in range(50):
    loss, grad = Opt.loss_and_grad(op, vn, rng.choice(NI, 512, replace=False), 1e-3, 50000)
for mode in ("after-numpy same", "after-numpy distinct"):
    ts = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20):
        op.loss_and_grad_host(vh, idx[0] if "same" in mode else idx[i + 5], 1e-3, gh, 50000)
    e1.record()
    torch.cuda.synchronize()
    print(NI, mode, "events ms per call", round(e0.elapsed_time(e1) / 20, 3))
del grad
for i in range(3):
    op.loss_and_grad_host(vh, idx[0], 1e-3, gh, 50000)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20):
    op.loss_and_grad_host(vh, idx[0], 1e-3, gh, 50000)
e1.record()
torch.cuda.synchronize()
print(NI, "after releasing the numpy result", "events ms per call", round(e0.elapsed_time(e1) / 20, 3))
