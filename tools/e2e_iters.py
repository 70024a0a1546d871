"""Per-call wall time of the reference-signature loss_and_grad (numpy complex128) in a fresh process."""
import time

import numpy as np
import torch

from paper_2311_16100_b200 import optim as Opt, synth
from paper_2311_16100_b200.forward import DatasetOperator

import sys
NI = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=NI)
op = DatasetOperator.from_engine(wl.engine)
v = (wl.v_true * 0.9).astype(np.complex128)
rng = np.random.default_rng(0)
ts = []
for i in range(50):
    rows = rng.choice(NI, 512, replace=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loss, grad = Opt.loss_and_grad(op, v, rows, 1e-3, 50000)
    ts.append((time.perf_counter() - t0) * 1e3)
print("per-call ms:", " ".join(f"{t:.2f}" for t in ts))
