"""Timeline of the numpy-signature host step (torch.profiler / CUPTI): copies and kernels of one call."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_16100_b200 import synth  # noqa: E402
from paper_2311_16100_b200.forward import DatasetOperator  # noqa: E402

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=4096)
op = DatasetOperator.from_engine(wl.engine)
v = (wl.v_true * 0.9).astype(np.complex128).reshape(-1)
gen = np.random.default_rng(1)
rows = [gen.choice(4096, 512, replace=False) for _ in range(8)]
for i in range(6):
    op.loss_and_grad_numpy(v, rows[i], 1e-3, 50000)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for i in range(2):
        op.loss_and_grad_numpy(v, rows[i], 1e-3, 50000)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t_first = evs[0].time_range.start
for e in evs:
    print(f"{(e.time_range.start - t_first):9.1f} {(e.time_range.end - t_first):9.1f} us  {e.name[:60]}")
