"""Timeline of the pipelined host step (torch.profiler / CUPTI): copies and kernels of one call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_16100_b200 import synth  # noqa: E402
from paper_2311_16100_b200.forward import DatasetOperator  # noqa: E402

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=4096)
op = DatasetOperator.from_engine(wl.engine)
M = 128
v_h = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).pin_memory()
g_h = torch.empty(M ** 3, dtype=torch.complex64).pin_memory()
gen = np.random.default_rng(1)
idx = [torch.from_numpy(gen.choice(4096, 512, replace=False).astype(np.int32)).pin_memory() for _ in range(8)]
for i in range(4):
    op.loss_and_grad_host(v_h, idx[i], 1e-3, g_h)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(4):
    op.loss_and_grad_host(v_h, idx[i], 1e-3, g_h)
print(f"wall per call {(time.perf_counter() - t0) / 4 * 1e3:.3f} ms")
t0 = time.perf_counter()
for i in range(20):
    op.engine.loss_grad_host(v_h, idx[i % 8], 98.0, 1e-3, g_h, op._host_stage["out_h"], op._host_stage)
print(f"enqueue only per call {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for i in range(2):
        op.loss_and_grad_host(v_h, idx[i], 1e-3, g_h)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t_first = evs[0].time_range.start
for e in evs:
    print(f"{(e.time_range.start - t_first):9.1f} {(e.time_range.end - t_first):9.1f} us  {e.name[:70]}")
