"""Time the binning kernels of a 20-batch plan (cfg3 shapes) -- run under ncu for per-kernel durations."""
import numpy as np
import torch
from paper_2311_16100_b200 import synth
wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=8192)
e = wl.engine
rng = np.random.default_rng(0)
b = np.stack([rng.choice(e.n_images, 512, replace=False) for _ in range(20)])
for rep in range(3):
    p = e.make_plan(b)
torch.cuda.synchronize()
a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a0.record()
p = e.make_plan(b)
a1.record()
torch.cuda.synchronize()
print("plan build ms", a0.elapsed_time(a1))
