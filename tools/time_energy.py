"""Device time of the planned projection-energy pass (the line-search gather) at cfg3, B=512."""
import numpy as np
import torch

from paper_2311_16100_b200 import synth

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=4096)
e = wl.engine
v = torch.from_numpy((wl.v_true * 0.5).astype(np.complex64)).cuda()
rng = np.random.default_rng(0)
batches = torch.stack([torch.from_numpy(rng.choice(e.n_images, 512, replace=False).astype(np.int32))
                       for _ in range(8)]).cuda()
plan = e.make_plan(batches)
for rep in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(8):
        q = e.proj_energy_planned(v, plan, k)
    b.record()
    torch.cuda.synchronize()
    print(f"proj_energy_planned {a.elapsed_time(b) / 8 * 1e3:.1f} us  {float(q):.9e}")
