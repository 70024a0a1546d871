"""Device time of the full-dataset loss pass (optim.run's per-epoch loss) at cfg3 (50,000 images)."""
import numpy as np
import torch

from paper_2311_16100_b200 import synth

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0)
e = wl.engine
v = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).cuda()
idx = e.all_indices()
for _ in range(2):
    e.loss(v, idx)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    sq = e.loss(v, idx)
b.record()
torch.cuda.synchronize()
print(f"full-dataset loss ({idx.numel()} images): {a.elapsed_time(b) / 5:.3f} ms  sq={float(sq):.6e}")
