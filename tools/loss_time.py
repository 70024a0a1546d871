"""Device time of the full-dataset loss (the epoch-end term of optim.run) at cfg3."""
import torch

from paper_2311_16100_b200 import synth

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0)
eng = wl.engine
v = torch.from_numpy((wl.v_true * 0.9).astype("complex64")).cuda()
idx = eng.all_indices()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sq = eng.loss(v, idx)
    e1.record()
    torch.cuda.synchronize()
    print(f"full loss over {idx.numel()} images: {e0.elapsed_time(e1):.3f} ms  sq {float(sq):.9e}")
b = idx[:512]
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    q = eng.proj_energy(v, b)
    e1.record()
    torch.cuda.synchronize()
    print(f"energy 512: {e0.elapsed_time(e1):.3f} ms")
