"""Host-side profile of optim.run at cfg3 (where the per-step wall time goes beyond the kernels)."""
import cProfile
import pstats
import sys
import time
from types import SimpleNamespace

import torch

from paper_2311_16100_b200 import optim, synth
from paper_2311_16100_b200.forward import DatasetOperator
from paper_2311_16100_b200.grid import GridSpec

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0)
eng = wl.engine
spec = GridSpec(eng.M)
stack = SimpleNamespace(spec=spec, mask_radius=eng.M // 2 - 1, n_images=eng.n_images, ctfs=wl.ctfs, poses=None)
op = DatasetOperator.from_engine(eng, spec)
alpha = optim.threshold_alpha(stack, None, 1e-3)
conf = optim.OptimConfig(lam=1e-3, batch_size=512, epochs=epochs, variant="estimated", seed=0)
optim.run(conf, stack, probes="device", op=op, alpha=alpha)
torch.cuda.synchronize()
t = time.perf_counter()
optim.run(conf, stack, probes="device", op=op, alpha=alpha)
torch.cuda.synchronize()
print("run s", time.perf_counter() - t, "per step ms", 1e3 * (time.perf_counter() - t) / (98 * epochs))
pr = cProfile.Profile()
pr.enable()
optim.run(conf, stack, probes="device", op=op, alpha=alpha)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
