"""Per-phase cycle accounting of the brick kernel's item loop (debug hook fsld_debug_phase_profile)."""
import ctypes

import numpy as np
import torch

from paper_2311_16100_b200 import synth, _capi as C
from paper_2311_16100_b200.engine import ctypes_ptr

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=4096)
eng = wl.engine
lib = C.load()
lib.fsld_debug_phase_profile.argtypes = [ctypes.c_void_p]
buf = torch.zeros(9, dtype=torch.int64, device="cuda")
v = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).cuda()
rng = np.random.default_rng(0)
for rep in range(2):
    idx = rng.choice(eng.n_images, 512, replace=False)
    eng.loss_grad(v, idx)
torch.cuda.synchronize()
lib.fsld_debug_phase_profile(ctypes_ptr(buf))
reps = 5
for rep in range(reps):
    idx = rng.choice(eng.n_images, 512, replace=False)
    eng.loss_grad(v, idx)
torch.cuda.synchronize()
lib.fsld_debug_phase_profile(None)
b = buf.cpu().numpy().astype(np.float64)
items = b[8]
names = ["setup", "bk+round", "pass1", "pass2", "-", "-", "-", "flush"]  # PHASE_MARK ids of fsld_brick_main.cuh
tot = b[:8].sum()
print(f"items/launch {items / reps:.0f}  cycles/item {tot / items:.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:12s} {b[i] / items:9.0f} cyc/item  {100 * b[i] / tot:5.1f}%")
