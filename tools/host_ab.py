"""Interleaved A/B of the host-buffer step (fsld_loss_grad_host) over slab counts, in one process:
PCIe rates drift between runs and boxes, so every configuration is timed in every round."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_16100_b200 import _capi as C  # noqa: E402
from paper_2311_16100_b200 import synth  # noqa: E402
from paper_2311_16100_b200.forward import DatasetOperator  # noqa: E402

slabs = [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "1,4,6,8,10,12,16").split(",")]
N_IMG = int(os.environ.get("FSLD_AB_IMAGES", "8192"))
wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=N_IMG)
op = DatasetOperator.from_engine(wl.engine)
M, B = 128, 512
v_h = C.host_empty(M ** 3, torch.complex64)
v_h.copy_(torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)))
g_h = C.host_empty(M ** 3, torch.complex64)
gen = np.random.default_rng(3)
idx = []
for _ in range(16):
    t = C.host_empty(B, torch.int32)
    t.copy_(torch.from_numpy(gen.choice(N_IMG, B, replace=False).astype(np.int32)))
    idx.append(t)
res = {n: [] for n in slabs}
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rnd in range(6):
    for n in slabs:
        op.engine.HOST_SLABS = n
        for i in range(3):
            op.loss_and_grad_host(v_h, idx[i], 1e-3, g_h)
        torch.cuda.synchronize()
        a.record()
        for i in range(16):
            op.loss_and_grad_host(v_h, idx[i], 1e-3, g_h)
        b.record()
        torch.cuda.synchronize()
        res[n].append(a.elapsed_time(b) / 16)
for n in slabs:
    r = sorted(res[n])
    print(f"slabs {n:3d}: median {r[len(r) // 2]:.4f} ms  min {r[0]:.4f}  max {r[-1]:.4f}")
