"""nn-mode loss+grad: table-driven brick kernel vs the per-pixel tile kernel (device ms per call, B images)."""
import sys

import numpy as np
import torch

from paper_2311_16100_b200 import synth
from paper_2311_16100_b200.engine import SliceEngine, records_for

M = int(sys.argv[1]) if len(sys.argv) > 1 else 128
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
cfg = synth.Config("nn", M, 4096, "nn", False, False, 0.1, B)
wl = synth.build_workload(cfg, seed=0)
e = wl.engine
tile = SliceEngine(M, "nn", e.mask, records_for(M, wl.quats), e.x_masked(), tile_path=True)
v = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).cuda()
rng = np.random.default_rng(0)
for name, eng in (("tables", e), ("tile", tile)):
    acc = eng.new_cacc()
    ts = []
    for rep in range(10):
        idx = eng.idx_tensor(rng.choice(eng.n_images, B, replace=False))
        acc.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.loss_grad(v, idx, acc=acc)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"M={M} B={B} {name:7s} ms median {np.median(ts[2:]):.4f} -> {B / np.median(ts[2:]) * 1e3 / 1e6:.2f} M img/s",
          flush=True)
