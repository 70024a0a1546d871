"""Device time of one fused loss+grad call (brick-sorted vs tile path), CUDA events around the C call only."""
import sys

import numpy as np
import torch

from paper_2311_16100_b200 import synth, _capi as C
from paper_2311_16100_b200.engine import SliceEngine, ctypes_ptr, _stream

M = int(sys.argv[1]) if len(sys.argv) > 1 else 128
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
cfg = synth.CONFIGS["cfg3"] if M == 128 else synth.Config("x", M, 4096, "tri", True, True, 0.05, B)
wl = synth.build_workload(cfg, seed=0, n_images=4096)
eng = wl.engine
lib = C.load()
v = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).cuda()
scr = eng.scratch(B)
for flags, name in ((0, "brick"), (C.TILE_PATH, "tile")):
    acc = torch.zeros(M ** 3, dtype=torch.complex64, device="cuda")
    sq = torch.zeros(1, dtype=torch.float64, device="cuda")
    rng = np.random.default_rng(0)
    ts = []
    for rep in range(12):
        idx = torch.from_numpy(rng.choice(eng.n_images, B, replace=False).astype(np.int32)).cuda()
        acc.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st = lib.fsld_loss_grad_sorted(M, 1, eng.n_mask, ctypes_ptr(eng.recs), ctypes_ptr(idx), B, ctypes_ptr(v),
                                       ctypes_ptr(eng.x), ctypes_ptr(eng.pc), ctypes_ptr(eng.ptab), ctypes_ptr(eng.seg_off),
                                       ctypes_ptr(eng.segs), ctypes_ptr(acc), ctypes_ptr(sq), flags, 0,
                                       ctypes_ptr(scr), scr.numel() * 8, _stream())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name:6s} status {st} ms min {min(ts):.4f} med {np.median(ts):.4f}  sq {float(sq):.6e} |acc| "
          f"{float(acc.abs().sum()):.6e}", flush=True)
