"""Debug: device time of one fsld_loss_grad call (brick vs tile) with CUDA events, repeated."""
import numpy as np
import torch

from paper_2311_16100_b200 import synth, _capi as C
from paper_2311_16100_b200.engine import SliceEngine, records_for, ctypes_ptr, _stream
from paper_2311_16100_b200.grid import disk_mask

M, B, N = 128, 512, 4096
mask = disk_mask(M, M // 2 - 1)
q = synth.haar_quaternions(N, 1)
recs = records_for(M, q, synth.normal_shifts(N, 2), synth.physical_ctfs(N, 3))
x = torch.randn((N, mask.size), dtype=torch.complex64, device="cuda")
lib = C.load()
v = torch.from_numpy(synth.gaussian_blob_volume(M, 1).astype(np.complex64)).cuda()
for flags, name in ((0, "brick"), (C.TILE_PATH, "tile")):
    eng = SliceEngine(M, "tri", mask, recs, x)
    scr = eng.scratch(B)
    acc = torch.zeros(M ** 3, dtype=torch.complex64, device="cuda")
    sq = torch.zeros(1, dtype=torch.float64, device="cuda")
    rng = np.random.default_rng(0)
    ts = []
    for rep in range(12):
        idx = torch.from_numpy(rng.choice(N, B, replace=False).astype(np.int32)).cuda()
        acc.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st = lib.fsld_loss_grad(M, 1, eng.n_mask, ctypes_ptr(eng.pix), ctypes_ptr(eng.recs), ctypes_ptr(idx), B,
                                ctypes_ptr(v), ctypes_ptr(eng.x), ctypes_ptr(acc), ctypes_ptr(sq), flags, 0,
                                ctypes_ptr(scr), scr.numel() * 8, _stream())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        nz = int((acc != 0).sum())
    print(name, "status", st, "ms", [round(t, 4) for t in ts], "nonzero", nz, "sq", float(sq), flush=True)
