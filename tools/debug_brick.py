"""Debug: run the brick loss+grad repeatedly on one engine and dump the work-item counters."""
import numpy as np
import torch

from paper_2311_16100_b200 import synth, _capi as C
from paper_2311_16100_b200.engine import SliceEngine, records_for
from paper_2311_16100_b200.grid import disk_mask

M, B, N = 128, 512, 2048
mask = disk_mask(M, M // 2 - 1)
q = synth.haar_quaternions(N, 1)
recs = records_for(M, q, synth.normal_shifts(N, 2), synth.physical_ctfs(N, 3))
x = torch.randn((N, mask.size), dtype=torch.complex64, device="cuda")
fast = SliceEngine(M, "tri", mask, recs, x)
tile = SliceEngine(M, "tri", mask, recs, x, tile_path=True)
v = torch.from_numpy(synth.gaussian_blob_volume(M, 1).astype(np.complex64)).cuda()
rng = np.random.default_rng(0)
lib = C.load()
nb = (M + 7) // 8
for rep in range(4):
    idx = rng.choice(N, B, replace=False)
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    sq1, a1, _ = fast.loss_grad(v, idx)
    t1.record()
    torch.cuda.synchronize()
    sq2, a2, _ = tile.loss_grad(v, idx)
    torch.cuda.synchronize()
    scr = fast._scratch
    # ctl lives at layout offset; recompute offsets like scratch_layout
    def al(x): return (x + 255) & ~255
    o = 0; o = al(o + 256); o = al(o + 4 * M * M); o = al(o + 4 * M); o = al(o + 4 * M)
    nbr = nb ** 3
    cnt_off = o; o = al(o + 4 * nbr); o = al(o + 4 * (nbr + 1)); o = al(o + 4 * nbr)
    capp = B * min(nbr, 4 * nb * nb); o = al(o + 4 * capp); capi = nbr + capp // 32 + 1; o = al(o + 16 * capi)
    ctl = scr.view(torch.int32)[o // 4: o // 4 + 4].cpu().numpy()
    cnt = scr.view(torch.int32)[cnt_off // 4: cnt_off // 4 + nbr].cpu().numpy()
    e1 = a1.cpu().numpy(); e2 = a2.cpu().numpy()
    print(rep, "ms", t0.elapsed_time(t1), "ctl", ctl, "pairs", cnt.sum(), "bricks", (cnt > 0).sum(),
          "sq rel", abs(float(sq1) - float(sq2)) / float(sq2),
          "acc rel", np.linalg.norm(e1 - e2) / np.linalg.norm(e2), flush=True)
