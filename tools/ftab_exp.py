"""EXPERIMENT: brick loss+grad with a precomputed per-pixel f table vs in-kernel CTF/phase."""
import ctypes
import numpy as np
import torch
from paper_2311_16100_b200 import synth, _capi as C
from paper_2311_16100_b200.engine import ctypes_ptr, _stream

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=4096)
e = wl.engine
lib = C.load()
lib.fsld_debug_ftab.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
ftab = torch.empty_like(e.x)
v = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).cuda()
rng = np.random.default_rng(0)
idxs = [torch.from_numpy(rng.choice(e.n_images, 512, replace=False).astype(np.int32)).cuda() for _ in range(12)]


def timeit():
    acc = torch.zeros(e.n_voxels, dtype=torch.complex64, device="cuda")
    ts = []
    sqs = []
    for idx in idxs:
        acc.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sq, _, _ = e.loss_grad(v, idx, acc=acc)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        sqs.append(float(sq))
    return np.min(ts), np.median(ts), sqs[-1], acc.clone()


t0 = timeit()
lib.fsld_debug_ftab(ctypes_ptr(e.recs), ctypes_ptr(e.pc), e.n_images, e.n_mask, ctypes_ptr(ftab))
t1 = timeit()
lib.fsld_debug_ftab(None, None, 0, 0, None)
print("in-kernel f: min %.4f med %.4f sq %.6e" % t0[:3])
print("f table    : min %.4f med %.4f sq %.6e" % t1[:3])
print("grad rel", float((t0[3] - t1[3]).abs().norm() / t0[3].abs().norm()))
