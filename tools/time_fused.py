"""Device time of the loss+grad step at cfg3 (B=512): accumulator path (planned brick pass + epilogue)
vs the fused-epilogue step (grad = lam v, brick pass adds scale * sums into grad, finalize)."""
import numpy as np
import torch

from paper_2311_16100_b200 import synth

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=8192)
e = wl.engine
v = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).cuda()
rng = np.random.default_rng(0)
K = 8
batches = np.stack([rng.choice(e.n_images, 512, replace=False) for _ in range(K)])
plan = e.make_plan(batches)
acc = torch.zeros(e.n_voxels, dtype=torch.complex64, device="cuda")
grad = torch.empty_like(acc)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
scale, lam = 50000 / 512, 1e-3


def old(k):
    sq = e.loss_grad_planned(v, plan, k, acc)
    e.epilogue(acc, v, scale, lam, sq, grad=grad)


def new(k):
    e.loss_grad_step_planned(v, plan, k, scale, lam, grad)


for name, fn in (("accumulator + epilogue", old), ("fused epilogue", new), ("accumulator + epilogue", old),
                 ("fused epilogue", new)):
    ts = []
    for k in range(K):
        flush.fill_(float(k))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(k)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{name:24s} {np.mean(ts[1:]) * 1e3:7.1f} us (mean of {K - 1})")
