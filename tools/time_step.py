"""Device time of each Algorithm-1 step kernel (CUDA events, warm, eager) on cfg3 with 4096 images."""
import numpy as np
import torch

from paper_2311_16100_b200 import synth, _capi as C

wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=4096)
e = wl.engine
M3 = e.M ** 3
B = 512
v = torch.from_numpy((wl.v_true * 0.5).astype(np.complex64)).cuda()
acc = torch.zeros(M3, dtype=torch.complex64, device="cuda")
fold = torch.zeros(M3, dtype=torch.float32, device="cuda")
d_avg = torch.zeros(M3, dtype=torch.float32, device="cuda")
d = torch.ones(M3, dtype=torch.float32, device="cuda")
dirv = torch.empty(M3, dtype=torch.complex64, device="cuda")
st = e.new_armijo_state(1.0)
idx = torch.from_numpy(np.random.default_rng(0).choice(e.n_images, B, replace=False).astype(np.int32)).cuda()
zb = e.gen_probes(1, 5)
p = C.StepParams(scale=8.0, lam=1e-3, beta=0.9, floor=1.0, w_old=0.5, w_new=0.5, hutch_scale=8.0, estimating=1)
sq = torch.zeros(1, dtype=torch.float64, device="cuda")


def tm(name, fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {a.elapsed_time(b) / reps * 1e3:9.1f} us", flush=True)


tm("gen_probes k=1", lambda: e.gen_probes(1, 5))
tm("hutch_fold k=1 (tile)", lambda: e.hutch_fold(zb, 1, idx, acc=fold))
tm("loss_grad_sorted", lambda: e.loss_grad(v, idx, acc=acc))
tm("loss_grad_hutch_sorted", lambda: e.loss_grad_hutch(v, idx, zb, acc, fold))
vol4 = e.precond_step(acc, v, p, dirv, fold=fold, d_avg=d_avg, d=d)
tm("precond_step", lambda: e.precond_step(acc, v, p, dirv, fold=fold, d_avg=d_avg, d=d))
p0 = C.StepParams(scale=8.0, lam=1e-3, beta=0.9, floor=1.0, w_old=0.5, w_new=0.5, hutch_scale=8.0, estimating=0)
tm("precond_step (fixed dhat)", lambda: e.precond_step(acc, v, p0, dirv))
tm("armijo_terms (tile)", lambda: e.armijo_terms(v, dirv, idx))
tm("proj_energy (brick)", lambda: e.proj_energy(dirv, idx))
qq = e.proj_energy(dirv, idx)
plan = e.make_plan(idx.view(1, -1))
tm("loss_grad_planned (+probe)", lambda: e.loss_grad_planned(v, plan, 0, acc, zbits=zb, fold=fold))
tm("proj_energy_planned", lambda: e.proj_energy_planned(dirv, plan, 0))
tm("armijo_select", lambda: e.armijo_select(sq, vol4[4:5], qq, vol4, 8.0, 1e-3, 0.5, st))
tm("apply_step", lambda: e.apply_step(v, dirv, st))
tm("norm2", lambda: e.norm2(v))
