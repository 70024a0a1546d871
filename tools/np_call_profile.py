import cProfile, pstats, sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2311_16100_b200 import synth, optim as Opt
from paper_2311_16100_b200.forward import DatasetOperator
wl = synth.build_workload(synth.CONFIGS["cfg3"], seed=0, n_images=4096)
op = DatasetOperator.from_engine(wl.engine)
v = (wl.v_true * 0.9).astype(np.complex128).reshape(-1)
rng = np.random.default_rng(0)
rows = [rng.choice(4096, 512, replace=False) for _ in range(300)]
for i in range(30):
    l, g = Opt.loss_and_grad(op, v, rows[i], 1e-3, 50000)
pr = cProfile.Profile()
pr.enable()
for i in range(30, 230):
    l, g = Opt.loss_and_grad(op, v, rows[i], 1e-3, 50000)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
