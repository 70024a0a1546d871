"""Relative L2 errors of the table-driven kernel against the fp64 oracle (cfg3 subset B=512, cfg2 subset,
golden M=16): the precision headroom of the fixed-point scatter."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
import cfg_data
from oracle import oracle as O
from conftest import load_golden
import paper_2311_16100_b200 as F

for name, (M, n, snr) in {"cfg3": (128, 1024, 0.05), "cfg2": (64, 2048, 0.05), "hisnr64": (64, 1024, 50.0)}.items():
    d = cfg_data.make(M, n, "tri", ctf=True, shifts=True, snr=snr)
    op = cfg_data.gpu_operator(d)
    batch = np.random.default_rng(1).permutation(n)[:512]
    for fac in (0.9, 0.999):
        v1 = (fac * d.v_true).astype(np.complex64).astype(np.complex128)
        lg, gg = F.loss_and_grad(op, v1, batch, 1e-3)
        lr, gr = O.loss_and_grad(d.oop, v1, batch, 1e-3)
        print(f"{name} v={fac}: loss rel {abs(lg - lr) / lr:.2e}  grad rel {O.relative_l2(gg, gr):.2e}", flush=True)
        if name == "hisnr64":  # the oracle on the device's inputs (images rounded to complex64)
            x64 = d.oop.x
            d.oop.x = x64.astype(np.complex64).astype(np.complex128)
            lr2, gr2 = O.loss_and_grad(d.oop, v1, batch, 1e-3)
            d.oop.x = x64
            print(f"{name} v={fac} (oracle on complex64 images): grad rel {O.relative_l2(gg, gr2):.2e}  "
                  f"|grad| / |lam v| {np.linalg.norm(gr) / (1e-3 * np.linalg.norm(v1)):.3e}", flush=True)
g = load_golden("dataset_m16_tri.npz")
