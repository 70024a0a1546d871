"""Repro: golden m16 tri SGD harness through the numpy loss_and_grad path (host step)."""
import faulthandler
import sys

faulthandler.enable()
sys.path.insert(0, "tests")
import numpy as np

from conftest import load_golden
from harness import sgd_harness
from test_gpu_parity import _GpuNS, golden_ops

g = load_golden("dataset_m16_tri.npz")
op, _ = golden_ops(g)
print("op ok", flush=True)
for rep in range(3):
    rec, v, st = sgd_harness(_GpuNS, op, op.spec.M ** 3, op.n_images, float(g["lam"]), float(g["alpha"]),
                             int(g["batch"].size), 4, 10)
    print("rep", rep, rec[:2, 1], flush=True)
