import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from oracle import oracle as O
import paper_2311_16100_b200 as F
from test_gpu_parity import golden_ops
g = dict(np.load("tests/golden/dataset_m16_tri.npz", allow_pickle=True))
op, oop = golden_ops(g)
lam = float(g["lam"]); idx = np.arange(op.n_images)
for name, z in (("z", g["z"]), ("v1", g["v1"])):
    a = op.hvp(z, idx, lam); b = oop.hvp(z, idx, lam)
    print(name, "rel", O.relative_l2(a, b), "repeat", O.relative_l2(op.hvp(z, idx, lam), a))
