"""`fsld` -- the reference package's import name, served by the B200 path (north_star: "keep the
reference package's Python API ... in pkg/src, so the new code is a drop-in for that path").

    PYTHONPATH=<repo>/pkg/src python -c "import fsld; print(fsld.loss_and_grad)"

resolves every public name of the reference's `fsld` (forward / optim / hessian / grid / metrics /
kernels / io / errors) to paper_2311_16100_b200, whose compute runs in the sm_100a kernels of
libfsld_b200.so (no CPU fallback).  The reference's CLI / config front-end (cli.py, config.py) is out
of scope and not provided.
"""
import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import paper_2311_16100_b200 as _b200  # noqa: E402
from paper_2311_16100_b200 import *  # noqa: E402,F401,F403

__all__ = list(_b200.__all__)
__version__ = _b200.__version__

# fsld.<submodule> -> paper_2311_16100_b200.<submodule> (import fsld.optim, from fsld.kernels import ...)
for _name in ("errors", "forward", "grid", "hessian", "io", "kernels", "metrics", "optim"):
    _mod = importlib.import_module(f"paper_2311_16100_b200.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
del _name, _mod
