"""Algorithm-1 step loop shared by the oracle and the GPU parity tests.

Mirrors optim.run's per-batch sequence (/root/reference/pkg/src/fsld/optim.py:362-382):
z -> hutchinson_update -> ema_and_threshold -> loss_and_grad -> armijo_search,
recording (f0, eta, f_next, backtracks) per step, which run() itself does not
(it records etas only).  ``ns`` supplies the five primitives plus
``rademacher``/``epoch_batches``/``z_stream``/``new_state``.
"""
import numpy as np


def sgd_harness(ns, op, n_voxels, n_images, lam, alpha, batch_size, seed, n_steps,
                beta=0.9, c=0.5, eta0=1.0):
    state = ns.new_state(n_voxels, alpha)
    z_rng = ns.z_stream(seed)
    v = np.zeros(n_voxels, dtype=np.complex128)
    eta = eta0
    rec = []
    step = 0
    epoch = 0
    while step < n_steps:
        for batch in ns.epoch_batches(n_images, batch_size, seed, epoch):
            if step == n_steps:
                break
            z = ns.rademacher(z_rng, n_voxels)
            ns.hutchinson_update(state, op, z, batch, lam)
            dhat = ns.ema_and_threshold(state, beta, alpha, True)
            f0, grad = ns.loss_and_grad(op, v, batch, lam)
            eta, v, f_next, nbt = ns.armijo_search(
                v, grad, dhat, lambda w: ns.batch_loss(op, w, batch, lam), eta, c, f0)
            rec.append((f0, eta, f_next, nbt))
            step += 1
        epoch += 1
    return np.array(rec), v, state
