"""GPU: the data-parallel step's default per-rank compute (B200 engine) at world size 1."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

import paper_2311_16100_b200 as F
from paper_2311_16100_b200 import dist as D
from paper_2311_16100_b200 import synth
from paper_2311_16100_b200.forward import DatasetOperator

pytestmark = pytest.mark.gpu


def test_sharded_step_world1_matches_loss_and_grad_and_probe_fold():
    wl = synth.build_workload(synth.CONFIGS["cfg2"], seed=0, n_images=256)
    op = DatasetOperator.from_engine(wl.engine)
    e = wl.engine
    batch = np.arange(0, 256, 3)
    lam = 1e-3
    v = torch.from_numpy((wl.v_true * 0.95).astype(np.complex64)).cuda()
    z = np.random.default_rng(0).integers(0, 2, size=(4, e.n_voxels)).astype(np.float64) * 2 - 1
    zbits, k = e.pack_probes(z)
    loss, grad, hs = D.sharded_step(op, v, batch, lam, zbits=zbits, k=k)
    loss_ref, grad_ref = F.loss_and_grad(op, v, torch.from_numpy(batch).cuda(), lam)
    assert abs(float(loss) - float(loss_ref)) / float(loss_ref) < 1e-6
    assert O.relative_l2(grad.cpu().numpy(), grad_ref.cpu().numpy()) < 1e-5  # two runs of fp32 atomics: order differs
    from paper_2311_16100_b200.optim import hutchinson_sample
    hs_ref, _ = hutchinson_sample(op, z, batch, lam)
    assert O.relative_l2(hs.cpu().numpy(), hs_ref) < 1e-6


def test_sharded_step_with_ball_compaction_matches_full_buffer():
    """The touched-ball compacted all-reduce buffer gives the same step as the full one (world 1)."""
    from paper_2311_16100_b200.grid import touched_ball
    wl = synth.build_workload(synth.CONFIGS["cfg2"], seed=1, n_images=256)
    op = DatasetOperator.from_engine(wl.engine)
    e = wl.engine
    batch = np.arange(1, 256, 3)
    lam = 1e-3
    v = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).cuda()
    zbits = e.gen_probes(1, 3)
    ball = touched_ball(e.M, e.M // 2 - 1)
    assert ball.size < e.n_voxels
    buf = D.PackedBuffer.new(e.n_voxels, True, torch.device("cuda"), ball=ball)
    assert buf.flat.numel() == 3 * ball.size + 2
    l1, g1, h1 = D.sharded_step(op, v, batch, lam, buf=buf, zbits=zbits, k=1)
    l2, g2, h2 = D.sharded_step(op, v, batch, lam, zbits=zbits, k=1)
    assert abs(float(l1) - float(l2)) / float(l2) < 1e-6
    assert O.relative_l2(g1.cpu().numpy(), g2.cpu().numpy()) < 1e-5
    assert O.relative_l2(h1.cpu().numpy(), h2.cpu().numpy()) < 1e-5


def _run_worker(rank, world_size, port, out_path, name, seed, shard=False):
    """One rank of a data-parallel optim.run (functional check: both ranks on cuda:0, gloo exchange)."""
    import torch.distributed as dist
    from conftest import load_golden
    from test_gpu_step import golden_stack
    from paper_2311_16100_b200 import optim as Opt
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world_size)
    g = load_golden(name)
    stack = golden_stack(g, seed)
    cfg = Opt.OptimConfig(lam=float(g["lam"]), batch_size=int(g["batch"].size), epochs=3, seed=seed,
                          mode=str(g["mode"]))
    vol, tr = Opt.run(cfg, stack, shard_dataset=shard)
    np.savez(out_path + f".{rank}.npz", v=vol.values, etas=np.array(tr.accepted_etas),
             f0=np.array(tr.step_f0), loss=tr.loss)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,seed,shard", [("dataset_m16_tri.npz", 4, False), ("dataset_m16_tri.npz", 4, True)])
def test_data_parallel_run_matches_single_process(golden, name, seed, shard):
    """optim.run with world_size 2 (each rank half of every batch, one compacted all-reduce per step;
    shard: each rank holds only half of the images and takes the batch images of its range)
    reproduces the single-process device run and the reference trajectory."""
    import os
    import socket
    import tempfile
    import torch.multiprocessing as mp
    from test_gpu_step import golden_stack
    from paper_2311_16100_b200 import optim as Opt
    g = golden(name)
    cfg = Opt.OptimConfig(lam=float(g["lam"]), batch_size=int(g["batch"].size), epochs=3, seed=seed,
                          mode=str(g["mode"]))
    vol1, tr1 = Opt.run(cfg, golden_stack(g, seed))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r")
        mp.start_processes(_run_worker, args=(2, port, out, name, seed, shard), nprocs=2, start_method="spawn")
        r0, r1 = np.load(out + ".0.npz"), np.load(out + ".1.npz")
    assert np.array_equal(r0["etas"], r1["etas"]) and np.array_equal(r0["v"], r1["v"])  # identical ranks
    assert np.array_equal(r0["etas"], np.array(tr1.accepted_etas))
    assert np.array_equal(r0["etas"][:10], g["sgd_rec"][:, 1])
    assert np.max(np.abs(r0["f0"] - np.array(tr1.step_f0)) / np.abs(np.array(tr1.step_f0))) < 1e-5
    assert O.relative_l2(r0["v"], vol1.values) < 1e-5
