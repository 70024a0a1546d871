"""GPU: bench.py's multi-rank modes, as the driver runs them.

* `python bench.py --gpus 2` with no torchrun environment re-launches itself under
  torch.distributed.run (2 ranks); on a 1-GPU box FSLD_BENCH_SINGLE_DEVICE=1 puts both ranks on
  cuda:0 with a gloo exchange (functional check: sharded dataset, the packed all-reduce, max-over-
  ranks timing, n_gpus = 2).
* FSLD_BENCH_FORCE_DP=1 runs the data-parallel step on a one-rank group, captured in one CUDA graph:
  with FSLD_COMM=nccl the packed NCCL all-reduce inside the graph, by default the NVLS exchange
  (multicast flush + barrier kernels; the graph the N-GPU run replays).
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SMALL = ["--steps", "2", "--warmup", "3", "--images", "2048", "--no-cpu-baseline", "--no-e2e", "--no-algo1",
         "--no-sweep"]


def _run(args, **env):
    e = dict(os.environ, PYTHONPATH=ROOT, **env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0]), r.stderr


def test_gpus2_self_launches_two_ranks():
    line, _ = _run(["--gpus", "2", *SMALL], FSLD_BENCH_SINGLE_DEVICE="1")
    assert line["n_gpus"] == 2
    assert line["config"]["parallelism"] == "dp2"
    assert line["details"]["allreduce_bytes"] > 0 and line["details"]["collectives_per_step"] == 1
    assert line["details"]["n_images_per_gpu"] == 1024  # 2,048 images sharded over 2 ranks
    assert line["value"] > 0 and line["scaling"] == "weak"


def test_dp_step_graph_with_nccl_collective():
    line, _ = _run(SMALL, FSLD_BENCH_FORCE_DP="1", FSLD_COMM="nccl")
    assert line["details"]["step"].startswith("CUDA graph replay"), line["details"]["step"]
    assert line["details"]["allreduce_bytes"] > 0
    assert line["value"] > 0


def test_dp_step_graph_with_nvls_exchange():
    """The default N > 1 exchange on NVSwitch: the brick pass flushes into the multicast accumulator
    (one-member team here), two barrier kernels, no all-reduce -- captured in the step's graph."""
    from paper_2311_16100_b200.dist import nvls_available

    line, _ = _run(SMALL, FSLD_BENCH_FORCE_DP="1")
    d = line["details"]
    assert d["step"].startswith("CUDA graph replay"), d["step"]
    assert line["value"] > 0
    if nvls_available(0):
        assert d["exchange"].startswith("NVLS"), d["exchange"]
        assert d["allreduce_bytes"] == 0 and d["collectives_per_step"] == 0
    else:  # no multicast on this box: the NCCL exchange, and the line says why
        assert d["exchange"].startswith("nccl ("), d["exchange"]
        assert d["allreduce_bytes"] > 0
