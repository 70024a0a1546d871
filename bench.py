"""Benchmark: image-slices/s of the fused project+CTF+adjoint (loss+grad) step on B200.

Workload (BASELINE.json configs[2], "cfg3"): M=128 complex64 Gaussian-blob
volume, 50,000 masked 128x128 images (12,645 px each), trilinear slicing,
physical astigmatic CTF, N(0,2px) shifts, SNR 0.05, batch 512 images PER GPU
(weak scaling).  One step = zero the gradient accumulator + the fused
slice->CTF/shift->residual->|r|^2->adjoint kernel over one batch + the
fixed-order loss reduction + ||v||^2 + the gradient epilogue
(scale*acc + lam*v), and for N>1 one NCCL all-reduce of the packed
[gradient | loss] buffer.  Inputs are synthetic (seeded).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config cfg3]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--images", type=int, default=0, help="override dataset size (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-algo1", action="store_true", help="skip the full Algorithm-1 step leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the cfg5 Hutchinson probe sweep leg")
    ap.add_argument("--run-epochs", type=int, default=20,
                    help="cfg3: epochs of the full Algorithm-1 run leg (optim.run; 0 = skip)")
    ap.add_argument("--lam", type=float, default=1e-3)
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def algorithmic_bytes(M, n_mask, B):
    """Compulsory HBM bytes of one fused loss+grad launch:
    B*(8 n_mask [x, complex64] + 128 [record]) + 16 M^3 [read v + write grad]."""
    return B * (8 * n_mask + 128) + 16 * M ** 3


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML every ~0.5 ms (the timed
    region of a default run is only a few ms), nvidia-smi as the fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        flag = lambda bit: "Active" if r & bit else "Not Active"  # noqa: E731
        return [str(sm), str(mx), hex(r), flag(0x8), flag(0x40), flag(0x20), flag(0x4)]

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self.samples.append(self._sample_nvml())
                    self._stop.wait(0.0005)
                    continue
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def poll_until(self, event):
        """Sample (NVML) on the calling thread until the CUDA event has completed."""
        if self._nvml is None:
            return
        while not event.query():
            try:
                self.samples.append(self._sample_nvml())
            except Exception:
                return
            time.sleep(0.0002)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------
# CPU legs (oracle port: test infrastructure, only the checker / baseline)
# ---------------------------------------------------------------------------

def cpu_workload(cfg, n_images, seed=0):
    """Host-side copy of the workload for the C oracle (same generators, fp64)."""
    from oracle import oracle as O
    from paper_2311_16100_b200 import synth

    M = cfg.M
    mask = O.disk_mask(M, M // 2 - 1)
    pix = O.mask_pix(M, mask)
    v = synth.gaussian_blob_volume(M, seed)
    q = synth.haar_quaternions(n_images, seed + 1)
    sh = synth.normal_shifts(n_images, seed + 2) if cfg.shifts else np.zeros((n_images, 2))
    ctab = (O.ctf_table_physical(synth.ctf_param_array(synth.physical_ctfs(n_images, seed + 3)), pix, M)
            if cfg.ctf else None)
    op = O.OracleOperator(M, cfg.mode, mask, q, sh, ctab, None)
    clean = op.project(v, np.arange(n_images))
    sigma = np.sqrt(np.mean(np.abs(clean) ** 2) / cfg.snr)
    rng = np.random.default_rng(seed + 100)
    op.x = clean + (sigma / np.sqrt(2)) * (rng.standard_normal(clean.shape) + 1j * rng.standard_normal(clean.shape))
    return op, v


def reference_package():
    """The unmodified reference package installed in baseline/_ref (pip install --target; git-ignored,
    travels to the GPU box), or None.  Its numba kernels are the reference's own CPU path."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "fsld")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import fsld  # noqa: F401
        import fsld.optim  # noqa: F401
        return fsld
    except Exception:  # numba missing / broken install: fall back to the C port
        return None


def reference_operator(fsld, cfg, n_images, seed=0):
    """The reference's own DatasetOperator on the workload's images: poses and images from the same
    generators as the GPU arm; the reference computes its phase tables itself; its CTF table is the
    builder-defined physical CTF (the reference's radial ctf_eval cannot express it)."""
    oop, v = cpu_workload(cfg, n_images, seed)
    M = cfg.M
    spec = fsld.GridSpec(M)
    from paper_2311_16100_b200 import synth
    q = synth.haar_quaternions(n_images, seed + 1)
    sh = synth.normal_shifts(n_images, seed + 2) if cfg.shifts else np.zeros((n_images, 2))
    poses = [fsld.Pose(q=q[i], t=sh[i]) for i in range(n_images)]
    images = np.zeros((n_images, M * M), dtype=np.complex128)
    images[:, oop.mask] = oop.x
    stack = fsld.ImageStack(spec=spec, images=images, poses=poses, ctfs=None, sigma=1.0, seed=seed,
                            mask_radius=M // 2 - 1, mode=cfg.mode)
    op = fsld.DatasetOperator(stack)
    if cfg.ctf:
        op.ctf_vals = np.ascontiguousarray(oop.ctf_vals)
    return op, v


def time_reference(fsld, op, v, batch, lam, n_total, steps, warmup):
    from fsld import optim as ref_optim
    rng = np.random.default_rng(7)
    for _ in range(warmup):  # the first call JIT-compiles the numba kernels
        ref_optim.loss_and_grad(op, v, rng.choice(op.n_images, batch, replace=False), lam, n_total)
    t0 = time.perf_counter()
    for _ in range(steps):
        ref_optim.loss_and_grad(op, v, rng.choice(op.n_images, batch, replace=False), lam, n_total)
    return (time.perf_counter() - t0) / steps


def time_cpu(op, v, batch, lam, n_total, steps, warmup):
    from oracle import oracle as O

    rng = np.random.default_rng(7)
    for _ in range(warmup):
        O.loss_and_grad(op, v, rng.choice(op.n_images, batch, replace=False), lam, n_total)
    t0 = time.perf_counter()
    for _ in range(steps):
        O.loss_and_grad(op, v, rng.choice(op.n_images, batch, replace=False), lam, n_total)
    return (time.perf_counter() - t0) / steps


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def op_n_mask(op):
    """n_mask of a reference / oracle operator."""
    return op.n_mask if hasattr(op, "n_mask") else op.x.shape[1]


def run_reference(args):
    """--impl reference: the reference's own CPU path (its numba kernels, installed in baseline/_ref,
    all host threads) on this config; the C oracle port when the install is unavailable."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2311_16100_b200 import synth

    cfg = synth.CONFIGS[args.config]
    B = cfg.batch
    n_sub = min(cfg.n_images, max(4 * B, 2048))
    fsld = reference_package()
    threads = os.cpu_count() or 1
    if fsld is not None:
        import numba
        numba.set_num_threads(numba.config.NUMBA_NUM_THREADS)
        threads = numba.get_num_threads()
        op, v = reference_operator(fsld, cfg, n_sub)
        per = time_reference(fsld, op, v * 0.9, B, args.lam, cfg.n_images, args.steps, max(args.warmup, 1))
        kind = "reference"
        sample = (f"{args.steps} steps x {B} images drawn from a {n_sub}-image host subset, the reference's "
                  f"fsld.optim.loss_and_grad (numba {numba.__version__}, {threads} threads, {cpu_model()}); "
                  f"physical CTF table injected as op.ctf_vals")
    else:
        from oracle import oracle as O
        op, v = cpu_workload(cfg, n_sub)
        threads = O.max_threads()
        per = time_cpu(op, v * 0.9, B, args.lam, cfg.n_images, args.steps, args.warmup)
        kind = "port"
        sample = (f"{args.steps} steps x {B} images drawn from a {n_sub}-image host subset, C oracle "
                  f"(fp64, OpenMP {threads} threads, {cpu_model()})")
    val = B / per
    line = {
        "impl": "reference", "metric": "image-slices/sec (fused project+CTF+adjoint, loss+grad)",
        "value": val, "unit": "images/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generators of BASELINE cfg; SURVEY.md 8d)",
        "config": bench_config(cfg, cfg.M, int(op_n_mask(op)), B, args.gpus),
        "details": {"images_sampled_from": n_sub},
        "cpu_baseline": {"value": val, "unit": "images/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": val, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def bench_config(cfg, M, n_mask, B, world):
    """The workload identity, the same keys in both arms (B200 and --impl reference)."""
    return {"workload": cfg.name, "M": M, "n_mask": n_mask, "mode": cfg.mode, "batch_per_gpu": B,
            "n_images": cfg.n_images, "ctf": "physical astigmatic" if cfg.ctf else "none",
            "shifts": bool(cfg.shifts), "parallelism": f"dp{world}"}


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2311_16100_b200 import synth
    from paper_2311_16100_b200.engine import _stream, ctypes_ptr
    from paper_2311_16100_b200 import _capi as C

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FSLD_BENCH_SINGLE_DEVICE=1 (functional check of the multi-rank code path on a 1-GPU box: all
    # ranks on cuda:0, host-side gloo exchange; never a reported number)
    single = os.environ.get("FSLD_BENCH_SINGLE_DEVICE") == "1"
    if single:
        local = 0
    torch.cuda.set_device(local)
    # the data-parallel step (ball gather, packed all-reduce, scatter); FSLD_BENCH_FORCE_DP=1 runs it
    # on a one-rank NCCL group (functional check of the captured collective on a 1-GPU box)
    dp = world > 1 or os.environ.get("FSLD_BENCH_FORCE_DP") == "1"
    if dp and world == 1:  # a one-rank group: rendezvous defaults
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    if dp:
        if single:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[args.config]
    # images sharded across ranks (rank r holds images [r N/W, (r+1) N/W) of the N-image dataset);
    # every rank takes a batch of B of its own images per step (weak scaling, B per GPU)
    wl = synth.build_workload(cfg, seed=0, n_images=args.images or None, shard=(rank, world))
    # cfg1/cfg2 are full-dataset passes in BASELINE; the timed step uses 1024-image batches
    B = min(cfg.batch if args.config not in ("cfg1", "cfg2") else 1024, wl.engine.n_images)
    eng = wl.engine
    M, n = eng.M, eng.n_mask
    lib = C.load()
    dev = eng.dev
    lam = args.lam
    n_total = wl.n_total
    scale = n_total / (B * world)

    v = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).to(dev)
    acc = torch.zeros(M ** 3, dtype=torch.complex64, device=dev)
    # N > 1: the all-reduce moves only the voxels a scatter can reach (grid.touched_ball, ~54 % at M=128)
    from paper_2311_16100_b200.grid import touched_ball
    ball = torch.from_numpy(touched_ball(M, M // 2 - 1)).to(dev)
    nball = int(ball.numel())
    packed = torch.zeros(2 * nball + 2, dtype=torch.float32, device=dev)
    grad = torch.empty(M ** 3, dtype=torch.complex64, device=dev)
    sq = torch.empty(1, dtype=torch.float64, device=dev)
    nrm = torch.empty(1, dtype=torch.float64, device=dev)
    scr = eng.scratch(B)
    nscr = eng._norm_scratch()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    flush_mode = os.environ.get("FSLD_BENCH_FLUSH", "clean")
    flush_rd = torch.ones(L2_FLUSH_BYTES // 8, dtype=torch.float32, device=dev) if flush_mode == "clean" else None

    def l2_flush(i):
        if flush_mode == "none":
            return
        flush.fill_(float(i))
        if flush_rd is not None:  # read > L2 afterwards: the fill's dirty lines are written back now
            flush_rd.sum()
    gen = np.random.default_rng(1234 + rank)
    n_steps = args.warmup + args.steps
    batches = [torch.from_numpy(gen.choice(eng.n_images, B, replace=False).astype(np.int32)).to(dev)
               for _ in range(n_steps)]
    stream = _stream()
    flags = C.TILE_PATH if os.environ.get("FSLD_TILE_PATH") else 0
    # loss_grad: count + scan + fill + brick kernel + reduce (5 kernels, + cnt memset); fused epilogue (2)
    launches_per_step = (7 if eng.brick_path and not flags else 4) + (2 if dp else 0)

    loss = torch.empty(1, dtype=torch.float64, device=dev)

    def step(idx, ev_k0=None, ev_k1=None):
        # acc is zero on entry (zeroed by the previous step's fused epilogue)
        stream = _stream()  # the current torch stream (the capture stream under CUDA-graph capture)
        if ev_k0 is not None:
            ev_k0.record()
        C.check(lib.fsld_loss_grad_sorted(M, eng.mode_id, n, ctypes_ptr(eng.recs), ctypes_ptr(idx), B,
                                          ctypes_ptr(v), ctypes_ptr(eng.x), ctypes_ptr(eng.pc), ctypes_ptr(eng.ptab),
                                          ctypes_ptr(eng.seg_off), ctypes_ptr(eng.segs), ctypes_ptr(acc),
                                          ctypes_ptr(sq), flags, 0, ctypes_ptr(scr), scr.numel() * 8, stream),
                "loss_grad")
        if ev_k1 is not None:
            ev_k1.record()
        return finish_step(stream)

    def finish_step(stream):
        if dp:  # one packed all-reduce: [grad accumulator on the touched ball | loss hi, lo]
            C.check(lib.fsld_ball_gather(nball, ctypes_ptr(ball), ctypes_ptr(acc), ctypes_ptr(packed), 8, stream),
                    "ball_gather")
            s32 = sq.float()
            packed[-2:-1].copy_(s32)
            packed[-1:].copy_((sq - s32.double()).float())
            dist.all_reduce(packed)
            C.check(lib.fsld_ball_scatter(nball, ctypes_ptr(ball), ctypes_ptr(packed), ctypes_ptr(acc), 8, stream),
                    "ball_scatter")
            sq.copy_(packed[-2:-1].double() + packed[-1:].double())
        C.check(lib.fsld_grad_epilogue(M ** 3, ctypes_ptr(acc), ctypes_ptr(v), scale, lam, ctypes_ptr(grad),
                                       ctypes_ptr(sq), ctypes_ptr(loss), 0, ctypes_ptr(nscr), nscr.numel() * 8,
                                       stream), "epilogue")
        return loss

    # Binning plans (default on the brick path): the batches of a run are known in advance, so their
    # brick binning is done K batches at a time (fsld_plan_build) and each step runs only the
    # work-item kernel.  The plan of the TIMED batches is built inside the measurement: its time is
    # added to the steps (t_plan / K per step).
    use_plan = flags == 0 and eng.brick_path and not os.environ.get("FSLD_NO_PLAN")
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t_plan = 0.0
    if use_plan:
        plan_w = eng.make_plan(torch.stack(batches[:args.warmup]))
        plan_t = eng.make_plan(torch.stack(batches[args.warmup:]), build=False)  # sized + allocated
        torch.cuda.synchronize()
        p0, p1 = E(), E()
        p0.record()
        eng.build_plan(plan_t)  # the binning work of the timed batches
        p1.record()
        torch.cuda.synchronize()
        t_plan = p0.elapsed_time(p1)
        # world 1: grad init + brick kernel + finalize (fused step); N > 1: brick kernel + reduce +
        # ball gather / scatter + epilogue (2)
        launches_per_step = 3 if not dp else 6

    # N > 1 on NVSwitch: the exchange rides on the brick pass (each item's flush is a multimem.red into
    # every rank's copy of the accumulator, dist.NvlsGroup) instead of the all-reduce after it;
    # FSLD_COMM=nccl keeps the packed NCCL all-reduce
    nvg, comm_note = None, "nccl"
    if dp and use_plan and eng.table_path and not single and os.environ.get("FSLD_COMM", "nvls") == "nvls":
        from paper_2311_16100_b200.dist import NvlsGroup, nvls_available

        ok = [nvls_available(local)]
        if world > 1:
            oks = [None] * world
            dist.all_gather_object(oks, ok[0])
            ok = oks
        if all(ok):
            try:
                nvg = NvlsGroup(M ** 3)
                comm_note = "nvls"
            except Exception as exc:  # (every rank raises together: NvlsGroup agrees on each phase)
                comm_note = f"nccl (NVLS set-up failed: {exc})"
        else:
            comm_note = "nccl (no multicast support reported)"
    sq_tot = torch.empty(1, dtype=torch.float64, device=dev)
    if nvg is not None:
        launches_per_step = 6  # barrier, brick kernel, loss reduce, barrier, epilogue (2)

    def planned_step(plan, k, ev_k0=None, ev_k1=None, fused=False):
        if nvg is not None:
            from paper_2311_16100_b200.dist import nvls_planned_step

            nvls_planned_step(eng, nvg, plan, k, v, scale, lam, grad, sq, sq_tot, loss, nscr,
                              events=(ev_k0, ev_k1) if ev_k0 is not None else None)
            return loss
        if fused and not dp:  # the whole step in one call: grad = lam v, brick pass adds s * sum, finalize
            eng.loss_grad_step_planned(v, plan, k, scale, lam, grad, sq=sq, loss=loss)
            return loss
        stream = _stream()
        if ev_k0 is not None:
            ev_k0.record()
        C.check(lib.fsld_loss_grad_planned(M, eng.mode_id, n, ctypes_ptr(eng.recs), ctypes_ptr(plan.buf), B, k,
                                           ctypes_ptr(v), ctypes_ptr(eng.x), ctypes_ptr(eng.pc), ctypes_ptr(eng.ptab),
                                           0, ctypes_ptr(acc),
                                           0, ctypes_ptr(sq), ctypes_ptr(scr), scr.numel() * 8, stream),
                "loss_grad_planned")
        if ev_k1 is not None:
            ev_k1.record()
        return finish_step(stream)

    for i in range(args.warmup):
        if use_plan:
            planned_step(plan_w, i)
        else:
            step(batches[i])
    torch.cuda.synchronize()
    # kernel-only timing (events around the fused loss+grad call, eager)
    kev = [(E(), E()) for _ in range(args.steps)]
    for i in range(args.steps):
        l2_flush(i)
        if use_plan:
            planned_step(plan_t, i, *kev[i])
        else:
            step(batches[args.warmup + i], *kev[i])
    torch.cuda.synchronize()
    kern_ms = [a_.elapsed_time(b_) for a_, b_ in kev]
    # the timed step runs as one CUDA graph replay; for N > 1 over NCCL the graph holds the whole
    # step -- brick pass, ball gather, the packed all-reduce, ball scatter, epilogue (the gloo
    # exchange of the single-device functional check cannot be captured and stays eager)
    idx_static = torch.empty(B, dtype=torch.int32, device=dev)
    graphs = None
    graph_note = "eager"
    if not (dp and single) and not os.environ.get("FSLD_NO_GRAPH"):
        graphs = []
        if use_plan:  # one graph per planned batch (the batch index is a kernel argument)
            try:
                for i in range(args.steps):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        planned_step(plan_t, i, fused=True)
                    graphs.append(g)
                graph_note = "CUDA graph replay"
            except Exception as exc:  # (a collective that refuses capture: fall back to eager steps)
                graphs = None
                graph_note = f"eager (graph capture failed: {type(exc).__name__})"
                torch.cuda.synchronize()
        else:
            idx_static.copy_(batches[0])
            step(idx_static)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step(idx_static)
            graphs = [g] * args.steps
            graph_note = "CUDA graph replay"
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(E(), E()) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for i in range(args.steps):
            l2_flush(i)  # L2 flush between timed steps (outside the step events)
            s0, s1 = ev[i]
            s0.record()
            if graphs is not None:
                if not use_plan:
                    idx_static.copy_(batches[args.warmup + i])
                graphs[i].replay()
            elif use_plan:
                planned_step(plan_t, i, fused=True)
            else:
                step(batches[args.warmup + i])
            s1.record()
        clk.poll_until(ev[-1][1])  # the host is ahead: sample clocks while the GPU runs the timed steps
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = [a_.elapsed_time(b_) for a_, b_ in ev]
    t_step = float(np.mean(step_ms)) + t_plan / args.steps
    t_kern = float(np.mean(kern_ms)) + t_plan / args.steps
    if world > 1:
        t = torch.tensor([t_step, t_kern], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step, t_kern = float(t[0]), float(t[1])
    value = world * B / (t_step * 1e-3)

    # e2e through the public API: host v in (pinned), host grad + loss out
    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(eng, wl, B, lam, n_total, args, world)

    hbm, src = peaks()
    abytes = algorithmic_bytes(M, n, B)
    achieved = abytes / (t_kern * 1e-3) / 1e9
    kname = ("brick_loss_grad_kernel" if eng.table_path else "sorted_loss_grad_kernel" if eng.brick_path
             else f"slice_kernel<{cfg.mode.upper()},LOSS_GRAD>")
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{cfg.name}/{kname}")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, B, lam)
    algo1 = None
    if world == 1 and not args.no_algo1 and eng.brick_path:  # the device step runs on binning plans
        algo1 = algo1_leg(eng, wl, B, lam, args)
    elif world == 1 and not args.no_algo1:
        algo1 = {"skipped": f"{cfg.mode} mode runs the per-pixel tile path; the device Algorithm-1 leg uses "
                            "brick binning plans (tri)"}
    run = None
    if world == 1 and args.run_epochs > 0 and args.config == "cfg3" and not args.no_algo1:
        run = run_leg(eng, wl, B, lam, args.run_epochs)
    nxt = None
    if world == 1 and args.config == "cfg3" and not args.no_algo1:
        nxt = next_rows_leg(eng, wl)
    sweep = None
    if world == 1 and rank == 0 and not args.no_sweep and args.config == "cfg3":
        _, n_sw, sw = hutch_sweep(argparse.Namespace(images=0, warmup=2, steps=8))
        sweep = {"workload": "cfg5_M128_hutch_sweep", "n_images": n_sw, "unit": "probe-images/s",
                 "kernel": "sorted_hutch_kernel (brick-sorted, bit-packed probes in smem, Q(c,c') = k - 2 popc(z_c xor z_c'))",
                 "k": [d["k"] for d in sw], "probe_images_per_s": [d["probe_images_per_s"] for d in sw],
                 "ms_per_pass": [d["ms_per_pass"] for d in sw],
                 "probe_bytes_per_probe": sw[0]["probe_bytes_per_probe"],
                 "rel_l2_vs_exact_M32": [d["rel_l2_vs_exact_M32"] for d in sw]}
    if rank == 0:
        line = {
            "metric": "image-slices/sec (fused project+CTF+adjoint, loss+grad)",
            "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded generators of BASELINE cfg; SURVEY.md 8d)",
            "config": bench_config(cfg, M, n, B, world),
            "details": {
                "arithmetic": ("complex64 images / volume / gradient, fp32 gather and residual; per-pixel CTF*phase and "
                               "trilinear footprint evaluated once in fp64 (dataset tables, stored fp32); int32 "
                               "fixed-point shared-memory adjoint, fp32 global reduction; fp64 loss sums"
                               if eng.table_path else
                               "complex64 images / volume / gradient, fp32 coordinates, CTF and shift phases as exact "
                               "64-bit fixed-point turns; int32 fixed-point shared-memory adjoint; fp64 loss sums"),
                "n_images_per_gpu": eng.n_images, "l2": {"write": "flushed between timed steps (512 MB write)", "none": "not flushed (inputs > L2)"}.get(flush_mode, "flushed between timed steps (512 MB write, then a 256 MB read: the flush's dirty lines are written back before the step, not during it)"),
                "allreduce_bytes": (8 * nball + 8) if dp and nvg is None else 0,
                "collectives_per_step": 1 if dp and nvg is None else 0,
                "exchange": (("NVLS: per-item multimem.red.add.v2.f32 flush into the multicast accumulator "
                              "(every rank's copy), 2 barrier kernels per step, |r|^2 slots summed in rank order")
                             if nvg is not None else comm_note if dp else "none (one GPU)"),
                "step": graph_note + (" of fsld_loss_grad_step_planned (grad = lam v, the brick pass adds scale * its "
                                      "sums into grad, loss finalize)" if use_plan and not dp else
                                      " of barrier + brick pass flushing into the NVLS multicast accumulator + "
                                      "barrier + epilogue" if nvg is not None else
                                      " of brick pass + ball gather + all_reduce([grad acc | sq]) + ball scatter + "
                                      "epilogue" if dp else ""),
                "binning": (f"plan of the {args.steps} timed batches (fsld_plan_build), built inside the "
                            f"measurement: {t_plan:.4f} ms, added as {t_plan / args.steps:.4f} ms per step")
                if use_plan else "per step (count -> scan -> fill kernels)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "peak_source": src,
                         "kernel": (f"fsld_loss_grad_planned: {kname} + loss reduce (+ the plan's binning / K)" if use_plan else (f"fsld_loss_grad_sorted: bin count/scan/fill + {kname} + loss reduce" if eng.brick_path else f"fsld {kname} (tile path)")),
                         "kernel_ms": t_kern, "algorithmic_bytes_per_launch": abytes},
            "gpu_launches": launches_per_step * args.steps + (5 if use_plan else 0),  # + plan build (2 memsets, 3 kernels)
            "clocks": clk.summary(),
        }
        if e2e is not None:
            line["e2e"] = e2e
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if algo1 is not None:
            line["algorithm1_step"] = algo1
        if run is not None:
            line["algorithm1_run"] = run
        if nxt is not None:
            line["next_rows"] = nxt
        if sweep is not None:
            line["hutchinson_sweep"] = sweep
        print(json.dumps(line), flush=True)
    if nvg is not None:
        nvg.check()
        nvg.close()
    if dp:
        dist.destroy_process_group()


def algo1_leg(eng, wl, B, lam, args):
    """One full Algorithm-1 step (optim.run, optim.py:362-382) resident on the device, estimated variant:
    probe generation + Hutchinson fold + fused loss+grad + precond/direction epilogue + projection of the
    direction + closed-form Armijo + update.  Reported beside the headline (which is loss+grad only)."""
    import torch

    from paper_2311_16100_b200 import _capi as C

    M3 = eng.M ** 3
    dev = eng.dev
    v = torch.from_numpy((wl.v_true * 0.5).astype(np.complex64)).to(dev)
    acc = torch.zeros(M3, dtype=torch.complex64, device=dev)
    fold = torch.zeros(M3, dtype=torch.float32, device=dev)
    d_avg = torch.zeros(M3, dtype=torch.float32, device=dev)
    d = torch.ones(M3, dtype=torch.float32, device=dev)
    dirv = torch.empty(M3, dtype=torch.complex64, device=dev)
    st = eng.new_armijo_state(1.0)
    hist = torch.zeros(5 * (args.warmup + args.steps + 1), dtype=torch.float64, device=dev)
    gen = np.random.default_rng(4321)
    n = eng.n_images
    batches = [torch.from_numpy(gen.choice(n, B, replace=False).astype(np.int32)).to(dev)
               for _ in range(args.warmup + args.steps)]
    scale = n / B
    alpha = 1.0

    plan_w = eng.make_plan(torch.stack(batches[:args.warmup]))
    plan_t = eng.make_plan(torch.stack(batches[args.warmup:]), build=False)

    def one(plan, pk, i, k):
        zb = eng.gen_probes(1, 77 + i)
        sq = eng.loss_grad_planned(v, plan, pk, acc, zbits=zb, fold=fold)
        p = C.StepParams(scale=scale, lam=lam, beta=0.9, floor=alpha, w_old=k / (k + 1), w_new=1.0 / (k + 1),
                         hutch_scale=scale, estimating=1)
        vol4 = eng.precond_step(acc, v, p, dirv, fold=fold, d_avg=d_avg, d=d)
        qq = eng.proj_energy_planned(dirv, plan, pk)
        eng.armijo_select(sq, vol4[4:5], qq, vol4, scale, lam, 0.5, st, hist)
        eng.apply_step(v, dirv, st)

    for i in range(args.warmup):
        one(plan_w, i, i, i)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    eng.build_plan(plan_t)  # the binning of the timed batches is part of the timed work
    for i in range(args.steps):
        one(plan_t, i, args.warmup + i, args.warmup + i)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    bt = hist.view(-1, 5)[: args.warmup + args.steps, 3].cpu().numpy()
    return {"ms_per_step": ms, "images_per_s": B / (ms * 1e-3), "batch": B, "probes_per_step": 1,
            "mean_backtracks": float(bt.mean()),
            "kernels": "plan build of the timed batches (3, once), per step: gen_probes, loss_grad_planned "
                       "(+probe, 3), precond_step (+reduce), proj_energy_planned (3), armijo_select, apply_step",
            "note": "eager launches, L2 not flushed; the reference runs (1 + backtracks) extra loss passes "
                    "per step where this runs one projection of the direction"}


def run_leg(eng, wl, B, lam, epochs):
    """The BASELINE cfg3 run itself: preconditioned SGD (Algorithm 1, estimated variant) over the whole
    dataset for `epochs` epochs through the public optim.run -- the reference's per-epoch batch
    permutation (97 full batches of 512 + one of 336 at 50,000 images), one Hutchinson probe per step
    generated on the device, a binning plan per epoch, closed-form Armijo, and the full-dataset loss
    at every epoch end.  Wall-clock seconds of the whole call (device-synchronised on both sides,
    host bookkeeping included)."""
    import time
    from types import SimpleNamespace

    import torch

    from paper_2311_16100_b200 import optim
    from paper_2311_16100_b200.forward import DatasetOperator
    from paper_2311_16100_b200.grid import GridSpec

    spec = GridSpec(eng.M)
    stack = SimpleNamespace(spec=spec, mask_radius=eng.M // 2 - 1, n_images=eng.n_images, ctfs=wl.ctfs,
                            poses=None)
    op = DatasetOperator.from_engine(eng, spec)
    conf = optim.OptimConfig(lam=lam, batch_size=B, epochs=epochs, variant="estimated", seed=0)
    ta = time.perf_counter()
    alpha = optim.threshold_alpha(stack, None, lam)  # host setup (CTF ring means of every image)
    t_alpha = time.perf_counter() - ta
    optim.run(optim.OptimConfig(lam=lam, batch_size=B, epochs=1, variant="estimated", seed=1), stack,
              probes="device", op=op, alpha=alpha)  # warm-up (allocations, plan sizing)
    loss0 = 0.5 * float(eng.loss(torch.zeros(eng.M ** 3, dtype=torch.complex64, device=eng.dev),
                                 eng.all_indices()).item())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, trace = optim.run(conf, stack, probes="device", op=op, alpha=alpha, reference=wl.v_true)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    steps = len(trace.accepted_etas)
    curve = trace.fsc_history[-1]
    below = np.flatnonzero(curve < 0.5)
    return {"epochs": epochs, "steps": steps, "batch": B, "n_images": eng.n_images, "seconds": sec,
            "ms_per_step": 1e3 * sec / steps, "images_per_s": epochs * eng.n_images / sec,
            "loss_v0": loss0, "loss_first_epoch": float(trace.loss[0]), "loss_last_epoch": float(trace.loss[-1]),
            "fsc_0.5_shell_last_epoch": int(below[0]) if below.size else len(curve),
            "fsc_shells": len(curve),
            "mean_backtracks": float(np.mean(trace.step_backtracks)),
            "path": "optim.run(OptimConfig(variant='estimated', batch_size=512), probes='device'): per step "
                    "probe + planned loss+grad + precond epilogue + direction energy + Armijo + update; "
                    "per epoch the full-dataset loss, the FSC against the generating volume and one host "
                    "read of the step records",
            "timing": "wall clock of the whole call, synchronised, host bookkeeping included",
            "setup_seconds": {"threshold_alpha": t_alpha,
                              "note": "per-image CTF ring power on the device (fsld_ctf_ring_power), before the call"}}


def next_rows_leg(eng, wl):
    """SURVEY 8f rows 3-4 (each with its parity test in tests/): full-dataset passes of the exact
    diagonal, the b-vector adjoint and one CG Hessian product (reference_solve), the device FSC, and
    the streaming FSD1 ingest (io.load_operator) -- device time per call with CUDA events (ingest:
    wall clock from file to device-resident dataset)."""
    import tempfile
    import time

    import torch

    from paper_2311_16100_b200 import io as fio
    from paper_2311_16100_b200.forward import ImageStack, Pose
    from paper_2311_16100_b200.grid import GridSpec, disk_mask
    from paper_2311_16100_b200.metrics import ShellIndex, fsc

    idx = eng.all_indices()
    n = idx.numel()
    dev = eng.dev
    z = torch.from_numpy((wl.v_true * 0.5).astype(np.complex64)).to(dev)

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    out = {"n_images": n}
    ms = timed(lambda: eng.exact_diag_acc(idx))
    brick_diag = eng.layout == "sorted" and eng.ptab is not None and eng.mode == "tri"
    out["exact_diag"] = {"ms": ms, "images_per_s": n / (ms * 1e-3),
                         "path": ("fsld_exact_diag_sorted_tab (table-driven brick kernel, DIAG pass; "
                                  "hessian.exact_diag)" if brick_diag else "fsld_exact_diag (hessian.exact_diag)")}
    if brick_diag:  # the deterministic call hessian.exact_diag makes, and the tile kernel it replaced
        from paper_2311_16100_b200 import _capi as C
        from paper_2311_16100_b200.engine import HITS_PER_IMAGE, ctypes_ptr, _stream

        lib = C.load()
        acc64 = torch.zeros(eng.n_voxels, dtype=torch.int64, device=dev)
        accf = torch.zeros(eng.n_voxels, dtype=torch.float32, device=dev)
        fxd = eng.fixed_scale(None, HITS_PER_IMAGE * n, 1.0)
        scr = eng.scratch(1024)

        def diag_det():
            for lo in range(0, n, 1024):
                sub = idx[lo:lo + 1024]
                C.check(lib.fsld_exact_diag_sorted_tab(eng.M, eng.mode_id, eng.n_mask, ctypes_ptr(eng.recs),
                                                       ctypes_ptr(sub), sub.numel(), ctypes_ptr(eng.pc),
                                                       ctypes_ptr(eng.ptab), ctypes_ptr(eng.seg_off),
                                                       ctypes_ptr(eng.segs), ctypes_ptr(acc64), C.DETERMINISTIC,
                                                       ctypes_ptr(fxd), ctypes_ptr(scr), scr.numel() * 8, _stream()),
                        "exact_diag_sorted_tab")

        def diag_tile():
            C.check(lib.fsld_exact_diag(eng.M, eng.mode_id, eng.n_mask, ctypes_ptr(eng.pix), ctypes_ptr(eng.recs),
                                        ctypes_ptr(idx), n, ctypes_ptr(accf), 0, None, _stream()), "exact_diag")

        out["exact_diag"]["deterministic_ms"] = timed(diag_det)
        out["exact_diag"]["tile_kernel_ms"] = timed(diag_tile)
    ms = timed(lambda: eng.backproject_dataset(idx))
    out["b_vector"] = {"ms": ms, "images_per_s": n / (ms * 1e-3), "path": "fsld_backproject_sorted (b_vector)"}
    ms = timed(lambda: eng.hvp_acc(z, idx))
    out["cg_hessian_product"] = {"ms": ms, "images_per_s": n / (ms * 1e-3),
                                 "path": "fsld_hvp over all images (one reference_solve CG iteration)"}
    shells = ShellIndex(eng.M, eng.M // 2 - 1, dev)
    ref = torch.from_numpy(wl.v_true.astype(np.complex64)).to(dev)
    ms = timed(lambda: fsc(z, ref, shells))
    out["fsc"] = {"ms": ms, "path": "metrics.fsc (device shell bincounts, one host read)"}
    # deterministic mode (FSLD_DETERMINISTIC) on the brick kernel: one B=512 loss+grad, against the
    # same call without the flag (both eager, binning included)
    if eng.ptab is not None and eng.mode == "tri":
        from paper_2311_16100_b200 import _capi as C
        from paper_2311_16100_b200.engine import ctypes_ptr, _stream

        lib = C.load()
        bsel = idx[:512].contiguous()
        v5 = torch.from_numpy((wl.v_true * 0.9).astype(np.complex64)).to(dev)
        acc64 = torch.zeros((eng.n_voxels, 2), dtype=torch.int64, device=dev)
        accf = torch.zeros(eng.n_voxels, dtype=torch.complex64, device=dev)
        fx = eng.fixed_scale(v5, 16 * 512, eng.x_maxabs)
        sqd = torch.empty(1, dtype=torch.float64, device=dev)
        scr = eng.scratch(512)

        def lg(flags, acc):
            C.check(lib.fsld_loss_grad_sorted(eng.M, eng.mode_id, eng.n_mask, ctypes_ptr(eng.recs), ctypes_ptr(bsel),
                                              512, ctypes_ptr(v5), ctypes_ptr(eng.x), ctypes_ptr(eng.pc),
                                              ctypes_ptr(eng.ptab), ctypes_ptr(eng.seg_off), ctypes_ptr(eng.segs),
                                              ctypes_ptr(acc), ctypes_ptr(sqd), flags, ctypes_ptr(fx),
                                              ctypes_ptr(scr), scr.numel() * 8, _stream()), "loss_grad_sorted")

        ms_d = timed(lambda: lg(C.DETERMINISTIC, acc64))
        ms_p = timed(lambda: lg(0, accf))
        out["deterministic_loss_grad"] = {
            "ms": ms_d, "images_per_s": 512 / (ms_d * 1e-3), "plain_ms": ms_p,
            "path": "fsld_loss_grad_sorted(FSLD_DETERMINISTIC), B=512: brick-ordered items, per-brick segment "
                    "sort, int64 fixed-point flush, per-item loss partials (bitwise independent of grid / batch "
                    "order, tests/test_gpu_det.py); plain_ms = the same call without the flag"}
    # ingest: a synthetic FSD1 file (the reference's on-disk format: complex128 full M^2 images)
    M, ni = eng.M, 1024
    rng = np.random.default_rng(7)
    mask = disk_mask(GridSpec(M), M // 2 - 1)
    imgs = np.zeros((ni, M * M), dtype=np.complex128)
    imgs[:, mask] = rng.standard_normal((ni, mask.size)) + 1j * rng.standard_normal((ni, mask.size))
    q = rng.standard_normal((ni, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    stack = ImageStack(spec=GridSpec(M), images=imgs, poses=[Pose(q=q[i], t=np.zeros(2)) for i in range(ni)],
                       ctfs=None, sigma=1.0, seed=7, mask_radius=M // 2 - 1, mode="tri")
    with tempfile.TemporaryDirectory() as td:
        path = fio.write_dataset(stack, f"{td}/ingest.fsd1")
        nbytes = path.stat().st_size
        fio.load_operator(path)  # warm (page cache, allocations)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op, _ = fio.load_operator(path)
        torch.cuda.synchronize()
        sec = time.perf_counter() - t0
    out["ingest"] = {"images": ni, "file_bytes": nbytes, "seconds": sec, "gb_per_s": nbytes / sec / 1e9,
                     "path": "io.load_operator: FSD1 chunks -> pinned -> HBM, complex64 masking and the one-time "
                             "brick sort on the device (file in the page cache)"}
    return out


def e2e_leg(eng, wl, B, lam, n_total, args, world):
    """End to end through the public API with HOST buffers, copies inside the timed region.

    Headline (the drop-in call): the reference's own call shape, optim.loss_and_grad(op, v, batch,
    lam) with a numpy complex128 v and numpy batch rows, returning (float, numpy complex128 grad) --
    per call: threaded cast into pinned complex64, the slab-pipelined host step, the cast back.
    Wall clock per call (the call returns host results, so it is synchronous).
    Beside it (`c_abi`): the C ABI's host-buffer entry fsld_loss_grad_host on pinned complex64
    buffers (DatasetOperator.loss_and_grad_host), timed with CUDA events."""
    import time

    import torch

    from paper_2311_16100_b200 import optim as Opt
    from paper_2311_16100_b200.forward import DatasetOperator

    op = DatasetOperator.from_engine(eng)
    M = eng.M
    from paper_2311_16100_b200 import _capi as C

    gen = np.random.default_rng(99)
    # (host-side timing: more calls than the device legs; the host pool, pinned output arrays and their
    # cached graphs settle over the first ~15 calls of a fresh process -- tools/e2e_iters.py)
    n_warm, n_time = max(args.warmup, 20), max(args.steps, 30)
    rows = [gen.choice(eng.n_images, B, replace=False).astype(np.int64) for _ in range(n_warm + n_time)]
    v_np = (wl.v_true * 0.9).astype(np.complex128)
    # (1) the reference's call shape
    # (the warm-up holds each result until the next call returns, exactly like the timed loop, so the
    # two recycled page-locked output arrays and their cached graphs both exist before timing starts)
    for i in range(n_warm):
        loss, grad = Opt.loss_and_grad(op, v_np, rows[i], lam, n_total)
    torch.cuda.synchronize()
    per_call = []
    t0 = time.perf_counter()
    for i in range(n_time):
        t1 = time.perf_counter()
        loss, grad = Opt.loss_and_grad(op, v_np, rows[n_warm + i], lam, n_total)
        per_call.append((time.perf_counter() - t1) * 1e3)
    sec = (time.perf_counter() - t0) / n_time
    assert grad.dtype == np.complex128 and np.isfinite(loss)
    # bytes over PCIe per call: the packed touched ball as complex64 in each direction, the batch
    # rows up; one flag per z-slab and [sum|r|^2, loss] down
    ball = eng.HOST_BALL
    n_ball = int(C.load().fsld_ball_voxels(M, float(eng.touch_radius))) if ball else M ** 3
    n_slabs = eng.NP_SLABS if ball else eng.HOST_SLABS
    out = {"value": world * B / sec, "unit": "images/s", "ms_per_step": sec * 1e3,
           "h2d_bytes_per_step": 8 * n_ball + 4 * B,
           "d2h_bytes_per_step": (8 * n_ball + 4 * n_slabs + 16) if ball else 16 * M ** 3 + 16,
           "ball_voxels": n_ball, "volume_voxels": M ** 3, "z_slabs": n_slabs,
           "path": ("optim.loss_and_grad(op, v: numpy complex128, batch: numpy, lam) -> (float, numpy complex128) "
                    "-- the reference's signature, through fsld_loss_grad_host_np_ball: the voxels a scatter can "
                    "reach (the touched ball) cast to complex64 and packed row by row on the library's native host "
                    "thread pool (streaming stores into page-locked staging), then the z-slab pipelined host step "
                    "(one contiguous copy per slab in each direction, overlapping the brick passes; each finished "
                    "gradient slab packed on the device, copied, and cast to complex128 into the returned array by "
                    "the host threads while later slabs are in flight; off the ball the host threads write "
                    "grad = lam v and sum ||v||^2 in fp64 meanwhile; cached CUDA graph)") if ball else
                   ("optim.loss_and_grad(op, v, batch, lam) through fsld_loss_grad_host_np with whole-plane copies "
                    "(FSLD_HOST_BALL=0)"),
           "timing": f"wall clock, mean of {n_time} calls after {n_warm} warm-up calls (host cast, PCIe copies and "
                     "kernels inside)",
           "per_call_ms": {"median": float(np.median(per_call)), "min": float(np.min(per_call)),
                           "max": float(np.max(per_call))}}
    # (2) the C ABI host-buffer entry on pinned complex64 buffers
    v_h = C.host_empty(M ** 3, torch.complex64)
    # (written with the library's streaming-store cast: a buffer filled with ordinary stores stays dirty
    # in the CPU caches and the copy engine then reads it at a fraction of the PCIe rate)
    from paper_2311_16100_b200.hostio import cast_native
    v_flat = np.ascontiguousarray(v_np, dtype=np.complex128).reshape(-1)
    cast_native(C.load().fsld_host_cast_f64_to_f32, v_flat.ctypes.data, v_h.data_ptr(), 2 * M ** 3, 8, 4)
    g_h = C.host_empty(M ** 3, torch.complex64)
    idx_h = []
    for r in rows:
        t = C.host_empty(B, torch.int32)
        t.copy_(torch.from_numpy(r.astype(np.int32)))
        idx_h.append(t)
    for i in range(args.warmup):
        op.loss_and_grad_host(v_h, idx_h[i], lam, g_h, n_total=n_total)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    cab_calls = []
    e0.record()
    for i in range(args.steps):
        t1 = time.perf_counter()
        op.loss_and_grad_host(v_h, idx_h[args.warmup + i], lam, g_h, n_total=n_total)
        cab_calls.append((time.perf_counter() - t1) * 1e3)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    out["c_abi"] = {"value": world * B / (ms * 1e-3), "unit": "images/s", "ms_per_step": ms,
                    "h2d_bytes_per_step": 8 * M ** 3 + 4 * B, "d2h_bytes_per_step": 8 * M ** 3 + 16,
                    "path": "DatasetOperator.loss_and_grad_host -> fsld_loss_grad_host (pinned complex64 host v / "
                            "idx in, pinned host grad + loss out; no casts)",
                    "host_buffers": "fsld_host_alloc (cudaHostAlloc)",
                    "per_call_ms": {"median": float(np.median(cab_calls)), "min": float(np.min(cab_calls)),
                                    "max": float(np.max(cab_calls))}}
    return out


def cpu_baseline(cfg, B, lam):
    """A bounded sample of the reference's own CPU path (baseline/_ref), else of the C oracle port."""
    n_sub = 2 * B
    steps = 4
    fsld = reference_package()
    if fsld is not None:
        import numba
        threads = numba.get_num_threads()
        op, v = reference_operator(fsld, cfg, n_sub)
        per = time_reference(fsld, op, v * 0.9, B, lam, cfg.n_images, steps, 1)
        return {"value": B / per, "unit": "images/s", "cores": threads, "kind": "reference",
                "sample": f"{steps} loss+grad steps x {B} images from a {n_sub}-image host subset, the reference's "
                          f"fsld.optim.loss_and_grad (numba {numba.__version__}, {threads} threads, {cpu_model()})"}
    from oracle import oracle as O
    op, v = cpu_workload(cfg, n_sub)
    threads = O.max_threads()
    per = time_cpu(op, v * 0.9, B, lam, cfg.n_images, steps, 1)
    return {"value": B / per, "unit": "images/s", "cores": threads, "kind": "port",
            "sample": f"{steps} loss+grad steps x {B} images from a {n_sub}-image host subset, C oracle "
                      f"(fp64, OpenMP {threads} threads, {cpu_model()})"}


def self_launch(args) -> int | None:
    """`python bench.py --gpus N` without a torchrun environment: re-run this script under
    torch.distributed.run with N local ranks (one per GPU, NCCL over NVLink), 127.0.0.1 rendezvous.
    Returns the launcher's exit code, or None when this process is already a rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    # NCCL's communicator init lines (one per rank) stay visible on stderr
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "cfg5":
        run_hutch_sweep(args)
    else:
        run_b200(args)



def hutch_sweep(args):
    """cfg5: Hutchinson probe-batching sweep at M=128 (4,096 images, physical CTF), k in {1,4,16,64,256}:
    per k the folded A*A z pass time, probe-images/s, probe bytes per probe (bit-packed: M^3/8 B) and
    the relative L2 of the estimated diagonal against the exact one at M=32 (same k, 4,096 images)."""
    import torch

    from paper_2311_16100_b200 import synth

    cfg = synth.CONFIGS["cfg5"]
    wl = synth.build_workload(cfg, seed=0, n_images=args.images or None)
    eng = wl.engine
    idx = eng.all_indices()
    n_img = idx.numel()
    sweep = []
    small = synth.build_workload(synth.Config("cfg5_M32_err", 32, 4096, "tri", True, True, 0.05, 4096), seed=1)
    se = small.engine
    exact_acc, fx = se.exact_diag_acc(se.all_indices())
    exact = se.finalize_r(exact_acc, fx, 1.0, 0.0).double()
    for k in (1, 4, 16, 64, 256):
        zb = eng.gen_probes(k, seed=1234 + k)
        acc = eng.new_racc()
        for _ in range(max(1, args.warmup // 2)):
            acc.zero_()
            eng.hutch_fold(zb, k, idx, acc=acc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(5, args.steps // 4)
        e0.record()
        for _ in range(reps):
            acc.zero_()
            eng.hutch_fold(zb, k, idx, acc=acc)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        zs = se.gen_probes(k, seed=99 + k)
        sacc, sfx = se.hutch_fold(zs, k, se.all_indices())
        est = se.finalize_r(sacc, sfx, 1.0 / k, 0.0).double()
        rel = float((est - exact).norm() / exact.norm())
        sweep.append({"k": k, "ms_per_pass": ms, "probe_images_per_s": k * n_img / (ms * 1e-3),
                      "probe_bytes_per_probe": eng.n_voxels / 8.0, "rel_l2_vs_exact_M32": rel})
    return cfg, n_img, sweep


def run_hutch_sweep(args):
    """bench.py --config cfg5: value = probe-images/s of the folded A*A z pass at k=64, plus the sweep."""
    rank = int(os.environ.get("RANK", "0"))
    cfg, n_img, sweep = hutch_sweep(args)
    if rank == 0:
        k64 = next(s for s in sweep if s["k"] == 64)
        print(json.dumps({
            "metric": "probe-images/s (folded Hutchinson A*A z, k=64)", "value": k64["probe_images_per_s"],
            "unit": "probe-images/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": k64["ms_per_pass"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 (bit-packed +-1 probes)", "data": "synthetic (seeded generators of BASELINE cfg5)",
            "config": {"workload": cfg.name, "M": cfg.M, "n_images": n_img, "mode": cfg.mode},
            "sweep": sweep}), flush=True)


if __name__ == "__main__":
    main()
