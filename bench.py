#!/usr/bin/env python3
"""PBAD hot-path benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

A bench "step" is one PBAD timestep (stepper.cpp:83-147) for the whole batch:
one k_chain_step (or general k_step) launch that runs begin_step, the
optimiser to completion and finish_step for every environment.  `value` is
device-timed simulated env-steps/s over all ranks (inputs resident in HBM),
`e2e` the same metric through the public C ABI call with host buffers
(pbad_gpu_rollout: H2D of q0/qdot0, D2H of the trajectory).  Multi-GPU is
weak scaling: every rank owns its own shard of `batch_per_gpu` independent
environments (no collective on the step path; one NCCL gather afterwards).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated env-steps/sec (batch×steps/s, device-timed) vs N links at 1/2/4/8 B200"
UNIT = "env-steps/s"

# BASELINE.json configs / SURVEY.md §8(d)
CONFIGS = {
    "C1": dict(scene="single_hinge", links=10, dt=0.01, batch=1024, opt="lbfgs", seed=0, lo=0.0, hi=0.0,
               desc="C1: 10-link planar single-hinge chain, PBAD energy form, L-BFGS, dt=0.01 (x1024 replicas)"),
    "C2": dict(scene="single_hinge", links=50, dt=0.033, batch=1024, opt="lbfgs", seed=0, lo=-0.3, hi=0.3,
               desc="C2: 1024 x 50-link single-hinge chains, L-BFGS, dt=0.033"),
    "C3": dict(scene="chain", links=100, dt=0.1, batch=4096, opt="lbfgs", seed=1, lo=-0.3, hi=0.3,
               desc="C3: 4096 x 200-DOF serial hinge chains (make_chain_scene(100)), L-BFGS, dt=0.1"),
    "C3LM": dict(scene="chain", links=100, dt=0.1, batch=4096, opt="lm", seed=1, lo=-0.3, hi=0.3,
                 desc="C3-LM: 4096 x 200-DOF serial hinge chains (make_chain_scene(100)), LM (Gauss-Newton + "
                      "Cholesky; the C3 'LM as variant' of SURVEY 8(d)), dt=0.1"),
    "C4": dict(scene="humanoid", links=18, dt=0.01, batch=4096, opt="lm", seed=2, lo=-0.1, hi=0.1,
               desc="C4: 4096 x 41-DOF humanoid trees, LM (Gauss-Newton + Cholesky), dt=0.01"),
    "C4b": dict(scene="humanoid_contact", links=18, dt=0.01, batch=4096, opt="lm", seed=2, lo=-0.1, hi=0.1,
                desc="C4b: 4096 x 41-DOF humanoid trees with ground contact (plane z=0, D1=2e4, D2=2e2), LM, "
                     "dt=0.01"),
    "C5": dict(scene="single_hinge", links=100, dt=0.01, batch=256, opt="lm", seed=3, lo=-0.3, hi=0.3, order=4,
               objective="residual",
               desc="C5: high-order collocation PBAD (K=4 residual form, U=300), 100-link chains, LM, dt=0.01, "
                    "256 per GPU (2048 over 8 B200)"),
}


def build_scene(cfg):
    from paper_1709_04145_b200 import scenes
    if cfg["scene"] == "chain":
        return scenes.make_chain_scene(cfg["links"])
    if cfg["scene"] == "single_hinge":
        return scenes.make_single_hinge_chain_scene(cfg["links"])
    sc = scenes.make_humanoid_scene()
    if cfg["scene"] == "humanoid_contact":
        from paper_1709_04145_b200.types import ContactModel
        sc.contact = ContactModel(plane_normal=(0.0, 0.0, 1.0), plane_offset=0.0, d1=2e4, d2=2e2)
    return sc


def initial_states(cfg, scene, n, first_env, count):
    """std::mt19937(seed) env-major draws (benchmark.cpp:278-288) for envs
    [first_env, first_env + count) of the global batch."""
    from paper_1709_04145_b200.scenes import mt19937_uniform
    if cfg["scene"].startswith("humanoid"):
        draws = mt19937_uniform(cfg["seed"], (first_env + count) * (n - 6), cfg["lo"], cfg["hi"])
        q = np.tile(scene.q0, (count, 1))
        q[:, 6:] = draws[first_env * (n - 6):].reshape(count, n - 6)
        return q
    if cfg["hi"] == cfg["lo"]:
        return np.tile(scene.q0, (count, 1))
    draws = mt19937_uniform(cfg["seed"], (first_env + count) * n, cfg["lo"], cfg["hi"])
    return draws[first_env * n:].reshape(count, n)


def sim_config(cfg, steps, fail_limit):
    from paper_1709_04145_b200.types import OptimizerKind, SimConfig
    from paper_1709_04145_b200.types import ObjectiveKind
    sim = SimConfig(dt=cfg["dt"], duration=cfg["dt"] * steps, consecutive_fail_limit=fail_limit,
                    order=cfg.get("order", 2),
                    objective=ObjectiveKind.residual_form if cfg.get("objective") == "residual"
                    else ObjectiveKind.energy_form)
    sim.optimizer.kind = OptimizerKind.lbfgs if cfg["opt"] == "lbfgs" else OptimizerKind.lm
    return sim


def flops_per_env_step(cfg, model, iters, accepted):
    """SURVEY.md §8(d) canonical FP64 FLOPs (FMA = 2): iterations x per-iteration
    cost + per-step overhead (construction eval, history precompute, energy audit).
    Dense linear algebra re-derived to the minimal counts:
    Cholesky n^3/3 (the survey's (2/3)n^3 is LU's count), the symmetric
    2 J^T J product U^2 (U + 1) (one triangle: the two reference chains are equal
    bit for bit) instead of a full 2 U^3 GEMM."""
    N, n = model.link_count(), model.total_dofs
    overhead = N * 481 + 240 * N + 205 * N
    if cfg["opt"] == "lbfgs":
        per_iter = N * (307 + 174) + n * (8 * 8 + 12)
        return iters * per_iter + overhead
    depth_dofs = []
    for i in range(N):
        d, k = 0, i
        while k >= 0:
            d += model.dof_count(k)
            k = model.parent(k)
        depth_dofs.append(model.dof_count(i) * d)
    P = sum(depth_dofs)
    if cfg.get("objective") == "residual":
        u = cfg["order"] - 1
        U = u * n
        rej = U ** 3 / 3.0 + 2 * U * U + u * N * 600
        acc_extra = U * U * (U + 1) + 2 * U * U + u * u * (320 * N + 48 * P)
        return iters * rej + accepted * acc_extra + acc_extra + u * N * 600 + 240 * N + 205 * N
    # LM energy form: n^3/3 + 2n^2 + Eonly + a (grad + GN)
    rej = n ** 3 / 3.0 + 2 * n * n + 307 * N
    acc_extra = (120 * N + 54 * n) + (320 * N + 24 * P)
    return iters * rej + accepted * acc_extra + overhead + 320 * N + 24 * P


def flops_total(cfg, model, iters, acc):
    """Sum of flops_per_env_step over the [B][K] iteration / accepted counts
    (one evaluation per distinct pair)."""
    pairs, counts = np.unique(np.stack([iters.ravel(), acc.ravel()], axis=1), axis=0, return_counts=True)
    return float(sum(c * flops_per_env_step(cfg, model, int(i), int(a)) for (i, a), c in zip(pairs, counts)))


def measured_dmma_peak(device):
    """FP64 tensor-core (DMMA) rate on this GPU (csrc/pbad_peak.cu), TFLOP/s."""
    import ctypes as C
    lib = C.CDLL(os.path.join(ROOT, "paper_1709_04145_b200", "libpbad_peak.so"))
    lib.pbad_peak_dmma.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    t, ms = C.c_double(), C.c_double()
    return t.value if lib.pbad_peak_dmma(device, C.byref(t), C.byref(ms)) == 0 else None


def measured_fp64_peak(device):
    import ctypes as C
    lib = C.CDLL(os.path.join(ROOT, "paper_1709_04145_b200", "libpbad_peak.so"))
    lib.pbad_peak_fp64.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    t, ms, lat = C.c_double(), C.c_double(), C.c_double()
    rc = lib.pbad_peak_fp64(device, C.byref(t), C.byref(ms), C.byref(lat))
    if rc != 0:
        return None, None
    return t.value, lat.value


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML
    through nvidia_ml_py, 5 ms period in a background thread; nvidia-smi
    fallback), so short timed regions still get samples."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = None
        self._thread = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.idx]) if vis and vis.split(",")[0].isdigit() else self.idx
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            return
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    for nm, bit in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(nm)
                except Exception:
                    pass
                self._stop.wait(0.005)

        self._thread = threading.Thread(target=run, daemon=True)
        self._thread.start()

    def stop(self):
        if not self._thread:
            return None
        self._stop.set()
        self._thread.join(timeout=2)
        if not self.samples:
            return None
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_baseline(cfg, scene, model_links, n, steps=1, sample=None, target_s=15.0):
    """The reference's own CPU batch_simulate (oracle/_ref: /root/reference
    sources compiled unmodified, kind "reference", its WorkerPool on all host
    threads) when built, else the C oracle port (kind "port"), over a bounded
    sample of the workload: one calibration round of `cores` environments x
    `steps` steps, then (if that took under ~10 s) a second round sized to
    about `target_s` seconds, which is the one reported."""
    import oracle
    cores = os.cpu_count() or 1
    forces = scene.forces()
    use_ref = oracle.ref_available()
    mo = oracle.RefModel(model_links) if use_ref else oracle.Model(model_links)
    run = oracle.ref_batch_simulate if use_ref else oracle.batch_simulate

    def timed(count, steps=steps):
        q0 = initial_states(cfg, scene, n, 0, count)
        sims = []
        for b in range(count):
            s = sim_config(cfg, steps, 1 << 30)
            s.q0 = q0[b]
            s.qdot0 = np.zeros(n)
            sims.append(s)
        t = time.perf_counter()
        trs = run(mo, forces, sims, workers=cores)
        el = time.perf_counter() - t
        return sum(tr.n_samples - 1 for tr in trs), el

    count = sample or min(cfg["batch"], cores)
    done, el = timed(count)
    if sample is None and el < 10.0 and count < cfg["batch"]:
        count = int(min(cfg["batch"], max(count + 1, count * target_s / max(el, 1e-3))))
        count = max(cores, (count // cores) * cores)
        done, el = timed(count)
        if el < 5.0:  # the whole batch is cheap: lengthen the rollout instead
            steps = int(min(50, max(2, steps * target_s / max(el, 1e-3))))
            done, el = timed(count, steps)
    kind = "reference" if use_ref else "port"
    what = ("reference batch_simulate (stepper.cpp:204-270, WorkerPool)" if use_ref
            else "C oracle batch_simulate")
    # the workers = 1 leg: one environment on one worker thread
    t1 = time.perf_counter()
    q1 = initial_states(cfg, scene, n, 0, 1)
    s1 = sim_config(cfg, steps, 1 << 30)
    s1.q0 = q1[0]
    s1.qdot0 = np.zeros(n)
    tr1 = run(mo, forces, [s1], workers=1)
    el1 = time.perf_counter() - t1
    one = (tr1[0].n_samples - 1) / el1
    res = {"value": done / el, "unit": UNIT, "cores": cores, "kind": kind,
           "sample": f"{count} envs x {steps} step(s) of {cfg['desc'].split(':')[0]} (first envs of the bench "
                     f"batch), {what}, {cores} threads, {el:.2f} s",
           "cpu_model": cpu_model(), "workers": cores,
           "workers_1": {"value": one, "unit": UNIT, "sample": f"env 0 x {steps} step(s), workers = 1, {el1:.2f} s"},
           "seconds": el}
    if cfg["opt"] == "lm":
        res["caveat"] = ("the reference build uses oracle/eigen_lite (Eigen3 is absent from the image): its dense "
                         "LLT and GEMM are naive loops, slower than real Eigen, so this CPU figure understates the "
                         "reference on the Newton path")
    return res


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or None


def _free_port():
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec this
    script as N ranks (one process per GPU) on this node and exit with the
    launcher's code.  Rank 0 prints the JSON line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


class Dist:
    """One process per GPU (torchrun env).  NCCL when every rank has its own
    device; when more ranks than visible devices share them (a dry run on a
    1-GPU box) the ranks map round-robin onto the devices and the
    collectives run on gloo over host tensors (`oversubscribed`)."""

    def __init__(self, ngpus):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != ngpus:
            raise SystemExit(f"bench.py: --gpus {ngpus} but WORLD_SIZE={self.world} (launch one rank per GPU)")
        import torch
        ndev = torch.cuda.device_count()
        if ndev < 1:
            raise SystemExit("bench.py: no CUDA device visible (the PBAD GPU path has no CPU fallback)")
        self.device = self.local % ndev
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(self.world)))
        self.oversubscribed = local_world > ndev
        self.backend = None
        if self.world > 1:
            import torch.distributed as dist
            torch.cuda.set_device(self.device)
            if self.oversubscribed:
                dist.init_process_group("gloo")
                self.backend = "gloo"
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
                self.backend = "nccl"

    def _dev(self):
        import torch
        return torch.device("cpu") if self.backend == "gloo" else torch.device("cuda", self.device)

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def reduce(self, x, op="max"):
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(x)], dtype=torch.float64, device=self._dev())
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    def gather_final(self, ctx, B, n, stream):
        """NCCL all-gather of every rank's final configurations [B][n] straight
        from device memory (pbad_gpu_final_state, no host bounce); returns
        (ms, gathered rows) or (None, None) at N = 1."""
        if self.world == 1:
            return None, None
        import torch
        import torch.distributed as dist
        fin = torch.empty((B, n), dtype=torch.float64, device=f"cuda:{self.device}")
        ctx.final_state(fin.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        self.barrier()
        g0 = time.perf_counter()
        if self.backend == "nccl":
            allq = torch.empty((self.world * B, n), dtype=torch.float64, device=f"cuda:{self.device}")
            dist.all_gather_into_tensor(allq, fin)
            torch.cuda.synchronize()
        else:
            parts = [torch.empty((B, n), dtype=torch.float64) for _ in range(self.world)]
            dist.all_gather(parts, fin.cpu())
            allq = torch.cat(parts)
        return (time.perf_counter() - g0) * 1e3, allq.shape[0]

    def close(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


def run_reference(args, cfg):
    world, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return
    scene = build_scene(cfg)
    from paper_1709_04145_b200.types import LinkSpec  # noqa: F401
    import oracle
    mo = oracle.Model(scene.links)
    n = mo.n_dofs
    cb = cpu_baseline(cfg, scene, scene.links, n, steps=max(1, min(args.steps, 2)))
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, args, world),
        "cpu_baseline": {k: v for k, v in cb.items() if k != "seconds"},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("reference arm = the reference's own C++ (oracle/_ref: /root/reference/proj/src compiled "
                 "unmodified against oracle/eigen_lite, Eigen3 being absent) on the host cores; falls back "
                 "to the C oracle port when oracle/_ref is not built (see DESIGN.md)"),
    }
    print(json.dumps(line), flush=True)


def config_block(cfg, args, world, D=None):
    c = {"workload": cfg["desc"], "batch_per_gpu": cfg["batch"], "global_batch": cfg["batch"] * world,
         "n_links": cfg["links"] * (2 if cfg["scene"] == "chain" else 1), "dt": cfg["dt"],
         "optimizer": cfg["opt"], "max_iters": 512, "consecutive_fail_limit": "unbounded (bench)",
         "parallelism": f"dp{world} (independent env shards, weak scaling)",
         "cache": "per-env solver state (~100 KB/env) > L2: inputs larger than L2, no flush needed"}
    if D is not None and D.world > 1:
        c["collective_backend"] = D.backend
        c["oversubscribed"] = D.oversubscribed
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("PBAD_BENCH_CONFIG", "C3"))
    ap.add_argument("--links", type=int, default=None,
                    help="chain configs: override the link count (the metric's 'vs N links' sweep)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if os.environ.get("PBAD_BENCH_BATCH"):  # experiments only: batch-size sweeps
        cfg["batch"] = int(os.environ["PBAD_BENCH_BATCH"])
    if args.links is not None:
        if not cfg["scene"] in ("chain", "single_hinge"):
            raise SystemExit("--links applies to the chain configurations (C1, C2, C3, C5)")
        cfg["links"] = args.links // 2 if cfg["scene"] == "chain" else args.links
        cfg["desc"] = cfg["desc"] + f" [link sweep: {args.links} links]"
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    relaunch_under_torchrun(args)

    D = Dist(args.gpus)
    world, rank, dev = D.world, D.rank, D.device
    import torch
    torch.cuda.set_device(dev)
    from paper_1709_04145_b200 import api, build as pbuild
    if not os.path.exists(pbuild.LIB):
        pbuild.build()

    scene = build_scene(cfg)
    model = api.build_model(scene.links)
    n = model.total_dofs
    B = cfg["batch"]
    W, K = args.warmup, args.steps
    total = W + K
    sim = sim_config(cfg, total, 1 << 30)
    ctx = api.GpuContext(model, scene.forces(), sim, device=dev, max_batch=B)
    q0 = initial_states(cfg, scene, n, rank * B, B)  # this rank's contiguous shard of the global batch
    # a dedicated stream: the legacy default stream has handle 0, which the C
    # ABI reads as "the context's own stream"; the inputs are written on it
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream
    with torch.cuda.stream(stream):
        dq0 = torch.from_numpy(q0).to(f"cuda:{dev}", non_blocking=False)
        dqd = torch.zeros_like(dq0)
    stream.synchronize()

    # warm-up steps (untimed)
    ctx.begin(B, dq0.data_ptr(), dqd.data_ptr(), sh)
    ctx.advance(W, sh)
    torch.cuda.synchronize()
    D.barrier()
    clocks = ClockSampler(dev)
    clocks.start()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.kernel_launches()
    e0.record(stream)
    ctx.advance(K, sh)
    e1.record(stream)
    launches = ctx.kernel_launches() - l0
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    ms = D.reduce(ms, "max")  # device time of the slowest rank
    out = ctx.sync_outputs(want_q=False, want_energy=False)
    iters = out["iterations"][:, W:W + K]
    acc = out["accepted"][:, W:W + K]
    st = out["status"]

    # NCCL gather of the final states, device to device (outside the timed region)
    gather_ms, gathered = D.gather_final(ctx, B, n, stream)

    # FLOP accounting for the roofline (per env, summed over all ranks' envs)
    fl = flops_total(cfg, model, iters, acc)
    fl = D.reduce(fl, "sum")
    value = world * B * K / (ms / 1e3)

    # end-to-end: every rank's public rollout call with host buffers (H2D +
    # kernels + D2H) started together; the job's time is the slowest rank's
    sim2 = sim_config(cfg, K, 1 << 30)
    ctx2 = api.GpuContext(model, scene.forces(), sim2, device=dev, max_batch=B)
    pq0 = torch.from_numpy(np.ascontiguousarray(q0)).pin_memory().numpy()
    pqd0 = torch.zeros(q0.shape, dtype=torch.float64).pin_memory().numpy()
    o2 = ctx2.make_outputs(B, want_q=True, want_energy=True, pinned=True)  # caller-owned, outside the clock
    ctx2.rollout(pq0, pqd0, out=o2)  # warm-up: lazy staging allocation, kernel attributes
    torch.cuda.synchronize()
    D.barrier()
    t0 = time.perf_counter()
    bufs = ctx2.rollout(pq0, pqd0, out=o2)
    el = D.reduce(time.perf_counter() - t0, "max")
    h2d = world * 2 * q0.nbytes
    d2h = world * sum(v.nbytes for v in bufs.values() if v is not None)
    e2e = {"value": world * B * K / el, "unit": UNIT, "h2d_bytes_per_step": int(h2d / K),
           "d2h_bytes_per_step": int(d2h / K),
           "note": (f"pbad_gpu_rollout (C ABI) on every rank concurrently: pinned host q0/qdot0 in, trajectory + "
                    f"solve reports out into caller-allocated pinned buffers; wall clock of the slowest of "
                    f"{world} rank(s) after one warm-up rollout; bytes summed over ranks")}
    del ctx2

    if rank != 0:
        D.close()
        return

    peak, lat = measured_fp64_peak(dev)
    peak_dmma = measured_dmma_peak(dev)
    achieved = fl / (ms / 1e3) / 1e12 / world  # per GPU
    # the CTA Newton kernel runs its J^T J and Cholesky updates on the FP64
    # tensor cores: its denominator is the larger of the two measured peaks
    uses_dmma = ctx.path == 4
    peak_used = max(peak, peak_dmma) if (uses_dmma and peak and peak_dmma) else peak
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", f"{args.config}_dram_per_launch.json")
    if os.path.exists(prof) and args.links is None:
        try:
            pj = json.load(open(prof))
            traffic = pj.get("dram_bytes_per_launch")
            traffic_src = "not measured in this run: from " + os.path.relpath(prof, ROOT) + ": " + pj.get("source", "")
        except Exception:
            traffic = None
    cb = None
    if not args.no_cpu_baseline and world == 1:  # the CPU baseline is an N=1, rank-0 measurement
        try:
            cb = cpu_baseline(cfg, scene, scene.links, n)
        except Exception as ex:  # the oracle must never block the GPU line
            cb = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {ex}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_block(cfg, args, world, D),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak_used, "unit": "TFLOP/s",
                     "frac": (achieved / peak_used) if peak_used else None, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "peak_dfma": peak, "peak_dmma": peak_dmma,
                     "peak_source": ("measured FP64 microbenchmarks (paper_1709_04145_b200/csrc/pbad_peak.cu) on "
                                     "this GPU: " + ("max(DFMA, DMMA) -- this kernel runs DMMA" if uses_dmma
                                                     else "DFMA")),
                     "flops_model": "SURVEY.md 8(d) canonical FP64 FLOPs per L-BFGS/LM iteration + per-step overhead",
                     "dfma_latency_cycles": lat},
        "cpu_baseline": cb,
        "e2e": e2e,
        "gpu_launches": launches,
        "kernel": {0: "pbad_gpu::k_step (general, thread per env)", 1: "pbad_gpu::k_chain_step (quad per env)",
                   2: "pbad_gpu::c4::k_chain4_step (warp-synchronous quads, TMA-fed adjoint)",
                   3: "pbad_gpu::tree::k_tree_step (warp per env, Newton/LM, in-SMEM Cholesky)",
                   4: "pbad_gpu::resid::k_resid_step (CTA per env, LM: residual form or large-n energy form, DMMA J^T J + blocked Cholesky)",
                   5: "pbad_gpu::c5::k_chain5_step (warp per env, shared-memory-resident L-BFGS, TMA-fed adjoint)",
                   6: "pbad_gpu::c6::k_chain6_step (8 lanes per env: two per transform row, TMA-fed adjoint)",
                   7: "pbad_gpu::c7::k_chain7_step (16 lanes per env: serial FK rows + link-parallel energy terms, TMA-fed adjoint)"
                   }.get(ctx.path),
        "clocks": clk,
        "mean_iterations_per_step": float(iters.mean()),
        "trajectories_ok": int(np.sum((st == 0) | (st == 4))),
        "gather_ms": gather_ms,
        "gathered_envs": gathered,
    }
    print(json.dumps(line), flush=True)
    D.close()


if __name__ == "__main__":
    main()
