#!/usr/bin/env python
"""Benchmark: one projected-EM iteration of 2-D SR-MRA (E-step + M-step over all N observations and
all L_high^2 shifts, finalize, projection) per step, through libsrmra.so's C ABI.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Metric (BASELINE.json): obs x shift likelihoods per second per EM iteration, N * L_high^2 / t.
Workload: BASELINE.json configs[3] by default (c3: L_high=128, L_low=32, K=4, N=100,000, sigma=0.125;
one of north_star's two targets, and the largest config the paper's metric names that is quoted on
1/2/4/8 GPUs), seeded synthetic data (synth/, the same data as tests/golden/c3_oracle.npz); c0..c4 via
--config.  Multi-GPU: STRONG scaling — the config's N observations are sharded in contiguous blocks
(paper_2204_04754_b200.shard.shard_bounds), one NCCL all-reduce of the sufficient statistics per
iteration (captured with the rest of the iteration in one CUDA graph).  `--gpus N` without torchrun
re-launches itself under torch.distributed.run with N ranks (and fails loudly when the node has fewer
than N GPUs).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "obs×shift likelihoods/sec per EM iteration (N·L_high^2/t), % of roofline"
UNIT = "obs*shift/s"
# FP32 SIMT peak: 148 SMs x 128 FP32 lanes x 2 FLOP (FMA) x 1.965 GHz (B200_PROFILING.md SM count and
# clocks.max.sm).
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
FLUSH_BYTES = 256 << 20


def flop_per_unit(path: str, L_low: int) -> float:
    """Algorithmic FLOP per (observation, shift) unit."""
    if path == "fft":
        return 10.0 * np.log2(L_low) + 17.0
    return 4.0 * L_low * L_low  # direct / gemm: 2 L_low^2 (E-step dot) + 2 L_low^2 (M-step)


def roof_kernel(path: str, L_low: int = 0) -> str:
    if path == "fft" and L_low == 128:
        return "k_fft_em128"
    return {"fft": "k_fft_em", "direct": "k_direct_em", "gemm": "k_gemm_em"}.get(path, path)


def ncu_traffic(kernel: str, cfg: str):
    """DRAM bytes (read + write) per launch of `kernel` from the latest committed `ncu --set full`
    capture (profiles/rNN_traffic.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    for f in reversed(files):
        try:
            v = json.load(open(f)).get(kernel, {}).get(cfg)
        except (OSError, ValueError):
            continue
        if v is not None:
            return v, os.path.relpath(f, ROOT)
    return None, None


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(p, world: int = 1) -> dict:
    return {"workload": p.name, "L_high": p.L_high, "L_low": p.L_low, "K": p.K, "global_N": p.N,
            "N_per_rank_max": -(-p.N // world), "sigma": p.sigma}


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, f[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------- oracle (CPU) legs
def oracle_rate(p, seconds: float, n_max: int | None = None):
    """Time the float64 oracle (as it stands) on a bounded sample of observations of p: one EM
    iteration from theta_0 on the first n observations, n sized for ~`seconds` of work."""
    import oracle
    oracle.build()
    n_probe = min(p.N, 64)
    t0 = time.perf_counter()
    oracle.em_iter(p.y[:n_probe], p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
    per_obs = (time.perf_counter() - t0) / n_probe
    n = int(max(n_probe, min(n_max or p.N, p.N, seconds / max(per_obs, 1e-9))))
    t0 = time.perf_counter()
    oracle.em_iter(p.y[:n], p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
    dt = time.perf_counter() - t0
    return n * p.L_high ** 2 / dt, n, dt, oracle.max_threads()


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import oracle
    oracle.build()
    p = synth.make_config(args.config)
    # per-step sample sized so warmup + steps finish in about `budget` seconds
    budget = float(os.environ.get("SRMRA_REF_BUDGET_S", 150))
    n_probe = min(p.N, 32)
    t0 = time.perf_counter()
    oracle.em_iter(p.y[:n_probe], p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
    per_obs = (time.perf_counter() - t0) / n_probe
    n = int(max(8, min(p.N, budget / (args.steps + args.warmup) / per_obs)))
    ys = p.y[:n]
    for _ in range(args.warmup):
        oracle.em_iter(ys, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.em_iter(ys, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n * p.L_high ** 2 * args.steps / tot
    sample = f"first {n} of {p.N} observations of {p.name}, one EM iteration from theta_0 per step"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload(p),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.max_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2204_04754_b200 as srm
    from paper_2204_04754_b200.shard import broadcast_nccl_id, shard_bounds

    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        nccl_id = broadcast_nccl_id(srm.srmra_nccl_unique_id)

    # strong scaling: every rank draws the same seeded config and keeps its contiguous shard
    p = synth.make_config(args.config)
    lo, hi = shard_bounds(p.N, world, rank)
    y_loc = np.ascontiguousarray(p.y[lo:hi])
    n_loc = hi - lo
    stream = torch.cuda.Stream(device=dev)
    ctx = srm.Context(y_loc, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=args.path,
                      proj_every=1, device=local, rank=rank, world=world, nccl_id=nccl_id,
                      stream=stream.cuda_stream, nccl_timeout_ms=600_000)
    path = ctx.path
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            ctx.em_iter(1)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    ctx.profile(True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with torch.cuda.stream(stream):
        for a, b in evs:
            flush.zero_()          # L2 flush (256 MiB write), outside the timed events
            a.record(stream)
            ctx.em_iter(1)
            b.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    em_ms, iter_ms, n_prof = ctx.profile_read()
    ctx.profile(False)
    ctx.get_estimate()  # raises SrmraError(NUMERIC) if any timed iteration produced a non-finite LL or estimate
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tot_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms, em_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t[0])
    units_step = p.N * p.L_high ** 2                     # the whole job's units (all ranks)
    value = units_step * args.steps / (tot_ms / 1e3)

    # roofline of the dominant kernel on this rank (measured live: the kernel's own globaltimer stamps
    # over the timed region, on the stream it is launched on); units = this rank's observations x shifts
    fpu = flop_per_unit(path, p.L_low)
    kern = roof_kernel(path, p.L_low)
    traffic, traffic_src = ncu_traffic(kern, p.name) if world == 1 else (None, None)
    em_avg_s = em_ms / 1e3 / max(n_prof, 1)
    achieved = fpu * n_loc * p.L_high ** 2 / em_avg_s / 1e12
    alg_bytes = int(n_loc * p.L_low * (p.L_low // 2 + 1) * 8) if path == "fft" else int(n_loc * p.L_low ** 2 * 4)
    hbm_peak = None
    try:
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except (OSError, ValueError):
        pass
    roof = {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": alg_bytes, "kernel": kern,
            "hbm_gbs": alg_bytes / em_avg_s / 1e9, "hbm_peak_gbs": hbm_peak,
            "hbm_frac": (alg_bytes / em_avg_s / 1e9 / hbm_peak) if hbm_peak else None,
            "flop_per_unit": fpu, "units_per_launch": n_loc * p.L_high ** 2, "kernel_ms_avg": em_avg_s * 1e3,
            "kernel_share_of_step": em_ms / max(float(sum(step_ms)), 1e-12),
            "rank": rank,
            "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x 1.965 GHz (B200_PROFILING.md)"}

    # end-to-end through the public API with pinned host buffers: load (H2D) + cfg.iters iterations + D2H
    e2e = None
    if args.e2e_jobs > 0:
        y_pin = torch.from_numpy(y_loc).pin_memory()
        y_np = y_pin.numpy()
        jt = []
        for j in range(args.e2e_jobs + 1):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            ctx.load_iterate(y_np, p.x0, p.rho1_0, p.rho2_0, p.iters)  # upload overlapped with the 1st E/M step
            ctx.get_estimate()
            dt = time.perf_counter() - t0
            if j > 0:
                jt.append(dt)
        tj = float(np.mean(jt))
        if world > 1:
            t = torch.tensor([tj], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tj = float(t[0])
        e2e = {"value": units_step * p.iters / tj, "unit": UNIT,
               "h2d_bytes_per_step": int(p.y.nbytes + world * (4 * p.L_high ** 2 + 16 * p.L_high)),
               "d2h_bytes_per_step": int(world * (4 * p.L_high ** 2 + 16 * p.L_high + 16)),
               "step": f"srmra_load_iterate (pinned host y shard, x0, rho; {p.iters} iteration(s), the first one's "
                       "E/M step per observation range as the range lands) + srmra_get_estimate on every rank "
                       "(bytes summed over ranks)",
               "timer": "host perf_counter, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, n, dt, cores = oracle_rate(p, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"first {n} of {p.N} observations of {p.name}, one EM iteration from theta_0 "
                         f"({dt:.1f} s)"}

    launches = ctx.launches_per_iter() * args.steps
    ctx.close()
    if rank == 0:
        cfg = workload(p, world)
        cfg.update({"path": path, "l2": "flushed before every timed step (256 MiB write, outside the events)",
                    "iters_per_step": 1, "parallelism": f"dp{world} (observations sharded, strong scaling)"})
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "gpu_launches_note": "libsrmra kernels only" + ("; + 1 NCCL all-reduce kernel per step" if world > 1 else ""),
                "clocks": clk, "step_ms_median": statistics.median(step_ms)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch_distributed(args) -> int:
    """`--gpus N` outside torchrun: re-run this script under torch.distributed.run with N ranks."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but this node has {have} visible GPU(s); "
                                   "refusing to measure fewer ranks than requested"}), flush=True)
        return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="auto", choices=["auto", "fft", "direct", "gemm"])
    ap.add_argument("--e2e-jobs", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args))
    run_ours(args)


if __name__ == "__main__":
    main()
