#!/usr/bin/env python
"""Benchmark: weighted particles/s of GPU importance sampling (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload linreg|poly|smc|mh|dsl-linreg] [--dry-run]

`--gpus N` outside a launcher re-executes the same command under torch.distributed.run, one
process per GPU (NCCL, rendezvous on 127.0.0.1, NCCL_DEBUG=INFO init lines on stderr); under a
launcher the world comes from WORLD_SIZE / RANK / LOCAL_RANK. `--dry-run` runs the multi-rank
orchestration (sharding, record all-gather, max-over-ranks timing) over gloo on CPU without
launching a kernel, for the CPU test suite.

Default workload (BASELINE.json configs[1]): Bayesian linear regression,
1e9 particles in total, strong-scaled (1e9/N per GPU), 1,000 synthetic points, prior
normal(0,10) on (a, b).
A step is one full importance-sampling pass over those particles: Philox draws, the model's
1,000 observe() terms, the fused log-sum-exp / ESS / moment / mode reduction, and (N > 1) the
per-rank record all-gather over NCCL. `--workload poly` runs the Fig.1 polynomial model
(configs[4], C5: 1.25e10 particles per GPU, 20 points); `--workload smc` the HMM particle
filter (configs[3], SMC time-steps/s on 1e8 particles) and `--workload mh` the 4096-chain LMH
sampler (configs[2], chain-steps/s).

`--impl reference` times the reference's CPU path — the C restatement in oracle/ (the
reference ships no executable engine) — on all host cores, rank 0 only.
One JSON line is printed by rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "weighted particles/sec (importance sampling)"

# C2 in CuPPL surface syntax (the dsl-linreg workload): xs / ys are bound from the host data
DSL_LINREG = """
model <- function() {
  a <- sample(normal(0, 10));
  b <- sample(normal(0, 10));
  factor(reduce(function(acc, i) { acc + dist-score(normal(a * xs[i] + b, 1), ys[i]) }, 0.0,
                repeat(function(i) { i }, length(xs))));
  [a, b]
};
importance(model, 1000000000)
"""
UNIT = "particles/s"

WORKLOADS = {
    "linreg": {
        "name": "C2: Bayesian linear regression IS, 1e9 particles in total (strong scaling over 1-8 GPUs), "
                "1k points (BASELINE configs[1])",
        "particles": 10**9,
        "scaling": "strong",
        "n_points": 1000,
    },
    "poly": {
        "name": "C5: Fig.1 polynomial regression IS, 1.25e10 particles/GPU (1e11 on 8 GPUs), 20 points "
                "(BASELINE configs[4])",
        "particles": 12_500_000_000,
        "scaling": "weak",
        "n_points": 20,
    },
    "smc": {
        "name": "C4: HMM S=50 bootstrap particle filter, 1e8 particles, T=1000, systematic resampling "
                "every step (BASELINE configs[3], single GPU)",
        "particles": 100_000_000,
        "scaling": "strong",
        "n_points": 1000,
    },
    "dsl-linreg": {
        "name": "C2 written in CuPPL and compiled (frontend.py -> NVRTC sm_100a): Bayesian linear regression IS, "
                "1e9 particles in total (strong scaling), 1k points",
        "particles": 10**9,
        "scaling": "strong",
        "n_points": 1000,
    },
    "mh": {
        "name": "C3: GMM K=5, 10k points, 4096 LMH chains x 10k steps (BASELINE configs[2])",
        "particles": 4096,
        "scaling": "weak",
        "n_points": 10_000,
    },
    "resample": {
        "name": "Generic systematic resampling (cuppl_resample) of C4's 1e8-particle population: fp32 "
                "log-weights + a 4-byte state payload per particle (BASELINE configs[3] population)",
        "particles": 100_000_000,
        "scaling": "weak",
        "n_points": 0,
    },
}
METRICS = {
    "linreg": (METRIC, UNIT),
    "poly": (METRIC, UNIT),
    "dsl-linreg": (METRIC, UNIT),
    "smc": ("SMC steps/sec", "time-steps/s"),
    "mh": ("MH chain-steps/sec", "chain-steps/s"),
    "resample": ("resampled particles/sec", "particles/s"),
}


def make_model(workload: str):
    from paper_2010_08454_b200 import models

    w = WORKLOADS[workload]
    if workload in ("linreg", "dsl-linreg"):
        return models.LinearRegression.synthetic(n_points=w["n_points"])
    if workload == "smc":
        return models.HiddenMarkovModel.synthetic(S=50, T=w["n_points"])
    if workload == "mh":
        return models.GaussianMixture.synthetic(n_points=w["n_points"])
    return models.PolyRegression.synthetic(n_points=w["n_points"])


def flops_per_particle(workload: str, n_points: int) -> float:
    """Algorithmic fp32 flops of one particle's model evaluation."""
    if workload in ("linreg", "dsl-linreg"):
        return 5.0 * n_points  # per point: (y - b) add, fma(-a, x, .), fma(r, r, acc)
    # poly, E[n] = 3: Horner (n-1) fma + (y - p) add + fma(r, r, acc) per point
    return n_points * (2 * 2 + 1 + 2)


# ----------------------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers --
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard(args, wl: dict, rank: int, world: int) -> tuple[int, int, int]:
    """(lo, hi, total): this rank's global particle ids [lo, hi) and the whole job's count.

    Strong-scaled workloads fix the total (C2: 1e9 over 1-8 GPUs, BASELINE configs[1]); weak-
    scaled ones fix the per-GPU share (C5: 1.25e10 per GPU, 1e11 on 8). Ranks own
    [floor(rN/R), floor((r+1)N/R)) like infer.shard_range."""
    n = args.particles or wl["particles"]
    total = n if wl["scaling"] == "strong" else n * world
    return total * rank // world, total * (rank + 1) // world, total


def relaunch(argv: list, gpus: int) -> int:
    """`--gpus N` without a launcher: the same command under torch.distributed.run, one process
    per GPU, rendezvous on 127.0.0.1; NCCL communicator init lines go to stderr."""
    from paper_2010_08454_b200.cli import relaunch_command

    cmd = relaunch_command(argv, gpus)
    i = cmd.index("-m", cmd.index("torch.distributed.run") + 1)
    cmd[i:i + 2] = [str(Path(__file__).resolve())]  # run bench.py, not the package CLI
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd + [f"--gpus={gpus}"], env=env)


def run_dry(args) -> dict | None:
    """Multi-rank orchestration without a GPU (gloo on CPU): the same sharding, the same 256-B
    rank-record all-gather and max-over-ranks timing as run_ours, no kernel launched."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    wl = WORKLOADS[args.workload]
    lo, hi, total = shard(args, wl, rank, world)
    rec = torch.zeros(256, dtype=torch.uint8)
    rec[:8] = torch.tensor(list((hi - lo).to_bytes(8, "little")), dtype=torch.uint8)
    gathered = torch.empty(world * 256, dtype=torch.uint8)
    t0 = time.perf_counter()
    if world > 1:
        dist.all_gather_into_tensor(gathered, rec)
    else:
        gathered.copy_(rec)
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    counts = [int.from_bytes(bytes(gathered[r * 256:r * 256 + 8].tolist()), "little") for r in range(world)]
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return None
    assert sum(counts) == total, (counts, total)
    return {"metric": METRICS[args.workload][0], "value": None, "unit": METRICS[args.workload][1],
            "n_gpus": world, "steps": 0, "warmup": 0, "dry_run": True, "scaling": wl["scaling"],
            "config": {"workload": wl["name"], "particles": total, "rank_shares": counts,
                       "parallelism": f"particle-sharded dp{world} (gloo dry run, no kernels)"},
            "max_rank_s": dt.item()}


def python_scalar_rate(workload: str, model, seconds: float = 3.0) -> dict:
    """SURVEY.md §8(d) CPU protocol item (i): the reference-arithmetic scalar Python rate on one
    core — per particle the reference's keyed split stream (rng.py:31-41) and draw algorithms
    (rng.py:43-117, restated in oracle/refstream.py) and the model's log-weight in Python floats,
    as the reference's (absent) VM would compute it."""
    from oracle import refstream

    xs = [float(x) for x in model.xs]
    ys = [float(y) for y in model.ys]
    base = refstream.key_of(1)
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < seconds:
        s = refstream.SplitMixStream(key=refstream.split_key(base, n))
        if workload in ("linreg", "dsl-linreg"):
            a, b = s.normal(0.0, 10.0), s.normal(0.0, 10.0)
            lw = 0.0
            for x, y in zip(xs, ys):
                z = (y - (a * x + b)) / model.sigma
                lw += -0.5 * z * z - math.log(model.sigma) - 0.5 * math.log(2 * math.pi)
        else:
            k = 2 + s.randint(3)
            c = [s.normal(0.0, 10.0) for _ in range(k)]
            lw = 0.0
            for x, y in zip(xs, ys):
                p = 0.0
                for cj in reversed(c):
                    p = p * x + cj
                lw -= (y - p) ** 2
        n += 1
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{n} particles in {dt:.1f} s: scalar Python, reference arithmetic (refstream SplitMix "
                      "streams and draw algorithms, fp64 log-weights)"}


def cpu_baseline(workload: str, model, target_s: float = 12.0, threads: int | None = None) -> dict:
    """Oracle (C port of the reference semantics) on the host cores, bounded sample."""
    from oracle import core

    core.build()
    threads = threads or os.cpu_count() or 1
    key = 0x9E0160293A33AAF7
    run = (lambda lo, hi: core.is_linreg(model.xs, model.ys, model.sigma, lo, hi, key, threads=threads)) \
        if workload in ("linreg", "dsl-linreg") else (lambda lo, hi: core.is_poly(model.xs, model.ys, lo, hi, key, threads=threads))
    n = 20_000 if workload in ("linreg", "dsl-linreg") else 500_000
    t0 = time.perf_counter()
    run(0, n)
    dt = time.perf_counter() - t0
    n2 = max(n, int(n * target_s / max(dt, 1e-3)))
    t0 = time.perf_counter()
    run(0, n2)
    dt = time.perf_counter() - t0
    return {"value": n2 / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n2} particles of the same model/data in {dt:.1f} s "
                      f"(oracle/cuppl_oracle.c, fp64, OpenMP {threads} threads)",
            "python_scalar_1core": python_scalar_rate(workload, model)}


def calibrate_philox(device) -> float:
    """Measured Philox4x32-10 blocks/s on this GPU (csrc/calib_kernels.cu kind 2)."""
    import torch

    from paper_2010_08454_b200 import _native as N

    L = N.lib()
    sink = torch.zeros(256, dtype=torch.float32, device=device)
    sm = torch.cuda.get_device_properties(device).multi_processor_count
    blocks, iters = sm * 16, 400
    st = N.stream_ptr(device)
    N.check(L.cuppl_calibrate(2, blocks, iters, N.ptr(sink), st))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    N.check(L.cuppl_calibrate(2, blocks, iters, N.ptr(sink), st))
    e1.record()
    torch.cuda.synchronize()
    return blocks * 256 * iters / (e0.elapsed_time(e1) / 1e3)


def calibrate_fp32(device) -> float:
    """Measured FFMA2 ceiling (FLOP/s) on this GPU (csrc/calib_kernels.cu kind 0)."""
    import torch

    from paper_2010_08454_b200 import _native as N

    L = N.lib()
    sink = torch.zeros(256, dtype=torch.float32, device=device)
    sm = torch.cuda.get_device_properties(device).multi_processor_count
    blocks, iters = sm * 8, 4000
    st = N.stream_ptr(device)
    for _ in range(2):
        N.check(L.cuppl_calibrate(0, blocks, iters, N.ptr(sink), st))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    N.check(L.cuppl_calibrate(0, blocks, iters, N.ptr(sink), st))
    e1.record()
    torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) / 1e3
    return blocks * 256 * iters * 512.0 / secs


def load_traffic(workload: str):
    """ncu-measured DRAM bytes (dram__bytes_read + write) per launch of the dominant kernel."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(workload)
        except json.JSONDecodeError:
            return None
    return None


# ----------------------------------------------------------------------------- arms -----
def run_ours(args) -> dict | None:
    import torch
    import torch.distributed as dist

    from paper_2010_08454_b200 import build as B

    B.build()
    from paper_2010_08454_b200 import Rng, infer

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    wl = WORKLOADS[args.workload]
    lo, hi, total = shard(args, wl, rank, world)
    per_gpu = hi - lo
    model = make_model(args.workload)
    if args.workload == "dsl-linreg":  # the same model and data, from CuPPL source
        from paper_2010_08454_b200 import frontend

        src_model, model = model, frontend.compile_program(DSL_LINREG, data={"xs": model.xs, "ys": model.ys})
        launcher = frontend.DslLauncher(model, device)
    else:
        src_model = model
        launcher = infer.IsLauncher(model, device)
    base = Rng(1)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=device)
    gathered = torch.empty(world * 256, dtype=torch.uint8, device=device)

    def step(k: int):
        launcher.launch(lo, hi, base.split(k).key)
        if world > 1:
            dist.all_gather_into_tensor(gathered, launcher.rec)

    for k in range(args.warmup):
        step(10_000 + k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the step events)
        starts[k].record()
        step(k)
        ends[k].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    t_ms = total_ms.item()
    value = total * args.steps / (t_ms / 1e3)

    # e2e: the public API from host data (model arrays in host memory -> kernel parameter
    # block; record + mode trace back to the host), same particle count and GPUs.
    e2e_steps = max(1, min(args.steps, 3))
    infer.run_importance(model, total, Rng(777))  # warm
    torch.cuda.synchronize()
    e2e_t = []
    for k in range(e2e_steps):
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        post = infer.run_importance(model, total, base.split(500 + k))
        e1.record()
        torch.cuda.synchronize()
        e2e_t.append(e0.elapsed_time(e1))
    e2e_ms = torch.tensor([sum(e2e_t)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = total * e2e_steps / (e2e_ms.item() / 1e3)
    h2d = src_model.xs.nbytes + src_model.ys.nbytes
    d2h = 256 * world + (16 if args.workload == "poly" else 8) + (4 if args.workload == "poly" else 0)

    result = None
    if rank == 0:
        peak = calibrate_fp32(device)
        fpp = flops_per_particle(args.workload, wl["n_points"])
        kernel_s = (sum(step_ms) / args.steps) / 1e3
        achieved = fpp * per_gpu / kernel_s
        sm_max = clk.get("sm_max_mhz") or 1965.0
        nominal = torch.cuda.get_device_properties(device).multi_processor_count * 128 * 2 * sm_max * 1e6
        roof = {
            "bound": "fp32",
            "achieved": achieved / 1e12,
            "peak": peak / 1e12,
            "unit": "TFLOP/s",
            "frac": achieved / peak,
            "traffic": (load_traffic(args.workload) or {}).get("bytes_per_launch"),
            "peak_source": "measured FFMA2 ceiling on this GPU (csrc/calib_kernels.cu kind 0); "
                           "MEASURED_PEAKS.json has no fp32 CUDA-core figure",
            "nominal_peak": nominal / 1e12,
            "frac_of_nominal": achieved / nominal,
            "flops_per_particle": fpp,
        }
        if args.workload == "poly":
            # SURVEY.md §8(d) C1/C5 roofline (fixed definition): issue-bound on the FMA pipe,
            # Philox at its MEASURED rate on this GPU (calib kind 2; the survey's 40-instruction
            # count is faster than the hardware's quarter-rate IMAD.WIDE) plus the algorithmic
            # I_fp32 = 86 FP32 instructions per particle (E[n] = 3: Horner 40 FFMA + 20 FADD +
            # 20 FFMA + 6) at 128 lanes/clk/SM, serialised (no credit for overlapping the two)
            ph = calibrate_philox(device)
            n_sm = torch.cuda.get_device_properties(device).multi_processor_count
            f_sm = (clk.get("sm_mhz") or sm_max) * 1e6
            i_fp32 = 86.0
            roof_rate = 1.0 / (1.0 / ph + i_fp32 / (128.0 * n_sm * f_sm))
            rate = per_gpu / kernel_s
            flop_roof = 1.0 / (1.0 / ph + fpp / peak)
            roof = {"bound": "issue (fma pipe: Philox IMAD.WIDE + fp32)", "achieved": rate,
                    "peak": roof_rate, "unit": "particles/s", "frac": rate / roof_rate,
                    "traffic": (load_traffic(args.workload) or {}).get("bytes_per_launch"),
                    "peak_source": f"SURVEY.md §8(d) C5: measured Philox {ph:.3g} blocks/s (calib kind 2) + "
                                   f"I_fp32 = 86 instr/particle at 128 lanes/clk x {n_sm} SMs x {f_sm / 1e6:.0f} MHz",
                    "flops_per_particle": fpp,
                    "flop_roof": flop_roof, "frac_of_flop_roof": rate / flop_roof,
                    "flop_roof_source": f"Philox + {fpp:.0f} flops/particle at the measured FFMA2 peak "
                                        f"{peak / 1e12:.1f} TFLOP/s (counts an FADD at half an FFMA's cost)"}
        result = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps,
            "higher_is_better": True,
            "scaling": wl["scaling"],
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (numpy seed 0, fp64 -> fp32; SURVEY.md §8(d)); Philox draws keyed by Rng(1).split(step)",
            "config": {
                "workload": wl["name"],
                "particles": total,
                "particles_rank0": per_gpu,
                "n_points": wl["n_points"],
                "parallelism": f"particle-sharded dp{world} (NCCL all-gather of 256 B rank records)",
                "l2": "flushed between timed steps (256 MiB write, excluded by per-step CUDA events)",
            },
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "paper_2010_08454_b200.infer.run_importance(model, n, rng)",
                    "log_z": post.log_z, "ess": post.ess},
            "gpu_launches": args.steps,
            "clocks": clk,
        }
        if args.workload == "dsl-linreg":
            result["config"]["particles_per_thread"] = launcher.lanes  # dsl_lanes.cuh build chosen
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline("linreg" if args.workload == "dsl-linreg" else args.workload,
                                                  src_model)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def _hbm_peak() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
        except (KeyError, ValueError, json.JSONDecodeError):
            pass
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def run_ours_engine(args) -> dict | None:
    """SMC (C4) and many-chain MH (C3) workloads on one GPU."""
    import torch

    from paper_2010_08454_b200 import build as B

    B.build()
    from paper_2010_08454_b200 import Rng, infer, smc

    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    wl = WORKLOADS[args.workload]
    model = make_model(args.workload)
    metric, unit = METRICS[args.workload]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=device)
    if args.workload == "smc":
        n = args.particles or wl["particles"]
        T = model.T
        # buffers built once; one process per GPU: the whole T-step run is one captured CUDA graph
        # (device-resident key), replayed per step; N > 1 launches step by step around NCCL
        runner = smc.SmcRunner(model, n, Rng(1), steps=T, device=device, graph=True)
        if runner.use_graph:
            runner.k6_events = []  # captured with the graph (event-record nodes) during warm-up
            runner.k6_every = 8    # K6 timed on every 8th time step (125 launches per run)

        def step(k):
            runner.reseed(Rng(1).split(k))
            runner.launch()
            return runner
        units_per_step = T  # time steps of the whole (strong-scaled) population
    else:
        chains = args.particles or wl["particles"]
        n_steps = args.mh_steps

        def step(k):  # weak scaling: `chains` chains per GPU, sharded by rank inside run_lmh
            return infer.run_lmh(model, n_steps, Rng(1).split(k), chains=chains * world, device=device)
        units_per_step = chains * n_steps * world
    for k in range(args.warmup):
        step(10_000 + k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    last = None
    k6_sum = k6_count = 0
    if args.workload == "smc" and not runner.use_graph:
        runner.k6_events = []  # dominant kernel (K6) timed live on its stream
    for k in range(args.steps):
        flush.zero_()
        starts[k].record()
        last = step(k)
        ends[k].record()
        if args.workload == "smc" and runner.use_graph:  # each replay re-records the same events
            torch.cuda.synchronize()
            k6_sum, k6_count = k6_sum + runner.k6_ms(), k6_count + len(runner.k6_events)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    t_ms = tot.item()
    value = units_per_step * args.steps / (t_ms / 1e3)
    if rank != 0:
        if args.workload == "smc":
            infer.run_smc(model, n, Rng(99))  # e2e leg is collective
        else:
            infer.run_lmh(model, args.mh_steps, Rng(99), chains=units_per_step // args.mh_steps)
        dist.barrier()
        dist.destroy_process_group()
        return None
    res = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
           "scaling": "strong" if args.workload == "smc" else "weak", "vs_baseline": None,
           "dtype": "f32", "data": "synthetic (numpy seed 0; SURVEY.md §8(d))",
           "config": {"workload": wl["name"], "l2": "flushed between timed steps (256 MiB write)"},
           "clocks": clk}
    if args.workload == "smc":
        peak, src = _hbm_peak()
        if runner.use_graph:
            k6_ms = k6_sum / k6_count
        else:
            k6 = [a.elapsed_time(b) for a, b in runner.k6_events]
            k6_ms = sum(k6) / len(k6)
        runner.k6_events = None
        # SURVEY.md §8(d) C4 per-unit figure, K6 share, s = 1 B state: reads lw_t (4) + ancestor
        # x_t (s), writes x_{t+1} (s) + lw_{t+1} (4). This build never stores a log-weight (a
        # state's weight is tabulated per step), so K6 moves ~1.6 B/particle (ncu traffic below)
        # and is bound by instruction issue, not HBM.
        k6_bytes = 10.0 * n / world
        achieved = k6_bytes / (k6_ms / 1e3) / 1e9
        tr = load_traffic("smc")
        res["config"].update({"particles": n, "time_steps": T, "state": "u8", "resampling": "systematic every step",
                              "launch": "one CUDA graph per run (init + T steps)" if runner.use_graph else "eager",
                              "parallelism": (f"particle-partitioned dp{world} (device-side peer exchanges: "
                                              "max + 32-B record all-gather per step over CUDA-IPC arenas, "
                                              "peer stores)") if world > 1 else "dp1"})
        res["roofline"] = {"bound": "hbm", "kernel": "smc_resample_kernel (K6)", "achieved": achieved, "peak": peak,
                           "unit": "GB/s", "frac": achieved / peak,
                           "traffic": None if tr is None else tr["bytes_per_launch"] * (n / tr["n"]),
                           "peak_source": src, "algorithmic_bytes_per_particle": 10,
                           "k6_ms_avg": k6_ms, "k6_share_of_step": k6_ms * T / (t_ms / args.steps),
                           "note": "state-only populations: measured DRAM traffic ~1.6 B/particle vs the "
                                   "survey's 10 B; K6 is issue-bound"}
        res["particle_steps_per_s"] = n * units_per_step * args.steps / (t_ms / 1e3)
        res["gpu_launches"] = args.steps * (1 + 2 * T)
        # e2e: public API from host data (model arrays host -> device tables), result to host
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = infer.run_smc(model, n, Rng(99))
        e1.record()
        torch.cuda.synchronize()
        res["e2e"] = {"value": T / (e0.elapsed_time(e1) / 1e3), "unit": unit,
                      "h2d_bytes_per_step": int(model.A.nbytes + model.ys.nbytes + model.mu.nbytes),
                      "d2h_bytes_per_step": int(T * 4 * 8 + T * 16 + T * 4 + 50 * 8),
                      "api": "paper_2010_08454_b200.infer.run_smc(model, n, rng)", "log_z": out.log_z}
    else:
        peak = calibrate_fp32(device)
        fl = 3.0 * wl["n_points"]  # per chain-step: per point (y - mu) add + fma(r, r, acc)
        achieved = fl * units_per_step / (t_ms / args.steps / 1e3)
        res["config"].update({"chains": units_per_step // args.mh_steps, "steps_per_chain": args.mh_steps,
                              "semantics": "full re-execution per step (reference LMH)"})
        res["roofline"] = {"bound": "fp32", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                           "frac": achieved / peak, "traffic": (load_traffic("mh") or {}).get("bytes_per_launch"),
                           "peak_source": "measured FFMA2 ceiling (csrc/calib_kernels.cu kind 0)",
                           "flops_per_chain_step": fl}
        res["gpu_launches"] = args.steps
        res["acceptance"] = last.acceptance
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = infer.run_lmh(model, args.mh_steps, Rng(99), chains=units_per_step // args.mh_steps)
        e1.record()
        torch.cuda.synchronize()
        res["e2e"] = {"value": units_per_step / (e0.elapsed_time(e1) / 1e3), "unit": unit,
                      "h2d_bytes_per_step": int(model.ys.nbytes), "d2h_bytes_per_step": int(units_per_step // args.mh_steps * 12 * 8),
                      "api": "paper_2010_08454_b200.infer.run_lmh(model, n, rng, chains=...)"}
    if not args.no_cpu_baseline and world == 1:
        res["cpu_baseline"] = cpu_baseline_engine(args, model)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return res


def cpu_baseline_engine(args, model) -> dict:
    from oracle import core

    core.build()
    threads = os.cpu_count() or 1
    if args.workload == "smc":
        n_full = args.particles or WORKLOADS["smc"]["particles"]
        n, T = 1_000_000, 50
        t0 = time.perf_counter()
        core.smc_run(model, n, 0x9E0160293A33AAF7, steps=T)
        dt = time.perf_counter() - t0
        return {"value": n * T / dt / n_full, "unit": "time-steps/s", "cores": threads, "kind": "port",
                "sample": f"{n} particles x {T} steps, oracle/cuppl_oracle.c or_smc_step (OpenMP {threads} "
                          f"threads): {n * T / dt:.3g} particle-steps/s, quoted per step of the "
                          f"{n_full}-particle filter (linear in particles)"}
    chains, steps = 64, 2000
    t0 = time.perf_counter()
    core.mh_gmm(model.ys, model.K, model.prior_sd, model.sigma, chains, steps, 0x9E0160293A33AAF7, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": chains * steps / dt, "unit": "chain-steps/s", "cores": threads, "kind": "port",
            "sample": f"{chains} chains x {steps} steps, oracle/cuppl_oracle.c or_mh_gmm (fp64, OpenMP {threads})"}


def run_ours_resample(args) -> dict | None:
    """Generic resampling (csrc/resample_kernels.cu) of a resident population: each step is one
    cuppl_resample call (max, quantise + scan, TMA-staged gather) over N particles."""
    import numpy as np
    import torch

    from paper_2010_08454_b200 import build as B

    B.build()
    from paper_2010_08454_b200 import Rng, resample
    from paper_2010_08454_b200 import _native as N
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    wl = WORKLOADS["resample"]
    n = args.particles or wl["particles"]
    gen = torch.Generator(device=device).manual_seed(1234 + rank)
    lw = (0.5 * torch.randn(n, device=device, generator=gen)).float()
    payload = torch.arange(n, dtype=torch.int32, device=device)
    out = torch.empty_like(payload)
    r = resample.Resampler(n, device)
    key = Rng(1).key
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=device)
    for k in range(args.warmup):
        r.launch(lw, payload, key, 1000 + k, out, None)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    for k in range(args.steps):
        flush.zero_()
        starts[k].record()
        r.launch(lw, payload, key, k, out, None)
        ends[k].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    t_ms = tot.item()
    value = world * n * args.steps / (t_ms / 1e3)
    # e2e: the public API from host (pinned) arrays: H2D of lw + payload, D2H of the new payload
    lw_h = lw.cpu().pin_memory()
    pay_h = payload.cpu().pin_memory()
    out_h = torch.empty_like(pay_h).pin_memory()
    resample.systematic(lw_h.to(device), pay_h.to(device), Rng(1), 499)  # warm (allocator, first touch)
    torch.cuda.synchronize()
    e2e_t = []
    for k in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = resample.systematic(lw_h.to(device, non_blocking=True), pay_h.to(device, non_blocking=True),
                                  Rng(1), 500 + k)
        out_h.copy_(res.payload, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        e2e_t.append(e0.elapsed_time(e1))
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return None
    peak, src = _hbm_peak()
    kernel_s = (t_ms / args.steps) / 1e3
    bpp = 20.0  # 12 + 2s B per particle-step, s = 4-byte state
    achieved = bpp * n / kernel_s / 1e9
    tr = load_traffic("resample")
    res_line = {
        "metric": METRICS["resample"][0], "value": value, "unit": "particles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64 (exact integer comb), f32 log-weights",
        "data": "synthetic: lw ~ 0.5 N(0,1) fp32, payload = int32 particle ids (torch seed 1234 + rank)",
        "config": {"workload": wl["name"], "particles_per_gpu": n, "payload_bytes": 4,
                   "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": f"replicas dp{world} (one population per GPU)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None if tr is None else tr["bytes_per_launch"] * (n / tr["n"]),
                     "peak_source": src, "algorithmic_bytes_per_particle": bpp,
                     "note": "one step = 3 kernels (RS1 max, RS2 quantise+scan, RS3 TMA-staged gather); "
                             "algorithmic bytes: lw read 3x (12) + payload read + write (8)"},
        "e2e": {"value": n * 2 / (sum(e2e_t) / 1e3), "unit": "particles/s",
                "h2d_bytes_per_step": int(lw_h.nbytes + pay_h.nbytes), "d2h_bytes_per_step": int(out_h.nbytes),
                "api": "paper_2010_08454_b200.resample.systematic(lw, payload, rng, t)"},
        "gpu_launches": 3 * args.steps,
        "clocks": clk,
    }
    if not args.no_cpu_baseline and world == 1:
        from oracle import core

        core.build()
        m = 10_000_000
        lw_c = lw[:m].cpu().numpy()
        pay_c = payload[:m].cpu().numpy()
        t0 = time.perf_counter()
        core.resample(lw_c, pay_c, key, 0)
        dt = time.perf_counter() - t0
        res_line["cpu_baseline"] = {"value": m / dt, "unit": "particles/s", "cores": os.cpu_count() or 1,
                                    "kind": "port", "sample": f"{m} particles, oracle/resample_oracle.c or_resample "
                                                              f"(OpenMP) in {dt:.2f} s"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return res_line


def run_reference(args) -> dict | None:
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    wl = WORKLOADS[args.workload]
    model = make_model(args.workload)
    metric, unit = METRICS[args.workload]
    from oracle import core

    core.build()
    threads = os.cpu_count() or 1
    key = 0x9E0160293A33AAF7
    if args.workload == "smc":
        per_step, cores = 1_000_000, threads
        n_full = args.particles or wl["particles"]
        sample = (f"{per_step} particles x 20 time steps per step (or_smc_step, OpenMP {threads}), rate quoted "
                  f"per time step of the {n_full}-particle filter (linear in particles)")

        def step(k):
            core.smc_run(model, per_step, key + k, steps=20)
        units = 20 * per_step / n_full
    elif args.workload == "resample":
        import numpy as np

        per_step, cores = 10_000_000, threads
        rs_ = np.random.default_rng(1234)
        lw_c = (0.5 * rs_.standard_normal(per_step)).astype(np.float32)
        pay_c = np.arange(per_step, dtype=np.int32)
        sample = f"{per_step} particles per step (oracle/resample_oracle.c or_resample, OpenMP {threads})"

        def step(k):
            core.resample(lw_c, pay_c, key, k)
        units = per_step
    elif args.workload == "mh":
        per_step, cores = 64, threads
        sample = f"{per_step} chains x 200 steps per step (or_mh_gmm, fp64, OpenMP {threads})"

        def step(k):
            core.mh_gmm(model.ys, model.K, model.prior_sd, model.sigma, per_step, 200, key + k, threads=threads)
        units = per_step * 200
    else:
        per_step, cores = (1_000_000 if args.workload in ("linreg", "dsl-linreg") else 20_000_000), threads
        sample = (f"{per_step} particles per step of the same workload (oracle/cuppl_oracle.c: C restatement of "
                  "the reference semantics; the reference ships no executable inference engine)")

        def step(k):
            if args.workload in ("linreg", "dsl-linreg"):
                core.is_linreg(model.xs, model.ys, model.sigma, k * per_step, (k + 1) * per_step, key, threads=threads)
            else:
                core.is_poly(model.xs, model.ys, k * per_step, (k + 1) * per_step, key, threads=threads)
        units = per_step
    for k in range(args.warmup):
        step(1000 + k)
    t0 = time.perf_counter()
    for k in range(args.steps):
        step(k)
    dt = time.perf_counter() - t0
    value = units * args.steps / dt
    return {
        "metric": metric, "value": value, "unit": unit, "n_gpus": max(world, args.gpus), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
        "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "impl": "reference",
        "config": {"workload": wl["name"], "units_per_step": units, "n_points": wl["n_points"]},
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="linreg")
    ap.add_argument("--particles", type=int, default=0, help="override particles per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mh-steps", type=int, default=10_000, help="MH steps per chain (workload mh)")
    ap.add_argument("--dry-run", action="store_true", help="gloo on CPU, no kernels (orchestration only)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return relaunch(sys.argv[1:], args.gpus)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.dry_run:
        res = run_dry(args)
    elif args.impl == "reference":
        res = run_reference(args)
    elif args.workload == "resample":
        res = run_ours_resample(args)
    elif args.workload in ("smc", "mh"):
        res = run_ours_engine(args)
    else:
        res = run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
