"""Command-line entry point (the reference's absent `cuppl.cli:main`,
pkg/pyproject.toml:16), over this package's GPU engines.

    python -m paper_2010_08454_b200 run --model poly --samples 100000 --seed 1 --format tsv
    python -m paper_2010_08454_b200 bench --filter smc --repeats 3

`run <file.cup>` compiles the program (its result must be importance(model, n)) to CUDA with
frontend.py / NVRTC; `run --model poly | linreg | gmm | hmm` runs one of the registered
hand-written engines (the BASELINE.json configs). The reference's flags, defaults and exit
codes are kept: 0 success, 1 usage / compile / configuration error, 2 runtime (inference)
error. `--seed` falls back to the CUPPL_SEED environment
variable. Posteriors are printed with posterior.serialize_posterior.

`bench` runs every selected workload `--repeats` times with fixed seeds after checking its
correctness predicate on the first run (SPEC.md: "timing never reported for an incorrect
run"), and prints one row per workload: mean and sd of the wall-clock seconds (device work
synchronised) and the rate.
"""

from __future__ import annotations

import argparse
import math
import os
import statistics
import sys
import time

import numpy as np

DEFAULT_SAMPLES = {"importance": 100_000, "mcmc": 10_000, "smc": 100_000}
DEFAULT_INFERENCE = {"poly": "importance", "linreg": "importance", "gmm": "mcmc", "hmm": "smc"}


def _model(name: str, points: int | None):
    from . import models

    if name == "poly":
        return models.PolyRegression.synthetic(n_points=points or 20)
    if name == "linreg":
        return models.LinearRegression.synthetic(n_points=points or 1000)
    if name == "gmm":
        return models.GaussianMixture.synthetic(n_points=points or 10_000)
    if name == "hmm":
        return models.HiddenMarkovModel.synthetic(S=50, T=points or 1000)
    raise ValueError(f"unknown model {name!r}")


class _Summary:
    """Posterior summary in the EmpiricalDistribution shape serialize_posterior expects."""

    def __init__(self, support, log_z, **extra):
        self.support = support
        self.log_z = log_z
        for k, v in extra.items():
            setattr(self, k, v)


def infer_once(model_name: str, inference: str, samples: int, seed: int, *, burn_in: int = 0, thin: int = 1,
               chains: int = 4096, points: int | None = None, smc_steps: int | None = None):
    """Run one inference; returns a posterior with .support / .log_z (and summaries)."""
    from . import infer
    from .rng import Rng

    model = _model(model_name, points)
    rng = Rng(seed)
    if inference == "importance":
        return infer.run_importance(model, samples, rng)
    if inference == "mcmc":
        r = infer.run_lmh(model, samples, rng, chains=chains, burn_in=burn_in, thin=thin)
        return _Summary([], None, n=r.n, mean={"sorted_mu": r.mean_vec.tolist()},
                        var=r.var_vec.tolist(), acceptance=r.acceptance)
    if inference == "smc":
        r = infer.run_smc(model, samples, rng, steps=smc_steps)
        t = max(r.filtering)
        f = r.filtering[t]
        return _Summary([(int(s), float(p)) for s, p in enumerate(f) if p > 0], r.log_z, n=r.n_particles,
                        ess=float(r.ess[t]))
    raise ValueError(f"inference {inference!r} is not available for this build (importance | mcmc | smc)")


def _seed(args) -> int:
    if args.seed is not None:
        return args.seed
    env = os.environ.get("CUPPL_SEED")
    return int(env) if env else 0


def _run_file(args) -> int:
    """`run <file.cup>`: compile the program's importance(model, n) for the GPU and run it."""
    from . import frontend, infer
    from .errors import CupError
    from .posterior import serialize_posterior
    from .rng import Rng

    try:
        src = open(args.file).read()
    except OSError:
        print(f"error: file not found: {args.file}", file=sys.stderr)
        return 1
    try:
        model = frontend.compile_program(src, max_depth=args.max_depth or 20)
    except CupError as e:
        print(e.render() if hasattr(e, "render") else f"error: {e}", file=sys.stderr)
        return 1
    if args.inference not in (None, model.engine):
        print(f"error: this program's engine is {model.engine} (its result expression)", file=sys.stderr)
        return 1
    try:
        if model.engine == "enumerate":
            # the program's own enumerate(model, n) bound unless --max-executions overrides it
            post = infer.run_enumeration(model, args.max_executions or model.default_n,
                                         args.max_depth or None)
        elif model.engine == "mcmc":
            post = infer.run_lmh(model, args.samples or model.default_n, Rng(_seed(args)), chains=args.chains,
                                 burn_in=args.burn_in, thin=args.thin)
        else:
            post = infer.run_importance(model, args.samples or model.default_n, Rng(_seed(args)))
        text = serialize_posterior(post, args.format)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except CupError as e:
        print(e.render() if hasattr(e, "render") else f"error: {e}", file=sys.stderr)
        return 2
    sys.stdout.write(text)
    sys.stdout.flush()
    return 0


def relaunch_command(argv: list, gpus: int) -> list:
    """`run --gpus N` outside a launcher: the same command, one process per GPU, under
    torch.distributed.run (rendezvous on 127.0.0.1)."""
    rest = []
    skip = False
    for a in argv:
        if skip:
            skip = False
            continue
        if a == "--gpus":
            skip = True
            continue
        if a.startswith("--gpus="):
            continue
        rest.append(a)
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "-m", "paper_2010_08454_b200"] + rest


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _join_world():
    """Under torch.distributed.run: one process per GPU, NCCL; only rank 0 prints. The engines
    shard particles / chains over the default group."""
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist.get_rank()


def cmd_run(args, argv=None) -> int:
    from .errors import CupError
    from .posterior import serialize_posterior

    if args.gpus > 1 and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        import subprocess

        return subprocess.call(relaunch_command(list(argv if argv is not None else sys.argv[1:]), args.gpus))
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and _join_world() != 0:
        sys.stdout = open(os.devnull, "w")  # ranks > 0 run their shard and stay silent
    if args.file:
        return _run_file(args)
    if not args.model:
        print("error: run needs a program file or --model", file=sys.stderr)
        return 1
    inference = args.inference or DEFAULT_INFERENCE[args.model]
    samples = args.samples or DEFAULT_SAMPLES.get(inference, 100_000)
    if samples < 1 or args.thin < 1:
        print("error: samples and thin must be >= 1", file=sys.stderr)
        return 1
    try:
        post = infer_once(args.model, inference, samples, _seed(args), burn_in=args.burn_in, thin=args.thin,
                          chains=args.chains, points=args.points, smc_steps=args.smc_steps)
        text = serialize_posterior(post, args.format)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except CupError as e:
        print(e.render() if hasattr(e, "render") else f"error: {e}", file=sys.stderr)
        return 2
    sys.stdout.write(text)
    sys.stdout.flush()
    return 0


# ----------------------------------------------------------------------------- bench ----
def _check(name: str, post) -> str | None:
    """Correctness predicate of a bench workload (closed forms computed here, in fp64)."""
    if name == "poly":
        s = sum(p for _, p in post.support)
        return None if abs(s - 1.0) < 1e-9 and math.isfinite(post.log_z) else f"degree masses sum to {s}"
    if name == "linreg":
        from . import models

        m = models.LinearRegression.synthetic(n_points=1000)
        X = np.stack([np.asarray(m.xs, float), np.ones(len(m.xs))], axis=1)
        prec = X.T @ X / m.sigma ** 2 + np.eye(2) / 100.0
        mean = np.linalg.solve(prec, X.T @ np.asarray(m.ys, float) / m.sigma ** 2)
        sd = np.sqrt(np.diag(np.linalg.inv(prec)))
        got = np.array([post.mean["a"], post.mean["b"]])
        err = np.abs(got - mean) / sd  # importance estimate within a few posterior sds
        return None if np.all(err < 3.0) else f"posterior mean {got} vs conjugate {mean} (sd {sd})"
    if name == "gmm":
        # 1000 single-site steps over 10,005 sites do not mix from a prior draw, so the check is
        # structural: finite, ordered pooled means and a proper acceptance rate
        mu = np.array(post.mean["sorted_mu"])
        ok = np.all(np.isfinite(mu)) and np.all(np.diff(mu) >= 0) and 0.0 < post.acceptance < 1.0
        return None if ok else f"sorted means {mu}, acceptance {post.acceptance}"
    if name == "hmm":
        from . import models

        m = models.HiddenMarkovModel.synthetic(S=50, T=1000)
        A, mu, y = np.asarray(m.A, float), np.asarray(m.mu, float), np.asarray(m.ys, float)
        alpha = np.log(np.asarray(m.pi0, float))
        lz = 0.0
        for t in range(len(y)):  # forward algorithm in log space
            if t:
                mx = alpha.max()
                alpha = np.log(np.exp(alpha - mx) @ A) + mx
            alpha = alpha - 0.5 * ((y[t] - mu) / m.sd) ** 2 - math.log(m.sd) - 0.5 * math.log(2 * math.pi)
            mx = alpha.max()
            c = mx + math.log(np.exp(alpha - mx).sum())
            lz += c
            alpha = alpha - c
        return None if abs(post.log_z - lz) < 2.0 else f"log Z {post.log_z} vs forward algorithm {lz}"
    return None


BENCH = {  # name: (model, inference, samples, unit, units per run)
    "poly": ("poly", "importance", 100_000_000, "particles/s", 100_000_000),
    "linreg": ("linreg", "importance", 100_000_000, "particles/s", 100_000_000),
    "gmm": ("gmm", "mcmc", 1000, "chain-steps/s", 4096 * 1000),
    "hmm": ("hmm", "smc", 1_000_000, "time-steps/s", 1000),
}


def cmd_bench(args) -> int:
    import torch

    rows, failed = [], False
    for name, (model, inference, samples, unit, units) in BENCH.items():
        if args.filter and args.filter not in name:
            continue
        seed = _seed(args)
        times, status = [], "ok"
        try:
            post = infer_once(model, inference, samples, seed)
            bad = _check(name, post)
            if bad:
                status, failed = f"FAILED: {bad}", True
            else:
                for r in range(args.repeats):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    infer_once(model, inference, samples, seed + 1 + r)
                    torch.cuda.synchronize()
                    times.append(time.perf_counter() - t0)
        except Exception as e:  # a failing workload is a row, not a crash
            status, failed = f"FAILED: {type(e).__name__}: {e}", True
        mean = statistics.mean(times) if times else float("nan")
        sd = statistics.stdev(times) if len(times) > 1 else 0.0
        rows.append((name, inference, samples, mean, sd, units / mean if times else float("nan"), unit, status))
    print(f"{'benchmark':10s} {'engine':11s} {'samples':>12s} {'mean s':>10s} {'sd s':>9s} {'rate':>12s}  unit / status")
    for name, inf, n, mean, sd, rate, unit, status in rows:
        print(f"{name:10s} {inf:11s} {n:12d} {mean:10.4f} {sd:9.4f} {rate:12.4g}  {unit} {status}")
    return 1 if failed else 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="cuppl-gpu", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="run one inference and print the posterior")
    r.add_argument("file", nargs="?", help="CuPPL program whose result is importance(model, n) (compiled for "
                   "the GPU by frontend.py)")
    r.add_argument("--model", choices=tuple(DEFAULT_INFERENCE))
    r.add_argument("--inference", choices=("importance", "mcmc", "smc", "enumerate"))
    r.add_argument("--max-executions", type=int, default=0,
                   help="enumeration: bound on the path index space (default: the program's enumerate(model, n))")
    r.add_argument("--max-depth", type=int, default=0,
                   help="enumeration: recursion / choice-point depth bound (SPEC.md RunConfig; default 20)")
    r.add_argument("--samples", "--particles", type=int, default=0,
                   help="particles (importance, smc) or steps per chain (mcmc)")
    r.add_argument("--smc-steps", type=int, default=None, help="smc: time steps to filter (default: all)")
    r.add_argument("--gpus", type=int, default=1, help="one process per GPU (NCCL; relaunched under "
                   "torch.distributed.run unless already inside it)")
    r.add_argument("--seed", type=int, default=None)
    r.add_argument("--burn-in", type=int, default=0)
    r.add_argument("--thin", type=int, default=1)
    r.add_argument("--chains", type=int, default=4096)
    r.add_argument("--points", type=int, default=None, help="data points (time steps for hmm)")
    r.add_argument("--format", choices=("tsv", "json"), default="tsv")
    b = sub.add_parser("bench", help="time the benchmark workloads (correctness checked first)")
    b.add_argument("--filter", default="")
    b.add_argument("--repeats", type=int, default=3)
    b.add_argument("--seed", type=int, default=None)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 1 if e.code else 0
    return cmd_run(args, argv) if args.cmd == "run" else cmd_bench(args)


if __name__ == "__main__":
    sys.exit(main())
