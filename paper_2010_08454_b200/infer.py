"""Inference entry points — the drop-in for `cuppl.infer`.

Signatures follow the SPEC: run_importance(model, n_samples, rng),
run_lmh(model, n_samples, rng), normalize(samples); `rng` is a
`cuppl.rng.Rng` (or this package's mirror, rng.py); `model` is a GPU model descriptor
(models.py) because the reference has no executable model form. Extra arguments are
keyword-only. Every engine runs in libcuppl_gpu.so; there is no CPU path.

Multi-GPU: when torch.distributed is initialised, rank r of R evaluates global particle ids
[floor(rN/R), floor((r+1)N/R)) (Philox counters use the global id, so draws do not depend on
R) and the fixed-size per-rank records are all-gathered and merged in rank order in fp64
(SPEC.md:449 ordered merge) — the only collective of importance sampling.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _native as N
from . import _nvtx
from .errors import AllZeroWeightError, InferRuntimeError
from .models import LinearRegression, PolyRegression
from .rng import key_of, seed_of


@dataclass
class WeightedSample:
    """(value, log_weight)."""

    value: Any
    log_weight: float


@dataclass
class EmpiricalDistribution:
    """Normalised posterior in compact form.

    support      merged (value, probability) pairs of the discrete part of the return value
                 (e.g. the polynomial degree) — real-valued returns have singleton support
                  and are summarised by `mean`, `mode` and, on request, traces
    log_z        log of the normalising-constant estimate: LSE(lw) - log n
    ess          effective sample size (sum w)^2 / sum w^2
    mode         return value of the highest-weight particle (ties -> lowest id, D7)
    """

    support: list = field(default_factory=list)
    n: int = 0
    log_z: float = -math.inf
    ess: float = 0.0
    mode: Any = None
    mode_log_weight: float = -math.inf
    mode_index: int = -1
    mean: dict = field(default_factory=dict)
    stats: dict = field(default_factory=dict)
    traces: dict = field(default_factory=dict)
    record: dict = field(default_factory=dict)

    def probability(self, value) -> float:
        for v, p in self.support:
            if v == value:
                return p
        return 0.0

    def expectation(self, name: str) -> float:
        return self.mean[name]


# ----------------------------------------------------------------------------- helpers --
def _world(group=None):
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return 0, 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Global particle ids owned by `rank`: [floor(rN/R), floor((r+1)N/R))."""
    return n * rank // world, n * (rank + 1) // world


def record_to_dict(rec: N.IsRecord) -> dict:
    d = {f: getattr(rec, f) for f, _ in N.IsRecord._fields_ if f not in ("stat_w", "bin_w")}
    d["stat_w"] = np.array(rec.stat_w[:])
    d["bin_w"] = np.array(rec.bin_w[:])
    return d


def records_from_bytes(buf: np.ndarray) -> list[N.IsRecord]:
    raw = np.ascontiguousarray(buf).view(np.uint8).reshape(-1, N.REC_BYTES)
    return [N.IsRecord.from_buffer_copy(r.tobytes()) for r in raw]


def merge_records(recs: list[N.IsRecord]) -> N.IsRecord:
    """Ordered fp64 merge (native, cuppl_is_record_merge)."""
    arr = (N.IsRecord * len(recs))(*recs)
    out = N.IsRecord()
    N.check(N.lib().cuppl_is_record_merge(arr, len(recs), C.byref(out)), "record_merge")
    return out


def _gather_records(rec_dev, group=None):
    """All-gather the per-rank device record (256 B) and merge in rank order."""
    import torch
    import torch.distributed as dist

    rank, world = _world(group)
    if world == 1:
        return records_from_bytes(rec_dev.cpu().numpy())
    backend = dist.get_backend(group)
    src = rec_dev if backend == "nccl" else rec_dev.cpu()
    out = torch.empty(world * src.numel(), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return records_from_bytes(out.cpu().numpy())


class IsLauncher:
    """Device-level importance-sampling launch for one model (stream-ordered, no sync).

    Keeps the model data on the host side of the ABI (it is passed by value into the kernel
    parameter block) and owns the workspace / record buffers for repeated launches.
    """

    def __init__(self, model, device=None):
        import torch

        self.model = model
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        L = N.lib()
        ws = L.cuppl_is_workspace_bytes_n(len(model.xs))
        self.ws = torch.empty(int(ws), dtype=torch.uint8, device=self.device)
        self.rec = torch.empty(N.REC_BYTES, dtype=torch.uint8, device=self.device)
        self._xs = np.ascontiguousarray(model.xs, dtype=np.float32)
        self._ys = np.ascontiguousarray(model.ys, dtype=np.float32)
        fp = C.POINTER(C.c_float)
        self._xp = self._xs.ctypes.data_as(fp)
        self._yp = self._ys.ctypes.data_as(fp)
        if model.kind not in ("poly", "linreg"):
            raise InferRuntimeError(f"importance sampling kernel for model kind {model.kind!r} not available")

    def launch(self, pid_begin: int, pid_end: int, key: int, injected=None, lw_out=None,
               deg_out=None, coef_out=None, rec_out=None, stream=None) -> None:
        L = N.lib()
        rec = self.rec if rec_out is None else rec_out
        st = stream if stream is not None else N.stream_ptr(self.device)
        m = self.model
        if m.kind == "poly":
            rc = L.cuppl_is_poly(self._xp, self._yp, len(self._xs), pid_begin, pid_end, key,
                                 N.ptr(injected), N.ptr(lw_out), N.ptr(deg_out), N.ptr(coef_out),
                                 N.ptr(rec), N.ptr(self.ws), self.ws.numel(), st)
        else:
            rc = L.cuppl_is_linreg(self._xp, self._yp, len(self._xs), float(m.sigma), pid_begin,
                                   pid_end, key, N.ptr(injected), N.ptr(lw_out), N.ptr(coef_out),
                                   N.ptr(rec), N.ptr(self.ws), self.ws.numel(), st)
        N.check(rc, f"is_{m.kind}")

    def trace_of(self, pid: int, key: int):
        """Re-run one particle to recover its return value (Philox is counter-based)."""
        import torch

        kind = self.model.kind
        coef = torch.empty(4 if kind == "poly" else 2, dtype=torch.float32, device=self.device)
        deg = torch.empty(1, dtype=torch.int32, device=self.device) if kind == "poly" else None
        rec = torch.empty(N.REC_BYTES, dtype=torch.uint8, device=self.device)
        self.launch(pid, pid + 1, key, coef_out=coef, deg_out=deg, rec_out=rec)
        c = coef.cpu().numpy().astype(float).tolist()
        if kind == "poly":
            n = int(deg.cpu().item())
            return c[:n]
        return tuple(c)


def _distribution_from_record(model, rec: N.IsRecord, n: int, launcher: IsLauncher, key: int,
                              traces: dict) -> EmpiricalDistribution:
    if rec.n_finite == 0:
        raise AllZeroWeightError("every particle has log-weight -inf (SPEC.md:421)")
    S, S2, M = rec.sum_w, rec.sum_w2, rec.max_lw
    out = EmpiricalDistribution(n=n, record=record_to_dict(rec), traces=traces)
    out.log_z = M + math.log(S) - math.log(n)
    out.ess = S * S / S2
    out.mode_log_weight = rec.argmax_lw
    out.mode_index = int(rec.argmax_pid)
    out.mode = launcher.trace_of(out.mode_index, key)
    st = np.array(rec.stat_w[:]) / S
    if model.kind == "linreg":
        out.mean = {"a": st[0], "b": st[1]}
        out.stats = {"var_a": st[2] - st[0] ** 2, "var_b": st[3] - st[1] ** 2,
                     "cov_ab": st[4] - st[0] * st[1]}
    else:
        bins = np.array(rec.bin_w[:3]) / S
        out.support = [(d, float(bins[d - 2])) for d in (2, 3, 4)]
        idx = {2: (0, 2), 3: (2, 5), 4: (5, 9)}
        for d, (a, b) in idx.items():
            w = rec.bin_w[d - 2]
            out.mean[f"c|n={d}"] = (np.array(rec.stat_w[a:b]) / w).tolist() if w > 0 else None
    return out


def normalize_tensors(lw, bins=None, n_bins: int = 1) -> dict:
    """K3 on device tensors: lw (fp32/fp64 CUDA tensor), bins (int32 value ids or None).

    Returns {"max_lw", "probs" (np.ndarray [n_bins]), "log_z", "ess", "argmax", "argmax_lw",
    "n_finite"}; raises AllZeroWeightError when every weight is -inf."""
    import torch

    L = N.lib()
    dev = lw.device
    lw = lw.contiguous()
    n = lw.numel()
    if bins is not None:
        bins = bins.to(torch.int32).contiguous()
    out_bins = torch.empty(n_bins, dtype=torch.int64, device=dev)
    out = torch.empty(6, dtype=torch.float64, device=dev)
    ws = torch.empty(int(L.cuppl_normalize_workspace_bytes()), dtype=torch.uint8, device=dev)
    sb = C.c_int(0)
    fn = L.cuppl_normalize_f64 if lw.dtype == torch.float64 else L.cuppl_normalize_f32
    if lw.dtype not in (torch.float64, torch.float32):
        lw = lw.to(torch.float64)
        fn = L.cuppl_normalize_f64
    N.check(fn(N.ptr(lw), N.ptr(bins), n, n_bins, N.ptr(out_bins), N.ptr(out), C.byref(sb), N.ptr(ws),
               ws.numel(), N.stream_ptr(dev)), "normalize")
    o = out.cpu().numpy()
    b = out_bins.cpu().numpy().view(np.uint64)
    nf = int(o[4:5].view(np.uint64)[0])
    if nf == 0:
        raise AllZeroWeightError("every weight is -inf (SPEC.md:421)")
    total = int(b.sum(dtype=np.uint64)) if n_bins > 1 else int(b[0])
    total_f = float(total) * 2.0 ** -sb.value
    M = float(o[0])
    probs = b.astype(np.float64) / float(total) if total > 0 else np.zeros(n_bins)
    return {"max_lw": M, "probs": probs, "log_z": M + math.log(total_f) - math.log(n),
            "ess": total_f * total_f / float(o[1]), "argmax": int(o[3:4].view(np.uint64)[0]),
            "argmax_lw": float(o[2]), "n_finite": nf, "scale_bits": sb.value}


@_nvtx.traced("cuppl.normalize")
def normalize(samples, *, device=None) -> EmpiricalDistribution:
    """normalize(samples): WeightedSample list (or (value, log_weight) pairs)
    -> EmpiricalDistribution. Support is merged by structural equality (value_key,
    cuppl/values.py:101-122) on the host; the log-sum-exp and the per-value masses run in K3."""
    import torch

    from .values import value_key

    if not samples:
        raise AllZeroWeightError("normalize of an empty sample")
    ids, values, lws = {}, [], []
    idx = []
    for s in samples:
        v, lw = (s.value, s.log_weight) if isinstance(s, WeightedSample) else s
        k = value_key(v)
        if k not in ids:
            ids[k] = len(values)
            values.append(v)
        idx.append(ids[k])
        lws.append(float(lw))
    dev = device or torch.device("cuda", torch.cuda.current_device())
    lw_t = torch.tensor(lws, dtype=torch.float64, device=dev)
    b_t = torch.tensor(idx, dtype=torch.int32, device=dev)
    r = normalize_tensors(lw_t, b_t, len(values))
    support = [(v, float(p)) for v, p in zip(values, r["probs"]) if p > 0]
    return EmpiricalDistribution(support=support, n=len(samples), log_z=r["log_z"], ess=r["ess"],
                                 mode=samples[r["argmax"]].value if isinstance(samples[r["argmax"]], WeightedSample)
                                 else samples[r["argmax"]][0],
                                 mode_log_weight=r["argmax_lw"], mode_index=r["argmax"], record=r)


@_nvtx.traced("cuppl.run_lmh")
def run_lmh(model, n_samples: int, rng, *, chains: int = 4096, burn_in: int = 0, thin: int = 1,
            return_trace: bool = False, group=None, device=None):
    """Lightweight Metropolis-Hastings as `chains` independent GPU chains of
    `n_samples` steps (mh.py, kernel K7; compiled programs: frontend.py)."""
    from .frontend import CompiledModel

    if isinstance(model, CompiledModel):
        return _run_compiled_lmh(model, n_samples, rng, chains=chains, burn_in=burn_in, thin=thin, group=group,
                                 device=device)
    from .mh import run_lmh as _run

    return _run(model, n_samples, rng, chains=chains, burn_in=burn_in, thin=thin,
                return_trace=return_trace, group=group, device=device)


@_nvtx.traced("cuppl.run_smc")
def run_smc(model, n_particles: int, rng, *, steps: int | None = None, record_ancestors: bool = False,
            hist_steps=None, group=None, device=None):
    """Bootstrap particle filter with systematic resampling every step (smc.py, K4-K6)."""
    from .smc import run_smc as _run

    return _run(model, n_particles, rng, steps=steps, record_ancestors=record_ancestors,
                hist_steps=hist_steps, group=group, device=device)


@_nvtx.traced("cuppl.run_importance")
def run_importance(model, n_samples: int, rng, *, return_traces: bool = False, group=None,
                   device=None) -> EmpiricalDistribution:
    """Likelihood-weighting importance sampling on the GPU.

    Each particle draws from the prior at every `sample` and adds `factor` terms to its
    log-weight; the result is normalised with a log-sum-exp. With
    torch.distributed initialised the particles are sharded over the ranks.
    """
    import torch

    if n_samples < 1:
        raise ValueError("n_samples must be >= 1")
    from .frontend import CompiledModel

    if isinstance(model, CompiledModel):
        return _run_compiled(model, n_samples, rng, return_traces=return_traces, group=group, device=device)
    if not isinstance(model, (PolyRegression, LinearRegression)):
        raise InferRuntimeError(f"no importance-sampling kernel for {type(model).__name__}")
    rank, world = _world(group)
    lo, hi = shard_range(n_samples, rank, world)
    key = key_of(rng)
    launcher = IsLauncher(model, device)
    dev = launcher.device
    traces = {}
    lw = deg = coef = None
    if return_traces:
        n_local = hi - lo
        lw = torch.empty(n_local, dtype=torch.float32, device=dev)
        coef = torch.empty((n_local, 4 if model.kind == "poly" else 2), dtype=torch.float32, device=dev)
        if model.kind == "poly":
            deg = torch.empty(n_local, dtype=torch.int32, device=dev)
        traces = {"log_weight": lw, "coef": coef, "pid_begin": lo}
        if deg is not None:
            traces["degree"] = deg
    try:
        launcher.launch(lo, hi, key, lw_out=lw, deg_out=deg, coef_out=coef)
        recs = _gather_records(launcher.rec, group)
    except InferRuntimeError as e:
        e.seed = seed_of(rng)
        raise
    rec = merge_records(recs)
    return _distribution_from_record(model, rec, n_samples, launcher, key, traces)


def _run_compiled(model, n_samples: int, rng, *, return_traces: bool, group, device) -> EmpiricalDistribution:
    """run_importance for a model compiled from CuPPL source (frontend.py, NVRTC)."""
    import torch

    from .frontend import MAX_TRACE_DRAWS, DslLauncher, distribution_from_record

    rank, world = _world(group)
    lo, hi = shard_range(n_samples, rank, world)
    key = key_of(rng)
    launcher = DslLauncher(model, device)
    traces, lw, draws = {}, None, None
    if return_traces:
        n_local = hi - lo
        lw = torch.empty(n_local, dtype=torch.float32, device=launcher.device)
        traces = {"log_weight": lw, "pid_begin": lo}
        if 0 < model.max_draws <= MAX_TRACE_DRAWS:
            draws = torch.zeros((n_local, model.max_draws), dtype=torch.float32, device=launcher.device)
            traces["draws"] = draws
    try:
        launcher.launch(lo, hi, key, lw_out=lw, draws_out=draws)
        recs = _gather_records(launcher.rec, group)
        launcher.check_errors()
    except InferRuntimeError as e:
        e.seed = seed_of(rng)
        raise
    out = distribution_from_record(model, merge_records(recs), n_samples, launcher, key)
    out.traces = traces
    return out


ENUM_INDEX_CAP = 1 << 36  # forced-choice indices one enumeration may launch (R^max choice points)
ENUM_BFS_CAP = 1 << 28    # indices whose completed paths are materialised for the breadth-first bound


@_nvtx.traced("cuppl.run_enumeration")
def run_enumeration(model, max_executions: int | None = None, max_depth: int | None = None, *, group=None,
                    device=None) -> EmpiricalDistribution:
    """run_enumeration of a compiled program `enumerate(model, n)` on the GPU.

    Every path through the model's choice points is executed as a forced-choice run (one GPU
    thread per index of the base-R choice space, fp64, frontend.py), weighted by the log-masses
    of its choices plus its factors. `max_executions` counts COMPLETED paths, as in the
    reference's breadth-first traversal (DESIGN DECISIONS "frontier order is FIFO;
    --max-executions counts completed paths"): when the program has more completed paths than
    that, the result keeps the first max_executions in breadth-first order — fewer choices
    first, then support order of the choices — and normalises over them. `max_depth` bounds the
    choice points. The index space R^depth is capped at ENUM_INDEX_CAP.
    """
    from .frontend import CompiledModel, DslLauncher, distribution_from_record

    if not isinstance(model, CompiledModel) or model.engine != "enumerate":
        raise InferRuntimeError("run_enumeration needs a program compiled from enumerate(model, n)")
    depth = model.max_draws
    if max_depth is not None and depth > max_depth:
        raise InferRuntimeError(f"the model has up to {depth} choice points > max_depth={max_depth}")
    n_paths = model.radix ** max(depth, 1)
    if n_paths > ENUM_INDEX_CAP:
        raise InferRuntimeError(f"{n_paths} forced-choice indices (radix {model.radix}, depth {depth}) exceed "
                                f"{ENUM_INDEX_CAP}")
    limit = max_executions if max_executions is not None else model.default_n
    rank, world = _world(group)
    lo, hi = shard_range(n_paths, rank, world)
    launcher = DslLauncher(model, device)
    if limit is not None and limit < n_paths:  # completed paths may exceed the bound: count them
        if world > 1 or n_paths > ENUM_BFS_CAP:
            raise InferRuntimeError(f"{n_paths} forced-choice indices: checking the breadth-first bound of "
                                    f"{limit} completed paths needs one process and <= {ENUM_BFS_CAP} indices; "
                                    f"pass max_executions >= {n_paths}")
        out = _enumeration_bfs(model, launcher, n_paths, int(limit))
        if out is not None:
            return out
    launcher.launch(lo, hi, 0)
    recs = _gather_records(launcher.rec, group)
    launcher.check_errors()
    rec = merge_records(recs)
    out = distribution_from_record(model, rec, n_paths, launcher, 0)
    out.log_z = rec.max_lw + math.log(rec.sum_w)  # exact evidence: the sum over paths
    return out


def _enumeration_bfs(model, launcher, n_paths: int, limit: int):
    """Breadth-first truncation (run_enumeration's docstring): None when every completed path
    fits in `limit` (the record of the whole space is then the result)."""
    import torch

    dev = launcher.device
    lw = torch.empty(n_paths, dtype=torch.float64, device=dev)
    nd = torch.empty(n_paths, dtype=torch.int32, device=dev)
    ret = torch.empty((n_paths, model.return_width), dtype=torch.float32, device=dev)
    rec = torch.empty_like(launcher.rec)
    launcher.launch(0, n_paths, 0, lw_out=lw, draws_out=nd, ret_out=ret, rec_out=rec)
    launcher.check_errors()
    R = model.radix
    p = torch.arange(n_paths, dtype=torch.int64, device=dev)
    ndl = nd.to(torch.int64)
    powR = torch.tensor([R ** k for k in range(max(model.max_draws, 1) + 1)], dtype=torch.int64, device=dev)
    # a path with k choices is index p < R^k (its unused digits zero): its canonical index
    canon = (ndl >= 0) & (p < powR[ndl.clamp(min=0)])
    if int(canon.sum()) <= limit:
        return None
    # breadth-first order: (choices, digits with the first choice most significant)
    lex = torch.zeros_like(p)
    rem = p.clone()
    for k in range(max(model.max_draws, 1)):
        dk = rem % R
        rem = rem // R
        lex = torch.where(k < ndl, lex + dk * powR[(ndl - 1 - k).clamp(min=0)], lex)
    key = ndl * (R ** max(model.max_draws, 1)) + lex
    key = torch.where(canon, key, torch.full_like(key, torch.iinfo(torch.int64).max))
    kept = torch.argsort(key)[:limit]
    # the path's own log-probability (the launch divided out the R^(MAXD - k) indices sharing it)
    lwp = lw[kept] + (model.max_draws - ndl[kept]).to(torch.float64) * math.log(R)
    keep_lw = lwp
    vals = ret[kept]
    out = EmpiricalDistribution(n=limit)
    m = float(keep_lw.max())
    if not math.isfinite(m):
        raise AllZeroWeightError("every kept path has probability 0 (SPEC.md:421)")
    w = torch.exp(keep_lw - m)
    z = float(w.sum())
    out.log_z = m + math.log(z)
    probs = w / z
    out.ess = z * z / float((w * w).sum())
    if model.return_kind in ("int", "bool"):
        v = vals[:, 0].to(torch.int64)
        lo_v = int(v.min())
        agg = torch.zeros(int(v.max()) - lo_v + 1, dtype=torch.float64, device=dev)
        agg.index_add_(0, v - lo_v, probs)
        conv = bool if model.return_kind == "bool" else int
        out.support = [(conv(lo_v + k), float(q)) for k, q in enumerate(agg.cpu().tolist()) if q > 0]
    names = [nm for nm in model.stat_names if not nm.endswith("^2")]
    for j, nm in enumerate(names[:model.return_width]):
        mean = float((probs * vals[:, j].to(torch.float64)).sum())
        out.mean[nm] = mean
        out.stats[f"var_{nm}"] = float((probs * vals[:, j].to(torch.float64) ** 2).sum()) - mean * mean
    out.stats["truncated_paths"] = int(canon.sum()) - limit
    out.record = {"bfs_limit": limit}
    return out


def _run_compiled_lmh(model, n_samples: int, rng, *, chains: int, burn_in: int, thin: int, group,
                      device) -> EmpiricalDistribution:
    """run_lmh of a program compiled from mcmc(model, n): `chains` chains, each recording the
    initial trace and the states after each of the following n_samples - 1 single-site steps;
    the chains are sharded over ranks and their statistics gathered (replicas)."""
    import torch

    from .frontend import run_mcmc

    if model.engine != "mcmc":
        raise InferRuntimeError("run_lmh needs a program compiled from mcmc(model, n)")
    if n_samples < 1 or chains < 1 or thin < 1:
        raise ValueError("n_samples, chains and thin must be >= 1")
    rank, world = _world(group)
    c0, c1 = shard_range(chains, rank, world)
    st = run_mcmc(model, n_samples, rng, chains=c1 - c0, burn_in=burn_in, thin=thin, chain_begin=c0,
                  device=device) if c1 > c0 else np.zeros((0, 1))
    if world > 1:  # replicas: per-chain statistics gathered in rank (= chain) order
        import torch.distributed as dist

        parts = [None] * world
        dist.all_gather_object(parts, st, group=group)
        st = np.concatenate([p for p in parts if len(p)])
    ns, nb = max(model.n_stats, 1), max(model.n_bins, 1)
    nrec = st[:, ns + nb].sum()
    if nrec <= 0:
        raise InferRuntimeError("no recorded samples (n_samples <= burn_in)")
    out = EmpiricalDistribution(n=int(nrec))
    means = st[:, :ns].sum(axis=0) / nrec
    out.mean = {name: float(v) for name, v in zip(model.stat_names, means) if not name.endswith("^2")}
    if model.stat_names and model.stat_names[-1].endswith("^2"):
        half = model.n_stats // 2
        out.stats = {f"var_{model.stat_names[k]}": float(means[half + k] - means[k] ** 2) for k in range(half)}
    if model.n_bins:
        probs = st[:, ns:ns + nb].sum(axis=0) / nrec
        conv = bool if model.return_kind == "bool" else int
        lo = getattr(model, "bin_lo", 0)
        out.support = [(conv(lo + k), float(p)) for k, p in enumerate(probs) if p > 0]
        out.support_truncated = bool(probs.sum() < 1.0 - 1e-9)  # values outside the chain histogram
    steps = max(n_samples - 1, 1)
    out.stats["acceptance"] = float(st[:, ns + nb + 1].sum() / (len(st) * steps))
    out.stats["chains"] = chains
    out.record = {"chain_stats": st}
    return out
