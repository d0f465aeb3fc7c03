"""Many-chain lightweight Metropolis-Hastings (K7) — the GPU form of run_lmh.

The reference runs ONE single-site LMH chain. Here `chains` independent chains
run in one kernel (one warp each: replicas — with torch.distributed the chains
are sharded over ranks and only the per-chain statistics are all-gathered at the end).
Every step re-executes the model (full log-likelihood, the reference's re-execution semantics)
and accepts with the single-site prior-proposal ratio. The oracle restatement is
oracle/cuppl_oracle.c or_mh_gmm.
"""

from __future__ import annotations

import math
import numpy as np

from . import _native as N
from .errors import InferRuntimeError
from .infer import EmpiricalDistribution
from .models import GaussianMixture
from .rng import key_of, seed_of


class ChainsDistribution(EmpiricalDistribution):
    """The EmpiricalDistribution of `chains` LMH chains' recorded
    return values — the sorted component means (label switching), a real vector: singleton
    support, summarised like a compiled model's vector return (mean["v<k>"],
    stats["var_v<k>"]), plus the chain diagnostics the many-chain form adds (per-chain means
    for Monte Carlo standard errors, acceptance rate, final states)."""

    @property
    def acceptance(self) -> float:
        return self.stats["acceptance"]

    @property
    def n_chains(self) -> int:
        return self.stats["chains"]

    @property
    def mean_vec(self) -> np.ndarray:
        return np.array([self.mean[f"v{k}"] for k in range(len(self.mean))])

    @property
    def var_vec(self) -> np.ndarray:
        return np.array([self.stats[f"var_v{k}"] for k in range(len(self.mean))])

    @property
    def chain_means(self) -> np.ndarray:
        return self.record["chain_means"]

    def mcse(self) -> np.ndarray:
        """Monte Carlo standard error of the mean from the between-chain spread."""
        cm = self.chain_means
        return cm.std(axis=0, ddof=1) / math.sqrt(len(cm))


def run_lmh(model: GaussianMixture, n_samples: int, rng, *, chains: int = 4096, burn_in: int = 0,
            thin: int = 1, return_trace: bool = False, group=None, device=None) -> ChainsDistribution:
    """`chains` independent LMH chains of `n_samples` steps each on the GPU; the result is the
    EmpiricalDistribution of the recorded sorted means."""
    import torch

    from .infer import _world, shard_range

    if not isinstance(model, GaussianMixture):
        raise InferRuntimeError(f"no MH kernel for {type(model).__name__}")
    if n_samples < 1 or chains < 1:
        raise ValueError("n_samples and chains must be >= 1")
    L = N.lib()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    rank, world = _world(group)
    c0, c1 = shard_range(chains, rank, world)
    nc = c1 - c0
    K, D = model.K, len(model.ys)
    dpad = L.cuppl_mh_padded_points(D)
    y = torch.zeros(dpad, dtype=torch.float32, device=dev)
    y[:D] = torch.from_numpy(np.ascontiguousarray(model.ys, dtype=np.float32)).to(dev)
    n_rec = 0 if n_samples <= burn_in else (n_samples - burn_in + thin - 1) // thin
    mu = torch.empty((max(nc, 1), K), dtype=torch.float32, device=dev)
    ll = torch.empty(max(nc, 1), dtype=torch.float32, device=dev)
    st = torch.zeros((max(nc, 1), 2 * K + 2), dtype=torch.float64, device=dev)
    tr = torch.empty((max(nc, 1), max(n_rec, 1), K), dtype=torch.float32, device=dev) if return_trace else None
    if nc:
        rc = L.cuppl_mh_gmm(N.ptr(y), D, K, float(model.prior_sd), float(model.sigma), nc, c0, n_samples,
                            burn_in, thin, key_of(rng), N.ptr(mu), N.ptr(ll), N.ptr(st), N.ptr(tr),
                            n_rec, N.stream_ptr(dev))
        N.check(rc, "mh_gmm", seed=seed_of(rng))
    stats = st[:nc]
    if world > 1:  # replicas: gather the per-chain statistics in rank (= chain) order
        import torch.distributed as dist

        sizes = [shard_range(chains, q, world)[1] - shard_range(chains, q, world)[0] for q in range(world)]
        tdev = dev if dist.get_backend(group) == "nccl" else torch.device("cpu")  # gloo: host tensors
        pad = torch.zeros((max(sizes), 2 * K + 2), dtype=torch.float64, device=tdev)
        pad[:nc] = stats.to(tdev)
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        stats = torch.cat([parts[q][:sizes[q]] for q in range(world)])
    s = stats.cpu().numpy()
    nrec = s[:, 2 * K]
    tot = nrec.sum()
    if tot <= 0:
        raise InferRuntimeError("no recorded samples (n_samples <= burn_in)")
    mean = s[:, :K].sum(axis=0) / tot
    var = s[:, K:2 * K].sum(axis=0) / tot - mean ** 2
    chain_means = s[:, :K] / np.maximum(nrec, 1)[:, None]
    acc = float(s[:, 2 * K + 1].sum() / (len(s) * n_samples))
    out = ChainsDistribution(n=int(tot))
    out.mean = {f"v{k}": float(mean[k]) for k in range(K)}
    out.stats = {f"var_v{k}": float(var[k]) for k in range(K)}
    out.stats.update({"acceptance": acc, "chains": chains, "steps": n_samples,
                      "recorded_per_chain": int(nrec[0]) if len(nrec) else 0})
    out.record = {"chain_stats": s, "chain_means": chain_means}
    out.traces = {"final_mu": mu[:nc], "final_log_lik": ll[:nc]}
    if tr is not None:
        out.traces["sorted_mu"] = tr[:nc]
    return out
