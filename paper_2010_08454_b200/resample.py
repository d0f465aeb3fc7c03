"""Generic systematic resampling on the GPU (C ABI cuppl_resample, csrc/resample_kernels.cu).

SMC is a non-goal of the reference; BASELINE's north_star names "resampling and
ancestor gather (TMA-staged cumulative weights, binary search, coalesced particle copy)". This
is that primitive for ANY population: fp32 log-weights plus an arbitrary per-particle payload
(a torch tensor whose first axis is the particle), resampled with the exact integer comb of
SURVEY.md Appendix A D6 — ancestors are bit-identical to oracle/resample_oracle.c for any
weights. The HMM filter (smc.py) applies the same rule to one-byte states with its fused
kernels; `GenericSmc` below runs a particle filter for any model whose propagation and
weighting are written as torch operations on the payload, with this primitive in between.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import _native as N
from .errors import AllZeroWeightError, InferRuntimeError
from .rng import key_of


@dataclass
class Resampled:
    payload: object       # torch tensor like the input payload (None when no payload)
    ancestors: object     # int64 tensor [n] (None unless requested)
    max_lw: float
    total: int            # T, the exact integer weight total
    ess: float            # (sum e)^2 / sum e^2
    log_z_increment: float  # M + ln(sum e / n): this step's log-evidence factor


class Resampler:
    """Device buffers for repeated resampling of populations of `n` particles."""

    def __init__(self, n: int, device=None):
        import torch

        if not 1 <= n < 2**31:
            raise ValueError("n must be in [1, 2^31)")
        self.n = n
        device = torch.device(device) if device is not None else torch.device("cuda")
        if device.type == "cuda" and device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        L = N.lib()
        self.ws = torch.empty(L.cuppl_resample_workspace_bytes(n), dtype=torch.uint8, device=self.device)
        self.stats = torch.empty(4, dtype=torch.float64, device=self.device)  # cuppl_resample_stats

    def launch(self, lw, payload, key: int, t: int, payload_out=None, ancestors_out=None) -> None:
        """Stream-ordered launch (no host sync); stats land in self.stats."""
        import torch

        if lw.dtype != torch.float32 or lw.numel() != self.n or not lw.is_contiguous():
            raise ValueError("lw must be a contiguous float32 tensor of n elements")
        bufs = [lw] + [b for b in (payload, payload_out, ancestors_out) if b is not None]
        if any(b.device != self.device for b in bufs):
            raise ValueError(f"every buffer must be on {self.device}")
        nbytes = 0
        if payload is not None:
            if payload.shape[0] != self.n or not payload.is_contiguous():
                raise ValueError("payload must be contiguous with the particle as its first axis")
            nbytes = payload.element_size() * payload[0].numel()
            if (payload_out is None or not payload_out.is_contiguous()
                    or payload_out.numel() * payload_out.element_size() != self.n * nbytes):
                raise ValueError("payload_out must be a contiguous buffer of the payload's size")
        if ancestors_out is not None and (ancestors_out.dtype != torch.int64 or ancestors_out.numel() != self.n
                                          or not ancestors_out.is_contiguous()):
            raise ValueError("ancestors_out must be a contiguous int64 tensor of n elements")
        L = N.lib()
        rc = L.cuppl_resample(N.ptr(lw), self.n, N.ptr(payload), nbytes, key, t, N.ptr(payload_out),
                              N.ptr(ancestors_out), N.ptr(self.stats), N.ptr(self.ws), self.ws.numel(),
                              N.stream_ptr(self.device))
        N.check(rc, "resample")

    def read_stats(self) -> tuple:
        import numpy as np

        raw = self.stats.cpu().numpy()
        total = int(raw[1:2].view(np.uint64)[0])
        return float(raw[0]), total, float(raw[2]), float(raw[3])


def systematic(lw, payload=None, rng=0, t: int = 0, *, ancestors: bool = False) -> Resampled:
    """Resample the population (lw, payload) once: returns the new payload (and ancestors)."""
    import torch

    n = lw.numel()
    r = Resampler(n, lw.device)
    out = torch.empty_like(payload) if payload is not None else None
    anc = torch.empty(n, dtype=torch.int64, device=lw.device) if ancestors else None
    r.launch(lw.contiguous(), None if payload is None else payload.contiguous(), key_of(rng), t, out, anc)
    m, total, s1, s2 = r.read_stats()
    if total == 0:
        raise AllZeroWeightError("every particle has weight 0 after quantisation (SPEC.md:421)")
    return Resampled(out, anc, m, total, s1 * s1 / s2, m + math.log(s1 / n))


@dataclass
class SmcRun:
    log_z: float
    log_z_steps: list
    ess: list
    payload: object  # final population (after the last reweighting, before resampling)
    log_weights: object


class GenericSmc:
    """Bootstrap particle filter for any model given as torch functions on the payload:

        init(n) -> payload                      (t = 0 draws)
        weight(payload, t) -> lw (float32 [n])  (log-likelihood of observation t)
        propagate(payload, t) -> payload        (transition t -> t + 1)

    Each step: weight, resample on the GPU (cuppl_resample, exact D6 comb keyed by the run's
    rng), propagate. log Z = sum over steps of M_t + ln(sum e / n)."""

    def __init__(self, init, weight, propagate, n: int, device=None):
        self.init, self.weight, self.propagate, self.n = init, weight, propagate, n
        self.r = Resampler(n, device)

    def run(self, steps: int, rng) -> SmcRun:
        import torch

        key = key_of(rng)
        x = self.init(self.n)
        out = torch.empty_like(x)
        log_z, lzs, esss = 0.0, [], []
        lw = None
        for t in range(steps):
            lw = self.weight(x, t).to(torch.float32).contiguous()
            if t + 1 == steps:  # final reweighting: the evidence increment without resampling
                m = float(lw.max())
                if not math.isfinite(m):
                    raise AllZeroWeightError("every particle has weight 0 (SPEC.md:421)")
                e = torch.exp(lw.double() - m)
                s1, s2 = float(e.sum()), float((e * e).sum())
                inc = m + math.log(s1 / self.n)
            else:
                self.r.launch(lw, x, key, t, out, None)
                m, total, s1, s2 = self.r.read_stats()
                if total == 0:
                    raise InferRuntimeError("every particle has weight 0", cause=AllZeroWeightError("all zero"),
                                            seed=None, step=t)
                inc = m + math.log(s1 / self.n)
                x, out = self.propagate(out, t), x
            log_z += inc
            lzs.append(inc)
            esss.append(s1 * s1 / s2)
        return SmcRun(log_z, lzs, esss, x, lw)
