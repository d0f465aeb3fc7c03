"""Built-in distributions: constructors, batch draws and scores on the GPU.

Constructors follow pkg/src/cuppl/builtins.py:86-94 (names with '-' become '_', parameter
order kept: normal(mean, sd), uniform_discrete(a, b) with support [a, b),
...). `sample` / `score` are the batch forms of `sample*` / `dist-score`
(builtins.py:97-99) and run in the K8 kernels of libcuppl_gpu.so;
`variance` is `dist-var`, an analytic host formula.
"""

from __future__ import annotations

import ctypes as C
import math

from . import _native as N
from .errors import InvalidDistParamError, UnsupportedDistError
from .rng import key_of
from .values import (BERNOULLI, BETA, CATEGORICAL, DISCRETE_TAGS, EXPONENTIAL, NORMAL, POISSON,
                     UNIFORM_CONTINUOUS, UNIFORM_DISCRETE, DistValue)


def normal(mean, sd):
    return DistValue(NORMAL, float(mean), float(sd))


def bernoulli(p):
    return DistValue(BERNOULLI, float(p))


def poisson(lam):
    return DistValue(POISSON, float(lam))


def uniform_discrete(a, b):
    return DistValue(UNIFORM_DISCRETE, int(a), int(b))


def uniform_continuous(a, b):
    return DistValue(UNIFORM_CONTINUOUS, float(a), float(b))


def beta(a, b):
    return DistValue(BETA, float(a), float(b))


def exponential(rate):
    return DistValue(EXPONENTIAL, float(rate))


def categorical(weights):
    """categorical(w): P(k) = w_k / sum(w). p0 holds the weight tuple."""
    w = tuple(float(x) for x in weights)
    if not w or any(not (x >= 0.0) or math.isinf(x) for x in w) or sum(w) <= 0.0:
        raise InvalidDistParamError(f"categorical{w}: weights must be finite, >= 0, not all 0")
    return DistValue(CATEGORICAL, w, len(w))


def categorical_thresholds(weights) -> list[int]:
    """u64 inverse-CDF thresholds: t_k = floor(cum_k / total * 2^32), k < K-1.

    A word w in [0, 2^32) selects the smallest k with w < t_k (K-1 if none), so category k
    is drawn with probability (t_k - t_{k-1}) / 2^32 and zero-weight categories never occur.
    """
    total = 0.0
    for v in weights:
        total += v
    out, cum = [], 0.0
    for v in weights[:-1]:
        cum += v
        out.append(min(max(math.floor(cum / total * 4294967296.0), 0), 1 << 32))
    return out


def alias_table(weights) -> list[int]:
    """Walker / Vose alias table with exact integer masses (used by the SMC kernels).

    Column k keeps k when the coin (low 32 bits of w*K for a u32 word w; the column is the high
    32 bits) is below thr_k in [0, 2^32], else yields alias_k; entries are thr | alias << 40.
    Masses m_k = floor(w_k / W * K * 2^32) sum to K * 2^32 after adding the rounding deficit to
    the first largest m_k; small / large stacks are popped LIFO in index order (the oracle's
    or_alias_build restates this exactly).
    """
    K = len(weights)
    unit = 1 << 32
    total = 0.0
    for v in weights:
        total += v
    m = [int(math.floor(float(v) / total * K * 4294967296.0)) for v in weights]
    kmax = 0
    for k in range(K):
        if m[k] > m[kmax]:
            kmax = k
    m[kmax] += K * unit - sum(m)
    small = [k for k in range(K) if m[k] < unit]
    large = [k for k in range(K) if m[k] >= unit]
    thr, alias = [0] * K, [0] * K
    while small and large:
        s, lg = small.pop(), large.pop()
        thr[s], alias[s] = m[s], lg
        m[lg] -= unit - m[s]
        (small if m[lg] < unit else large).append(lg)
    for k in large + small:
        thr[k], alias[k] = unit, k
    return [thr[k] | (alias[k] << 40) for k in range(K)]


def variance(d: DistValue) -> float:
    """dist-var."""
    t = d.tag
    if t == NORMAL:
        return d.p1 ** 2
    if t == BERNOULLI:
        return d.p0 * (1.0 - d.p0)
    if t == POISSON:
        return d.p0
    if t == UNIFORM_DISCRETE:
        n = d.p1 - d.p0
        return (n * n - 1) / 12.0
    if t == UNIFORM_CONTINUOUS:
        return (d.p1 - d.p0) ** 2 / 12.0
    if t == BETA:
        a, b = d.p0, d.p1
        return a * b / ((a + b) ** 2 * (a + b + 1.0))
    if t == EXPONENTIAL:
        return 1.0 / d.p0 ** 2
    if t == CATEGORICAL:
        w = d.p0
        s = sum(w)
        m = sum(k * x for k, x in enumerate(w)) / s
        return sum(x * (k - m) ** 2 for k, x in enumerate(w)) / s
    raise UnsupportedDistError(f"unsupported distribution tag {t}")


def _to_native(d: DistValue, device):
    """Build a cuppl_dist; categorical tables are uploaded to `device` (kept alive by caller)."""
    import torch

    nd = N.Dist()
    nd.tag = d.tag
    keep = None
    if d.tag == CATEGORICAL:
        thr = categorical_thresholds(d.p0)
        nd.n_table = len(d.p0)
        if thr:
            keep = torch.tensor(thr, dtype=torch.int64, device=device)  # values <= 2^32 fit
            nd.table = keep.data_ptr()
        else:
            keep = torch.zeros(1, dtype=torch.int64, device=device)
            nd.table = keep.data_ptr()
    else:
        nd.p0 = float(d.p0)
        nd.p1 = float(d.p1)
        nd.p2 = float(d.p2)
    return nd, keep


def sample(d: DistValue, n: int, rng, first_id: int = 0, device=None):
    """n draws of `sample*(d)` on the GPU; draw i uses Philox stream (first_id + i, TAG_DIST).

    Returns a CUDA tensor: float32 for continuous kinds, int32 for discrete kinds.
    """
    import torch

    device = device or torch.device("cuda", torch.cuda.current_device())
    L = N.lib()
    dtype = torch.int32 if d.tag in DISCRETE_TAGS else torch.float32
    out = torch.empty(n, dtype=dtype, device=device)
    nd, keep = _to_native(d, device)
    rc = L.cuppl_dist_sample(C.byref(nd), key_of(rng), N.TAG_DIST, first_id, n, N.ptr(out),
                             N.stream_ptr(device))
    N.check(rc, "dist_sample")
    del keep  # stream-ordered: the kernel was enqueued before the caching allocator reuses it
    return out


def score(d: DistValue, x):
    """dist-score(d, x) for a CUDA tensor x (float32 or int32 per kind) -> float32 tensor."""
    import torch

    L = N.lib()
    want = torch.int32 if d.tag in DISCRETE_TAGS else torch.float32
    x = x.to(want).contiguous()
    out = torch.empty(x.numel(), dtype=torch.float32, device=x.device)
    nd, keep = _to_native(d, x.device)
    rc = L.cuppl_dist_score(C.byref(nd), N.ptr(x), x.numel(), N.ptr(out), N.stream_ptr(x.device))
    N.check(rc, "dist_score")
    del keep
    return out
