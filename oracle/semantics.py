"""numpy fp64 restatement of the distribution and normalisation semantics.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  dist_score   SPEC.md:312-320 (natural log density/mass, -inf outside the support)
  dist_var
  normalize    SPEC.md:417-425 (log-sum-exp shifted by the max; support merged by
               structural equality, cuppl/values.py:101-122; -inf weights excluded;
               all -inf raises AllZeroWeightError, cuppl/errors.py:119)
  categorical  SURVEY.md Appendix A D5: inverse CDF on u32 words with u64 thresholds
"""

from __future__ import annotations

import math

import numpy as np

NORMAL, BERNOULLI, POISSON, UNIFORM_DISCRETE, UNIFORM_CONTINUOUS, BETA, EXPONENTIAL, CATEGORICAL = range(8)
HALF_LOG_2PI = 0.5 * math.log(2.0 * math.pi)


def dist_score(tag: int, params, x) -> float:
    p = list(params)
    if tag == NORMAL:
        mu, sd = p[0], p[1]
        z = (x - mu) / sd
        return -0.5 * z * z - math.log(sd) - HALF_LOG_2PI
    if tag == BERNOULLI:
        return math.log(p[0]) if x else math.log1p(-p[0])
    if tag == POISSON:
        k = int(x)
        if k < 0:
            return -math.inf
        lam = p[0]
        return (k * math.log(lam) if k else 0.0) - lam - math.lgamma(k + 1)
    if tag == UNIFORM_DISCRETE:
        a, b = int(p[0]), int(p[1])
        return -math.log(b - a) if a <= int(x) < b else -math.inf
    if tag == UNIFORM_CONTINUOUS:
        a, b = p[0], p[1]
        return -math.log(b - a) if a <= x <= b else -math.inf
    if tag == BETA:
        a, b = p[0], p[1]
        if not (0.0 <= x <= 1.0):
            return -math.inf
        return ((a - 1) * math.log(x) + (b - 1) * math.log1p(-x)
                - (math.lgamma(a) + math.lgamma(b) - math.lgamma(a + b)))
    if tag == EXPONENTIAL:
        r = p[0]
        return math.log(r) - r * x if x >= 0 else -math.inf
    if tag == CATEGORICAL:
        w = np.asarray(p[0], dtype=np.float64)
        k = int(x)
        if 0 <= k < len(w) and w[k] > 0:
            return math.log(w[k] / w.sum())
        return -math.inf
    raise ValueError(tag)


def dist_var(tag: int, params) -> float:
    p = list(params)
    if tag == NORMAL:
        return p[1] ** 2
    if tag == BERNOULLI:
        return p[0] * (1 - p[0])
    if tag == POISSON:
        return p[0]
    if tag == UNIFORM_DISCRETE:
        n = int(p[1]) - int(p[0])
        return (n * n - 1) / 12.0
    if tag == UNIFORM_CONTINUOUS:
        return (p[1] - p[0]) ** 2 / 12.0
    if tag == BETA:
        a, b = p[0], p[1]
        return a * b / ((a + b) ** 2 * (a + b + 1))
    if tag == EXPONENTIAL:
        return 1.0 / p[0] ** 2
    if tag == CATEGORICAL:
        w = np.asarray(p[0], dtype=np.float64)
        q = w / w.sum()
        k = np.arange(len(w))
        m = (q * k).sum()
        return float((q * (k - m) ** 2).sum())
    raise ValueError(tag)


def categorical_thresholds(weights) -> np.ndarray:
    """u64 thresholds t_k = floor(cum_k / P * 2^32), k < K-1 (left-fold cumsum in fp64)."""
    w = np.asarray(weights, dtype=np.float64)
    total = 0.0
    for v in w:
        total += v
    out = np.zeros(max(len(w) - 1, 0), dtype=np.uint64)
    cum = 0.0
    for k in range(len(w) - 1):
        cum += w[k]
        t = math.floor(cum / total * 4294967296.0)
        out[k] = min(max(t, 0), 1 << 32)
    return out


def categorical_from_word(thresholds: np.ndarray, w: int) -> int:
    for k, t in enumerate(thresholds):
        if w < int(t):
            return k
    return len(thresholds)


def value_key(v):
    """Structural identity (restates cuppl/values.py:101-122 for scalars/tuples/lists)."""
    if v is None:
        return ("u",)
    if v is True or v is False:
        return ("b", v)
    if isinstance(v, int):
        return ("i", v)
    if isinstance(v, float):
        return ("r", v)
    if isinstance(v, str):
        return ("s", v)
    if isinstance(v, tuple):
        return ("t",) + tuple(value_key(x) for x in v)
    if isinstance(v, list):
        return ("v",) + tuple(value_key(x) for x in v)
    raise TypeError(type(v))


def normalize(samples):
    """samples: list of (value, log_weight). Returns ({value_key: (value, prob)}, log_z)."""
    lws = np.array([lw for _, lw in samples], dtype=np.float64)
    finite = np.isfinite(lws)
    if not finite.any():
        raise ZeroDivisionError("all weights are -inf")
    m = lws[finite].max()
    s = np.exp(lws[finite] - m).sum()
    lse = m + math.log(s)
    out: dict = {}
    for (v, lw) in samples:
        if not math.isfinite(lw):
            continue
        k = value_key(v)
        p = math.exp(lw - lse)
        if k in out:
            out[k] = (out[k][0], out[k][1] + p)
        else:
            out[k] = (v, p)
    return out, lse - math.log(len(samples))
