"""Closed-form oracles (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

  linreg_posterior  conjugate Gaussian linear regression: a, b ~ normal(0, s0);
                    y_i ~ normal(a x_i + b, sigma)
  poly_posterior    Fig.1 model: for each degree n the
                    factor exp(-||y - Phi_n c||^2) is a Gaussian kernel in c, so the
                    per-degree evidence and the coefficient posterior are closed form
  hmm_forward       forward algorithm for the SMC HMM: log p(y_{0:T})
                    and the filtering marginals p(x_t | y_{0:t})
  kalman_loglik     Kalman filter of a 1-D linear-Gaussian state-space model: the exact log
                    p(y_{0:T}) a particle filter on a continuous state estimates
"""

from __future__ import annotations

import math

import numpy as np


def _log_mvn0(y: np.ndarray, cov: np.ndarray) -> float:
    L = np.linalg.cholesky(cov)
    z = np.linalg.solve(L, y)
    return float(-0.5 * z @ z - np.log(np.diag(L)).sum() - 0.5 * len(y) * math.log(2 * math.pi))


def linreg_posterior(xs, ys, sigma: float = 1.0, prior_sd: float = 10.0):
    """Returns (mean[a, b], cov 2x2, log_evidence)."""
    x = np.asarray(xs, dtype=np.float64)
    y = np.asarray(ys, dtype=np.float64)
    X = np.stack([x, np.ones_like(x)], axis=1)
    prec = np.eye(2) / prior_sd**2 + X.T @ X / sigma**2
    cov = np.linalg.inv(prec)
    mean = cov @ (X.T @ y) / sigma**2
    logz = _log_mvn0(y, prior_sd**2 * X @ X.T + sigma**2 * np.eye(len(y)))
    return mean, cov, logz


def poly_posterior(xs, ys, prior_sd: float = 10.0, degrees=(2, 3, 4)):
    """Posterior over degree n (uniform prior over `degrees`) and E[c | n].

    Weight of a trace: exp(-||y - Phi c||^2) = pi^{D/2} N(y; Phi c, I/2), so
    Z_n = pi^{D/2} N(y; 0, s0^2 Phi Phi^T + I/2) and c | n ~ N(m_n, S_n) with
    S_n^{-1} = I/s0^2 + 2 Phi^T Phi, m_n = S_n 2 Phi^T y.
    Returns (p_n dict, {n: m_n}, {n: S_n}, log_z) where log_z = log mean weight.
    """
    x = np.asarray(xs, dtype=np.float64)
    y = np.asarray(ys, dtype=np.float64)
    D = len(x)
    logZ, means, covs = {}, {}, {}
    for n in degrees:
        Phi = np.stack([x**j for j in range(n)], axis=1)
        logZ[n] = 0.5 * D * math.log(math.pi) + _log_mvn0(
            y, prior_sd**2 * Phi @ Phi.T + 0.5 * np.eye(D))
        S = np.linalg.inv(np.eye(n) / prior_sd**2 + 2 * Phi.T @ Phi)
        means[n] = S @ (2 * Phi.T @ y)
        covs[n] = S
    lz = np.array([logZ[n] for n in degrees])
    m = lz.max()
    p = np.exp(lz - m)
    p /= p.sum()
    log_z = m + math.log(np.exp(lz - m).sum() / len(degrees))
    return {n: float(pi) for n, pi in zip(degrees, p)}, means, covs, log_z


def hmm_forward(A, pi0, mu, sd, y):
    """Exact filter for x_0 ~ pi0, x_t ~ A[x_{t-1}], y_t ~ normal(mu[x_t], sd).

    Returns (log p(y_{0:T-1}), filtering marginals [T, S]).
    """
    A = np.asarray(A, dtype=np.float64)
    pi0 = np.asarray(pi0, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    T = len(y)
    S = len(pi0)
    filt = np.zeros((T, S))
    logp = 0.0
    pred = pi0
    for t in range(T):
        le = -0.5 * ((y[t] - mu) / sd) ** 2 - math.log(sd) - 0.5 * math.log(2 * math.pi)
        m = le.max()
        a = pred * np.exp(le - m)
        s = a.sum()
        logp += m + math.log(s)
        filt[t] = a / s
        pred = filt[t] @ A
    return logp, filt


def kalman_loglik(y, a: float, q: float, r: float, s0: float):
    """x_0 ~ N(0, s0^2), x_{t+1} = a x_t + N(0, q^2), y_t = x_t + N(0, r^2): log p(y_{0:T-1}) and
    the filtering means E[x_t | y_{0:t}]."""
    m, P = 0.0, s0 * s0
    ll = 0.0
    means = []
    for t, yt in enumerate(np.asarray(y, dtype=np.float64)):
        if t > 0:
            m, P = a * m, a * a * P + q * q
        S = P + r * r
        ll += -0.5 * (math.log(2 * math.pi * S) + (yt - m) ** 2 / S)
        K = P / S
        m, P = m + K * (yt - m), (1 - K) * P
        means.append(m)
    return ll, np.array(means)
