"""GPU model descriptors.

The reference runs a model as a compiled bytecode closure through sample/factor shifts
(cuppl/lowering.py:489-508); its executable form (vm, prelude) is not
shipped. On the GPU a model is a descriptor naming a compiled kernel plus
its data; `run_importance` / `run_lmh` / `run_smc` accept these in place of the closure.
Each docstring gives the CuPPL source the kernel executes.

Synthetic data generators follow SURVEY.md §8(d): generated in fp64 from numpy seed 0,
stored as fp32; both the GPU and the oracle read the same fp32 values.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64), dtype=np.float32)


@dataclass
class PolyRegression:
    """Fig.1 model:

        model <- function() {
          n <- sample(uniform-discrete(2,5));
          line <- repeat(function(i) { sample(normal(0,10)) }, n);
          factor(-distance(line, data));
          line }

    with distance(c, data) = sum_i (y_i - sum_{j<n} c_j x_i^j)^2 and support
    [2, 5) for n (D1). Returns the coefficient vector.
    """

    xs: np.ndarray
    ys: np.ndarray
    kind: str = field(default="poly", init=False)

    def __post_init__(self):
        self.xs, self.ys = _f32(self.xs), _f32(self.ys)
        if self.xs.shape != self.ys.shape or self.xs.ndim != 1:
            raise ValueError("xs and ys must be 1-D arrays of equal length")

    @classmethod
    def synthetic(cls, n_points: int = 20, seed: int = 0) -> "PolyRegression":
        """C1/C5 data: x_i = -1 + 2i/(D-1); y = 1 - 2x + 0.5x^2 + 0.1 eps."""
        rs = np.random.default_rng(seed)
        x = -1.0 + 2.0 * np.arange(n_points) / (n_points - 1)
        y = 1.0 - 2.0 * x + 0.5 * x * x + 0.1 * rs.standard_normal(n_points)
        return cls(x, y)


@dataclass
class LinearRegression:
    """Bayesian linear regression:

        model <- function() {
          a <- sample(normal(0,10)); b <- sample(normal(0,10));
          map(function(i) { observe(normal(a*x[i] + b, sigma), y[i]) }, ...);
          (a, b) }
    """

    xs: np.ndarray
    ys: np.ndarray
    sigma: float = 1.0
    kind: str = field(default="linreg", init=False)

    def __post_init__(self):
        self.xs, self.ys = _f32(self.xs), _f32(self.ys)
        if self.xs.shape != self.ys.shape or self.xs.ndim != 1:
            raise ValueError("xs and ys must be 1-D arrays of equal length")

    @classmethod
    def synthetic(cls, n_points: int = 1000, seed: int = 0) -> "LinearRegression":
        """C2 data: x ~ U(-1, 1); y = 2x - 1 + eps."""
        rs = np.random.default_rng(seed)
        x = rs.uniform(-1.0, 1.0, n_points)
        y = 2.0 * x - 1.0 + rs.standard_normal(n_points)
        return cls(x, y, 1.0)


@dataclass
class GaussianMixture:
    """GMM for many-chain LMH:

        mu_k ~ normal(0, prior_sd), k < K;  z_i ~ categorical(1/K ...);
        observe(normal(mu[z_i], sigma), y_i);  returns mu
    """

    ys: np.ndarray
    K: int = 5
    prior_sd: float = 10.0
    sigma: float = 1.0
    kind: str = field(default="gmm", init=False)

    def __post_init__(self):
        self.ys = _f32(self.ys)

    @classmethod
    def synthetic(cls, n_points: int = 10_000, K: int = 5, seed: int = 0) -> "GaussianMixture":
        """C3 data: mu = (-8, -4, 0, 4, 8); z_i uniform; y_i = mu_{z_i} + N(0, 1)."""
        rs = np.random.default_rng(seed)
        mu = np.linspace(-8.0, 8.0, K) if K == 5 else np.linspace(-2.0 * K, 2.0 * K, K)
        z = rs.integers(0, K, n_points)
        y = mu[z] + rs.standard_normal(n_points)
        return cls(y, K)


@dataclass
class HiddenMarkovModel:
    """HMM for the bootstrap particle filter:

        x_0 ~ categorical(pi0); x_t ~ categorical(A[x_{t-1}]);
        observe(normal(mu[x_t], sd), y_t)
    """

    A: np.ndarray
    pi0: np.ndarray
    mu: np.ndarray
    sd: float
    ys: np.ndarray
    states: np.ndarray | None = None  # simulated truth, when synthetic
    kind: str = field(default="hmm", init=False)

    def __post_init__(self):
        self.A = np.asarray(self.A, dtype=np.float64)
        self.pi0 = np.asarray(self.pi0, dtype=np.float64)
        self.mu = _f32(self.mu)
        self.ys = _f32(self.ys)
        S = len(self.pi0)
        if self.A.shape != (S, S) or len(self.mu) != S:
            raise ValueError("A must be SxS and mu length S")

    @property
    def n_states(self) -> int:
        return len(self.pi0)

    @property
    def T(self) -> int:
        return len(self.ys)

    @classmethod
    def synthetic(cls, S: int = 50, T: int = 1000, seed: int = 0) -> "HiddenMarkovModel":
        """C4 data: A = 0.9 I + (0.1/(S-1))(11^T - I); pi0 uniform; mu_k = k; sd = 1."""
        rs = np.random.default_rng(seed)
        A = np.full((S, S), 0.1 / (S - 1))
        np.fill_diagonal(A, 0.9)
        pi0 = np.full(S, 1.0 / S)
        mu = np.arange(S, dtype=np.float64)
        x = np.zeros(T, dtype=np.int64)
        x[0] = rs.integers(0, S)
        for t in range(1, T):
            x[t] = rs.choice(S, p=A[x[t - 1]])
        y = mu[x] + rs.standard_normal(T)
        return cls(A, pi0, mu, 1.0, y, x)
