"""Generic systematic resampling (C ABI cuppl_resample, csrc/resample_kernels.cu): GPU ancestors
and payloads bit-exact against oracle/resample_oracle.c for any weights and payload shapes; the
oracle's own properties on CPU; a particle filter on a continuous-state model (GenericSmc)
against the Kalman filter."""

import math

import numpy as np
import pytest

KEY = 0x9E0160293A33AAF7


# ---------------------------------------------------------------- CPU: the oracle ----------
@pytest.mark.parametrize("n", [1, 5, 1000, 40_000])
def test_oracle_systematic_properties(oracle_lib, n):
    """Systematic resampling: ancestors non-decreasing, every offspring count within 1 of
    N w_i / sum w (w the exactly quantised weights), payload rows copied from the ancestors."""
    rs = np.random.default_rng(n)
    lw = (3 * rs.standard_normal(n)).astype(np.float32)
    pay = rs.standard_normal((n, 3)).astype(np.float32)
    out, anc, st = oracle_lib.resample(lw, pay, KEY, 4)
    assert st["status"] == 0 and st["T"] > 0
    assert np.all(np.diff(anc.astype(np.int64)) >= 0)
    assert np.array_equal(out, pay[anc.astype(np.int64)])
    e = np.exp(lw.astype(np.float64) - lw.max())
    cnt = np.bincount(anc.astype(np.int64), minlength=n)
    assert np.all(np.abs(cnt - n * e / e.sum()) < 1.0 + 1e-6)


def test_oracle_all_zero_weights(oracle_lib):
    lw = np.full(10, -np.inf, dtype=np.float32)
    _, _, st = oracle_lib.resample(lw, np.zeros(10, np.int32), KEY, 0)
    assert st["status"] == 2 and st["T"] == 0


def test_kalman_oracle_matches_brute_force_gaussian():
    """The Kalman log-likelihood equals the joint Gaussian density of y (small T)."""
    from oracle import exact

    a, q, r, s0, T = 0.9, 0.5, 0.7, 1.3, 6
    y = np.array([0.3, -0.2, 1.1, 0.4, -0.9, 0.05])
    cov_x = np.zeros((T, T))
    var = [s0 * s0]
    for t in range(1, T):
        var.append(a * a * var[-1] + q * q)
    for i in range(T):
        for j in range(T):
            cov_x[i, j] = a ** abs(i - j) * var[min(i, j)]
    cov = cov_x + r * r * np.eye(T)
    ll, _ = exact.kalman_loglik(y, a, q, r, s0)
    assert ll == pytest.approx(exact._log_mvn0(y, cov), rel=1e-12)


# ---------------------------------------------------------------- GPU: bit-exactness -------
def _lw(kind, n, rs):
    if kind == "normal":
        return (3 * rs.standard_normal(n)).astype(np.float32)
    if kind == "wide":  # many particles far below the maximum (quantised to 0)
        return (40 * rs.standard_normal(n)).astype(np.float32)
    if kind == "degenerate":  # one particle holds (almost) all the weight
        lw = np.full(n, -200.0, dtype=np.float32)
        lw[rs.integers(n)] = 0.0
        return lw
    if kind == "equal":
        return np.zeros(n, dtype=np.float32)
    if kind == "special":  # -inf, NaN and +-0 entries
        lw = rs.standard_normal(n).astype(np.float32)
        lw[rs.random(n) < 0.2] = -np.inf
        lw[rs.random(n) < 0.05] = np.nan
        lw[rs.random(n) < 0.05] = -0.0
        return lw
    raise ValueError(kind)


def _gpu(lw, pay, t, ancestors=True):
    import torch

    from paper_2010_08454_b200 import resample

    dev = torch.device("cuda")
    lw_d = torch.from_numpy(lw).to(dev)
    pay_d = None if pay is None else torch.from_numpy(pay).to(dev)
    r = resample.Resampler(len(lw), dev)
    out = None if pay is None else torch.empty_like(pay_d)
    anc = torch.empty(len(lw), dtype=torch.int64, device=dev) if ancestors else None
    r.launch(lw_d, pay_d, KEY, t, out, anc)
    m, total, s1, s2 = r.read_stats()
    return (None if out is None else out.cpu().numpy(), None if anc is None else anc.cpu().numpy(),
            (m, total, s1, s2))


PAYLOADS = {
    "f32": lambda n, rs: rs.standard_normal(n).astype(np.float32),
    "i64": lambda n, rs: rs.integers(-2**40, 2**40, n),
    "f32x3": lambda n, rs: rs.standard_normal((n, 3)).astype(np.float32),
    "u8x5": lambda n, rs: rs.integers(0, 256, (n, 5)).astype(np.uint8),
    "f32x16": lambda n, rs: rs.standard_normal((n, 16)).astype(np.float32),  # 64 B: not staged
    "none": lambda n, rs: None,
}


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 2048, 2049, 8193, 100_003, 1_000_000])
@pytest.mark.parametrize("kind", ["normal", "wide", "degenerate", "equal", "special"])
def test_gpu_resample_bit_exact(cuda, oracle_lib, n, kind):
    rs = np.random.default_rng(n + len(kind))
    lw = _lw(kind, n, rs)
    pay = PAYLOADS["f32x3"](n, rs)
    out, anc, (m, total, s1, s2) = _gpu(lw, pay, 11)
    ref_out, ref_anc, st = oracle_lib.resample(lw, pay, KEY, 11)
    assert total == st["T"] and np.float32(m) == np.float32(st["M"])
    assert np.array_equal(anc.astype(np.uint64), ref_anc)
    assert np.array_equal(out, ref_out)
    assert s1 == pytest.approx(st["s1"], rel=1e-7) and s2 == pytest.approx(st["s2"], rel=1e-7)  # fp32 over 8, fp64 above


@pytest.mark.gpu
@pytest.mark.parametrize("payload", sorted(PAYLOADS))
def test_gpu_resample_payload_shapes(cuda, oracle_lib, payload):
    n = 50_001
    rs = np.random.default_rng(3)
    lw = _lw("normal", n, rs)
    pay = PAYLOADS[payload](n, rs)
    out, anc, (m, total, _, _) = _gpu(lw, pay, 2)
    ref_out, ref_anc, st = oracle_lib.resample(lw, np.zeros(n, np.int32) if pay is None else pay, KEY, 2)
    assert total == st["T"] and np.array_equal(anc.astype(np.uint64), ref_anc)
    if pay is not None:
        assert np.array_equal(out, ref_out)


@pytest.mark.gpu
def test_gpu_resample_at_c4_scale(cuda, oracle_lib):
    """1e8 particles (BASELINE configs[3]'s population) with a 4-byte payload: T ~ N 2^31 ~ 2^57,
    where the fp64 rank estimates and the 128-bit fix-ups carry real magnitudes."""
    n = 100_000_000
    rs = np.random.default_rng(0)
    lw = (0.5 * rs.standard_normal(n)).astype(np.float32)
    pay = np.arange(n, dtype=np.int32)
    out, anc, (m, total, _, _) = _gpu(lw, pay, 7, ancestors=False)
    ref_out, ref_anc, st = oracle_lib.resample(lw, pay, KEY, 7)
    assert total == st["T"] and total > 2**53  # beyond exact fp64 integers
    assert np.array_equal(out, ref_out)


@pytest.mark.gpu
def test_gpu_resample_all_zero_raises(cuda):
    import torch

    from paper_2010_08454_b200 import resample
    from paper_2010_08454_b200.errors import AllZeroWeightError

    with pytest.raises(AllZeroWeightError):
        resample.systematic(torch.full((100,), -math.inf, device="cuda"), None, 1)


@pytest.mark.gpu
def test_gpu_generic_smc_linear_gaussian_matches_kalman(cuda):
    """A continuous-state model — outside the HMM filter's one-byte states — filtered with torch
    propagation and the GPU resampler: log Z within Monte Carlo error of the Kalman filter, and
    the run is bit-reproducible."""
    import torch

    from oracle import exact
    from paper_2010_08454_b200 import Rng, resample

    a, q, r, s0, T = 0.95, 0.3, 0.5, 1.0, 60
    rs = np.random.default_rng(5)
    x, ys = rs.normal(0, s0), []
    for t in range(T):
        if t:
            x = a * x + rs.normal(0, q)
        ys.append(x + rs.normal(0, r))
    ys = np.array(ys, dtype=np.float32).astype(np.float64)
    ll_ref, _ = exact.kalman_loglik(ys, a, q, r, s0)
    y_d = torch.tensor(ys, dtype=torch.float32, device="cuda")

    def make(seed):
        g = torch.Generator(device="cuda").manual_seed(seed)
        init = lambda n: s0 * torch.randn(n, device="cuda", generator=g)  # noqa: E731
        weight = lambda x, t: -0.5 * ((y_d[t] - x) / r) ** 2 - math.log(r) - 0.5 * math.log(2 * math.pi)  # noqa: E731
        prop = lambda x, t: a * x + q * torch.randn(x.shape, device="cuda", generator=g)  # noqa: E731
        return resample.GenericSmc(init, weight, prop, 200_000)

    runs = [make(9).run(T, Rng(3)) for _ in range(2)]
    assert runs[0].log_z == runs[1].log_z  # same seeds: the same bits
    assert abs(runs[0].log_z - ll_ref) < 0.05, (runs[0].log_z, ll_ref)


@pytest.mark.gpu
def test_gpu_resampler_rejects_mismatched_buffers(cuda):
    """Buffer checks before the launch: a short output buffer, a wrong ancestor dtype or a
    mismatched payload would otherwise be written out of bounds by the kernels."""
    import torch

    from paper_2010_08454_b200 import resample

    n = 1000
    r = resample.Resampler(n)
    lw = torch.zeros(n, dtype=torch.float32, device="cuda")
    pay = torch.zeros((n, 3), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        r.launch(lw, pay, 1, 0, torch.empty((n - 1, 3), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        r.launch(lw, pay, 1, 0, None)
    with pytest.raises(ValueError):
        r.launch(lw, None, 1, 0, None, torch.empty(n, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        r.launch(lw[:-1], None, 1, 0)
    with pytest.raises(ValueError):
        r.launch(lw, pay.cpu(), 1, 0, torch.empty_like(pay))
    r.launch(lw, pay, 1, 0, torch.empty_like(pay), torch.empty(n, dtype=torch.int64, device="cuda"))
    m, total, s1, s2 = r.read_stats()
    assert total == n * 2**31 and s1 == n
