"""GPU parity tests for K8 (Philox, draws, scores) and K1/K2 (importance sampling), through
the C ABI, against the CPU oracle."""

import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KEY = 0x9E0160293A33AAF7  # Rng(1).key


def tol_ok(got, ref):
    """D11: |lw_gpu - lw_cpu| <= 1e-5 |lw_cpu| + 1e-6."""
    return np.abs(got - ref) <= 1e-5 * np.abs(ref) + 1e-6


def test_philox_bit_exact(cuda, oracle_lib):
    import torch

    from paper_2010_08454_b200 import _native as N

    L = N.lib()
    for first, blk, tag in [(0, 0, 1), ((1 << 32) - 3, 5, 3), (10**11, 2, 7)]:
        out = torch.empty((4096, 4), dtype=torch.int32, device=cuda)
        N.check(L.cuppl_philox_blocks(KEY, first, blk, tag, 4096, N.ptr(out), N.stream_ptr()))
        got = out.cpu().numpy().view(np.uint32)
        ref = oracle_lib.philox_blocks(KEY, first, blk, tag, 4096)
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("name,args", [
    ("uniform_discrete", (2, 5)), ("bernoulli", (0.3,)), ("categorical", ([0.1, 0.0, 0.6, 0.3],)),
    ("poisson", (4.0,)), ("poisson", (75.0,)),
])
def test_discrete_draws_bit_exact(cuda, oracle_lib, name, args):
    """Integer draws are exact functions of the Philox words: identical on GPU and oracle."""
    from oracle import semantics as S
    from paper_2010_08454_b200 import dists

    d = getattr(dists, name)(*args)
    got = dists.sample(d, 20000, KEY, first_id=123).cpu().numpy()
    table = S.categorical_thresholds(args[0]) if name == "categorical" else None
    p0 = d.p0 if name != "categorical" else 0
    ref = oracle_lib.dist_sample(d.tag, p0, d.p1 if name != "categorical" else 0, KEY, 7, 123, 20000, table=table)
    assert np.array_equal(got, ref)  # poisson too: its products of uniforms are fp64 on the GPU


@pytest.mark.parametrize("name,args", [("normal", (1.5, 10.0)), ("uniform_continuous", (-2.0, 3.0)),
                                       ("exponential", (2.0,)), ("beta", (2.0, 3.0)), ("beta", (0.5, 0.7))])
def test_continuous_draws_match_oracle(cuda, oracle_lib, name, args):
    from paper_2010_08454_b200 import dists

    d = getattr(dists, name)(*args)
    got = dists.sample(d, 20000, KEY).cpu().numpy().astype(np.float64)
    f32 = lambda v: float(np.float32(v))  # the parameters as the kernel receives them
    ref = oracle_lib.dist_sample(d.tag, f32(d.p0), f32(d.p1), KEY, 7, 0, 20000)
    # fp64 on the GPU like the reference (gamma's Marsaglia-Tsang decisions, the fp64 normal
    # pairs and their shared spare): the fp32 rounding of the same double, up to a last-bit
    # difference of the libm functions (log, pow, sin, cos)
    bad = np.abs(got - ref) > 2.0 * np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    assert not bad.any(), (int(bad.sum()), np.flatnonzero(bad)[:5].tolist(), got[bad][:5].tolist(), ref[bad][:5].tolist())


def test_dist_sample_spec_rows(cuda):
    from paper_2010_08454_b200 import dists

    assert (dists.sample(dists.bernoulli(1.0), 1000, KEY).cpu() == 1).all()
    u = dists.sample(dists.uniform_discrete(2, 5), 100000, KEY).cpu().numpy()
    assert set(np.unique(u)) == {2, 3, 4}
    z = dists.sample(dists.normal(0, 10), 10**6, KEY).cpu().double()
    assert abs(z.mean().item()) < 0.05 and abs(z.std().item() - 10) < 0.1


def test_dist_score_matches_oracle(cuda):
    import torch

    from oracle import semantics as S
    from paper_2010_08454_b200 import dists

    cases = [(dists.normal(0, 1), [0.0, 1.3, -4.0]), (dists.bernoulli(0.5), [1, 0]),
             (dists.uniform_discrete(2, 5), [1, 2, 4, 5, 7]), (dists.poisson(4.0), [0, 3, 11, -1]),
             (dists.beta(2.0, 3.0), [0.2, 0.9, 1.5]), (dists.exponential(2.0), [0.0, 1.0, -1.0]),
             (dists.uniform_continuous(-1, 3), [0.0, 3.5]), (dists.categorical([1, 0, 3]), [0, 1, 2, 3])]
    for d, xs in cases:
        discrete = d.tag in (1, 2, 3, 7)
        x = torch.tensor(xs, dtype=torch.int32 if discrete else torch.float32, device=cuda)
        got = dists.score(d, x).cpu().numpy().astype(np.float64)
        params = [d.p0, d.p1] if d.tag != 7 else [list(d.p0)]
        ref = np.array([S.dist_score(d.tag, params, v) for v in xs])
        assert np.array_equal(np.isinf(got), np.isinf(ref)), (d, got, ref)
        fin = np.isfinite(ref)
        assert np.allclose(got[fin], ref[fin], rtol=1e-5, atol=1e-5), (d, got, ref)


def _run_traced(model, n, key, first=0, injected=None):
    import torch

    from paper_2010_08454_b200 import infer

    la = infer.IsLauncher(model)
    dev = la.device
    lw = torch.empty(n, dtype=torch.float32, device=dev)
    coef = torch.empty((n, 4 if model.kind == "poly" else 2), dtype=torch.float32, device=dev)
    deg = torch.empty(n, dtype=torch.int32, device=dev) if model.kind == "poly" else None
    la.launch(first, first + n, key, injected=injected, lw_out=lw, deg_out=deg, coef_out=coef)
    rec = infer.records_from_bytes(la.rec.cpu().numpy())[0]
    return (lw.cpu().numpy().astype(np.float64), None if deg is None else deg.cpu().numpy(),
            coef.cpu().numpy(), infer.record_to_dict(rec))


@pytest.mark.parametrize("n,D", [(1, 20), (31, 20), (1000, 20), (65537, 20), (4099, 65), (4099, 500)])
def test_poly_injected_draws_parity(cuda, oracle_lib, n, D):
    """Fixed injected draws: GPU log-weights == oracle fp64 within 1e-5 relative (D11); data
    sets above 64 points take the device-memory path."""
    import torch

    from paper_2010_08454_b200 import models

    m = models.PolyRegression.synthetic(n_points=D)
    rs = np.random.default_rng(n)
    inj = np.zeros((n, 5), dtype=np.float32)
    inj[:, 0] = rs.integers(2, 5, n)
    inj[:, 1:] = (10 * rs.standard_normal((n, 4))).astype(np.float32)
    lw, deg, coef, rec = _run_traced(m, n, KEY, injected=torch.tensor(inj, device=cuda))
    ref, (lw_ref, deg_ref, _) = oracle_lib.is_poly(m.xs, m.ys, 0, n, KEY, injected=inj, traces=True)
    assert tol_ok(lw, lw_ref).all()
    assert np.array_equal(deg, deg_ref)
    assert rec["n_total"] == n and rec["n_finite"] == n
    assert rec["argmax_pid"] == ref["argmax_pid"] or math.isclose(
        lw_ref[rec["argmax_pid"]], ref["argmax_lw"], rel_tol=1e-5)
    assert rec["max_lw"] == pytest.approx(ref["max_lw"], rel=1e-5, abs=1e-5)
    # normaliser and per-degree mass
    assert rec["sum_w"] * math.exp(rec["max_lw"] - ref["max_lw"]) == pytest.approx(ref["sum_w"], rel=1e-4)
    assert np.allclose(np.array(rec["bin_w"][:3]) / rec["sum_w"], np.array(ref["bin_w"][:3]) / ref["sum_w"],
                       rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("D", [1, 20, 1000, 3000, 3969, 10_000, 100_000])
def test_linreg_injected_draws_parity(cuda, oracle_lib, D):
    """Up to 3968 points the data ride in the kernel-parameter block; larger data sets are read
    from device memory (the workspace tail)."""
    import torch

    from paper_2010_08454_b200 import models

    m = models.LinearRegression.synthetic(n_points=D)
    n = 4099
    rs = np.random.default_rng(D)
    inj = (rs.standard_normal((n, 2)) * [0.5, 0.5] + [2, -1]).astype(np.float32)
    inj[::7] = (10 * rs.standard_normal((len(inj[::7]), 2))).astype(np.float32)
    lw, _, coef, rec = _run_traced(m, n, KEY, injected=torch.tensor(inj, device=cuda))
    ref, (lw_ref, _) = oracle_lib.is_linreg(m.xs, m.ys, 1.0, 0, n, KEY, injected=inj, traces=True)
    assert tol_ok(lw, lw_ref).all(), np.max(np.abs(lw - lw_ref) / np.abs(lw_ref))
    assert np.array_equal(coef, inj)
    # the record's normaliser is the fp64 sum over its own log-weights ...
    own = np.exp(lw - rec["max_lw"]).sum()
    assert rec["sum_w"] == pytest.approx(own, rel=1e-5)
    # ... and the oracle's within what the per-particle fp32 evaluation error moves it (at large D
    # an error of 1e-5 |lw| ~ 1e-1 absolute changes a weight by that fraction)
    S = rec["sum_w"] * math.exp(rec["max_lw"] - ref["max_lw"])
    dom = lw_ref > lw_ref.max() - 20.0
    rel = 1e-3 + 2.0 * float(np.abs(lw - lw_ref)[dom].max())
    assert S == pytest.approx(ref["sum_w"], rel=rel)


# particle-id windows: small ids, one crossing 2^32 (the counter's high word), and C5's range
# (1e11 particles: ids above 2^36)
PID_WINDOWS = [12345, (1 << 32) - 40_000, 10**11 - 7]


@pytest.mark.parametrize("first", PID_WINDOWS)
def test_poly_philox_traces_match_oracle(cuda, oracle_lib, first):
    """Philox mode: the degree draws are bit-exact; coefficients agree to fp32 SFU accuracy; the
    log-weight of the GPU's own trace agrees with the oracle fp64 evaluation (D11)."""
    from paper_2010_08454_b200 import models

    m = models.PolyRegression.synthetic()
    n = 100_000
    lw, deg, coef, rec = _run_traced(m, n, KEY, first=first)
    _, (lw_ref, deg_ref, coef_ref) = oracle_lib.is_poly(m.xs, m.ys, first, first + n, KEY, traces=True)
    assert np.array_equal(deg, deg_ref)
    # fp32 SFU Box-Muller: lg2.approx's absolute error (~2^-22) is a large relative error of the
    # radius when u1 -> 1, so normals near 0 carry |dz| up to ~4e-5 (x sd = 10 here)
    assert np.all(np.abs(coef - coef_ref) <= 1e-4 * np.abs(coef_ref) + 5e-4)
    inj = np.concatenate([deg[:, None].astype(np.float32), coef], axis=1)
    _, (lw_inj, _, _) = oracle_lib.is_poly(m.xs, m.ys, first, first + n, KEY, injected=inj, traces=True)
    assert tol_ok(lw, lw_inj).all()


@pytest.mark.parametrize("first", [0] + PID_WINDOWS[1:])
def test_linreg_philox_traces_match_oracle(cuda, oracle_lib, first):
    from paper_2010_08454_b200 import models

    m = models.LinearRegression.synthetic()
    n = 50_000
    lw, _, coef, rec = _run_traced(m, n, KEY, first=first)
    _, (lw_ref, coef_ref) = oracle_lib.is_linreg(m.xs, m.ys, 1.0, first, first + n, KEY, traces=True)
    assert np.all(np.abs(coef - coef_ref) <= 1e-4 * np.abs(coef_ref) + 5e-4)  # see the poly test
    _, (lw_inj, _) = oracle_lib.is_linreg(m.xs, m.ys, 1.0, first, first + n, KEY, injected=coef, traces=True)
    assert tol_ok(lw, lw_inj).all()
    # the record's mode is a global particle id (u64)
    k = int(np.argmax(lw))
    assert rec["argmax_pid"] == first + k or lw[int(rec["argmax_pid"]) - first] == lw[k]


def test_is_deterministic_and_traces_do_not_change_record(cuda):
    import torch

    from paper_2010_08454_b200 import infer, models

    m = models.PolyRegression.synthetic()
    la = infer.IsLauncher(m)
    la.launch(0, 3_000_000, KEY)
    a = la.rec.clone()
    la.launch(0, 3_000_000, KEY)
    b = la.rec.clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_run_importance_poly_against_exact(cuda):
    from oracle import exact
    from paper_2010_08454_b200 import Rng, infer, models

    m = models.PolyRegression.synthetic()
    post = infer.run_importance(m, 20_000_000, Rng(1))
    p_exact, means, covs, logz = exact.poly_posterior(m.xs.astype(float), m.ys.astype(float))
    for d, p in post.support:
        se = math.sqrt(max(p_exact[d] * (1 - p_exact[d]), 1e-8) / post.ess)
        assert abs(p - p_exact[d]) < 5 * se + 1e-4
    assert abs(post.log_z - logz) < 5 / math.sqrt(post.ess) + 0.01
    n_best = max(p_exact, key=p_exact.get)
    mean = np.array(post.mean[f"c|n={n_best}"])
    sd = np.sqrt(np.diag(covs[n_best]))
    assert np.all(np.abs(mean - means[n_best]) < 6 * sd / math.sqrt(post.ess * p_exact[n_best]) + 1e-3)
    assert len(post.mode) in (2, 3, 4)


def test_run_importance_linreg_against_exact(cuda):
    from oracle import exact
    from paper_2010_08454_b200 import Rng, infer, models

    m = models.LinearRegression.synthetic(n_points=100)
    post = infer.run_importance(m, 50_000_000, Rng(2))
    mean, cov, logz = exact.linreg_posterior(m.xs.astype(float), m.ys.astype(float), 1.0)
    est = np.array([post.mean["a"], post.mean["b"]])
    sd = np.sqrt(np.diag(cov))
    assert post.ess > 100
    assert np.all(np.abs(est - mean) < 6 * sd / math.sqrt(post.ess) + 1e-3)
    assert abs(post.log_z - logz) < 6 / math.sqrt(post.ess) + 0.01


def test_all_zero_weights_raise(cuda):
    """-inf everywhere: a data point the polynomial can never fit finitely."""
    from paper_2010_08454_b200 import Rng, errors, infer, models

    m = models.LinearRegression([0.0, 1.0], [np.inf, 0.0])
    with pytest.raises(errors.AllZeroWeightError):
        infer.run_importance(m, 1000, Rng(1))


def test_normalize_spec_rows(cuda):
    from paper_2010_08454_b200 import errors, infer

    d = infer.normalize([("x", math.log(0.2)), ("y", math.log(0.2))])
    assert d.support == [("x", 0.5), ("y", 0.5)]
    d = infer.normalize([infer.WeightedSample("x", -1000.0), infer.WeightedSample("y", -1001.0)])
    assert d.probability("x") == pytest.approx(math.e / (math.e + 1), abs=1e-9)
    assert d.probability("y") == pytest.approx(1 / (math.e + 1), abs=1e-9)
    d = infer.normalize([("x", -math.inf), ("y", 0.0)])
    assert d.support == [("y", 1.0)]
    with pytest.raises(errors.AllZeroWeightError):
        infer.normalize([("x", -math.inf), ("y", -math.inf)])


def test_normalize_merges_support_and_is_permutation_invariant(cuda, oracle_lib):
    from oracle import semantics as S
    from paper_2010_08454_b200 import infer

    rs = np.random.default_rng(0)
    vals = [int(v) for v in rs.integers(0, 20, 5000)] + [(1, 2.0), True, None]
    lws = list(rs.normal(-3, 2, len(vals)))
    samples = list(zip(vals, lws))
    d = infer.normalize(samples)
    ref, lz = S.normalize(samples)
    assert abs(sum(p for _, p in d.support) - 1) < 1e-12
    for v, p in d.support:
        assert p == pytest.approx(ref[S.value_key(v)][1], abs=1e-9)
    assert d.log_z == pytest.approx(lz, abs=1e-9)
    perm = rs.permutation(len(samples))
    d2 = infer.normalize([samples[i] for i in perm])
    assert sorted(d.support, key=repr) == sorted(d2.support, key=repr)  # identical bytes


def test_normalize_tensors_matches_is_record(cuda):
    """K3 over IS traces reproduces the fused K2 record (degree histogram, log Z, mode)."""
    import torch

    from paper_2010_08454_b200 import Rng, infer, models

    m = models.PolyRegression.synthetic()
    post = infer.run_importance(m, 2_000_000, Rng(4), return_traces=True)
    lw = post.traces["log_weight"]
    deg = post.traces["degree"] - 2
    r = infer.normalize_tensors(lw, deg, 3)
    for d, p in post.support:
        assert r["probs"][d - 2] == pytest.approx(p, rel=1e-4, abs=1e-7)
    assert r["log_z"] == pytest.approx(post.log_z, abs=1e-4)
    assert r["argmax"] == post.mode_index


CURAND_CHECK = r"""
#define MAXD 1
#include <curand_philox4x32_x.h>
#include "cuppl_device.cuh"
extern "C" __global__ void philox_vs_curand(const uint4* ctr, const unsigned int* keys, uint4* ours,
                                            uint4* theirs, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint2 k = make_uint2(keys[2 * i], keys[2 * i + 1]);
  theirs[i] = curand_Philox4x32_10(ctr[i], k);
  ours[i] = cuppl::philox4x32_10(ctr[i], k.x, k.y);
}
"""


def test_philox_matches_curand(cuda):
    """the Philox4x32-10 block function equals cuRAND's
    curand_Philox4x32_10 (curand_philox4x32_x.h of this CUDA toolkit) on random counters and keys,
    including counter words at 2^32 - 1."""
    import ctypes as C

    import torch
    from cuda.bindings import driver as cu

    from paper_2010_08454_b200 import frontend

    cubin = frontend._nvrtc_cubin(CURAND_CHECK, 1, ("-I/usr/local/cuda/include",))
    torch.cuda.init()
    err, mod = cu.cuModuleLoadData(cubin)
    assert err == cu.CUresult.CUDA_SUCCESS
    err, fn = cu.cuModuleGetFunction(mod, b"philox_vs_curand")
    assert err == cu.CUresult.CUDA_SUCCESS
    n = 1 << 16
    rs = np.random.default_rng(3)
    ctr = rs.integers(0, 2**32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    ctr[:64] = 0xFFFFFFFF  # all-ones words
    ctr[64:128, 0] = 0xFFFFFFFF
    keys = rs.integers(0, 2**32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    d_ctr = torch.from_numpy(ctr.view(np.int32)).to(cuda)
    d_keys = torch.from_numpy(keys.view(np.int32)).to(cuda)
    ours = torch.zeros((n, 4), dtype=torch.int32, device=cuda)
    theirs = torch.ones((n, 4), dtype=torch.int32, device=cuda)
    vals = [C.c_uint64(d_ctr.data_ptr()), C.c_uint64(d_keys.data_ptr()), C.c_uint64(ours.data_ptr()),
            C.c_uint64(theirs.data_ptr()), C.c_int32(n)]
    ptrs = (C.c_void_p * len(vals))(*[C.addressof(v) for v in vals])
    st = torch.cuda.current_stream().cuda_stream
    err, = cu.cuLaunchKernel(fn, n // 256, 1, 1, 256, 1, 1, 0, st, C.addressof(ptrs), 0)
    assert err == cu.CUresult.CUDA_SUCCESS
    torch.cuda.synchronize()
    assert torch.equal(ours, theirs)
    cu.cuModuleUnload(mod)


def _is_ranks_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # both ranks share the test box's GPU
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_08454_b200 import Rng, infer, models

        out = []
        for m in (models.LinearRegression.synthetic(n_points=200), models.PolyRegression.synthetic()):
            post = infer.run_importance(m, 2_000_003, Rng(3))
            out.append((post.log_z, post.ess, dict(post.mean), post.mode_index, post.mode_log_weight,
                        list(post.support)))
        q.put((rank, out))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_is_two_ranks_match_one(cuda):
    """Particle sharding over two processes (gloo, one GPU): both ranks merge
    the gathered records to the same posterior, whose mode is the single-process run's
    particle (per-particle log-weights do not depend on the partition) and whose log Z, ESS,
    moments and degree masses equal it to fp32-accumulation accuracy."""
    import multiprocessing as mp
    import socket

    from paper_2010_08454_b200 import Rng, infer, models

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_is_ranks_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1]  # identical merges on every rank
    for j, m in enumerate((models.LinearRegression.synthetic(n_points=200), models.PolyRegression.synthetic())):
        one = infer.run_importance(m, 2_000_003, Rng(3))
        lz, ess, mean, mi, mlw, sup = res[0][1][j]
        assert mi == one.mode_index and mlw == one.mode_log_weight
        assert abs(lz - one.log_z) <= 1e-6 * abs(one.log_z) + 1e-6
        assert ess == pytest.approx(one.ess, rel=1e-5)
        for k, v in one.mean.items():
            assert mean[k] == pytest.approx(v, rel=1e-5, abs=1e-6)
        for (v1, p1), (v2, p2) in zip(sup, one.support):
            assert v1 == v2 and p1 == pytest.approx(p2, rel=1e-5, abs=1e-9)
