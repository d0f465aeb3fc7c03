"""GPU tests of the many-chain LMH engine (K7) against the CPU restatement and closed forms."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KEY = 0x9E0160293A33AAF7


def test_mh_initial_trace_and_short_chain_match_oracle(cuda, oracle_lib):
    """Zero steps: initial means / log-likelihood equal the oracle's; a few steps: identical
    accept decisions except where fp32 vs fp64 re-execution straddles log u (rare)."""
    import torch

    from oracle import core
    from paper_2010_08454_b200 import _native as N
    from paper_2010_08454_b200 import models

    m = models.GaussianMixture.synthetic(n_points=1000)
    L = N.lib()
    K, D = m.K, len(m.ys)
    y = torch.zeros(L.cuppl_mh_padded_points(D), device=cuda)
    y[:D] = torch.tensor(m.ys, device=cuda)
    nc = 64
    mu = torch.empty((nc, K), device=cuda)
    ll = torch.empty(nc, device=cuda)
    st = torch.zeros((nc, 2 * K + 2), dtype=torch.float64, device=cuda)
    N.check(L.cuppl_mh_gmm(N.ptr(y), D, K, 10.0, 1.0, nc, 0, 0, 0, 1, KEY, N.ptr(mu), N.ptr(ll), N.ptr(st),
                           None, 0, N.stream_ptr()))
    mu0, ll0 = mu.cpu().numpy(), ll.cpu().numpy()
    y64 = np.asarray(m.ys, dtype=np.float32).astype(np.float64)
    for c in range(nc):
        z, mref, lref = core.mh_gmm_init(m.ys, K, 10.0, 1.0, c, KEY)
        # means: fp32 SFU Box-Muller against fp64 (the D11 note of test_gpu_is.py)
        assert np.allclose(mu0[c], mref, rtol=1e-5, atol=1e-4)
        # log-likelihood: D11 against the fp64 re-evaluation of the GPU's own trace (labels are
        # integer draws, bit-exact; means the GPU's)
        r = y64 - mu0[c].astype(np.float64)[z]
        l64 = -0.5 * float(np.dot(r, r)) - D * 0.5 * math.log(2 * math.pi)
        assert abs(ll0[c] - l64) <= 1e-5 * abs(l64) + 1e-6, (c, ll0[c], l64)
    steps = 200
    N.check(L.cuppl_mh_gmm(N.ptr(y), D, K, 10.0, 1.0, nc, 0, steps, 0, 1, KEY, N.ptr(mu), N.ptr(ll), N.ptr(st),
                           None, 0, N.stream_ptr()))
    mref, lref, sref = core.mh_gmm(m.ys, K, 10.0, 1.0, nc, steps, KEY)
    got = st.cpu().numpy()
    same = np.all(np.isclose(mu.cpu().numpy(), mref, rtol=1e-4, atol=1e-3), axis=1)
    assert same.mean() >= 0.98, same.mean()  # chains whose decisions never straddled
    assert np.array_equal(got[same, 2 * K + 1], sref[same, 2 * K + 1])


def test_mh_single_component_matches_conjugate_posterior(cuda):
    """K = 1: mu | y ~ normal with precision 1/prior_sd^2 + D. Single-site LMH with prior
    proposals mixes slowly on the mean (it is 1 of K + D sites), so the data set is small."""
    from paper_2010_08454_b200 import Rng, infer, models

    rs = np.random.default_rng(3)
    y = 1.7 + rs.standard_normal(20)
    m = models.GaussianMixture(y, K=1, prior_sd=2.0)
    prec = 1 / 4 + len(y)
    mean = y.astype(np.float32).astype(float).sum() / prec
    post = infer.run_lmh(m, 40_000, Rng(5), chains=256, burn_in=10_000)
    assert abs(post.mean_vec[0] - mean) < 5 * post.mcse()[0] + 1e-3
    assert abs(post.var_vec[0] - 1 / prec) < 0.2 / prec
    assert 0.0 < post.acceptance < 1.0


def test_mh_gmm_recovers_separated_means(cuda):
    from paper_2010_08454_b200 import Rng, infer, models

    rs = np.random.default_rng(4)
    z = rs.integers(0, 2, 40)
    y = np.where(z == 0, -3.0, 3.0) + rs.standard_normal(40)
    m = models.GaussianMixture(y, K=2, prior_sd=5.0)
    post = infer.run_lmh(m, 60_000, Rng(1), chains=256, burn_in=20_000)
    good = np.all(np.abs(post.chain_means - np.array([-3, 3])) < 1.0, axis=1)
    assert good.mean() > 0.8
    assert np.all(np.abs(np.median(post.chain_means[good], axis=0) - [-3, 3]) < 0.5)


def test_mh_statistics_match_oracle_chains(cuda, oracle_lib):
    """Same model, same chains: GPU and oracle posterior summaries agree within MC error."""
    from oracle import core
    from paper_2010_08454_b200 import Rng, infer, models

    m = models.GaussianMixture.synthetic(n_points=300, K=3)
    rng = Rng(11)
    post = infer.run_lmh(m, 3000, rng, chains=128, burn_in=1000)
    assert isinstance(post, infer.EmpiricalDistribution)  # SPEC.md:408-413's result type
    assert post.n == 128 * 2000 and set(post.mean) == {"v0", "v1", "v2"}
    mref, lref, sref = core.mh_gmm(m.ys, 3, 10.0, 1.0, 128, 3000, rng.key, burn_in=1000)
    ref_chain = sref[:, :3] / sref[:, [6]]
    se = np.sqrt(post.chain_means.var(axis=0, ddof=1) / 128 + ref_chain.var(axis=0, ddof=1) / 128)
    assert np.all(np.abs(post.chain_means.mean(axis=0) - ref_chain.mean(axis=0)) < 5 * se + 0.05)
    acc_ref = sref[:, 7].sum() / (128 * 3000)
    assert abs(post.acceptance - acc_ref) < 0.02


@pytest.mark.parametrize("D", [7, 20_000])
def test_mh_data_shapes_match_oracle_initial_trace(cuda, oracle_lib, D):
    """Tiny and large data sets (1 to 4 register groups of points per thread): the initial
    traces and log-likelihoods equal the oracle's."""
    import torch

    from oracle import core
    from paper_2010_08454_b200 import _native as N
    from paper_2010_08454_b200 import models

    m = models.GaussianMixture.synthetic(n_points=D)
    L = N.lib()
    K = m.K
    y = torch.zeros(L.cuppl_mh_padded_points(D), device=cuda)
    y[:D] = torch.tensor(m.ys, device=cuda)
    nc = 40
    mu = torch.empty((nc, K), device=cuda)
    ll = torch.empty(nc, device=cuda)
    st = torch.zeros((nc, 2 * K + 2), dtype=torch.float64, device=cuda)
    N.check(L.cuppl_mh_gmm(N.ptr(y), D, K, 10.0, 1.0, nc, 0, 0, 0, 1, KEY, N.ptr(mu), N.ptr(ll), N.ptr(st),
                           None, 0, N.stream_ptr()))
    mu0, ll0 = mu.cpu().numpy(), ll.cpu().numpy()
    y64 = np.asarray(m.ys, dtype=np.float32).astype(np.float64)
    for c in range(nc):
        z, mref, lref = core.mh_gmm_init(m.ys, K, 10.0, 1.0, c, KEY)
        # means: fp32 SFU Box-Muller against fp64 (the D11 note of test_gpu_is.py)
        assert np.allclose(mu0[c], mref, rtol=1e-5, atol=1e-4)
        # log-likelihood: D11 against the fp64 re-evaluation of the GPU's own trace (labels are
        # integer draws, bit-exact; means the GPU's)
        r = y64 - mu0[c].astype(np.float64)[z]
        l64 = -0.5 * float(np.dot(r, r)) - D * 0.5 * math.log(2 * math.pi)
        assert abs(ll0[c] - l64) <= 1e-5 * abs(l64) + 1e-6, (c, ll0[c], l64)


GMM_PROG = """
ys <- [1.2, -0.7, 3.1, 2.2, -1.9, 0.4, 2.8, -0.3];
model <- function() {
  mu <- sample(normal(0, 3));
  reduce(function(acc, y) { observe(normal(mu, 1), y); acc }, 0, ys);
  mu
};
mcmc(model, 400)
"""


def _mh_ranks_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # both ranks share the test box's GPU
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_08454_b200 import Rng, frontend, infer, models

        m = models.GaussianMixture.synthetic(n_points=500, K=3)
        post = infer.run_lmh(m, 300, Rng(11), chains=70, burn_in=100)
        cm = frontend.compile_program(GMM_PROG)
        post2 = infer.run_lmh(cm, 400, Rng(12), chains=50, burn_in=100)
        q.put((rank, post.record["chain_stats"], dict(post.mean), post.stats["acceptance"],
               post2.record["chain_stats"], dict(post2.mean)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_mh_two_ranks_equal_one(cuda):
    """MH is replicas: chains sharded over two processes (gloo, one GPU)
    gather to exactly the per-chain statistics and posterior of a single-process run — the
    hand-written K7 GMM chains and a compiled mcmc program."""
    import multiprocessing as mp
    import socket

    from paper_2010_08454_b200 import Rng, frontend, infer, models

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mh_ranks_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    m = models.GaussianMixture.synthetic(n_points=500, K=3)
    one = infer.run_lmh(m, 300, Rng(11), chains=70, burn_in=100)
    one2 = infer.run_lmh(frontend.compile_program(GMM_PROG), 400, Rng(12), chains=50, burn_in=100)
    for o in out:
        assert np.array_equal(o[1], one.record["chain_stats"])
        assert o[2] == dict(one.mean) and o[3] == one.stats["acceptance"]
        assert np.array_equal(o[4], one2.record["chain_stats"])
        assert o[5] == dict(one2.mean)
