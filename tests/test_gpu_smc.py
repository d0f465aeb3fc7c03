"""GPU parity tests of the SMC engine (K4/K5/K6) against the exact CPU restatement
(oracle/cuppl_oracle.c or_smc_*) and the HMM forward algorithm."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KEY = 0x9E0160293A33AAF7


def _gpu_run(model, n, steps, local_world=None, record_ancestors=True, hist_steps=None):
    import torch

    from paper_2010_08454_b200 import smc

    r = smc.SmcRunner(model, n, KEY, record_ancestors=record_ancestors, local_world=local_world,
                      steps=steps, hist_steps=hist_steps)
    res = r.run()
    torch.cuda.synchronize()
    x = np.concatenate([t.cpu().numpy() for t in res.states]).astype(np.int32)
    lw = np.concatenate([t.cpu().numpy() for t in res.log_weights])
    anc = [np.concatenate([a.cpu().numpy() for a in step]).astype(np.uint64) for step in res.ancestors]
    return res, x, lw, anc


@pytest.mark.parametrize("n,S,steps", [(100_000, 50, 12), (8 * 1031, 7, 20), (64, 3, 10), (262_144, 50, 5),
                                       (70_001, 100, 6), (20_000, 256, 4),
                                       (16, 4, 5), (17, 3, 6), (33, 2, 4), (4097, 2, 5)])
def test_smc_bit_exact_single_rank(cuda, oracle_lib, n, S, steps):
    from paper_2010_08454_b200 import models

    m = models.HiddenMarkovModel.synthetic(S=S, T=steps, seed=1)
    res, x, lw, anc = _gpu_run(m, n, steps, hist_steps=list(range(steps)))
    ref = oracle_lib.smc_run(m, n, KEY, record_ancestors=True, hist_steps=list(range(steps)))
    assert np.array_equal(res.total_weight, ref["T"]), "integer weight totals differ"
    assert np.array_equal(res.max_log_weight.astype(np.float32), ref["M"])
    for t in range(steps - 1):
        assert np.array_equal(anc[t], ref["ancestors"][t]), f"ancestors differ at step {t}"
    assert np.array_equal(x, ref["x"])
    assert np.array_equal(lw.view(np.uint32), ref["lw"].view(np.uint32))
    for t in range(steps):
        assert np.array_equal(res.filtering_int[t], ref["hist"][t])
    # s1 is summed in fp32 per thread on the GPU, fp64 sequentially in the oracle
    assert np.allclose(res.log_z_steps, ref["log_z_steps"], rtol=1e-7, atol=1e-7)


@pytest.mark.parametrize("R", [2, 3, 4, 8])
def test_smc_rank_partition_invariance(cuda, oracle_lib, R):
    """Virtual ranks on one GPU: identical bits for every partition of the particles."""
    from paper_2010_08454_b200 import models

    n, steps = 50_000, 10
    m = models.HiddenMarkovModel.synthetic(S=50, T=steps, seed=2)
    res, x, lw, anc = _gpu_run(m, n, steps, local_world=R)
    ref = oracle_lib.smc_run(m, n, KEY, record_ancestors=True)
    assert np.array_equal(res.total_weight, ref["T"])
    for t in range(steps - 1):
        assert np.array_equal(anc[t], ref["ancestors"][t]), f"R={R}: ancestors differ at step {t}"
    assert np.array_equal(x, ref["x"]) and np.array_equal(lw.view(np.uint32), ref["lw"].view(np.uint32))


def test_smc_population_below_rank_granule_is_refused(cuda):
    """Rank boundaries are multiples of 16 particles (16-byte state stores): fewer than 16 per
    rank is refused up front rather than run on empty ranks."""
    from paper_2010_08454_b200 import models, smc

    m = models.HiddenMarkovModel.synthetic(S=4, T=3, seed=6)
    for n, R in ((1, 1), (15, 1), (127, 8)):
        with pytest.raises(ValueError):
            smc.SmcRunner(m, n, KEY, local_world=R if R > 1 else None, steps=3)


@pytest.mark.parametrize("n,R", [(128, 8), (131, 8), (4096 * 3 + 1, 3)])
def test_smc_small_rank_shares(cuda, oracle_lib, n, R):
    """The smallest rank shares (16 particles, ragged last rank) and tile-boundary splits stay
    bit-exact."""
    from paper_2010_08454_b200 import models

    steps = 6
    m = models.HiddenMarkovModel.synthetic(S=5, T=steps, seed=6)
    res, x, lw, anc = _gpu_run(m, n, steps, local_world=R)
    ref = oracle_lib.smc_run(m, n, KEY, record_ancestors=True)
    assert np.array_equal(res.total_weight, ref["T"])
    for t in range(steps - 1):
        assert np.array_equal(anc[t], ref["ancestors"][t]), f"ancestors differ at step {t}"
    assert np.array_equal(x, ref["x"]) and np.array_equal(lw.view(np.uint32), ref["lw"].view(np.uint32))


def _snapshot(res):
    x = np.concatenate([t.cpu().numpy() for t in res.states])
    lw = np.concatenate([t.cpu().numpy() for t in res.log_weights]).view(np.uint32)
    return (x, lw, np.asarray(res.total_weight).copy(), np.asarray(res.log_z_steps).copy(),
            {t: np.asarray(h).copy() for t, h in res.filtering_int.items()})


@pytest.mark.parametrize("R", [None, 3])
def test_smc_graph_replay_matches_eager(cuda, R):
    """One captured CUDA graph of the whole run (init + T steps), the Philox key read from device
    memory: replays under two different keys are bit-identical to eager runs; K6 is timed
    inside the graph by event-record nodes."""
    import torch

    from paper_2010_08454_b200 import models, smc

    steps, n = 12, 100_000
    m = models.HiddenMarkovModel.synthetic(S=50, T=steps, seed=7)
    g = smc.SmcRunner(m, n, KEY, steps=steps, graph=True, hist_steps=[5, 11], local_world=R)
    assert g.use_graph
    g.k6_events = []
    for key in (KEY, KEY ^ 0x5555_0000_1234):
        g.reseed(key)
        got = _snapshot(g.run())
        ref = _snapshot(smc.SmcRunner(m, n, key, steps=steps, hist_steps=[5, 11], local_world=R).run())
        for a, b in zip(got[:4], ref[:4]):
            assert np.array_equal(a, b)
        assert all(np.array_equal(got[4][t], ref[4][t]) for t in (5, 11))
    torch.cuda.synchronize()
    assert len(g.k6_events) == steps - 1 and g.k6_ms() > 0  # one pair per time step


@pytest.mark.parametrize("graph", [False, True])
def test_smc_reseeded_runner_matches_fresh(cuda, oracle_lib, graph):
    """A runner reused under other keys (reseed) equals fresh runs and the oracle: per-step state
    (maxima, histograms) is reset by init. Small populations make the per-step maximum depend
    on the key, so stale maxima would show."""
    from paper_2010_08454_b200 import models, smc

    steps, n = 10, 64
    m = models.HiddenMarkovModel.synthetic(S=50, T=steps, seed=8)
    r = smc.SmcRunner(m, n, KEY, steps=steps, graph=graph, hist_steps=[steps - 1])
    for key in (KEY, KEY + 1, KEY + 2, KEY + 3):
        r.reseed(key)
        got = _snapshot(r.run())
        ref = oracle_lib.smc_run(m, n, key, record_ancestors=False, hist_steps=[steps - 1])
        assert np.array_equal(got[2], ref["T"]), key
        assert np.array_equal(got[0].astype(np.int32), ref["x"]) and np.array_equal(got[1], ref["lw"].view(np.uint32))
        assert np.array_equal(got[4][steps - 1], ref["hist"][steps - 1])


@pytest.mark.parametrize("R", [None, 3])
def test_smc_snapshot_resume_bit_identical(cuda, tmp_path, R):
    """Checkpoint / resume: stop after 5 of 12 steps, save the snapshot to disk,
    restore it into a fresh runner and finish — bit-identical to the uninterrupted run."""
    import torch

    from paper_2010_08454_b200 import models, smc

    steps, n = 12, 50_000
    m = models.HiddenMarkovModel.synthetic(S=20, T=steps, seed=9)
    kw = dict(steps=steps, hist_steps=[3, steps - 1], record_ancestors=True, local_world=R)
    full_res = smc.SmcRunner(m, n, KEY, **kw).run()
    full = _snapshot(full_res)
    full_anc = [[a.cpu().numpy() for a in step] for step in full_res.ancestors]
    a = smc.SmcRunner(m, n, KEY, **kw)
    a.advance(5)
    torch.save(a.snapshot(), tmp_path / "smc.pt")
    del a
    b = smc.SmcRunner(m, n, 12345, **kw)  # another key: restore brings the snapshot's
    b.restore(torch.load(tmp_path / "smc.pt"))
    res = b.resume()
    got = _snapshot(res)
    for x, y in zip(got[:4], full[:4]):
        assert np.array_equal(x, y)
    assert all(np.array_equal(got[4][t], full[4][t]) for t in (3, steps - 1))
    anc = [[a.cpu().numpy() for a in step] for step in res.ancestors]
    assert len(anc) == len(full_anc) == steps - 1
    assert all(np.array_equal(p, q) for s1, s2 in zip(anc, full_anc) for p, q in zip(s1, s2))


def test_smc_degenerate_weights(cuda, oracle_lib):
    """An observation only one state explains: a few particles get all the offspring."""
    from paper_2010_08454_b200 import models

    m = models.HiddenMarkovModel.synthetic(S=50, T=6, seed=3)
    m.ys[2] = 49.0 + 6.0  # far above every mean but the last: weights collapse
    m.ys[4] = -7.0
    n = 40_000
    res, x, lw, anc = _gpu_run(m, n, 6)
    ref = oracle_lib.smc_run(m, n, KEY, record_ancestors=True)
    for t in range(5):
        assert np.array_equal(anc[t], ref["ancestors"][t])
    assert np.array_equal(x, ref["x"])
    assert res.ess.min() < 0.05 * n


def test_smc_log_evidence_matches_forward_algorithm(cuda):
    from oracle import exact
    from paper_2010_08454_b200 import Rng, models, smc

    m = models.HiddenMarkovModel.synthetic(S=50, T=200, seed=0)
    lz, filt = exact.hmm_forward(m.A, m.pi0, m.mu.astype(float), m.sd, m.ys.astype(float))
    res = smc.run_smc(m, 2_000_000, Rng(7))
    # PF log-evidence standard error ~ 0.03 at this size (measured on the oracle)
    assert abs(res.log_z - lz) < 0.25
    f = res.filtering[199]
    assert np.abs(f - filt[199]).sum() < 0.05


def test_smc_deterministic(cuda):
    from paper_2010_08454_b200 import models

    m = models.HiddenMarkovModel.synthetic(S=50, T=8, seed=4)
    _, x1, lw1, _ = _gpu_run(m, 300_000, 8, record_ancestors=False)
    _, x2, lw2, _ = _gpu_run(m, 300_000, 8, record_ancestors=False)
    assert np.array_equal(x1, x2) and np.array_equal(lw1.view(np.uint32), lw2.view(np.uint32))


def _mp_worker(rank, world, port, n, steps, q, exchange="collective", graph=False):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # both ranks share the one GPU of the test box; peers via CUDA IPC
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_08454_b200 import models, smc

        m = models.HiddenMarkovModel.synthetic(S=50, T=steps, seed=5)
        r = smc.SmcRunner(m, n, KEY, record_ancestors=not graph, steps=steps, exchange=exchange, graph=graph)
        if graph:  # a first replay under another key: the second one must still be exact
            assert r.use_graph
            r.reseed(KEY ^ 0x5555)
            r.run()
            r.reseed(KEY)
        res = r.run()
        torch.cuda.synchronize()
        q.put((rank, r.bounds[rank], res.states[0].cpu().numpy(), res.log_weights[0].cpu().numpy(),
               [a[0].cpu().numpy() for a in res.ancestors], res.total_weight, res.log_z))
        dist.barrier()
        r.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange,graph", [("collective", False), ("peer", False), ("peer", True)])
def test_smc_multiprocess_ipc_matches_oracle(cuda, oracle_lib, exchange, graph):
    """Two processes sharing the GPU, CUDA-IPC peer stores for the particles; the per-step
    exchanges either through torch.distributed (gloo here) or device-side over the peer-mapped
    arenas (cuppl_peer_exchange) — then the whole run of each rank is also one CUDA graph,
    replayed twice: the same bits as the single-rank oracle."""
    import multiprocessing as mp
    import socket

    from paper_2010_08454_b200 import models

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    n, steps = 40_000, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mp_worker, args=(r, 2, port, n, steps, q, exchange, graph)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    m = models.HiddenMarkovModel.synthetic(S=50, T=steps, seed=5)
    ref = oracle_lib.smc_run(m, n, KEY, record_ancestors=True)
    x = np.concatenate([o[2] for o in out]).astype(np.int32)
    lw = np.concatenate([o[3] for o in out])
    assert np.array_equal(out[0][5], ref["T"]) and np.array_equal(out[1][5], ref["T"])
    for t in range(steps - 1 if not graph else 0):
        anc = np.concatenate([o[4][t] for o in out]).astype(np.uint64)
        assert np.array_equal(anc, ref["ancestors"][t]), f"ancestors differ at step {t}"
    assert np.array_equal(x, ref["x"]) and np.array_equal(lw.view(np.uint32), ref["lw"].view(np.uint32))
    assert out[0][6] == out[1][6]
