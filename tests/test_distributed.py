"""Multi-process host logic on CPU (gloo, world size 2): rank sharding and the ordered merge of
per-rank importance-sampling records — the only collective of the IS path."""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import core, refstream
        from paper_2010_08454_b200 import infer, models

        m = models.PolyRegression.synthetic()
        n, key = 30_001, refstream.key_of(9)
        r, w = infer._world()
        lo, hi = infer.shard_range(n, r, w)
        d, _ = core.is_poly(m.xs, m.ys, lo, hi, key, threads=1)
        rec = infer.N.IsRecord()
        for k, v in d.items():
            if k in ("stat_w", "bin_w"):
                getattr(rec, k)[:] = list(v)
            else:
                setattr(rec, k, v)
        buf = torch.frombuffer(bytearray(bytes(rec)), dtype=torch.uint8)
        recs = infer._gather_records(buf)  # all-gather over gloo + rank-order list
        merged = infer.record_to_dict(infer.merge_records(recs))
        out_q.put((rank, merged["sum_w"], merged["argmax_pid"], merged["n_total"], list(merged["bin_w"][:3])))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_record_gather_and_merge(oracle_lib, native_lib):
    import multiprocessing as mp

    from oracle import refstream
    from paper_2010_08454_b200 import models

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    m = models.PolyRegression.synthetic()
    full, _ = oracle_lib.is_poly(m.xs, m.ys, 0, 30_001, refstream.key_of(9), threads=1)
    for rank, sw, amax, ntot, bins in res:
        assert ntot == 30_001
        assert amax == full["argmax_pid"]
        assert sw == pytest.approx(full["sum_w"], rel=1e-12)
        assert np.allclose(bins, full["bin_w"][:3], rtol=1e-12)
    assert res[0][1:] == res[1][1:]  # every rank merges to identical bytes


def test_rank_partitions():
    """IS / MH shard contiguous ranges of near-equal size; SMC rank boundaries are multiples of
    16 (16-byte state stores) that cover the population in order."""
    from paper_2010_08454_b200 import infer, smc

    rs = np.random.default_rng(0)
    for world in range(1, 9):
        for n in [world, 16 * world, 1000, 10**9 + 7, int(rs.integers(1, 10**12))]:
            parts = [infer.shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[r][1] == parts[r + 1][0] for r in range(world - 1))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1
            if n >= 16 * world and n < 2**31:
                b = smc.rank_boundaries(n, world)
                assert b[0] == 0 and b[-1] == n and len(b) == world + 1
                assert all(x % 16 == 0 for x in b[:-1]) and all(b[r] < b[r + 1] for r in range(world))
