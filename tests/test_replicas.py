"""Replica host logic on CPU with gloo, world size 2: query
sharding, the result all-gather (bit-exact scores), max-over-ranks timing.
No GPU compute: each rank fabricates the answers its shard would produce."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_02171_b200.replicas import shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_answers(lo, hi, k):
    rng = np.random.Generator(np.random.PCG64(lo))
    ids = (np.arange(lo, hi)[:, None] * 100 + np.arange(k)[None, :]).astype(np.uint32)
    sc = rng.standard_normal((hi - lo, k)).astype(np.float32)
    sc[:, -1] = np.float32(-0.0)  # signed zero must survive the gather
    cnt = (np.arange(lo, hi) % (k + 1)).astype(np.uint32)
    return ids, sc, cnt


def _worker(rank, world, port, nq, k, q):
    import torch.distributed as dist

    from paper_2605_02171_b200.replicas import gather_results, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(nq, world, rank)
    ids, sc, cnt = fake_answers(lo, hi, k)
    a_ids, a_sc, a_cnt = gather_results(ids, sc, cnt, nq)
    t = max_over_ranks(1.5 + rank)
    q.put((rank, a_ids, a_sc.view(np.uint32), a_cnt, t))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_cover_exactly():
    for nq in (0, 1, 7, 10000):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(nq, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nq
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("nq", [9, 1000])
def test_gloo_world2_gather_is_exact(nq):
    k, world = 10, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nq, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_ids, want_sc, want_cnt = fake_answers(0, nq, k)
    # fake_answers is seeded per shard start: rebuild expected per shard
    parts = [fake_answers(*shard_bounds(nq, world, r), k) for r in range(world)]
    want_ids = np.concatenate([p[0] for p in parts])
    want_sc = np.concatenate([p[1] for p in parts]).view(np.uint32)
    want_cnt = np.concatenate([p[2] for p in parts])
    for rank, ids, sc_bits, cnt, t in got:
        assert np.array_equal(ids, want_ids)
        assert np.array_equal(sc_bits, want_sc)
        assert np.array_equal(cnt, want_cnt)
        assert t == 2.5  # max over ranks of 1.5 + rank
