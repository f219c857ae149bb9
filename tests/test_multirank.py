"""Pair sharding for batched independent products across ranks (world_size 2, gloo, CPU).
The per-rank multiply is replaced by Python's int product here; on the GPU box the same
code path calls the batched device multiply."""
import os
import random
import socket

import pytest
import torch.multiprocessing as mp

from paper_1503_04955_b200.parallel import shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(n, r, world)
                seen.extend(range(lo, hi))
                assert hi - lo in (n // world, n // world + 1)
            assert seen == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1503_04955_b200.parallel import dmul_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = random.Random(42)
    pairs = [(rng.getrandbits(3000), rng.getrandbits(3000)) for _ in range(13)]
    calls = []

    def fake(pp):
        calls.append(len(pp))
        return [a * b for a, b in pp]

    got = dmul_sharded(pairs, rank, world, multiply=fake)
    q.put((rank, got == [a * b for a, b in pairs], calls))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_gloo_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert [ok for _, ok, _ in res] == [True, True]
    assert [c for _, _, c in res] == [[7], [6]]
