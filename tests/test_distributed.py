"""world_size-2 gloo test of the multi-GPU sharding (CPU, no GPU needed).

The data path has no collective: every rank computes the same global order
from (seed, epoch) and takes positions [r*B, (r+1)*B) of each global batch.
The only cross-rank traffic is the optional one-time seed broadcast."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, bs, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_12517_b200.loader import LoaderConfig, _dist_info, shard_batches
        from paper_2306_12517_b200.traversal import OrderKind, TraversalOrder

        seed = torch.tensor([1234 if rank == 0 else -1])
        dist.broadcast(seed, src=0)             # one-time seed agreement
        cfg = LoaderConfig(batch_size=bs, distributed=True, seed=int(seed.item()), order=OrderKind.QUASI_RANDOM)
        r, w = _dist_info(cfg)
        assert (r, w) == (rank, world)
        pm = [i // 7 for i in range(n)]
        gb = TraversalOrder(cfg.order, cfg.seed).epoch_batches(1, n, bs * w, pm)
        mine = shard_batches(gb, r, w, bs)
        gathered = [None] * w
        dist.all_gather_object(gathered, mine)
        if rank == 0:
            result_q.put((gb, gathered))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_partition_each_global_batch():
    world, n, bs = 2, 301, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, bs, q)) for r in range(world)]
    for p in procs:
        p.start()
    gb, parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(i for part in parts for b in part for i in b) == list(range(n))
    for g, batch in enumerate(gb):
        union = []
        for r in range(world):
            if g < len(parts[r]):
                union += parts[r][g]
        assert union == batch


def _seed_worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_12517_b200.loader import LoaderConfig, agree_seed

        cfg = LoaderConfig(batch_size=4, distributed=True, seed=100 + rank)   # ranks disagree locally
        result_q.put((rank, agree_seed(cfg)))
    finally:
        dist.destroy_process_group()


def test_gloo_one_time_seed_agreement():
    """distributed=True: every rank adopts rank 0's seed with one broadcast at
    Loader construction (north_star: the only collective of the path)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seed_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: 100, 1: 100}
