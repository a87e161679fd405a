"""world_size-2 gloo test of the multi-GPU sharding (CPU, no GPU needed).

The data path has no collective: every rank computes the same global order
from (seed, epoch) and takes positions [r*B, (r+1)*B) of each global batch; a
short tail global batch is padded by wrap-around to a multiple of the world
size and split evenly, so every rank sees the same number of batches (a DDP
loop would hang at epoch end otherwise).  The only cross-rank traffic is the
one-time seed broadcast."""

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


def _worker(rank, world, port, n, bs, result_q, drop_last=False):
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
        gb = TraversalOrder(cfg.order, cfg.seed).epoch_batches(1, n, bs * w, pm, drop_last)
        mine = [list(map(int, b)) for b in shard_batches(gb, r, w, bs)]
        counts = [None] * w
        dist.all_gather_object(counts, len(mine))
        assert len(set(counts)) == 1, counts      # equal batch counts on every rank
        gathered = [None] * w
        dist.all_gather_object(gathered, mine)
        if rank == 0:
            result_q.put((gb, gathered))
    finally:
        dist.destroy_process_group()


def _run_partition(world, n, bs, drop_last=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, bs, q, drop_last)) for r in range(world)]
    for p in procs:
        p.start()
    gb, parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [list(map(int, b)) for b in gb], parts


@pytest.mark.parametrize("n", [301, 297, 320, 5])
def test_gloo_two_ranks_partition_each_global_batch(n):
    """n=297, B=8, W=2: the tail global batch has 9 positions (< B + 1), which the
    rank-slice rule alone would give to rank 0 only (one extra batch there)."""
    world, bs = 2, 8
    gb, parts = _run_partition(world, n, bs)
    assert len(parts[0]) == len(parts[1]) == -(-n // (world * bs))
    flat = [i for part in parts for b in part for i in b]
    assert set(flat) == set(range(n))
    pad = len(flat) - n                              # duplicates: only the wrap-around padding
    assert 0 <= pad < world
    order = [i for b in gb for i in b]
    for g, batch in enumerate(gb):
        union = [i for r in range(world) for i in parts[r][g]]
        if len(batch) == world * bs:
            assert union == batch
        else:                                        # even split of the padded tail
            assert union == batch + order[:len(union) - len(batch)]
            assert len(parts[0][g]) == len(parts[1][g])


def test_gloo_two_ranks_drop_last():
    gb, parts = _run_partition(2, 297, 8, drop_last=True)
    assert len(parts[0]) == len(parts[1]) == 297 // 16
    for g, batch in enumerate(gb):
        assert parts[0][g] + parts[1][g] == batch


def _seed_worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_12517_b200.loader import LoaderConfig, agree_seed

        cfg = LoaderConfig(batch_size=4, distributed=True, seed=100 + rank)   # ranks disagree locally
        big = LoaderConfig(batch_size=4, distributed=True, seed=(1 << 64) - 5 if rank == 0 else 7)   # bit 63 set
        result_q.put((rank, (agree_seed(cfg), agree_seed(big))))
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
    assert got == {0: (100, (1 << 64) - 5), 1: (100, (1 << 64) - 5)}
