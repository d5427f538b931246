"""CPU, world_size 2 over gloo: the plumbing of bench.py's multi-GPU modes
without a device -- the strong split of one batch into contiguous shards and
the all-gather that puts the shards' costs back in batch order (BASELINE
configs 3-4), and the max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PMB_DIST_BACKEND="gloo")
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import importlib
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    bench = importlib.import_module("bench")
    count = 1024
    lo, hi = bench.shard(count, world, rank)
    # stand-in costs: each chromosome's own index, computed by its rank only
    costs = torch.arange(lo, hi, dtype=torch.int64) * 3 + 1
    out = torch.empty(count, dtype=torch.int64)
    bench.allgather_into(out, costs)
    slowest = bench.max_over_ranks(10.0 + rank, world)
    q.put((rank, lo, hi, bool(torch.equal(out, torch.arange(count, dtype=torch.int64) * 3 + 1)), slowest))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_strong_split_gathers_costs_in_batch_order(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(60)
    per = 1024 // world
    for rank, lo, hi, ordered, slowest in res:
        assert (lo, hi) == (rank * per, (rank + 1) * per)
        assert ordered
        assert slowest == 10.0 + world - 1  # the max over ranks


def test_shard_rejects_uneven_split():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    with pytest.raises(ValueError):
        bench.shard(1000, 3, 0)
