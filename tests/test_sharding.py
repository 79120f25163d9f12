"""Multi-process (gloo, world_size 2, CPU) checks of the batch×head sharding
used by bench.py for N>1 GPUs: the per-rank unit ranges tile the global units
exactly once, and the step time reported is the max over ranks."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2512_16615_b200.sharding import shard_units


def test_shard_units_partition():
    for total in (1, 16, 17, 128):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_units(total, world, r) for r in range(world)]
            covered = [u for s, c in spans for u in range(s, s + c)]
            assert covered == list(range(total))
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    assert shard_units(128, 8, 3) == (48, 16)   # C4: 128 units over 8 GPUs
    with pytest.raises(ValueError):
        shard_units(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2512_16615_b200.sharding import max_over_ranks, shard_units
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, count = shard_units(32, world, rank)
    spans = [None] * world
    dist.all_gather_object(spans, (start, count))
    t = max_over_ranks(1.0 + rank)
    # per-rank work is independent: sum of unit ids over the whole job
    local = torch.tensor([sum(range(start, start + count))], dtype=torch.int64)
    dist.all_reduce(local)
    q.put((rank, spans, t, int(local.item())))
    dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, spans, t, total in res:
        assert spans == [(0, 16), (16, 16)]
        assert t == 2.0                      # max over ranks
        assert total == sum(range(32))
