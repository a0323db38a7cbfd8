"""Multi-rank (gloo, world_size 2, CPU) check of the batch-sharding logic bench.py uses:
every member owned once, shards reproduce the single-rank instances exactly (seeding is by
member index), max/sum reductions and trace gathering behave."""
import os
import socket

import numpy as np
import pytest

from paper_2603_18527_b200.sharding import shard_members


def test_shard_members_partition():
    for total in (64, 7, 9, 128):
        for world in (1, 2, 4, 8):
            if total < world:
                continue
            seen = []
            for r in range(world):
                first, count = shard_members(total, world, r)
                seen.extend(range(first, first + count))
            assert seen == list(range(total))
    assert shard_members(64, 8, 3) == (24, 8)  # config 1: 8 per GPU at 8 GPUs
    with pytest.raises(ValueError):
        shard_members(3, 4, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2603_18527_b200 as bs
    from paper_2603_18527_b200.sharding import gather_traces, max_over_ranks, sum_over_ranks
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total = 6
    first, count = shard_members(total, world, rank)
    spec = bs.InstanceSpec(n=16, ppw=8.0, contrast=0.5)
    k2, f, k0, eta = bs.make_instances(spec, first, count)
    mx = max_over_ranks(float(rank + 1))
    sm = sum_over_ranks(float(count))
    gathered = gather_traces([first + i for i in range(count)])
    if rank == 0:
        q.put((mx, sm, gathered, k2, k0))
    else:
        q.put((None, None, None, k2, k0))
    dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    head = [r for r in results if r[0] is not None][0]
    mx, sm, gathered, _, _ = head
    assert mx == 2.0 and sm == 6.0 and gathered == list(range(6))
    import paper_2603_18527_b200 as bs
    k2_all, _, k0_all, _ = bs.make_instances(bs.InstanceSpec(n=16, ppw=8.0, contrast=0.5), 0, 6)
    shards = sorted(results, key=lambda r: r[4][0] != k0_all[0])  # rank 0's shard first
    k2_cat = np.concatenate([shards[0][3], shards[1][3]])
    assert np.array_equal(k2_cat, k2_all)  # sharded synthesis == single-rank synthesis
