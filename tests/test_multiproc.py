"""The N>1 path on CPU: world_size-2 gloo processes shard images and reduce
their timings with a max (the bench's only collective)."""
import os
import socket

from paper_1311_5304_b200 import shard


def test_lpt_balances_and_covers():
    costs = [9, 7, 6, 5, 4, 3, 2, 2, 1]
    parts = shard.assign_lpt(costs, 2)
    assert sorted(i for p in parts for i in p) == list(range(len(costs)))
    loads = [sum(costs[i] for i in p) for p in parts]
    assert abs(loads[0] - loads[1]) <= max(costs)
    assert shard.assign_lpt(costs, 1) == [list(range(len(costs)))]


def test_split_rows_and_context():
    for rows in (1, 7, 68, 250):
        for world in (1, 2, 3, 8):
            spans = shard.split_rows(rows, world)
            assert sum(n for _, n in spans) == rows
            assert all(spans[k][0] + spans[k][1] == spans[k + 1][0] for k in range(world - 1))
    assert shard.chroma_context(0, 4, 10) == (0, 5)
    assert shard.chroma_context(4, 6, 10) == (3, 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    costs = [1920 * 1080] * 5 + [4096 * 4096] * 2 + [512 * 512] * 9
    mine = shard.assign_lpt(costs, world)[rank]
    t = float(sum(costs[i] for i in mine))  # stand-in for this rank's device time
    q.put((rank, mine, shard.max_over_ranks(t)))
    dist.destroy_process_group()


def test_gloo_world2_shard_and_max():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    res = [q.get(timeout=120) for _ in procs]
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    res.sort()
    items = res[0][1] + res[1][1]
    assert sorted(items) == list(range(16)) and not set(res[0][1]) & set(res[1][1])
    assert res[0][2] == res[1][2] == max(res[0][2], res[1][2])
