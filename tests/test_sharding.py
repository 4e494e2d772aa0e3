"""Multi-rank sharding logic on CPU: world size 2 over gloo, with the CPU oracle
standing in for each rank's GPU (the data path has no collective; only the
accept bitmap words are gathered)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1809_07858_b200.shard import shard_bounds


def test_bounds_are_word_aligned_and_cover():
    for n in [1, 31, 32, 33, 1000, 4097, 100_003]:
        for parts in [1, 2, 3, 8]:
            b = shard_bounds(n, parts)
            assert b[0] == 0 and b[-1] == n and b == sorted(b)
            assert all(x % 32 == 0 for x in b[:-1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, queue):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_1809_07858_b200.shard import filter_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    t, p = o.generate_pairs(123, n, 100, 0, 10)
    fn = lambda tt, pp, e, w: o.shouji_batch(tt, pp, e, w, estimates=False)[0]  # noqa: E731
    full = filter_sharded(t, p, 5, rank, world, fn)
    if rank == 0:
        queue.put(full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [4097, 10_000])
def test_gloo_world2_matches_single_process(n):
    from oracle.oracle import Oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    full = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    o = Oracle()
    t, p = o.generate_pairs(123, n, 100, 0, 10)
    ref, _, _ = o.shouji_batch(t, p, 5)
    assert (full == ref).all()
