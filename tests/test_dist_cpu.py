"""Multi-process (world size 2, gloo on CPU) coverage of the N > 1 bench path:
per-rank timings reduce to their max, the job value counts every replica, and
the reference arm runs on rank 0 only (2D configs are replicas,
no data-path collective)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = 3.0 + rank  # rank 1 is slower
    m = bench.reduce_max(ms)
    v = bench.aggregate(1000, world, m)
    tdist.barrier()
    q.put((rank, m, v))
    tdist.destroy_process_group()


def test_reduce_max_and_aggregate_two_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m, v in out:
        assert m == 4.0                       # max over ranks
        assert v == pytest.approx(1000 * 2 / 4e-3)


def test_single_process_identity():
    import bench
    assert bench.reduce_max(2.5) == 2.5
    assert bench.aggregate(100, 1, 1.0) == pytest.approx(1e5)
