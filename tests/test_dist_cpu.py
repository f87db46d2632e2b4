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


# ------------------------------------------ z-slab exchange plan (§8e) ----
CASES = [(nz, G, h, ga) for nz in (8, 24, 32, 48) for G in (2, 4, 8) if nz % G == 0
         for h in (0, 1, 2, 3, 5) for ga in (0, 1)]


def _check_plans(nz, G, h, ga, plans):
    """plans[r] = list of (peer, z0, z1, send) of rank r (fmg_slab_plan)."""
    slab = nz // G
    for r in range(G):
        recv = [(s, a, b) for s, a, b, snd in plans[r] if not snd]
        # every receive is matched by the owner's send, in the same per-pair order
        for s in range(G):
            if s == r:
                continue
            mine = [(a, b) for ss, a, b in recv if ss == s]
            theirs = [(a, b) for pp, a, b, snd in plans[s] if snd and pp == r]
            assert mine == theirs, (nz, G, h, ga, r, s)
            for a, b in mine:  # the sender owns what it sends
                assert s * slab <= a < b <= (s + 1) * slab
        # the receives cover exactly the ghost planes (or every foreign plane)
        got = sorted(z for _, a, b in recv for z in range(a, b))
        lo, hi = r * slab, (r + 1) * slab
        if ga:
            need = [z for z in range(nz) if not lo <= z < hi]
        else:
            need = list(range(max(0, lo - h), lo)) + list(range(hi, min(nz, hi + h)))
        assert got == need, (nz, G, h, ga, r)


def test_slab_plan_all_ranks_in_process():
    import paper_2511_19036_b200 as P
    for nz, G, h, ga in CASES:
        plans = [P.slab_plan(nz, G, r, h, bool(ga)) for r in range(G)]
        _check_plans(nz, G, h, ga, plans)
    with pytest.raises(P.FmgError):
        P.slab_plan(10, 4, 0, 1)


def _plan_worker(rank, world, port, q):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_19036_b200 as P
    ok = True
    for nz, G, h, ga in CASES:
        if G != world:
            continue
        mine = P.slab_plan(nz, G, rank, h, bool(ga))
        allp = [None] * world
        tdist.all_gather_object(allp, mine)  # what each rank would post to NCCL
        try:
            _check_plans(nz, G, h, ga, allp)
        except AssertionError:
            ok = False
    tdist.barrier()
    q.put((rank, ok))
    tdist.destroy_process_group()


def test_slab_plan_two_ranks_gloo():
    """The N > 1 exchange path as two processes: each rank builds its own
    send/recv list (as fmg_create_dist does before posting grouped NCCL
    send/recv); the lists gathered over gloo pair up exactly."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in out)
