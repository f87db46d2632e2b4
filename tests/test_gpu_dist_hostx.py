"""Two processes, one GPU: z slabs with a real data plane.

Each process is one slab rank of fmg_create_hostx.  Every ghost-plane exchange
(BFP sections of u_L, FP64 coarse planes, the gathered coarse residual) and
the norm sum really cross the process boundary: device -> host -> gloo over
127.0.0.1 -> host -> device.  The ranks never wait on each other inside a
kernel, only in the host transport.  The sections the ranks own, assembled
plane by plane, must be bit-identical to the undecomposed solve (and so to the
oracle), and the norms equal within the slab-sum reassociation."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, d, p, levels, outdir):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_19036_b200 as P
    torch.cuda.set_device(0)
    s = P.Solver(d, p, levels, hostx=(rank, world, P.host_transport_gloo()))
    s.solve()
    norms = s.norms()
    out = {"norms": norms}
    for l in range(levels):
        for which in (0, 1):
            m, e, w = s.section(which, l)
            out[f"m{which}_{l}"], out[f"e{which}_{l}"], out[f"w{which}_{l}"] = m, e, np.array(w)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    s.close()
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("d,p,levels", [(3, 1, 6), (3, 3, 4)])
def test_two_process_host_transport_bit_identical(tmp_path, d, p, levels):
    import torch.multiprocessing as mp
    import paper_2511_19036_b200 as P
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=_worker, args=(r, world, port, d, p, levels, str(tmp_path))) for r in range(world)]
    for q in ps:
        q.start()
    for q in ps:
        q.join(timeout=600)
        assert q.exitcode == 0
    ranks = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    ref = P.Solver(d, p, levels)
    ref.solve()
    n1 = ref.norms()
    for r in range(world):
        m = n1 != 0
        assert np.all(np.abs(ranks[r]["norms"][m] - n1[m]) <= 1e-12 * n1[m])
    for l in range(levels):
        nz = ref.geom(l)[0]
        for which in (0, 1):
            mr, er, wr = ref.section(which, l)
            assert all(int(ranks[r][f"w{which}_{l}"]) == wr for r in range(world))
            bpp = len(er) // nz  # blocks per plane
            for z in range(nz):
                o = ranks[z // (nz // world)]  # plane z from its owner
                sl = slice(z * bpp, (z + 1) * bpp)
                assert np.array_equal(o[f"e{which}_{l}"][sl], er[sl]), (which, l, z)
                assert np.array_equal(o[f"m{which}_{l}"][z * bpp * wr:(z + 1) * bpp * wr],
                                      mr[z * bpp * wr:(z + 1) * bpp * wr]), (which, l, z)
