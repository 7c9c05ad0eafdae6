"""Sharded pipeline on the device: two ranks (gloo; both processes on cuda:0,
exchanging through host memory, no kernel waits on another process) must
reproduce the single-process result exactly."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1903_12359_b200 as pg
        from paper_1903_12359_b200 import generators as gen
        from paper_1903_12359_b200.dist import parameterize_distributed
        if mode == "sphere":
            V, F, cuts = _sphere_case()
            gp, rep = parameterize_distributed(pg.TriMesh(V, F), cuts, "sphere")
        else:
            V, F, cuts = gen.height_field_case(65, 4, seed=2)
            gp, rep = parameterize_distributed(pg.TriMesh(V, F), cuts, mode,
                                               pairs=gen.row_tree_schedule_order(4, 4))
        q.put((rank, np.asarray(gp.coords), rep.flips, rep.solver.get("shard")))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover
        q.put((rank, "error", repr(exc), None))


def _sphere_case():
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sphere4.npz"))
    return z["V"], z["F"], z["cuts"]


@pytest.mark.parametrize("mode", ["free", "disk", "sphere"])
def test_two_rank_shards_match_single_gpu(cuda, mode):
    import multiprocessing as mp
    import paper_1903_12359_b200 as pg
    from paper_1903_12359_b200 import generators as gen

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r in res.values():
        assert not isinstance(r[1], str), r[2]
    if mode == "sphere":
        V, F, cuts = _sphere_case()
        gp, rep = pg.parameterize(pg.TriMesh(V, F), cuts, "sphere")
    else:
        V, F, cuts = gen.height_field_case(65, 4, seed=2)
        gp, rep = pg.parameterize(pg.TriMesh(V, F), cuts, mode, pairs=gen.row_tree_schedule_order(4, 4))
    ref = np.asarray(gp.coords)
    s0, s1 = res[0][3], res[1][3]
    assert s0 and s1 and sorted(s0 + s1) == list(range(rep.n_submeshes))
    for r in (0, 1):
        assert res[r][2] == rep.flips == 0
        # disjoint sums are exact: identical up to the sign of zero
        assert np.array_equal(res[r][1], ref)
