"""Sharded pipeline on the device: two ranks (gloo; both processes on cuda:0,
exchanging through host memory, no kernel waits on another process) must
reproduce the single-process result: the boundary all-gather feeds the
replicated weld, every rank solves its own subdomains, and the assembled
UV (gather_coords) equals the one-GPU UV bit for bit; every rank's report
carries the whole mesh's flips, repairs and distortion summary (order
statistics exact, sums to rounding)."""

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
        from paper_1903_12359_b200.dist import Shard, gather_coords
        shard = Shard()
        V, F, cuts, m, kw = _case(mode)
        gp, rep = pg.parameterize(pg.TriMesh(V, F), cuts, m, shard=shard, **kw)
        full = gather_coords(gp, shard)
        q.put((rank, full, rep.flips, rep.solver.get("shard"), rep.distortion, rep.repairs,
               rep.solver.get("exchanged_bytes"), np.asarray(gp.coords)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover
        q.put((rank, "error", repr(exc), None))


def _golden(name):
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"{name}.npz"))


def _case(mode):
    from paper_1903_12359_b200 import generators as gen
    if mode == "sphere":
        z = _golden("sphere4")
        return z["V"], z["F"], z["cuts"], "sphere", {}
    if mode == "fold":  # jittered strips whose harmonic maps fold: the repair path
        z = _golden("repair_strips3")
        return z["V"], z["F"], z["cuts"], str(z["mode"]), {}
    V, F, cuts = gen.height_field_case(65, 4, seed=2)
    return V, F, cuts, mode, {"pairs": gen.row_tree_schedule_order(4, 4)}


@pytest.mark.parametrize("mode", ["free", "disk", "sphere", "fold"])
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
    V, F, cuts, m, kw = _case(mode)
    gp, rep = pg.parameterize(pg.TriMesh(V, F), cuts, m, **kw)
    ref = np.asarray(gp.coords)
    s0, s1 = res[0][3], res[1][3]
    assert s0 and s1 and sorted(s0 + s1) == list(range(rep.n_submeshes))
    assert np.array_equal(res[0][1], ref)  # assembled on rank 0 from both ranks' own vertices
    nb = sum(len(c) for c in pg.partition_mesh(pg.TriMesh(V, F), cuts).boundary_cycles)
    for r in (0, 1):
        flips, d, reps, xb, own = res[r][2], res[r][4], res[r][5], res[r][6], res[r][7]
        assert flips == rep.flips
        assert [x["flips_before"] for x in reps] == [x["flips_before"] for x in rep.repairs]
        assert [x.get("remaining") for x in reps] == [x.get("remaining") for x in rep.repairs]
        for key in ("median", "iqr"):  # per-corner |d| are the same numbers: exact order statistics agree
            assert d["angular_abs"][key] == rep.distortion["angular_abs"][key]
            # area ratios are normalised by summed areas (summation order differs)
            assert abs(d["area_abs"][key] - rep.distortion["area_abs"][key]) <= 1e-12
        for key in ("mean", "sd"):
            assert abs(d["angular_abs"][key] - rep.distortion["angular_abs"][key]) <= 1e-12 * max(
                1.0, abs(rep.distortion["angular_abs"][key]))
        assert d["angular_histogram"] == rep.distortion["angular_histogram"]
        assert d["excluded_corners"] == rep.distortion["excluded_corners"]
        # the rank's own coordinates (the seams included) are the one-GPU ones
        ok = ~np.isnan(own.real if own.ndim == 1 else own[:, 0])
        assert np.array_equal(own[ok], ref[ok])
        # exchange: the boundary all-gather (2 blocks of the longest rank's
        # slots) plus the small summary / metric reductions
        assert xb < 16 * (2 * nb + 4096) + 160_000, xb


def _nccl_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        import paper_1903_12359_b200 as pg
        from paper_1903_12359_b200.dist import Shard, gather_coords
        shard = Shard()
        V, F, cuts, m, kw = _case("free")
        gp, rep = pg.parameterize(pg.TriMesh(V, F), cuts, m, shard=shard, **kw)
        q.put((rank, gather_coords(gp, shard), rep.flips, rep.distortion["angular_abs"]["median"]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover
        q.put((rank, "error", repr(exc), None))


def test_two_gpu_nccl_matches_single_gpu(cuda):
    """The production transport: two ranks on two GPUs over NCCL (one
    all-gather + the small reductions). Runs where two GPUs are visible."""
    import multiprocessing as mp
    import torch
    import paper_1903_12359_b200 as pg
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r) for r in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
    for r in res.values():
        assert not isinstance(r[1], str), r[2]
    V, F, cuts, m, kw = _case("free")
    gp, rep = pg.parameterize(pg.TriMesh(V, F), cuts, m, **kw)
    assert np.array_equal(res[0][1], np.asarray(gp.coords))
    assert res[0][2] == res[1][2] == rep.flips == 0
    assert res[0][3] == res[1][3] == rep.distortion["angular_abs"]["median"]
