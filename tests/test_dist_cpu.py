"""Multi-rank host logic of dist.py on CPU (gloo, world_size 2).

The device solves are replaced by the oracle (this is test infrastructure).
Each rank solves its LPT shard; the boundary-loop values of its own
submeshes go through the one exchange of the design, `Shard.slot_layout` +
`Shard.all_gather_` (each rank's slots packed, gathered, scattered into
slot order); each rank then solves its own Dirichlet problems and fills the
other ranks' loops with the welded values (pipeline._fill_foreign_loops).
The tests check that the exchanged boundary values equal the
single-process ones bit for bit, that every rank's own vertices (seams
included) stitch to the single-process result, and that the exchange moves
one padded block per rank.
"""

import os
import socket

import numpy as np
import pytest

from paper_1903_12359_b200.dist import lpt_shards, subdomain_cost


def test_lpt_covers_and_balances():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        sizes = list(rng.integers(50, 5000, size=37))
        sh = lpt_shards(sizes, world)
        flat = sorted(i for s in sh for i in s)
        assert flat == list(range(37))
        loads = [sum(subdomain_cost(sizes[i]) for i in s) for s in sh]
        assert max(loads) - min(loads) <= max(subdomain_cost(x) for x in sizes) + 1e-6
        assert sh == lpt_shards(sizes, world)  # deterministic


def test_lpt_equal_sizes_round_robin_and_empty_ranks():
    sh = lpt_shards([100] * 64, 8)
    assert [len(s) for s in sh] == [8] * 8
    sh = lpt_shards([10, 20], 4)
    assert sorted(len(s) for s in sh) == [0, 0, 1, 1]
    with pytest.raises(ValueError):
        lpt_shards([1], 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import oracle
    from paper_1903_12359_b200 import generators as gen
    from paper_1903_12359_b200.dist import Shard
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        V, F, cuts = gen.height_field_case(25, 3, seed=1)
        sp = oracle.split_mesh(V, F, cuts)
        sizes = [len(v) for v in sp.sub_V]
        voff = np.concatenate([[0], np.cumsum(sizes)])
        nb = [len(l) for l in sp.loops]
        loff = np.concatenate([[0], np.cumsum(nb)])
        shard = Shard()
        own = shard.comps(sizes)
        # flatten own submeshes, embeddings over all local vertices
        z0 = np.zeros(voff[-1], np.complex128)
        for c in own:
            z0[voff[c]:voff[c + 1]] = oracle.dncp_flatten(sp.sub_V[c], sp.sub_F[c], sp.loops[c])
        # the exchange: own slots packed, all-gathered, scattered to slot order
        loop_gid = np.concatenate([voff[c] + np.asarray(sp.loops[c]) for c in range(sp.n_sub)])
        own_slots, smap, blk = shard.slot_layout(loff)
        send = torch.zeros(blk, dtype=torch.complex128)
        send[:len(own_slots)] = torch.from_numpy(z0[loop_gid[own_slots]])
        recv = torch.empty(world * blk, dtype=torch.complex128)
        shard.all_gather_(send, recv)
        tv_ext = np.zeros(loff[-1] + 1, np.complex128)
        tv_ext[smap] = recv.numpy()
        tvn = tv_ext[:-1]
        # harmonic of own submeshes with the exchanged boundary values, then
        # the other ranks' loops := their Dirichlet values
        z = np.full(voff[-1], np.nan + 0j)
        for c in own:
            g = tvn[loff[c]:loff[c + 1]]
            z[voff[c]:voff[c + 1]] = oracle.dirichlet_extend(sp.sub_V[c], sp.sub_F[c], sp.loops[c], g)
        foreign = np.setdiff1d(np.arange(len(loop_gid)), own_slots)
        z[loop_gid[foreign]] = tvn[foreign]
        q.put((rank, own, tvn.copy(), z, shard.exchanged_bytes, blk))
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, "error", repr(exc), None, None, None))


def test_shard_exchange_gloo_matches_single_process():
    import multiprocessing as mp
    import oracle
    from paper_1903_12359_b200 import generators as gen

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=240)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r in res.values():
        assert r[1] != "error", r[2]
    # the two shards partition the submeshes
    assert sorted(res[0][1] + res[1][1]) == list(range(9))
    assert res[0][1] and res[1][1]
    # single-process reference of the same data flow
    V, F, cuts = gen.height_field_case(25, 3, seed=1)
    sp = oracle.split_mesh(V, F, cuts)
    flat = [oracle.dncp_flatten(sp.sub_V[c], sp.sub_F[c], sp.loops[c]) for c in range(sp.n_sub)]
    tv = np.concatenate([flat[c][sp.loops[c]] for c in range(sp.n_sub)])
    loff = np.concatenate([[0], np.cumsum([len(l) for l in sp.loops])])
    zref = np.concatenate([oracle.dirichlet_extend(sp.sub_V[c], sp.sub_F[c], sp.loops[c],
                                                   tv[loff[c]:loff[c + 1]]) for c in range(sp.n_sub)])
    voff = np.concatenate([[0], np.cumsum([len(v) for v in sp.sub_V])])
    for r in (0, 1):
        assert np.array_equal(res[r][2], tv)
        z = res[r][3]
        known = ~np.isnan(z.real)
        assert np.array_equal(z[known], zref[known])
        # own submeshes complete, every seam copy known
        for c in res[r][1]:
            assert known[voff[c]:voff[c + 1]].all()
        loop_gid = np.concatenate([voff[c] + np.asarray(sp.loops[c]) for c in range(sp.n_sub)])
        assert known[loop_gid].all()
        assert res[r][4] == 2 * res[r][5] * 16  # one all-gather of two padded blocks
        assert 2 * res[r][5] <= len(tv) + max(len(l) for l in sp.loops)
