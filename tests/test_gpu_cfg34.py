"""Stage-wise parity on the irregular BASELINE configurations (cfg 3:
Delaunay disk, cfg 4: spherical-harmonic icosphere) at test sizes, against
the oracle. The reference cannot weld these layouts end to end (ragged
k-means cuts), so, as in SURVEY, parity is stage-wise:
partition integers (bit-exact), cotangent Laplacian (bit-exact off-diagonals),
DNCP flatten and the Dirichlet solve (<= 1e-6 x diameter)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(name):
    from paper_1903_12359_b200 import generators as gen
    if name == "cfg3s":
        return gen.cfg3(seed=0, n_points=20000, n_clusters=16)
    return gen.cfg4(seed=0, subdiv=5, n_clusters=16)


@pytest.fixture(scope="module", params=["cfg3s", "cfg4s"])
def setup(request, cuda):
    import oracle
    from paper_1903_12359_b200 import TriMesh, partition_mesh
    V, F, cuts = _case(request.param)
    part = partition_mesh(TriMesh(V, F), cuts)
    sp = oracle.split_mesh(V, F, cuts)
    return request.param, V, F, cuts, part, sp


def test_partition_bit_exact(setup):
    name, V, F, cuts, part, sp = setup
    assert part.n_submeshes == sp.n_sub
    assert np.array_equal(part.face_assignment, sp.face_assignment)
    for a, b in zip(part.vertex_maps, sp.vertex_maps):
        assert np.array_equal(a, b)
    for a, b in zip(part.boundary_cycles, sp.boundary_cycles):
        assert np.array_equal(a, b)
    for a, b in zip(part.local_loops, sp.loops):
        assert np.array_equal(a, b)


def test_laplacian_bit_exact(setup):
    import torch
    import oracle
    from paper_1903_12359_b200 import _native as nat
    name, V, F, cuts, part, sp = setup
    b = part.batch
    b.laplacian()
    rp = b.host(nat.ARR_L_ROWPTR, torch.int64)
    col = b.host(nat.ARR_L_COL, torch.int32)
    val = b.host(nat.ARR_L_VAL, torch.float64)
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    for c in range(sp.n_sub):
        L = oracle.cotan_laplacian(sp.sub_V[c], sp.sub_F[c])
        r = rp[voff[c]:voff[c + 1] + 1]
        assert np.array_equal((r - r[0]).astype(np.int32), L.indptr)
        assert np.array_equal(col[r[0]:r[-1]], L.indices)
        v = val[r[0]:r[-1]]
        rows = np.repeat(np.arange(L.shape[0]), np.diff(L.indptr))
        off = L.indices != rows
        assert np.array_equal(v[off], L.data[off])


def test_flatten_and_dirichlet_match_oracle(setup):
    import torch
    import oracle
    from paper_1903_12359_b200 import _native as nat
    name, V, F, cuts, part, sp = setup
    b = part.batch
    z, st = b.flatten()
    assert all(s["status"] == 0 for s in st)
    z = z.cpu().numpy()
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    comps = range(0, sp.n_sub, 3)
    for c in comps:
        ref = oracle.dncp_flatten(sp.sub_V[c], sp.sub_F[c], sp.loops[c])
        got = z[voff[c]:voff[c + 1]]
        diam = 2 * np.max(np.abs(ref - ref.mean()))
        assert np.max(np.abs(got - ref)) <= 1e-6 * diam, (name, c)
    # Dirichlet solve with the flattened boundary values, all subdomains
    loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
    lp = b.host(nat.ARR_LOOP, torch.int32)
    gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
    vals = z[gid]
    zh, sth = b.harmonic(gid, vals)
    assert all(s["status"] == 0 for s in sth)
    zh = zh.cpu().numpy()
    for c in comps:
        g = z[voff[c] + sp.loops[c]]
        ref = oracle.dirichlet_extend(sp.sub_V[c], sp.sub_F[c], sp.loops[c], g)
        got = zh[voff[c]:voff[c + 1]]
        diam = 2 * np.max(np.abs(ref - ref.mean()))
        assert np.max(np.abs(got - ref)) <= 1e-6 * diam, (name, c)
