"""The multifrontal direct solver (csrc/direct.cu), the default behind
`flatten` (flatten.py:125-188) and the Dirichlet solve (assemble.py:23-50):
per-subdomain agreement with SuperLU through the oracle, with the PCG path,
across leaf sizes, run to run, and on the irregular meshes of cfg 3 / cfg 4.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _diam(z):
    return 2 * np.max(np.abs(z - z.mean()))


def _batch(V, F, cuts):
    from paper_1903_12359_b200 import TriMesh, partition_mesh
    return partition_mesh(TriMesh(V, F, check=False), cuts).batch


def _loops(b):
    import torch
    from paper_1903_12359_b200 import _native as nat
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
    lp = b.host(nat.ARR_LOOP, torch.int32)
    return voff, [lp[loff[c]:loff[c + 1]] for c in range(b.K)]


def _check_vs_oracle(V, F, cuts, flat_tol, harm_tol, sample=None):
    import oracle
    b = _batch(V, F, cuts)
    z, st = b.flatten(solver="direct")
    assert all(s["status"] == 0 for s in st)
    d = b.last_solve(0)
    assert d["solver"] == "direct" and d["fmas"] > 0
    z = z.cpu().numpy()
    voff, loops = _loops(b)
    gid = np.concatenate([voff[c] + loops[c] for c in range(b.K)]).astype(np.int32)
    zh, sth = b.harmonic(gid, z[gid], solver="direct")
    assert all(s["status"] == 0 for s in sth)
    assert b.last_solve(1)["solver"] == "direct"
    zh = zh.cpu().numpy()
    sp = oracle.split_mesh(V, F, cuts)
    cs = range(b.K) if sample is None else sample
    for c in cs:
        rf = oracle.dncp_flatten(sp.sub_V[c], sp.sub_F[c], sp.loops[c])
        ef = np.max(np.abs(z[voff[c]:voff[c + 1]] - rf)) / _diam(rf)
        assert ef <= flat_tol, (c, ef)
        rh = oracle.dirichlet_extend(sp.sub_V[c], sp.sub_F[c], sp.loops[c], z[voff[c] + sp.loops[c]])
        eh = np.max(np.abs(zh[voff[c]:voff[c + 1]] - rh)) / _diam(rh)
        assert eh <= harm_tol, (c, eh)
    return b, z


def test_direct_height_field_matches_superlu(cuda):
    """Both solves of every subdomain of a 129^2 height field (4x4 blocks)
    agree with SuperLU to round-off: the flatten to 1e-9 of the diameter
    (the pinned DNCP system has condition ~1e6), the Dirichlet solve to 1e-12."""
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.height_field_case(129, 4, seed=1)
    _check_vs_oracle(V, F, cuts, 1e-9, 1e-12)


def test_direct_irregular_meshes(cuda):
    """Delaunay disk (cfg 3 construction) and icosphere (cfg 4 construction)
    at test size: k-means subdomains with ragged boundaries."""
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.cfg3(seed=0, n_points=20000, n_clusters=16)
    _check_vs_oracle(V, F, cuts, 1e-9, 1e-12, sample=range(0, 16, 3))
    V, F, cuts = gen.cfg4(seed=0, subdiv=5, n_clusters=16)
    _check_vs_oracle(V, F, cuts, 1e-9, 1e-12, sample=range(0, 16, 3))


def test_direct_matches_pcg(cuda):
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.height_field_case(257, 4)
    b = _batch(V, F, cuts)
    zd, _ = b.flatten(solver="direct")
    zp, _ = b.flatten(solver="pcg")
    zd, zp = zd.cpu().numpy(), zp.cpu().numpy()
    voff, _ = _loops(b)
    for c in range(b.K):
        a, e = zd[voff[c]:voff[c + 1]], zp[voff[c]:voff[c + 1]]
        assert np.max(np.abs(a - e)) <= 1e-7 * _diam(e), c


@pytest.mark.parametrize("leaf", ["4", "17", "300"])
def test_direct_leaf_size_invariant(cuda, monkeypatch, leaf):
    """The dissection depth changes the elimination order, not the answer."""
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.height_field_case(97, 3, seed=2)
    b = _batch(V, F, cuts)
    z0, _ = b.flatten(solver="direct")
    monkeypatch.setenv("PGCP_DIRECT_LEAF", leaf)
    z1, st = b.flatten(solver="direct")
    assert all(s["status"] == 0 for s in st)
    z0, z1 = z0.cpu().numpy(), z1.cpu().numpy()
    assert np.max(np.abs(z0 - z1)) <= 1e-9 * _diam(z0)


def test_direct_bitwise_repeatable(cuda):
    """Fixed-order extend-add and reductions: two factorizations and solves
    of the same batch are bit-identical."""
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.height_field_case(129, 4, seed=5)
    b = _batch(V, F, cuts)
    z0, _ = b.flatten(solver="direct")
    z1, _ = b.flatten(solver="direct")
    assert np.array_equal(z0.cpu().numpy(), z1.cpu().numpy())


def test_direct_is_default_and_pcg_selectable(cuda, monkeypatch):
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.height_field_case(65, 2)
    b = _batch(V, F, cuts)
    b.flatten()
    assert b.last_solve(0)["solver"] == "direct"
    b.flatten(maxit=100000)          # an iteration cap asks for PCG
    assert b.last_solve(0)["solver"] == "pcg"
    monkeypatch.setenv("PGCP_SOLVER", "pcg")
    b.flatten()
    assert b.last_solve(0)["solver"] == "pcg"
    b.flatten(solver="direct")       # explicit beats the environment
    assert b.last_solve(0)["solver"] == "direct"


def test_boundary_last_factor_serves_dirichlet(cuda, monkeypatch):
    """PGCP_DIRECT_BLAST=1: the DNCP system is factored with every boundary
    loop last; the Dirichlet solve then runs on the interior block of that
    factor (no factorization of its own) and still matches SuperLU."""
    from paper_1903_12359_b200 import generators as gen
    monkeypatch.setenv("PGCP_DIRECT_BLAST", "1")
    V, F, cuts = gen.height_field_case(97, 3, seed=4)
    b, z = _check_vs_oracle(V, F, cuts, 1e-9, 1e-12)
    assert b.last_solve(1)["borrowed"] and b.last_solve(1)["fmas"] == 0


@pytest.mark.parametrize("switch", ["PGCP_DIRECT_TWO_STREAMS", "PGCP_DIRECT_WSPLIT", "PGCP_DIRECT_NO_WARP"])
def test_direct_front_scheduling_is_result_neutral(cuda, monkeypatch, switch):
    """How the fronts of a level are scheduled -- complex fronts on a second
    stream, warp-sized fronts split off a list of larger ones and packed into
    CTAs by size -- does not change a front's arithmetic: the flatten and the
    Dirichlet solve are bit-identical with each option off (257^2 subdomains:
    the upper lists mix warp-sized and larger fronts, real and complex)."""
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.height_field_case(513, 2, seed=4)
    b = _batch(V, F, cuts)
    voff, loops = _loops(b)
    gid = np.concatenate([voff[c] + loops[c] for c in range(b.K)]).astype(np.int32)

    def run():
        z, st = b.flatten(solver="direct")
        assert all(s["status"] == 0 for s in st)
        z = z.cpu().numpy()
        zh, sth = b.harmonic(gid, z[gid], solver="direct")
        assert all(s["status"] == 0 for s in sth)
        return z, zh.cpu().numpy()

    z0, h0 = run()
    monkeypatch.setenv(switch, "1" if switch == "PGCP_DIRECT_NO_WARP" else "0")
    z1, h1 = run()
    if switch == "PGCP_DIRECT_NO_WARP":  # another kernel's summation order: agreement, not identity
        assert np.max(np.abs(z0 - z1)) <= 1e-9 * _diam(z0)
        assert np.max(np.abs(h0 - h1)) <= 1e-9 * _diam(h0)
    else:
        assert np.array_equal(z0, z1) and np.array_equal(h0, h1)
