"""GPU parity of the hot-path stages against the reference goldens and the
oracle: partition integers, CSR patterns (bit-exact), Laplacian values,
DNCP flatten and harmonic solves, system patterns (C_ff / L_II)."""

import numpy as np
import pytest

from conftest import load_golden, unpack, unpack_csr

pytestmark = pytest.mark.gpu

CUT_CASES = ["cfg1", "strips4", "blocks3x3", "disk2x2", "flat2x2", "sphere2", "sphere4", "tree4x4", "ptree4x4", "qtree4x4"]
ALL_CASES = CUT_CASES + ["k1free", "k1disk"]


def _mesh_part(case):
    from paper_1903_12359_b200.mesh import TriMesh
    from paper_1903_12359_b200.partition import partition_mesh
    z = load_golden(case)
    mesh = TriMesh(z["V"], z["F"])
    if len(z["cuts"]):
        part = partition_mesh(mesh, z["cuts"])
        batch = part.batch
    else:
        part = None
        batch = mesh.batch()
    return z, mesh, part, batch


@pytest.mark.parametrize("case", CUT_CASES)
def test_partition_integers(cuda, case):
    z, mesh, part, _ = _mesh_part(case)
    assert part.n_submeshes == len(unpack(z, "vertex_maps"))
    assert np.array_equal(part.face_assignment, z["face_assignment"])
    for a, b in zip(part.vertex_maps, unpack(z, "vertex_maps")):
        assert np.array_equal(a, b)
    for a, b in zip(part.boundary_cycles, unpack(z, "cycles")):
        assert np.array_equal(a, b)
    for a, b in zip(part.local_loops, unpack(z, "loops")):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("case", ["cfg1", "blocks3x3", "sphere4"])
def test_local_faces_match_oracle(cuda, case):
    import oracle
    z, mesh, part, _ = _mesh_part(case)
    sp = oracle.split_mesh(z["V"], z["F"], z["cuts"])
    for sub, f in zip(part.submeshes, sp.sub_F):
        assert np.array_equal(sub.faces, f)


@pytest.mark.parametrize("case", ALL_CASES)
def test_laplacian_csr(cuda, case):
    import torch
    from paper_1903_12359_b200 import _native as nat
    z, mesh, part, batch = _mesh_part(case)
    batch.laplacian()
    rp = batch.host(nat.ARR_L_ROWPTR, torch.int64)
    col = batch.host(nat.ARR_L_COL, torch.int32)
    val = batch.host(nat.ARR_L_VAL, torch.float64)
    voff = batch.host(nat.ARR_VERT_OFF, torch.int64)
    for c, L in enumerate(unpack_csr(z, "L")):
        r = rp[voff[c]:voff[c + 1] + 1]
        ip = (r - r[0]).astype(np.int32)
        assert np.array_equal(ip, L.indptr), "indptr"
        assert np.array_equal(col[r[0]:r[-1]], L.indices), "indices"
        v = val[r[0]:r[-1]]
        rows = np.repeat(np.arange(L.shape[0]), np.diff(L.indptr))
        off = L.indices != rows
        assert np.array_equal(v[off], L.data[off]), "off-diagonal values must be bit-exact"
        assert np.max(np.abs(v - L.data)) <= 1e-14 * np.max(np.abs(L.data))
        assert np.sum(v == 0) == np.sum(L.data == 0)


@pytest.mark.parametrize("case", ALL_CASES)
def test_flatten_matches_reference(cuda, case):
    z, mesh, part, batch = _mesh_part(case)
    zz, stats = batch.flatten()
    zz = zz.cpu().numpy()
    import torch
    from paper_1903_12359_b200 import _native as nat
    voff = batch.host(nat.ARR_VERT_OFF, torch.int64)
    for c, ref in enumerate(unpack(z, "flat")):
        got = zz[voff[c]:voff[c + 1]]
        diam = np.max(np.abs(ref - ref[:, None])) if len(ref) < 3000 else 2 * np.max(np.abs(ref - ref.mean()))
        assert np.max(np.abs(got - ref)) <= 1e-6 * diam, (c, stats[c])
        assert stats[c]["status"] == 0
    # pinned systems: C_ff pattern bit-exact, rhs equal
    for c, (Cref, rref) in enumerate(zip(unpack_csr(z, "Cff", values=False), unpack(z, "rhs_f"))):
        C, rhs = batch.export_system(0, c)
        assert np.array_equal(C.indptr, Cref.indptr) and np.array_equal(C.indices, Cref.indices)
        assert np.allclose(rhs, rref, rtol=0, atol=1e-14)


@pytest.mark.parametrize("case", [c for c in ALL_CASES if c != "k1free"])
def test_harmonic_matches_reference(cuda, case):
    import torch
    from paper_1903_12359_b200 import _native as nat
    z, mesh, part, batch = _mesh_part(case)
    voff = batch.host(nat.ARR_VERT_OFF, torch.int64)
    loops = unpack(z, "loops")
    g = unpack(z, "harm_g")
    gid = np.concatenate([voff[c] + loops[c] for c in range(len(loops))]).astype(np.int32)
    zz, stats = batch.harmonic(gid, np.concatenate(g))
    zz = zz.cpu().numpy()
    for c, ref in enumerate(unpack(z, "harm")):
        got = zz[voff[c]:voff[c + 1]]
        scale = np.max(np.abs(ref))
        assert np.max(np.abs(got - ref)) <= 1e-7 * scale, (c, stats[c])
    for c, (Lref, rref) in enumerate(zip(unpack_csr(z, "Lii", values=False), unpack(z, "rhs_h"))):
        L, rhs = batch.export_system(1, c)
        assert np.array_equal(L.indptr, Lref.indptr) and np.array_equal(L.indices, Lref.indices)
        assert np.allclose(rhs, rref, rtol=0, atol=1e-13 * max(1.0, np.max(np.abs(rref))))


def test_api_single_mesh(cuda):
    import oracle
    from paper_1903_12359_b200 import flatten as fl
    from paper_1903_12359_b200.assemble import harmonic_solve
    from paper_1903_12359_b200.mesh import TriMesh, boundary_loops
    z = load_golden("k1free")
    mesh = TriMesh(z["V"], z["F"])
    L = fl.cotangent_laplacian(mesh)
    Lo = oracle.cotan_laplacian(z["V"], z["F"])
    assert np.array_equal(L.indptr, Lo.indptr) and np.array_equal(L.indices, Lo.indices)
    loop = boundary_loops(mesh)[0]
    assert np.array_equal(loop, unpack(z, "loops")[0])
    w = fl.flatten_free_boundary(mesh)
    ref = unpack(z, "flat")[0]
    assert np.max(np.abs(w - ref)) < 1e-8
    h = harmonic_solve(mesh, loop, ref[loop])
    assert np.max(np.abs(h - ref)) < 1e-8  # DNCP interior rows are L u = 0


def test_solve_determinism(cuda):
    z, mesh, part, batch = _mesh_part("blocks3x3")
    a, _ = batch.flatten()
    b, _ = batch.flatten()
    assert bool((a == b).all())


def test_partition_errors(cuda):
    from paper_1903_12359_b200.errors import MeshError, PartitionError
    from paper_1903_12359_b200.mesh import TriMesh
    from paper_1903_12359_b200.partition import partition_mesh
    z = load_golden("cfg1")
    mesh = TriMesh(z["V"], z["F"])
    cuts = z["cuts"]
    with pytest.raises(PartitionError, match="duplicate"):
        partition_mesh(mesh, np.concatenate([cuts, cuts[:1, ::-1]]))
    with pytest.raises(PartitionError, match="not a mesh edge"):
        partition_mesh(mesh, np.concatenate([cuts, [[0, 5000]]]))
    from paper_1903_12359_b200.generators import cuts_from_face_labels
    cell = np.arange(len(z["F"])) // 2
    ix, iy = cell % 99, cell // 99
    hole = ((ix > 30) & (ix < 60) & (iy > 30) & (iy < 60)).astype(int)
    with pytest.raises(PartitionError, match=r"component 0 is unsupported \(chi=0, 2 loops\)"):
        partition_mesh(mesh, cuts_from_face_labels(z["F"], hole))  # annulus, as the reference
    with pytest.raises(MeshError):
        TriMesh(z["V"], np.array([[0, 1, 1]]))
    with pytest.raises(MeshError):
        TriMesh(z["V"][:3], np.array([[0, 1, 5]]))


@pytest.mark.slow
def test_cfg2_stagewise(cuda):
    """BASELINE cfg 2 (1024^2, 8x8): partition integers vs the oracle at full
    size; DNCP of three subdomains vs the oracle's SuperLU solve."""
    import oracle
    from paper_1903_12359_b200 import generators as gen
    from paper_1903_12359_b200.mesh import TriMesh
    from paper_1903_12359_b200.partition import partition_mesh
    V, F, cuts = gen.cfg2(0)
    mesh = TriMesh(V, F, check=False)
    part = partition_mesh(mesh, cuts)
    sp = oracle.split_mesh(V, F, cuts)
    assert np.array_equal(part.face_assignment, sp.face_assignment)
    for a, b in zip(part.boundary_cycles, sp.boundary_cycles):
        assert np.array_equal(a, b)
    zz, stats = part.batch.flatten()
    zz = zz.cpu().numpy()
    import torch
    from paper_1903_12359_b200 import _native as nat
    voff = part.batch.host(nat.ARR_VERT_OFF, torch.int64)
    for c in (0, 27, 63):
        ref = oracle.dncp_flatten(sp.sub_V[c], sp.sub_F[c], sp.loops[c])
        got = zz[voff[c]:voff[c + 1]]
        assert np.max(np.abs(got - ref)) <= 1e-6 * 2 * np.max(np.abs(ref - ref.mean()))


def test_harmonic_prepare_then_solve_equals_harmonic(cuda):
    """The two-call harmonic API (structure first, values later) gives the
    same embedding as the one-call solve, bit for bit."""
    import torch
    from paper_1903_12359_b200 import TriMesh, partition_mesh
    from paper_1903_12359_b200 import _native as nat
    z = load_golden("blocks3x3")
    part = partition_mesh(TriMesh(z["V"], z["F"]), z["cuts"])
    b = part.batch
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
    lp = b.host(nat.ARR_LOOP, torch.int32)
    gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
    vals = np.exp(2j * np.pi * np.linspace(0, 1, len(gid), endpoint=False))
    z1, _ = b.harmonic(gid, vals)
    b.harmonic_prepare(gid)
    z2, st = b.harmonic_solve(vals)
    assert all(s["status"] == 0 for s in st)
    assert torch.equal(z1, z2)
