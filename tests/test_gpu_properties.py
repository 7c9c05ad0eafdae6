"""Size-independent properties at BASELINE sizes and SPEC acceptance checks
(SURVEY §4): the flatten / harmonic consistency on every cfg-2 subdomain,
the planar-grid acceptance criterion, a Beltrami known answer, sphere unit
norm."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_harmonic_reproduces_flatten_interior_cfg2(cuda):
    """The DNCP interior rows are exactly L u = 0 (M touches only boundary
    rows), so the Dirichlet solve with a flatten's own boundary values
    reproduces its interior -- for all 64 cfg-2 subdomains at full size."""
    import torch
    from paper_1903_12359_b200 import TriMesh, partition_mesh
    from paper_1903_12359_b200 import _native as nat
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.cfg2(0)
    b = partition_mesh(TriMesh(V, F, check=False), cuts).batch
    z, st = b.flatten()
    assert all(s["status"] == 0 for s in st)
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
    lp = b.host(nat.ARR_LOOP, torch.int32)
    gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
    zh, sth = b.harmonic(gid, z[torch.as_tensor(gid, device=z.device).long()])
    assert all(s["status"] == 0 for s in sth)
    zf, zh = z.cpu().numpy(), zh.cpu().numpy()
    for c in range(b.K):
        a, e = zf[voff[c]:voff[c + 1]], zh[voff[c]:voff[c + 1]]
        diam = 2 * np.max(np.abs(a - a.mean()))
        assert np.max(np.abs(a - e)) <= 1e-7 * diam, c


def test_planar_grid_acceptance(cuda):
    """SPEC acceptance: a 64 x 64 planar grid parameterizes with mean
    angular distortion below 0.01 degrees and no flips."""
    from paper_1903_12359_b200 import TriMesh, parameterize
    from paper_1903_12359_b200 import generators as gen
    V, F = gen.flat_grid_arrays(63)
    cuts = gen.cuts_from_face_labels(F, gen.block_face_labels(64, 2))
    gp, rep = parameterize(TriMesh(V, F), cuts, "free")
    assert rep.flips == 0
    assert rep.distortion["angular_abs"]["mean"] < 0.01


def test_beltrami_known_answer(cuda):
    """mu of z -> z + conj(z) / 2 is 1/2 on every triangle."""
    from paper_1903_12359_b200 import beltrami_per_face
    rng = np.random.default_rng(0)
    src = rng.normal(size=(50, 3)) + 1j * rng.normal(size=(50, 3))
    tgt = src + 0.5 * np.conj(src)
    mu = beltrami_per_face(src, tgt)
    assert np.max(np.abs(mu - 0.5)) <= 1e-12


def test_sphere_unit_norm(cuda):
    """SPEC acceptance: spherical parameterizations lie on the unit sphere."""
    from conftest import load_golden
    from paper_1903_12359_b200 import TriMesh, parameterize
    z = load_golden("sphere4")
    gp, rep = parameterize(TriMesh(z["V"], z["F"]), z["cuts"], "sphere")
    assert np.max(np.abs(np.linalg.norm(gp.coords, axis=1) - 1.0)) <= 1e-9

def test_coarse_start_same_solution_fewer_iterations(cuda, monkeypatch):
    """The coarse start (x0 = Q b) changes the CG path,
    not the answer: flatten from x = 0 and from x0 agree to 1e-7 x diameter
    per subdomain, and the coarse start needs fewer iterations in total."""
    import torch
    from paper_1903_12359_b200 import TriMesh, partition_mesh
    from paper_1903_12359_b200 import _native as nat
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.height_field_case(257, 4)
    b = partition_mesh(TriMesh(V, F, check=False), cuts).batch
    monkeypatch.setenv("PGCP_SOLVER", "pcg")
    out = {}
    for x0 in ("0", "1"):
        monkeypatch.setenv("PGCP_PCG_X0", x0)
        z, st = b.flatten()
        assert all(s["status"] == 0 for s in st)
        out[x0] = (z.cpu().numpy(), b.last_solve(0)["iters_sum"])
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    for c in range(b.K):
        a, e = out["0"][0][voff[c]:voff[c + 1]], out["1"][0][voff[c]:voff[c + 1]]
        diam = 2 * np.max(np.abs(a - a.mean()))
        assert np.max(np.abs(a - e)) <= 1e-7 * diam, c
    assert out["1"][1] < out["0"][1]
