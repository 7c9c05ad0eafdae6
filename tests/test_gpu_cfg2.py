"""The benchmarked run, pinned end to end against the reference.

`tests/golden/cfg2_qtree.npz` holds what the reference `pgcp.parameterize`
(`pipeline.py:119-271`) produced on BASELINE cfg 2 (1024^2 height field,
seed 0, 8x8 blocks, 64 subdomains) with the quadtree weld order that
bench.py uses (`make_goldens.py cfg2_qtree`, run in the build container
with the reference on 8 processes). These tests run the device path exactly
as bench.py does and compare:

  * partition integers (face labels, boundary cycles, local loops, vertex
    maps) and the weld plan (every step's cycles) bit for bit;
  * all 64 DNCP flattens (`flatten.py:125-188`) on every boundary-loop
    vertex and every 61st local vertex, <= 1e-6 x the subdomain diameter;
  * all 64 Dirichlet solves (`assemble.py:23-50`) from the reference's
    welded boundary values, same sample and tolerance;
  * the largest weld of each of the 6 levels (k up to 1024), <= 1e-9
    relative, as in test_gpu_pipeline.test_welds_match_reference;
  * the final UV (every 61st parent vertex) <= 1e-6 x diameter, 0 flips,
    angular mean / sd / median / IQR within 1e-3 degrees, seam residuals.
"""

import json

import numpy as np
import pytest

from conftest import load_golden, unpack


@pytest.fixture(scope="module")
def golden():
    return load_golden("cfg2_qtree")


@pytest.fixture(scope="module")
def cfg2():
    from paper_1903_12359_b200 import generators as gen
    V, F, cuts = gen.cfg2(0)
    return V, F, cuts, gen.quadtree_schedule_order(8, 8)


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def _diam(z):
    return 2 * np.max(np.abs(z - z.mean()))


def test_cfg2_inputs_are_the_golden_inputs(golden, cfg2):
    V, F, cuts, _ = cfg2
    assert _sha(np.asarray(V, np.float64)) == str(golden["V_sha"])
    assert _sha(np.asarray(F, np.int32)) == str(golden["F_sha"])
    assert _sha(np.asarray(cuts, np.int64)) == str(golden["cuts_sha"])


@pytest.fixture(scope="module")
def part(cfg2):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1903_12359_b200.mesh import TriMesh
    from paper_1903_12359_b200.partition import partition_mesh
    V, F, cuts, _ = cfg2
    return partition_mesh(TriMesh(V, F), cuts)


@pytest.mark.gpu
def test_cfg2_partition_and_plan_bit_exact(golden, cfg2, part):
    from paper_1903_12359_b200.partition import plan_weld_schedule
    assert part.n_submeshes == 64
    assert np.array_equal(part.face_assignment, golden["face_assignment"].astype(np.int64))
    assert _sha(np.concatenate(part.vertex_maps).astype(np.int64)) == str(golden["vertex_maps_sha"])
    for a, b in zip(part.boundary_cycles, unpack(golden, "cycles")):
        assert np.array_equal(a, b)
    for a, b in zip(part.local_loops, unpack(golden, "loops")):
        assert np.array_equal(a, b)
    steps = plan_weld_schedule(part, "free", pairs=cfg2[3])
    assert len(steps) == 63
    for st, meta, sha in zip(steps, golden["step_meta"], golden["step_sha"]):
        assert [st.comp_a, st.comp_b, st.k, int(st.closed)] == list(meta)
        assert _sha(np.asarray(st.a_cycle, np.int64)) == str(sha[0])
        assert _sha(np.asarray(st.b_cycle, np.int64)) == str(sha[1])
        assert _sha(np.asarray(st.merged_cycle, np.int64)) == str(sha[2])


def _voff(batch):
    import torch
    from paper_1903_12359_b200 import _native as nat
    return batch.host(nat.ARR_VERT_OFF, torch.int64)


@pytest.mark.gpu
def test_cfg2_all_64_flattens_match_reference(golden, part):
    b = part.batch
    z, stats = b.flatten()
    z = z.cpu().numpy()
    voff = _voff(b)
    stride = int(golden["stride"])
    loops = unpack(golden, "loops")
    worst = 0.0
    for c, (ref_loop, ref_samp) in enumerate(zip(unpack(golden, "flat_loop"), unpack(golden, "flat_samp"))):
        got = z[voff[c]:voff[c + 1]]
        diam = _diam(ref_loop)  # the boundary carries the subdomain's extent
        err = max(np.max(np.abs(got[loops[c]] - ref_loop)), np.max(np.abs(got[::stride] - ref_samp))) / diam
        worst = max(worst, err)
        assert err <= 1e-6, (c, err)
    assert all(s["status"] == 0 for s in stats)
    print(f"cfg2 flatten: worst err/diam {worst:.2e} over 64 subdomains")


@pytest.mark.gpu
def test_cfg2_all_64_harmonic_solves_match_reference(golden, part):
    b = part.batch
    voff = _voff(b)
    loops = unpack(golden, "loops")
    gid = np.concatenate([voff[c] + loops[c] for c in range(64)]).astype(np.int32)
    vals = golden["harm_g"]
    z, stats = b.harmonic(gid, vals)
    z = z.cpu().numpy()
    stride = int(golden["stride"])
    worst = 0.0
    for c, (g, ref_samp) in enumerate(zip(unpack(golden, "harm_g"), unpack(golden, "harm_samp"))):
        got = z[voff[c]:voff[c + 1]]
        diam = _diam(g)
        assert np.array_equal(got[loops[c]], g)  # Dirichlet values held exactly
        err = np.max(np.abs(got[::stride] - ref_samp)) / diam
        worst = max(worst, err)
        assert err <= 1e-6, (c, err)
    assert all(s["status"] == 0 for s in stats)
    print(f"cfg2 harmonic: worst err/diam {worst:.2e} over 64 subdomains")


@pytest.mark.gpu
def test_cfg2_largest_weld_per_level_matches_reference(cuda, golden):
    from paper_1903_12359_b200 import partial_weld
    ks = golden["weld_k"][golden["big_weld"]]
    assert ks.max() >= 1000
    for k, a, b, oa, ob, i in zip(ks, unpack(golden, "big_in_a"), unpack(golden, "big_in_b"),
                                  unpack(golden, "big_out_a"), unpack(golden, "big_out_b"), golden["big_weld"]):
        r = partial_weld(a, b, int(k))
        sc = max(np.max(np.abs(oa)), np.max(np.abs(ob)))
        ea = np.max(np.abs(r.a - oa)) / sc
        eb = np.max(np.abs(r.b - ob)) / sc
        assert ea <= 1e-9 and eb <= 1e-9, (int(k), ea, eb)
        assert abs(r.seam_error - golden["weld_seam"][i]) <= 1e-9 * sc


@pytest.mark.gpu
def test_cfg2_end_to_end_matches_reference(golden, cfg2):
    """parameterize exactly as bench.py calls it (e2e leg: host arrays in,
    host coordinates out)."""
    from paper_1903_12359_b200 import TriMesh, parameterize
    V, F, cuts, pairs = cfg2
    gp, rep = parameterize(TriMesh(V, F.astype(np.int32)), cuts, "free", pairs=pairs)
    stride = int(golden["stride"])
    got = np.asarray(gp.coords)[::stride]
    ref = golden["coords_samp"]
    err = np.max(np.abs(got - ref)) / float(golden["coords_diam"])
    assert err <= 1e-6, err
    assert rep.flips == int(golden["flips"]) == 0
    rd = json.loads(str(golden["distortion_json"]))
    for key in ("mean", "sd", "median", "iqr"):
        assert abs(rep.distortion["angular_abs"][key] - rd["angular_abs"][key]) <= 1e-3, key
    assert rep.distortion["excluded_corners"] == rd["excluded_corners"]
    assert len(rep.seam_residuals) == len(golden["seam_residuals"]) == 63
    assert rep.ok == bool(golden["ok"])
    ref_rep = json.loads(str(golden["repairs_json"]))
    assert [r["flips_before"] for r in rep.repairs] == [r["flips_before"] for r in ref_rep]
    print(f"cfg2 end to end: uv err/diam {err:.2e}, mean |d| {rep.distortion['angular_abs']['mean']:.6f} "
          f"(reference {rd['angular_abs']['mean']:.6f})")
