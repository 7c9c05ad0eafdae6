"""Pin the CPU oracle against the reference's own outputs (CPU, no GPU).

The golden fixtures were produced by running the reference package
(tests/golden/make_goldens.py); the oracle must reproduce them bit for bit
(the oracle calls numpy/scipy exactly as the reference does). When the
reference itself is importable (build container), it is also compared live.
"""

import json
import os

import numpy as np
import pytest

from conftest import PIPELINE_CASES, REPAIR_CASES, case_pairs, load_golden, unpack, unpack_csr

import oracle
from oracle import planner as opl

REF = "/root/reference/pkg/src"


@pytest.mark.parametrize("case", PIPELINE_CASES + REPAIR_CASES)
def test_oracle_pipeline_bitwise(case):
    z = load_golden(case)
    mode = str(z["mode"])
    cuts = z["cuts"] if len(z["cuts"]) else None
    kw = {}
    if case_pairs(case) is not None:
        kw = dict(schedule="pairs", pairs=case_pairs(case))
    out = oracle.run_parameterize(z["V"], z["F"], cuts, mode, **kw)
    coords = np.asarray(out["coords"])
    assert np.array_equal(coords, z["coords"])
    assert out["flips"] == int(z["flips"])
    assert out["distortion"] == json.loads(str(z["distortion_json"]))
    assert out["seam_residuals"] == list(z["seam_residuals"])
    part = out["partition"]
    assert np.array_equal(part.face_assignment, z["face_assignment"])
    for a, b in zip(part.vertex_maps, unpack(z, "vertex_maps")):
        assert np.array_equal(a, b)
    for a, b in zip(part.boundary_cycles, unpack(z, "cycles")):
        assert np.array_equal(a, b)
    for st, a, b, mg, meta in zip(out["steps"], unpack(z, "step_a"), unpack(z, "step_b"),
                                  unpack(z, "step_merged"), z["step_meta"]):
        assert np.array_equal(st.a_cycle, a) and np.array_equal(st.b_cycle, b)
        assert np.array_equal(st.merged_cycle, mg)
        assert [st.comp_a, st.comp_b, st.k, int(st.closed)] == list(meta)
    for f, g in zip(out["flat"], unpack(z, "flat")):
        assert np.array_equal(f, g)
    if "repairs_json" in z.files:
        ref = json.loads(str(z["repairs_json"]))
        assert [{k: v for k, v in r.items() if k != "submesh"} for r in ref] == out["repairs"]
    if "harm" in z.files:
        for a, b in zip(out["embeddings_local"], unpack(z, "harm")):
            assert np.array_equal(a, b)


def test_oracle_qc_correct_bitwise():
    """oracle.repair restates assemble.py:53-217 call for call: the repaired
    embeddings, iteration counts and remaining faces of the reference's
    qc_correct (tests/golden/qc_direct.npz), the per-face layout, and the
    degenerate-triangle error."""
    from oracle.repair import OracleRepairError, isometric_layout, repair_folds
    z = load_golden("qc_direct")
    for i in range(int(z["count"])):
        assert np.array_equal(isometric_layout(z[f"V{i}"], z[f"F{i}"]), z[f"layout{i}"])
        args = (z[f"layout{i}"], z[f"F{i}"], z[f"z{i}"], z[f"fixed{i}"])
        if f"err{i}" in z.files:
            with pytest.raises(OracleRepairError, match="degenerate source triangle"):
                repair_folds(*args, max_iter=int(z[f"max_iter{i}"]))
            continue
        out, it, ok, left, n0 = repair_folds(*args, max_iter=int(z[f"max_iter{i}"]))
        assert [it, int(ok), n0] == list(z[f"res{i}"])
        assert np.array_equal(left, z[f"remaining{i}"])
        assert np.array_equal(out, z[f"out{i}"])


@pytest.mark.parametrize("case", ["cfg1", "blocks3x3", "flat2x2", "sphere4"])
def test_oracle_systems_bitwise(case):
    z = load_golden(case)
    sp = oracle.split_mesh(z["V"], z["F"], z["cuts"]) if len(z["cuts"]) else \
        oracle.surface.single_domain(z["V"], z["F"])
    Ls = unpack_csr(z, "L")
    Cff = unpack_csr(z, "Cff", values=False)
    Lii = unpack_csr(z, "Lii", values=False)
    for i in range(sp.n_sub):
        L, C, rhs, *_ = oracle.dncp_system(sp.sub_V[i], sp.sub_F[i], sp.loops[i])
        assert np.array_equal(L.indptr, Ls[i].indptr) and np.array_equal(L.indices, Ls[i].indices)
        assert np.array_equal(L.data, Ls[i].data)
        assert np.array_equal(C.indptr, Cff[i].indptr) and np.array_equal(C.indices, Cff[i].indices)
        assert np.array_equal(rhs, unpack(z, "rhs_f")[i])
        if "harm_g_off" in z.files:
            _, Li, rh, _ = oracle.harmonic_system(sp.sub_V[i], sp.sub_F[i], sp.loops[i],
                                                  unpack(z, "harm_g")[i])
            assert np.array_equal(Li.indptr, Lii[i].indptr) and np.array_equal(Li.indices, Lii[i].indices)
            assert np.array_equal(rh, unpack(z, "rhs_h")[i])


def test_flat_grid_explicit_zeros():
    """Right angles give exact-zero cot weights: kept in L, dropped in C_ff
    (SURVEY §0 fact 3)."""
    z = load_golden("flat2x2")
    L = unpack_csr(z, "L")[0]
    C = unpack_csr(z, "Cff", values=False)[0]
    assert np.sum(L.data == 0) > 0
    n = L.shape[0]
    assert C.nnz < 2 * (L.nnz - np.sum(L.data == 0)) + 4 * n


def test_hermitian_form():
    """C_ff (real 2|U| form) equals H = L_UU + 2i M_xy on complex vectors,
    and -C_f,fixed t equals the complex RHS the device builds (pcg.cu)."""
    z = load_golden("cfg1")
    sp = oracle.split_mesh(z["V"], z["F"], z["cuts"])
    i = 2
    L, C, rhs, free, fixed, fv, (p0, p1) = oracle.dncp_system(sp.sub_V[i], sp.sub_F[i], sp.loops[i])
    n = L.shape[0]
    U = np.setdiff1d(np.arange(n), [p0, p1])
    loop = sp.loops[i]
    nxt = dict(zip(loop.tolist(), np.roll(loop, -1).tolist()))
    prv = dict(zip(loop.tolist(), np.roll(loop, 1).tolist()))
    pos = {int(u): r for r, u in enumerate(U)}
    t = {p0: 0j, p1: 1 + 0j}
    rng = np.random.default_rng(0)
    x = rng.normal(size=len(U)) + 1j * rng.normal(size=len(U))
    Hx = L[U][:, U] @ x
    b = -(L[U][:, [p0, p1]] @ np.array([t[p0], t[p1]]))
    for r, u in enumerate(U):
        if u in nxt:
            a, c = nxt[u], prv[u]
            Hx[r] += 0.5j * ((x[pos[a]] if a in pos else 0) - (x[pos[c]] if c in pos else 0))
            b[r] -= 0.5j * (t[a] if a in t else 0) - 0.5j * (t[c] if c in t else 0)
    y = C @ np.concatenate([x.real, x.imag])
    nu = len(U)
    assert np.allclose(y[:nu], Hx.real, atol=1e-12) and np.allclose(y[nu:], Hx.imag, atol=1e-12)
    assert np.allclose(rhs[:nu], b.real, atol=1e-14) and np.allclose(rhs[nu:], b.imag, atol=1e-14)


def test_known_answers():
    """SPEC.md worked examples as evaluated by the reference."""
    ka = load_golden("known_answers")
    s3 = np.sqrt(3.0)
    V = np.array([[0, 0, 0], [1, 0, 0], [0.5, s3 / 2, 0]], float)
    L = oracle.cotan_laplacian(V, np.array([[0, 1, 2]])).toarray()
    assert np.array_equal(L, ka["equilateral_L"])
    assert abs(L[0, 1] - (-0.2886751345948128)) < 1e-15
    assert abs(L[0, 0] - 0.5773502691896257) < 1e-15
    Vr = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    Lr = oracle.cotan_laplacian(Vr, np.array([[0, 1, 2]]))
    assert Lr.nnz == int(ka["right_L_nnz"]) == 9  # hypotenuse entry kept as explicit zero
    assert np.array_equal(Lr.toarray(), ka["right_L_dense"])
    Vs = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], float)
    M = oracle.area_form(4, [np.array([0, 1, 2, 3])])
    xy = np.concatenate([Vs[:, 0], Vs[:, 1]])
    assert xy @ (M @ xy) == float(ka["unit_square_area"]) == 1.0
    st = oracle.summary_stats([1.0, 2.0, 3.0, 4.0])
    assert [st["mean"], st["sd"], st["median"], st["iqr"]] == list(ka["summ_1234"])
    assert oracle.summary_stats(np.arange(1.0, 9.0))["iqr"] == float(ka["iqr_1to8"]) == 3.5
    d, valid = oracle.angle_distortion(Vr, np.array([[0, 1, 2]]), np.array([0, 2, 1j]), "free")
    assert np.allclose(d, ka["stretch_distortion"], atol=0, rtol=0)
    P = oracle.stereo_inverse(np.array([0, oracle.zipper.INF, 1.0]))
    assert np.array_equal(P, ka["stereo_inv"])


def test_weld_corpus():
    """Oracle partial_weld reproduces the reference on random Jordan pairs
    (SPEC acceptance criterion 1 corpus)."""
    z = load_golden("weld_corpus")
    A, B = unpack(z, "a"), unpack(z, "b")
    OA, OB = unpack(z, "oa"), unpack(z, "ob")
    for a, b, k, oa, ob, seam in zip(A, B, z["k"], OA, OB, z["seam"]):
        r = oracle.partial_weld(a, b, int(k))
        assert np.array_equal(r.a, oa) and np.array_equal(r.b, ob)
        assert r.seam_error == seam
        # the logs replay the transformation on the inputs
        ra, _ = oracle.replay(r.log_a, a)
        assert np.allclose(ra, r.a, rtol=0, atol=1e-9 * np.max(np.abs(r.a)))


def test_pipeline_welds_match_golden():
    for case in ["cfg1", "blocks3x3", "sphere4", "disk2x2"]:
        z = load_golden(case)
        ins_a, ins_b = unpack(z, "weld_in_a"), unpack(z, "weld_in_b")
        outs_a, outs_b = unpack(z, "weld_out_a"), unpack(z, "weld_out_b")
        for a, b, k, cl, oa, ob in zip(ins_a, ins_b, z["weld_k"], z["weld_closed"], outs_a, outs_b):
            r = oracle.closed_weld(a, b) if cl else oracle.partial_weld(a, b, int(k))
            assert np.array_equal(r.a, oa) and np.array_equal(r.b, ob)
        if "geo_in" in z.files:
            circ, _ = oracle.geodesic_to_circle(z["geo_in"])
            assert np.array_equal(circ, z["geo_out"])


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
def test_oracle_vs_live_reference_strips():
    import sys
    sys.path.insert(0, REF)
    import pgcp
    from paper_1903_12359_b200.generators import height_field_case
    V, F, cuts = height_field_case(41, 5, layout="strips", seed=9)
    gp, rep = pgcp.parameterize(pgcp.TriMesh(V, F), cuts, "free")
    out = oracle.run_parameterize(V, F, cuts, "free")
    assert np.array_equal(out["coords"], gp.coords)


def test_planner_error_paths():
    # two components sharing only a corner: no open arc -> PartitionError
    with pytest.raises(Exception):
        opl.greedy_schedule([np.array([0, 1, 2]), np.array([2, 3, 4])], np.zeros((0, 2), np.int64))
