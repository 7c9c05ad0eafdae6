"""GPU parity of the quasi-conformal fold-over repair (repair.cu) against the
reference: `qc_correct` called directly (tests/golden/qc_direct.npz) and
the pipeline cases whose harmonic maps fold (repair_*.npz, the per-submesh
repair of pipeline.py:88-102). UV within 1e-6 of the parameter-domain
diameter; iteration counts, cleared flags, remaining faces and flip counts
equal; angle-distortion mean/sd within 1e-3 degrees."""

import json
import re

import numpy as np
import pytest

from conftest import REPAIR_CASES, load_golden, unpack

pytestmark = pytest.mark.gpu


def _diam(z):
    z = np.asarray(z)
    return 2 * np.max(np.abs(z - z.mean()))


def test_face_layout_matches_reference(cuda):
    from paper_1903_12359_b200 import TriMesh, face_layout
    z = load_golden("qc_direct")
    for i in range(int(z["count"])):
        lay = face_layout(TriMesh(z[f"V{i}"], z[f"F{i}"], check=False))
        assert np.array_equal(lay, z[f"layout{i}"])  # numpy's evaluation order, bit for bit


def test_beltrami_matches_oracle(cuda):
    from oracle.repair import face_beltrami
    from paper_1903_12359_b200 import beltrami_per_face
    z = load_golden("qc_direct")
    for i in range(3):
        src, F, lay = z[f"z{i}"], z[f"F{i}"], z[f"layout{i}"]
        ref = face_beltrami(src[F], lay)  # per-face corner form
        got = beltrami_per_face(src[F], lay)
        fin = np.isfinite(ref)
        assert np.array_equal(fin, np.isfinite(got))
        assert np.max(np.abs(got[fin] - ref[fin])) <= 1e-12 * max(1.0, np.max(np.abs(ref[fin])))
        # per-vertex form with faces: the identity map has mu == 0
        assert np.max(np.abs(beltrami_per_face(src, src, F))) <= 1e-12


def test_beltrami_degenerate_raises(cuda):
    from paper_1903_12359_b200 import SolveError, beltrami_per_face
    src = np.array([[0, 1, 2]], dtype=np.complex128)  # collinear
    tgt = np.array([[0, 1, 1j]], dtype=np.complex128)
    with pytest.raises(SolveError, match="degenerate source triangle 0"):
        beltrami_per_face(src, tgt)


def test_check_bijectivity():
    from paper_1903_12359_b200 import check_bijectivity
    rep = check_bijectivity(np.array([0.1, 0.995, np.inf, 0.5j, np.nan]), threshold=0.99)
    assert list(rep.bad_faces) == [1, 2, 4]
    assert rep.max_mu == np.inf and not rep.ok


def test_qc_correct_matches_reference(cuda):
    from paper_1903_12359_b200 import SolveError, qc_correct
    z = load_golden("qc_direct")
    for i in range(int(z["count"])):
        args = (z[f"layout{i}"], z[f"F{i}"], z[f"z{i}"], z[f"fixed{i}"])
        if f"err{i}" in z.files:
            with pytest.raises(SolveError, match="degenerate source triangle"):
                qc_correct(*args, max_iter=int(z[f"max_iter{i}"]))
            continue
        out, rep = qc_correct(*args, max_iter=int(z[f"max_iter{i}"]))
        it, cleared, n0 = z[f"res{i}"]
        assert (rep.iterations, int(rep.cleared), rep.initial_flips) == (it, cleared, n0), i
        assert np.array_equal(np.sort(rep.remaining_faces), z[f"remaining{i}"]), i
        ref = z[f"out{i}"]
        assert np.max(np.abs(out - ref)) <= 1e-6 * _diam(ref), i


def test_qc_correct_no_flips_is_identity(cuda):
    from paper_1903_12359_b200 import qc_correct
    z = load_golden("qc_direct")
    V, F = z["V0"], z["F0"]
    emb = V[:, 0] + 1j * V[:, 1]
    out, rep = qc_correct(z["layout0"], F, emb, z["fixed0"])
    assert rep.iterations == 0 and rep.cleared and rep.initial_flips == 0
    assert np.array_equal(out, emb)


@pytest.mark.parametrize("case", REPAIR_CASES)
def test_pipeline_repair_matches_reference(cuda, case):
    from paper_1903_12359_b200 import TriMesh, parameterize
    z = load_golden(case)
    mesh = TriMesh(z["V"], z["F"])
    cuts = z["cuts"] if len(z["cuts"]) else None
    gp, rep = parameterize(mesh, cuts, str(z["mode"]))
    ref = z["coords"]
    got = np.asarray(gp.coords)
    assert np.max(np.abs(got - ref)) <= 1e-6 * _diam(ref), case
    assert rep.flips == int(z["flips"])
    refrep = json.loads(str(z["repairs_json"]))
    assert rep.repairs == refrep
    rd = json.loads(str(z["distortion_json"]))
    for key in ("mean", "sd"):
        assert abs(rep.distortion["angular_abs"][key] - rd["angular_abs"][key]) <= 1e-3
    assert rep.ok == bool(z["ok"])


def test_stitch_global_matches_reference(cuda):
    from paper_1903_12359_b200 import TriMesh, partition_mesh, stitch_global
    z = load_golden("repair_strips3")
    part = partition_mesh(TriMesh(z["V"], z["F"]), z["cuts"])
    gp = stitch_global(part, unpack(z, "harm"), "free")
    ref = z["coords"]
    assert np.max(np.abs(gp.coords - ref)) <= 1e-12 * _diam(ref)
    assert len(gp.flipped_faces) == int(z["flips"])


def test_intermediate_form_matches_reference(cuda):
    """intermediate_form (welding.py:578-602) on the weld corpus boundaries,
    both branches: values within 1e-9 of the scale, side tags and record
    counts equal; error paths with the reference's messages."""
    from paper_1903_12359_b200 import WeldError, intermediate_form
    z = load_golden("intermediate")
    for pts, vals, sides, nrec, k, br in zip(unpack(z, "pts"), unpack(z, "vals"), unpack(z, "sides"), z["nrec"],
                                             z["k"], z["branch"]):
        r = intermediate_form(pts, int(k), int(br))
        assert np.array_equal(r.sides, sides)
        assert len(r.log) == nrec
        fin = np.isfinite(vals)
        assert np.array_equal(fin, np.isfinite(r.values))
        sc = np.max(np.abs(vals[fin]))
        assert np.max(np.abs(r.values[fin] - vals[fin])) <= 1e-9 * sc
    cases = (([0, 1, 2], 0), ([0, 1], 2), ([1, 1, 2, 3], 2), ([0, 1, 1j, 2], 3))
    for (pts, k), msg in zip(cases, z["errors"]):
        if str(msg):
            with pytest.raises(WeldError, match=re.escape(str(msg))):
                intermediate_form(np.asarray(pts, np.complex128), k)
        else:
            intermediate_form(np.asarray(pts, np.complex128), k)
