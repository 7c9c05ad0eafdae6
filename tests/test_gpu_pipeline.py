"""GPU parity of the weld engine and of the end-to-end device pipeline
against the reference goldens (UV within 1e-6 of the parameter-domain
diameter, 0 flips, angle-distortion mean/sd within 1e-3 degrees, exact
median/IQR agreement to rounding)."""

import json

import numpy as np
import pytest

from conftest import case_pairs, load_golden, unpack

pytestmark = pytest.mark.gpu

CASES = ["cfg1", "strips4", "blocks3x3", "disk2x2", "k1free", "k1disk", "flat2x2", "sphere2", "sphere4",
         "tree4x4", "ptree4x4", "qtree4x4"]


def _diam(z):
    z = np.asarray(z)
    if z.ndim == 2:  # sphere: chordal diameter 2
        return 2.0
    zz = z[np.isfinite(z)]
    c = zz.mean()
    return 2 * np.max(np.abs(zz - c))


@pytest.mark.parametrize("case", ["cfg1", "blocks3x3", "sphere4", "disk2x2", "tree4x4", "ptree4x4", "qtree4x4"])
def test_welds_match_reference(cuda, case):
    from paper_1903_12359_b200 import closed_weld, partial_weld
    z = load_golden(case)
    ins_a, ins_b = unpack(z, "weld_in_a"), unpack(z, "weld_in_b")
    outs_a, outs_b = unpack(z, "weld_out_a"), unpack(z, "weld_out_b")
    for a, b, k, cl, oa, ob, seam in zip(ins_a, ins_b, z["weld_k"], z["weld_closed"], outs_a, outs_b,
                                         z["weld_seam"]):
        r = closed_weld(a, b) if cl else partial_weld(a, b, int(k))
        sc = max(np.max(np.abs(oa)), np.max(np.abs(ob)))
        assert np.max(np.abs(r.a - oa)) <= 1e-9 * sc
        assert np.max(np.abs(r.b - ob)) <= 1e-9 * sc
        assert abs(r.seam_error - seam) <= 1e-9 * sc


def test_weld_corpus(cuda):
    from paper_1903_12359_b200 import apply_log, partial_weld
    z = load_golden("weld_corpus")
    for a, b, k, oa, ob in zip(unpack(z, "a"), unpack(z, "b"), z["k"], unpack(z, "oa"), unpack(z, "ob")):
        r = partial_weld(a, b, int(k))
        sc = max(np.max(np.abs(oa)), np.max(np.abs(ob)))
        assert np.max(np.abs(r.a - oa)) <= 1e-9 * sc
        assert np.max(np.abs(r.b - ob)) <= 1e-9 * sc
        # SPEC acceptance 1: shared samples coincide
        assert np.max(np.abs(r.a[:k + 1] - r.b[:k + 1])) <= 1e-8 * sc
        ra, _ = apply_log(r.log_a, a)
        assert np.max(np.abs(ra - r.a)) <= 1e-9 * sc


def test_geodesic_matches_reference(cuda):
    from paper_1903_12359_b200 import geodesic_to_circle
    for case in ["disk2x2", "k1disk"]:
        z = load_golden(case)
        circ, log = geodesic_to_circle(z["geo_in"])
        assert np.max(np.abs(circ - z["geo_out"])) <= 1e-9
        assert np.max(np.abs(np.abs(circ) - 1)) <= 1e-9


@pytest.mark.parametrize("case", CASES)
def test_pipeline_matches_reference(cuda, case):
    from paper_1903_12359_b200 import TriMesh, parameterize
    z = load_golden(case)
    mesh = TriMesh(z["V"], z["F"])
    cuts = z["cuts"] if len(z["cuts"]) else None
    kw = {}
    if case_pairs(case) is not None:
        kw["pairs"] = case_pairs(case)
    gp, rep = parameterize(mesh, cuts, str(z["mode"]), **kw)
    ref = z["coords"]
    got = np.asarray(gp.coords)
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref)) <= 1e-6 * _diam(ref), case
    assert rep.flips == int(z["flips"]) == 0
    rd = json.loads(str(z["distortion_json"]))
    for key in ("mean", "sd", "median", "iqr"):
        assert abs(rep.distortion["angular_abs"][key] - rd["angular_abs"][key]) <= 1e-3
    assert rep.distortion["excluded_corners"] == rd["excluded_corners"]
    assert rep.ok == bool(z["ok"])
    if rd["conformal_energy"] is not None:
        assert abs(rep.distortion["conformal_energy"] - rd["conformal_energy"]) <= 1e-6 * max(
            1.0, abs(rd["conformal_energy"]))
    assert len(rep.seam_residuals) == len(z["seam_residuals"])


def test_pipeline_determinism(cuda):
    from paper_1903_12359_b200 import TriMesh, parameterize
    z = load_golden("blocks3x3")
    mesh = TriMesh(z["V"], z["F"])
    g1, _ = parameterize(mesh, z["cuts"], "free")
    g2, _ = parameterize(mesh, z["cuts"], "free")
    assert np.array_equal(g1.coords, g2.coords)


def test_distortion_report_exact_order_stats(cuda):
    """median / IQR from the device radix select equal numpy's percentile
    on the same |d| values."""
    from paper_1903_12359_b200 import TriMesh
    from paper_1903_12359_b200.metrics import DeviceDistortion
    z = load_golden("cfg1")
    mesh = TriMesh(z["V"], z["F"])
    dd = DeviceDistortion(z["V"], z["F"], z["coords"], "free")
    d = dd.d.cpu().numpy()
    v = dd.valid.cpu().numpy().astype(bool)
    a = np.abs(d[v])
    q25, q50, q75 = np.percentile(a, [25, 50, 75])
    assert dd.stats("angular")["median"] == q50
    assert dd.stats("angular")["iqr"] == q75 - q25
    rd = json.loads(str(z["distortion_json"]))
    assert abs(dd.stats("angular")["mean"] - rd["angular_abs"]["mean"]) < 1e-12
    assert dd.hist == rd["angular_histogram"]["counts"]


def test_weld_error_propagates(cuda):
    from paper_1903_12359_b200 import WeldError, partial_weld
    a = np.array([0, 1, 1 + 1j, 1j], dtype=complex)
    with pytest.raises(WeldError, match="zip points 0 and 1 coincide"):
        partial_weld(np.array([0, 0, 1 + 1j, 1j]), a, 2)
    with pytest.raises(WeldError, match="out of range"):
        partial_weld(a, a, 7)


def test_two_level_falls_back_to_jacobi(cuda, monkeypatch):
    """A slot the two-level PCG does not finish within its cap is re-solved
    with Jacobi-PCG on the device; the result still matches the reference."""
    from paper_1903_12359_b200 import TriMesh, parameterize
    monkeypatch.setenv("PGCP_SOLVER", "pcg")
    monkeypatch.setenv("PGCP_PCG_COARSE_MAXIT", "5")
    z = load_golden("blocks3x3")
    gp, rep = parameterize(TriMesh(z["V"], z["F"]), z["cuts"], str(z["mode"]))
    ref = z["coords"]
    assert np.max(np.abs(np.asarray(gp.coords) - ref)) <= 1e-6 * _diam(ref)
    assert max(rep.solver["flatten_iters"]) > 5


@pytest.mark.parametrize("every", ["1", "3", "64"])
def test_streamed_replay_equals_serial_replay(cuda, monkeypatch, every):
    """The streamed weld replay runs concurrently with phase 1 and applies
    each record once its counter covers it. It must give the serial replay's
    result bit for bit, whatever the counter publishing interval."""
    from paper_1903_12359_b200 import TriMesh, parameterize
    z = load_golden("qtree4x4")
    mesh = TriMesh(z["V"], z["F"])
    kw = {"pairs": case_pairs("qtree4x4")}
    monkeypatch.setenv("PGCP_WELD_STREAM", "0")
    g0, r0 = parameterize(mesh, z["cuts"], str(z["mode"]), **kw)
    monkeypatch.setenv("PGCP_WELD_STREAM", "1")
    monkeypatch.setenv("PGCP_WELD_PROG_EVERY", every)
    g1, r1 = parameterize(mesh, z["cuts"], str(z["mode"]), **kw)
    assert np.array_equal(g0.coords, g1.coords)
    assert r0.seam_residuals == r1.seam_residuals


def test_streamed_replay_failed_step(cuda, monkeypatch):
    """A weld step that fails in phase 1 publishes its final counter; the
    streamed replay leaves its points alone and the error surfaces as in
    the serial replay."""
    from paper_1903_12359_b200 import WeldError, partial_weld
    a = np.array([0, 1, 1 + 1j, 1j], dtype=complex)
    for mode in ("0", "1"):
        monkeypatch.setenv("PGCP_WELD_STREAM", mode)
        with pytest.raises(WeldError, match="zip points 0 and 1 coincide"):
            partial_weld(np.array([0, 0, 1 + 1j, 1j]), a, 2)


@pytest.mark.parametrize("env", [{"PGCP_PCG_COARSE": "0"}, {"PGCP_COARSE_FP64": "1"}, {"PGCP_PCG2_NT": "256"},
                                 {"PGCP_PCG_GMAX": "4"}, {"PGCP_PCG_ORDER": "rev"}, {"PGCP_PCG_ORDER": "prev"},
                                 {"PGCP_PCG_X0": "0"}, {"PGCP_OVERLAP_HPREP": "0"}])
def test_solver_switches_match_reference(cuda, monkeypatch, env):
    """Every A/B switch of the PCG solver (PGCP_SOLVER=pcg): plain Jacobi-PCG,
    fp64 E^-1, 256-thread CTAs, a coarser coarse grid, both launch orders,
    the start from zero, the non-overlapped harmonic preparation -- each
    must still give the reference's UV."""
    from paper_1903_12359_b200 import TriMesh, parameterize
    monkeypatch.setenv("PGCP_SOLVER", "pcg")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for case in ("qtree4x4", "disk2x2"):
        z = load_golden(case)
        kw = {"pairs": case_pairs(case)} if case_pairs(case) is not None else {}
        gp, rep = parameterize(TriMesh(z["V"], z["F"]), z["cuts"], str(z["mode"]), **kw)
        ref = z["coords"]
        assert np.max(np.abs(np.asarray(gp.coords) - ref)) <= 1e-6 * _diam(ref), (case, env)
        assert rep.flips == 0


@pytest.mark.parametrize("case", ["qtree4x4", "cfg1", "sphere4", "disk2x2", "tree4x4"])
def test_wave_weld_equals_barrier_weld(cuda, monkeypatch, case):
    """The wavefront phase 1 (k_phase1w, default) applies the same records in
    the same order as the per-record-barrier kernel (PGCP_WELD_WAVE=0): the
    welded map is bit-identical, and so are the seam residuals."""
    from paper_1903_12359_b200 import TriMesh, parameterize
    z = load_golden(case)
    mesh = TriMesh(z["V"], z["F"])
    kw = {"pairs": case_pairs(case)} if case_pairs(case) is not None else {}
    cuts = z["cuts"] if len(z["cuts"]) else None
    monkeypatch.setenv("PGCP_WELD_WAVE", "0")
    g0, r0 = parameterize(mesh, cuts, str(z["mode"]), **kw)
    monkeypatch.setenv("PGCP_WELD_WAVE", "1")
    g1, r1 = parameterize(mesh, cuts, str(z["mode"]), **kw)
    assert np.array_equal(np.asarray(g0.coords), np.asarray(g1.coords))
    assert r0.seam_residuals == r1.seam_residuals


def test_prepared_schedule_equals_single_call(cuda, monkeypatch):
    """pgcp_weld_schedule_prepare + _execute (the pipeline's default: prepared
    on the planning thread during the flatten) is the same weld as the single
    pgcp_weld_schedule_run call, bit for bit, and a prepared schedule refuses a
    second run."""
    from paper_1903_12359_b200 import TriMesh, parameterize
    from paper_1903_12359_b200.welding import PreparedSchedule
    z = load_golden("qtree4x4")
    mesh = TriMesh(z["V"], z["F"])
    kw = {"pairs": case_pairs("qtree4x4")}
    monkeypatch.setenv("PGCP_WELD_PREPARE", "0")
    g0, r0 = parameterize(mesh, z["cuts"], str(z["mode"]), **kw)
    monkeypatch.setenv("PGCP_WELD_PREPARE", "1")
    g1, r1 = parameterize(mesh, z["cuts"], str(z["mode"]), **kw)
    assert np.array_equal(np.asarray(g0.coords), np.asarray(g1.coords))
    assert r0.seam_residuals == r1.seam_residuals
    # an unused handle is released without a run
    info = np.array([[2, 0, 3, 3, 0, 1]], dtype=np.int32)
    ps = PreparedSchedule(info, np.arange(6, dtype=np.int32), np.array([0, 0], dtype=np.int64),
                          np.zeros((0, 2), dtype=np.int32))
    ps.close()
    ps.close()


def test_wave_weld_errors(cuda, monkeypatch):
    """Weld failures inside the wavefront loops surface as the same
    WeldError as with the barrier kernel, on every weld size."""
    from paper_1903_12359_b200 import WeldError, partial_weld
    z = load_golden("weld_corpus")
    a, b, k = unpack(z, "a")[0], unpack(z, "b")[0], int(z["k"][0])
    bad = a.copy()
    bad[3] = bad[2]  # two zip points coincide -> the Open chain fails
    msgs = []
    for mode in ("0", "1"):
        monkeypatch.setenv("PGCP_WELD_WAVE", mode)
        with pytest.raises(WeldError) as ei:
            partial_weld(bad, b, k)
        msgs.append(str(ei.value))
    assert msgs[0] == msgs[1]
