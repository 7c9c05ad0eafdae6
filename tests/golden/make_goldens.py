"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_goldens.py

Every number stored here comes from the reference package `pgcp`
(`/root/reference/pkg/src/pgcp`). Stage-wise intermediates are captured by
wrapping the reference's own batch seam `pipeline._run_tasks`
(`pipeline.py:105-109`) and its weld entry points as the pipeline calls them
(`pipeline.py:184-204`), so nothing is re-derived outside the reference.
Inputs are the repo's seeded generators (`paper_1903_12359_b200.generators`).
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import pgcp  # noqa: E402  (the reference)
from pgcp import pipeline as ref_pipeline  # noqa: E402
from pgcp import shapes as ref_shapes  # noqa: E402
from scipy import sparse  # noqa: E402

from paper_1903_12359_b200 import generators as gen  # noqa: E402


def pack(out, name, arrays, dtype=None):
    arrays = [np.asarray(a) if dtype is None else np.asarray(a, dtype=dtype) for a in arrays]
    off = np.zeros(len(arrays) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(a) for a in arrays])
    out[name + "_off"] = off
    out[name] = np.concatenate(arrays) if arrays else np.zeros(0)


def pack_csr(out, name, mats, values=True):
    pack(out, name + "_indptr", [m.indptr for m in mats], np.int32)
    pack(out, name + "_indices", [m.indices for m in mats], np.int32)
    if values:
        pack(out, name + "_data", [m.data for m in mats], np.float64)


def capture_run(V, F, cuts, mode, schedule_pairs=None, workers=1):
    """Run pgcp.parameterize and capture every stage's inputs/outputs."""
    cap = {"tasks": [], "welds": [], "geo": None}
    orig_run = ref_pipeline._run_tasks
    orig_pw = ref_pipeline.partial_weld
    orig_cw = ref_pipeline.closed_weld
    orig_geo = ref_pipeline.geodesic_to_circle
    orig_plan = ref_pipeline.plan_weld_schedule

    def run_tasks(task, argslist, workers):
        res = orig_run(task, argslist, workers)
        cap["tasks"].append((task.__name__, argslist, res))
        return res

    def pw(a, b, k, hard_tol=1e-6):
        r = orig_pw(a, b, k, hard_tol=hard_tol)
        cap["welds"].append(("partial", np.array(a), np.array(b), k, r))
        return r

    def cw(a, b, hard_tol=1e-6):
        r = orig_cw(a, b, hard_tol=hard_tol)
        cap["welds"].append(("closed", np.array(a), np.array(b), len(a) - 1, r))
        return r

    def geo(points, interior=None):
        r = orig_geo(points, interior)
        cap["geo"] = (np.array(points), r[0])
        return r

    def plan(part, mode="free"):
        if schedule_pairs is None:
            steps = orig_plan(part, mode)
        else:
            steps = pairs_plan(part, schedule_pairs)
        cap["steps"] = steps
        return steps

    ref_pipeline._run_tasks = run_tasks
    ref_pipeline.partial_weld = pw
    ref_pipeline.closed_weld = cw
    ref_pipeline.geodesic_to_circle = geo
    ref_pipeline.plan_weld_schedule = plan
    try:
        mesh = pgcp.TriMesh(V, F)
        gp, rep = pgcp.parameterize(mesh, cuts, mode, workers=workers)
    finally:
        ref_pipeline._run_tasks = orig_run
        ref_pipeline.partial_weld = orig_pw
        ref_pipeline.closed_weld = orig_cw
        ref_pipeline.geodesic_to_circle = orig_geo
        ref_pipeline.plan_weld_schedule = orig_plan
    return mesh, gp, rep, cap


def pairs_plan(part, pairs):
    """WeldSteps for an explicit merge order, built from the reference's own
    planner primitives (`partition._cyclic_runs`, `_rotate_to`, `WeldStep`)."""
    from pgcp import partition as P
    cycles = {i: list(map(int, c)) for i, c in enumerate(part.boundary_cycles)}
    steps = []
    for ca, cb in pairs:
        runs = P._cyclic_runs(cycles[ca], cycles[cb])
        chain = min(runs, key=lambda ch: (-len(ch), ch[0]))
        a_cycle = P._rotate_to(cycles[ca], chain[0])
        b_cycle = P._rotate_to(list(reversed(cycles[cb])), chain[0])
        k = len(chain) - 1
        merged = [chain[-1]] + a_cycle[k + 1:] + [chain[0]] + list(reversed(b_cycle[k + 1:]))
        steps.append(P.WeldStep(ca, cb, np.array(a_cycle), np.array(b_cycle), k, False,
                                np.array(merged)))
        del cycles[cb]
        cycles[ca] = merged
    return steps


def stagewise_systems(sub_meshes, pins_list, g_list):
    """Reference-built L, C_ff and L_II for each submesh, via the reference's
    functions and the exact expressions of `flatten.py:157-166` /
    `assemble.py:34-41`."""
    Ls, Cffs, rhs_f, Liis, rhs_h = [], [], [], [], []
    for sub, pins, g in zip(sub_meshes, pins_list, g_list):
        n = sub.n_vertices
        loops = pgcp.boundary_loops(sub)
        L = pgcp.cotangent_laplacian(sub)
        M = pgcp.area_matrix(sub, loops)
        C = sparse.block_diag([L, L], format="csr") - 2.0 * M
        p0, p1 = pins
        fixed = np.array([p0, p1, p0 + n, p1 + n])
        free = np.setdiff1d(np.arange(2 * n), fixed)
        Cff = C[free][:, free]
        rf = -C[free][:, fixed] @ np.array([0.0, 1.0, 0.0, 0.0])
        loop = loops[0]
        interior = np.setdiff1d(np.arange(n), loop)
        Lii = L[interior][:, interior]
        rh = -(L[interior][:, loop] @ g) if g is not None else np.zeros(len(interior), complex)
        Ls.append(L)
        Cffs.append(Cff.tocsr())
        rhs_f.append(rf)
        Liis.append(Lii.tocsr())
        rhs_h.append(rh)
    return Ls, Cffs, rhs_f, Liis, rhs_h


def pipeline_case(name, V, F, cuts, mode, schedule_pairs=None, stagewise=True):
    out = {"V": V, "F": np.asarray(F, dtype=np.int32),
           "cuts": np.zeros((0, 2), np.int64) if cuts is None else np.asarray(cuts, np.int64),
           "mode": np.array(mode)}
    mesh, gp, rep, cap = capture_run(V, F, cuts, mode, schedule_pairs)
    if cuts is None or len(cuts) == 0:
        subs = [mesh]
        vmaps = [np.arange(mesh.n_vertices)]
        fa = np.zeros(mesh.n_faces, np.int64)
        cycles = [pgcp.boundary_loops(mesh)[0]]
    else:
        part = pgcp.partition_mesh(mesh, cuts)
        subs, vmaps, fa, cycles = part.submeshes, part.vertex_maps, part.face_assignment, part.boundary_cycles
    out["face_assignment"] = fa
    pack(out, "vertex_maps", vmaps, np.int64)
    pack(out, "cycles", cycles, np.int64)
    pack(out, "loops", [pgcp.boundary_loops(s)[0] for s in subs], np.int64)
    steps = cap.get("steps", [])
    out["step_meta"] = np.array([[s.comp_a, s.comp_b, s.k, int(s.closed)] for s in steps],
                                dtype=np.int64).reshape(-1, 4)
    pack(out, "step_a", [s.a_cycle for s in steps], np.int64)
    pack(out, "step_b", [s.b_cycle for s in steps], np.int64)
    pack(out, "step_merged", [s.merged_cycle for s in steps], np.int64)
    tasks = {t[0]: t for t in cap["tasks"]}
    flat = tasks["_dncp_task"][2]
    pack(out, "flat", flat, np.complex128)
    pins = [pgcp.flatten.default_pins(pgcp.boundary_loops(s)[0], s.vertices) for s in subs]
    out["pins"] = np.array(pins, dtype=np.int64).reshape(-1, 2)
    g_list = [None] * len(subs)
    if "_harmonic_task" in tasks:
        hargs = tasks["_harmonic_task"][1]
        g_list = [a[3] for a in hargs]
        pack(out, "harm_g", g_list, np.complex128)
        pack(out, "harm", [r[0] for r in tasks["_harmonic_task"][2]], np.complex128)
        out["flips_before"] = np.array([r[1]["flips_before"] for r in tasks["_harmonic_task"][2]])
    # welds: inputs and outputs of every partial/closed weld as the pipeline called it
    pack(out, "weld_in_a", [w[1] for w in cap["welds"]], np.complex128)
    pack(out, "weld_in_b", [w[2] for w in cap["welds"]], np.complex128)
    pack(out, "weld_out_a", [w[4].a for w in cap["welds"]], np.complex128)
    pack(out, "weld_out_b", [w[4].b for w in cap["welds"]], np.complex128)
    out["weld_k"] = np.array([w[3] for w in cap["welds"]], dtype=np.int64)
    out["weld_closed"] = np.array([w[0] == "closed" for w in cap["welds"]])
    out["weld_seam"] = np.array([w[4].seam_error for w in cap["welds"]])
    if cap["geo"] is not None:
        out["geo_in"], out["geo_out"] = cap["geo"]
    if stagewise:
        Ls, Cffs, rf, Liis, rh = stagewise_systems(subs, pins, g_list)
        pack_csr(out, "L", Ls)
        pack_csr(out, "Cff", Cffs, values=False)
        pack(out, "rhs_f", rf, np.float64)
        pack_csr(out, "Lii", Liis, values=False)
        pack(out, "rhs_h", rh, np.complex128)
    out["coords"] = np.asarray(gp.coords)
    out["repairs_json"] = np.array(json.dumps(rep.repairs))
    out["flips"] = np.array(rep.flips)
    out["seam_residuals"] = np.array(rep.seam_residuals, dtype=np.float64)
    out["distortion_json"] = np.array(json.dumps(rep.distortion))
    out["ok"] = np.array(rep.ok)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {os.path.getsize(path) / 1e3:.0f} KB  mode={mode} K={len(subs)} "
          f"flips={rep.flips} mean|d|={rep.distortion['angular_abs']['mean']:.6f}")


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def cfg2_qtree_case(stride=61, workers=None):
    """The benchmarked run itself: cfg 2 (1024^2 height field, 8x8 blocks,
    seed 0) welded in the quadtree order, free mode, run by the reference
    `pgcp.parameterize` (`pipeline.py:119-271`) with `workers` processes.

    The full run is ~1M vertices, so the fixture keeps, exactly as the
    reference produced them:
      * integer outputs: face labels (uint8), boundary cycles and local loops
        (full), per-step (comp_a, comp_b, k) and sha256 of every step's
        a/b/merged cycle;
      * the flatten of every subdomain on its whole boundary loop plus every
        `stride`-th local vertex; the welded Dirichlet values g of every
        subdomain (full; the product of the whole weld chain) and the
        harmonic solution on every `stride`-th local vertex;
      * the inputs and outputs of the largest weld of each of the 6 levels
        (k up to 1024) and every weld's seam error;
      * the final UV on every `stride`-th parent vertex, flips, seam
        residuals and the full distortion report;
      * the reference's own stage timings on this host (`report.timings`).
    """
    import time as _time
    workers = workers or os.cpu_count() or 1
    V, F, cuts = gen.cfg2(0)
    pairs = gen.quadtree_schedule_order(8, 8)
    t0 = _time.perf_counter()
    mesh, gp, rep, cap = capture_run(V, F, cuts, "free", schedule_pairs=pairs, workers=workers)
    wall = _time.perf_counter() - t0
    part = pgcp.partition_mesh(mesh, cuts)
    out = {"mode": np.array("free"), "stride": np.array(stride),
           "V_sha": np.array(_sha(np.asarray(V, np.float64))),
           "F_sha": np.array(_sha(np.asarray(F, np.int32))),
           "cuts_sha": np.array(_sha(np.asarray(cuts, np.int64))),
           "face_assignment": np.asarray(part.face_assignment, np.uint8),
           "vertex_maps_sha": np.array(_sha(np.concatenate(part.vertex_maps).astype(np.int64))),
           "sub_n": np.array([m.n_vertices for m in part.submeshes], np.int64)}
    pack(out, "cycles", part.boundary_cycles, np.int64)
    loops = [pgcp.boundary_loops(s)[0] for s in part.submeshes]
    pack(out, "loops", loops, np.int64)
    steps = cap["steps"]
    out["step_meta"] = np.array([[s.comp_a, s.comp_b, s.k, int(s.closed)] for s in steps], np.int64)
    out["step_sha"] = np.array([[_sha(np.asarray(s.a_cycle, np.int64)), _sha(np.asarray(s.b_cycle, np.int64)),
                                 _sha(np.asarray(s.merged_cycle, np.int64))] for s in steps])
    # level of each weld: 1 + the deeper of the two components' last merges
    depth, lev = {}, []
    for s in steps:
        lv = 1 + max(depth.get(s.comp_a, 0), depth.get(s.comp_b, 0))
        depth[s.comp_a] = lv
        lev.append(lv)
    out["step_level"] = np.array(lev, np.int64)
    tasks = {t[0]: t for t in cap["tasks"]}
    flat = tasks["_dncp_task"][2]
    samp = [np.arange(0, len(z), stride) for z in flat]
    pack(out, "flat_loop", [z[lp] for z, lp in zip(flat, loops)], np.complex128)
    pack(out, "flat_samp", [z[s] for z, s in zip(flat, samp)], np.complex128)
    hres = tasks["_harmonic_task"][2]
    pack(out, "harm_g", [a[3] for a in tasks["_harmonic_task"][1]], np.complex128)
    pack(out, "harm_samp", [r[0][s] for r, s in zip(hres, samp)], np.complex128)
    out["flips_before"] = np.array([r[1]["flips_before"] for r in hres], np.int64)
    welds = cap["welds"]
    out["weld_k"] = np.array([w[3] for w in welds], np.int64)
    out["weld_seam"] = np.array([w[4].seam_error for w in welds])
    big = []
    for lv in sorted(set(lev)):
        idx = [i for i in range(len(welds)) if lev[i] == lv]
        big.append(max(idx, key=lambda i: (welds[i][3], -i)))
    out["big_weld"] = np.array(big, np.int64)
    pack(out, "big_in_a", [welds[i][1] for i in big], np.complex128)
    pack(out, "big_in_b", [welds[i][2] for i in big], np.complex128)
    pack(out, "big_out_a", [welds[i][4].a for i in big], np.complex128)
    pack(out, "big_out_b", [welds[i][4].b for i in big], np.complex128)
    coords = np.asarray(gp.coords)
    out["coords_samp"] = coords[::stride]
    cen = coords.mean()
    out["coords_diam"] = np.array(2 * np.max(np.abs(coords - cen)))
    out["flips"] = np.array(rep.flips)
    out["seam_residuals"] = np.array(rep.seam_residuals, np.float64)
    out["distortion_json"] = np.array(json.dumps(rep.distortion))
    out["repairs_json"] = np.array(json.dumps(rep.repairs))
    out["ok"] = np.array(rep.ok)
    tm = dict(rep.timings)
    tm["wall"] = wall
    tm["workers"] = workers
    out["ref_timings_json"] = np.array(json.dumps(tm))
    path = os.path.join(HERE, "cfg2_qtree.npz")
    np.savez_compressed(path, **out)
    print(f"cfg2_qtree: {os.path.getsize(path) / 1e6:.2f} MB flips={rep.flips} "
          f"mean|d|={rep.distortion['angular_abs']['mean']:.6f} timings={tm}")


def known_answers():
    """SPEC.md worked examples evaluated by the reference."""
    out = {}
    s3 = np.sqrt(3.0)
    eq = pgcp.TriMesh(np.array([[0, 0, 0], [1, 0, 0], [0.5, s3 / 2, 0]], float),
                      np.array([[0, 1, 2]]))
    out["equilateral_L"] = pgcp.cotangent_laplacian(eq).toarray()
    ri = pgcp.TriMesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), np.array([[0, 1, 2]]))
    Lri = pgcp.cotangent_laplacian(ri)
    out["right_L_dense"] = Lri.toarray()
    out["right_L_nnz"] = np.array(Lri.nnz)
    sq = pgcp.TriMesh(np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], float),
                      np.array([[0, 1, 2], [0, 2, 3]]))
    M = pgcp.area_matrix(sq)
    xy = np.concatenate([sq.vertices[:, 0], sq.vertices[:, 1]])
    out["unit_square_area"] = np.array(xy @ (M @ xy))
    out["mobius_to_unit_1pi"] = pgcp.mobius_apply(pgcp.mobius_to_unit(1 + 1j), 1 + 1j)
    out["pair_align_identity"] = np.array(pgcp.mobius_pair_align(1j, -1j), dtype=complex)
    out["opening_1"] = pgcp.opening_map(1.0)
    out["opening_0"] = pgcp.opening_map(0.0)
    out["closing_pm_i"] = pgcp.closing_map(np.array([1j, -1j]))
    out["stereo_inv"] = pgcp.stereographic_inverse(np.array([0, pgcp.INF, 1.0]))
    v = np.array([1.0, 2.0, 3.0, 4.0])
    st = pgcp.summarize(v)
    out["summ_1234"] = np.array([st["mean"], st["sd"], st["median"], st["iqr"]])
    out["iqr_1to8"] = np.array(pgcp.summarize(np.arange(1.0, 9.0))["iqr"])
    # stretch x2 of the unit right triangle: corner distortions
    tri = pgcp.TriMesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), np.array([[0, 1, 2]]))
    d, valid = pgcp.angular_distortion(tri, np.array([0, 2, 1j]))
    out["stretch_distortion"] = d
    np.savez_compressed(os.path.join(HERE, "known_answers.npz"), **out)
    print("known_answers written")


def qc_cases():
    """Direct `qc_correct` calls of the reference (assemble.py:174-217):
    (0) a grid embedding with one interior vertex dragged across a
    neighbour (clears), (1)-(2) the folded harmonic maps of the repair
    pipeline cases' submeshes as `_harmonic_task` hands them to qc_correct
    (pipeline.py:90-97), (3) a degenerate embedded triangle (SolveError)."""
    from pgcp.assemble import face_layout, qc_correct
    out = {"count": 0}

    def put(i, V, F, z, fixed, max_iter=5):
        sub = pgcp.TriMesh(V, F, check=False)
        lay = face_layout(sub)
        try:
            zo, rep = qc_correct(lay, F, z, fixed, max_iter=max_iter)
            res = np.array([rep.iterations, int(rep.cleared), rep.initial_flips])
            rem = np.asarray(rep.remaining_faces, np.int64)
        except pgcp.SolveError as e:
            zo, res, rem = np.zeros(0, complex), np.array([-1, 0, 0]), np.zeros(0, np.int64)
            out[f"err{i}"] = np.array(str(e))
        out[f"V{i}"], out[f"F{i}"], out[f"z{i}"] = V, np.asarray(F, np.int32), z
        out[f"fixed{i}"], out[f"layout{i}"], out[f"max_iter{i}"] = np.asarray(fixed, np.int64), lay, np.array(max_iter)
        out[f"out{i}"], out[f"res{i}"], out[f"remaining{i}"] = zo, res, rem
        out["count"] = i + 1

    Vg, Fg = gen.flat_grid_arrays(12)
    Vg[:, 2] = 0.05 * np.sin(3 * Vg[:, 0]) * np.cos(2 * Vg[:, 1])
    z = Vg[:, 0] + 1j * Vg[:, 1]
    z[13 * 6 + 6] += (1.3 + 0.2j) / 12
    put(0, Vg, Fg, z, pgcp.boundary_loops(pgcp.TriMesh(Vg, Fg))[0])
    for i, (strips, mode, seed) in enumerate([(0, "disk", 1), (3, "free", 1)], start=1):
        V, F, cuts = gen.jittered_grid_case(25, seed=seed, strips=strips)
        _, _, _, cap = capture_run(V, F, cuts, mode)
        hargs = [t for t in cap["tasks"] if t[0] == "_harmonic_task"][0][1]
        j = 0 if strips == 0 else 2
        sv, sf, bd, bv = hargs[j][:4]
        z0 = pgcp.harmonic_solve(pgcp.TriMesh(sv, sf, check=False), bd, bv)
        put(i, sv, sf, z0, bd)
    zd = Vg[:, 0] + 1j * Vg[:, 1]
    v00, v10, v11 = 13 * 6 + 6, 13 * 6 + 7, 13 * 7 + 7  # face [v00, v10, v11] made collinear
    zd[v11] = zd[v10] + 0.5 * (zd[v10] - zd[v00])
    put(3, Vg, Fg, zd, pgcp.boundary_loops(pgcp.TriMesh(Vg, Fg))[0])
    np.savez_compressed(os.path.join(HERE, "qc_direct.npz"), **out)
    print("qc_direct:", [tuple(out[f"res{i}"]) for i in range(out["count"])])


def intermediate_cases():
    """`intermediate_form` (welding.py:578-602) of the weld corpus boundaries
    on both branches, plus its error paths."""
    w = np.load(os.path.join(HERE, "weld_corpus.npz"))
    a_off, b_off = w["a_off"], w["b_off"]
    out = {"vals": [], "sides": [], "nrec": [], "k": [], "branch": [], "pts": []}
    for i in range(len(w["k"])):
        for pts, br in ((w["a"][a_off[i]:a_off[i + 1]], pgcp.welding.UPPER),
                        (w["b"][b_off[i]:b_off[i + 1]], pgcp.welding.LOWER)):
            k = int(w["k"][i])
            r = pgcp.intermediate_form(pts, k, br)
            out["pts"].append(pts)
            out["vals"].append(r.values)
            out["sides"].append(r.sides)
            out["nrec"].append(len(r.log))
            out["k"].append(k)
            out["branch"].append(br)
    res = {}
    pack(res, "pts", out["pts"], np.complex128)
    pack(res, "vals", out["vals"], np.complex128)
    pack(res, "sides", out["sides"], np.int8)
    for key in ("nrec", "k", "branch"):
        res[key] = np.array(out[key], dtype=np.int64)
    errs = []
    for pts, k in (([0, 1, 2], 0), ([0, 1], 2), ([1, 1, 2, 3], 2), ([0, 1, 1j, 2], 3)):
        try:
            pgcp.intermediate_form(np.asarray(pts, np.complex128), k)
            errs.append("")
        except pgcp.WeldError as e:
            errs.append(str(e))
    res["errors"] = np.array(errs)
    np.savez_compressed(os.path.join(HERE, "intermediate.npz"), **res)
    print("intermediate:", len(out["k"]), "forms; errors", errs)


def weld_corpus(seed=0, count=12):
    """Random Jordan polygon pairs welded by the reference `partial_weld`
    (SPEC acceptance criterion 1 shape): two star-shaped regions sharing an
    arc of a common chord-split disk."""
    rng = np.random.default_rng(seed)
    out = {"a": [], "b": [], "k": [], "oa": [], "ob": [], "seam": []}
    made = 0
    while made < count:
        m = int(rng.integers(20, 120))
        k = int(rng.integers(2, m // 2))
        # shared arc along the real axis from 1 to -1 (k+1 samples), region a
        # above (boundary ccw: arc then upper curve back), region b below
        # shared arc along the real axis from -1 to 1 (k+1 samples); region a
        # above it (boundary ccw: arc, then the upper curve back to -1),
        # region b below it (arc in the same order, region on the right)
        x = np.sort(rng.uniform(-0.95, 0.95, k - 1))
        arc = np.concatenate([[-1.0], x, [1.0]]) + 0j
        tu = np.sort(rng.uniform(0.05, np.pi - 0.05, m - k))
        upper = (1.0 + 0.3 * rng.uniform(-1, 1, len(tu))) * np.exp(1j * tu)
        tl = np.sort(rng.uniform(np.pi + 0.05, 2 * np.pi - 0.05, m - k))[::-1]
        lower = (1.0 + 0.3 * rng.uniform(-1, 1, len(tl))) * np.exp(1j * tl)
        a = np.concatenate([arc, upper])
        b = np.concatenate([arc, lower])
        try:
            r = pgcp.partial_weld(a, b, k)
        except pgcp.WeldError:
            continue
        out["a"].append(a)
        out["b"].append(b)
        out["k"].append(k)
        out["oa"].append(r.a)
        out["ob"].append(r.b)
        out["seam"].append(r.seam_error)
        made += 1
    res = {}
    pack(res, "a", out["a"], np.complex128)
    pack(res, "b", out["b"], np.complex128)
    pack(res, "oa", out["oa"], np.complex128)
    pack(res, "ob", out["ob"], np.complex128)
    res["k"] = np.array(out["k"], dtype=np.int64)
    res["seam"] = np.array(out["seam"])
    np.savez_compressed(os.path.join(HERE, "weld_corpus.npz"), **res)
    print(f"weld_corpus: {count} welds")


def _cases():
    def c_cfg1():
        V, F, cuts = gen.cfg1(seed=0)
        pipeline_case("cfg1", V, F, cuts, "free")

    def c_strips4():
        V, F, cuts = gen.height_field_case(33, 4, layout="strips", seed=3)
        pipeline_case("strips4", V, F, cuts, "free")

    def c_blocks3x3():
        V, F, cuts = gen.height_field_case(31, 3, seed=5)
        pipeline_case("blocks3x3", V, F, cuts, "free")

    def c_disk2x2():
        V, F, cuts = gen.height_field_case(30, 2, seed=7)
        pipeline_case("disk2x2", V, F, cuts, "disk")

    def c_k1():
        V, F = gen.height_field_grid(25, seed=11)
        pipeline_case("k1free", V, F, None, "free")
        pipeline_case("k1disk", V, F, None, "disk")

    def c_flat2x2():
        Vf, Ff = gen.flat_grid_arrays(20)
        cf = gen.cuts_from_face_labels(Ff, gen.block_face_labels(21, 2))
        pipeline_case("flat2x2", Vf, Ff, cf, "free")

    def c_sphere():
        sph = ref_shapes.icosphere(3)
        lab = ref_shapes.hemisphere_labels(sph)
        pipeline_case("sphere2", np.array(sph.vertices), np.array(sph.faces),
                      ref_shapes.cuts_from_face_labels(sph, lab), "sphere")
        lab = ref_shapes.azimuth_labels(sph, 4)
        pipeline_case("sphere4", np.array(sph.vertices), np.array(sph.faces),
                      ref_shapes.cuts_from_face_labels(sph, lab), "sphere")

    def c_tree4x4():
        # balanced rows->strips->tree schedule on 4x4 blocks (documented deviation)
        V, F, cuts = gen.height_field_case(41, 4, seed=2)
        pipeline_case("tree4x4", V, F, cuts, "free",
                      schedule_pairs=gen.row_tree_schedule_order(4, 4))

    def c_ptree4x4():
        # fully pairwise tree (blocks -> pairs -> rows -> strips)
        V, F, cuts = gen.height_field_case(41, 4, seed=2)
        pipeline_case("ptree4x4", V, F, cuts, "free",
                      schedule_pairs=gen.pairwise_tree_schedule_order(4, 4))

    def c_qtree4x4():
        # quadtree order (alternating horizontal / vertical pairwise merges), the bench's order
        V, F, cuts = gen.height_field_case(41, 4, seed=2)
        pipeline_case("qtree4x4", V, F, cuts, "free",
                      schedule_pairs=gen.quadtree_schedule_order(4, 4))

    def c_repair():
        # jittered grids whose harmonic maps fold: the per-submesh repair of pipeline.py:88-102 runs
        for name, strips, mode, seed in [("repair_k1disk", 0, "disk", 1), ("repair_strips3", 3, "free", 1),
                                         ("repair_disk2", 2, "disk", 1)]:
            V, F, cuts = gen.jittered_grid_case(25, seed=seed, strips=strips)
            pipeline_case(name, V, F, cuts, mode)

    return {"known_answers": known_answers, "weld_corpus": weld_corpus, "intermediate": intermediate_cases,
            "qc": qc_cases, "repair": c_repair,
            "cfg1": c_cfg1, "strips4": c_strips4,
            "blocks3x3": c_blocks3x3, "disk2x2": c_disk2x2, "k1": c_k1, "flat2x2": c_flat2x2,
            "sphere": c_sphere, "tree4x4": c_tree4x4, "ptree4x4": c_ptree4x4,
            "qtree4x4": c_qtree4x4, "cfg2_qtree": cfg2_qtree_case}


def main():
    """python make_goldens.py [case ...]  (default: every case)"""
    cases = _cases()
    names = sys.argv[1:] or [c for c in cases if c != "cfg2_qtree"]  # cfg2_qtree: ~5 min, run by name
    for n in names:
        cases[n]()


if __name__ == "__main__":
    main()
