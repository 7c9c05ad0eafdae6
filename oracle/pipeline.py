"""Oracle: end-to-end PGCP driver (restates `pipeline.py:82-297`).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Also the CPU arm of
bench.py (`--impl reference` and the `cpu_baseline` field): the per-subdomain
solves fan out over a process pool exactly like `_run_tasks`
(`pipeline.py:105-109`).
"""

import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from .assembly import distortion_summary, stitch
from .laplace import conformal_energy, cotan_laplacian, dirichlet_extend, dncp_flatten
from .planner import greedy_schedule, pair_schedule
from .repair import isometric_layout, planar_flips, repair_folds
from .surface import single_domain, split_mesh, topology_class
from .zipper import closed_weld, geodesic_to_circle, interior_point, partial_weld, replay


def _poly_area(z):
    return 0.5 * float(np.sum(z.real * np.roll(z, -1).imag - z.imag * np.roll(z, -1).real))


def _flatten_job(args):
    V, F, loop = args
    return dncp_flatten(V, F, loop)


def _dirichlet_job(args):
    """The Dirichlet solve alone (`assemble.py:23-50`) of one submesh:
    (V, F, loop, boundary values) -> complex embedding."""
    V, F, loop, g = args
    return dirichlet_extend(V, F, loop, g)


def _harmonic_job(args):
    """`_harmonic_task` (pipeline.py:88-102): harmonic extension, flip check,
    and the quasi-conformal repair of a folded submesh. Returns (z, info)."""
    V, F, loop, g = args[:4]
    repair_iters = args[4] if len(args) > 4 else 5
    z = dirichlet_extend(V, F, loop, g)
    nf = len(planar_flips(z, F))
    info = {"flips_before": nf, "repair_iterations": 0, "cleared": nf == 0}
    if nf:
        z, it, ok, left, n0 = repair_folds(isometric_layout(V, F), F, z, loop, max_iter=repair_iters)
        info = {"flips_before": n0, "repair_iterations": it, "cleared": ok, "remaining": [int(x) for x in left]}
    return z, info


def _fan_out(fn, jobs, workers):
    if workers <= 1 or len(jobs) <= 1:
        return [fn(j) for j in jobs]
    with ProcessPoolExecutor(max_workers=min(workers, len(jobs))) as ex:
        return list(ex.map(fn, jobs))


def subdomain_solves(split, workers=1, boundary_values=None):
    """The hot path alone: DNCP flatten of every submesh, then (if
    `boundary_values` is given, one complex array per submesh in loop order)
    the harmonic solve. Returns (flat, harm)."""
    flat = _fan_out(_flatten_job, [(split.sub_V[i], split.sub_F[i], split.loops[i])
                                   for i in range(split.n_sub)], workers)
    harm = None
    if boundary_values is not None:
        harm = _fan_out(_harmonic_job, [(split.sub_V[i], split.sub_F[i], split.loops[i],
                                         boundary_values[i]) for i in range(split.n_sub)],
                        workers)
    return flat, harm


def run_parameterize(V, F, cuts=None, mode="free", workers=1, schedule="greedy",
                     pairs=None, hard_tol=1e-6, snap_tol=1e-8, keep=False):
    """`parameterize` (`pipeline.py:119-271`). `schedule` = "greedy" (the
    reference planner) or "pairs" (explicit merge order `pairs`).

    Returns a dict with coords, flips, distortion, timings, the partition,
    the steps, the flatten embeddings and the welded boundary values.
    """
    V = np.asarray(V, dtype=np.float64)
    F = np.asarray(F, dtype=np.int64)
    timings = {}
    chi, nl, cls = topology_class(len(V), F)
    if mode in ("free", "disk") and cls != "disk_type":
        raise ValueError(f"mode {mode!r} needs a disk-type mesh, got {cls}")
    if mode == "sphere" and cls != "sphere_type":
        raise ValueError(f"sphere mode needs a genus-0 closed mesh, got {cls}")
    t0 = time.perf_counter()
    if cuts is None or len(cuts) == 0:
        if mode == "sphere":
            raise ValueError("sphere mode requires a cut set (K >= 2)")
        part = single_domain(V, F)
        steps = []
    else:
        part = split_mesh(V, F, cuts)
        if schedule == "greedy":
            steps = greedy_schedule(part.boundary_cycles, part.cuts, mode)
        else:
            steps = pair_schedule(part.boundary_cycles, part.cuts, pairs, mode)
    timings["partition"] = time.perf_counter() - t0

    t0 = time.perf_counter()
    flat, _ = subdomain_solves(part, workers)
    timings["flatten"] = time.perf_counter() - t0
    out = {"partition": part, "steps": steps, "flat": flat, "timings": timings,
           "seam_residuals": []}

    if part.n_sub == 1 and mode == "free":
        embeddings = [flat[0]]
    else:
        vals = {}
        members = {}
        for i in range(part.n_sub):
            vals[i] = dict(zip(part.boundary_cycles[i].tolist(), flat[i][part.loops[i]]))
            members[i] = [i]
        exterior = []
        t0 = time.perf_counter()
        for st in steps:
            A, B = vals[st.comp_a], vals[st.comp_b]
            al = np.array([A[int(p)] for p in st.a_cycle], dtype=np.complex128)
            bl = np.array([B[int(p)] for p in st.b_cycle], dtype=np.complex128)
            res = closed_weld(al, bl, hard_tol) if st.closed else partial_weld(al, bl, st.k, hard_tol)
            sc = max(float(np.max(np.abs(res.a))), float(np.max(np.abs(res.b))))
            out["seam_residuals"].append(res.seam_error / sc if sc else 0.0)
            new = dict(zip(st.b_cycle.tolist(), res.b))
            new.update(zip(st.a_cycle.tolist(), res.a))
            for side, lg in ((A, res.log_a), (B, res.log_b)):
                rest = [p for p in side if p not in new]
                if rest:
                    z, _ = replay(lg, np.array([side[p] for p in rest]))
                    new.update(zip(rest, z))
            if st.closed:
                ext = st.comp_b if _poly_area(res.a) > 0 else st.comp_a
                exterior = list(members[ext])
            vals[st.comp_a] = new
            members[st.comp_a] += members[st.comp_b]
            del vals[st.comp_b], members[st.comp_b]
        timings["weld"] = time.perf_counter() - t0
        tracked = vals[next(iter(vals))]

        if mode == "disk":
            gc = [int(p) for p in (steps[-1].merged_cycle if steps else part.boundary_cycles[0])]
            bv = np.array([tracked[p] for p in gc], dtype=np.complex128)
            if _poly_area(bv) < 0:
                gc = [gc[0]] + gc[:0:-1]
                bv = np.array([tracked[p] for p in gc], dtype=np.complex128)
            circ, lg = geodesic_to_circle(bv)
            new = dict(zip(gc, circ))
            rest = [p for p in tracked if p not in new]
            if rest:
                z, _ = replay(lg, np.array([tracked[p] for p in rest]))
                new.update(zip(rest, z))
            tracked = new

        t0 = time.perf_counter()
        ext = set(exterior)
        center = None
        if mode == "sphere" and ext:
            sv = np.array([tracked[int(p)] for p in steps[-1].a_cycle])
            if _poly_area(sv) < 0:
                sv = sv[::-1]
            center = interior_point(sv)
        g_all = []
        for i in range(part.n_sub):
            g = np.array([tracked[int(p)] for p in part.boundary_cycles[i]], dtype=np.complex128)
            if i in ext:
                g = 1.0 / (g - center)
            g_all.append(g)
        harm = _fan_out(_harmonic_job, [(part.sub_V[i], part.sub_F[i], part.loops[i], g_all[i])
                                        for i in range(part.n_sub)], workers)
        embeddings = []
        out["flips_before"] = []
        out["repairs"] = []
        out["embeddings_local"] = []
        for i, (z, info) in enumerate(harm):
            out["flips_before"].append(info["flips_before"])
            out["repairs"].append(info)
            out["embeddings_local"].append(z)
            if i in ext:
                z = center + 1.0 / z
            embeddings.append(z)
        timings["harmonic"] = time.perf_counter() - t0
        out["welded"] = tracked
        out["harmonic_g"] = g_all
        out["center"] = center

    t0 = time.perf_counter()
    gp = stitch(len(V), F, part.vertex_maps, embeddings, mode, hard_tol=hard_tol)
    timings["stitch"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    energy = None
    if mode in ("free", "disk"):
        energy = float(sum(conformal_energy(cotan_laplacian(part.sub_V[i], part.sub_F[i]),
                                            embeddings[i], [part.loops[i]])
                           for i in range(part.n_sub)))
    out["distortion"] = distortion_summary(V, F, gp.coords, mode, energy)
    timings["metrics"] = time.perf_counter() - t0
    out["coords"] = gp.coords
    out["flips"] = int(len(gp.flipped_faces))
    out["embeddings"] = embeddings
    out["stitched"] = gp
    out["ok"] = out["flips"] == 0 and all(r <= snap_tol for r in out["seam_residuals"])
    return out


def default_workers():
    return os.cpu_count() or 1
