"""Oracle: stitching, sphere projection, flip checks and distortion metrics
(restates `assemble.py:97-102,252-337` and `metrics.py:22-176`).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np

from .laplace import OracleSolveError
from .surface import boundary_loop_list


def planar_signed_areas(z, F):
    """`assemble.py:97-102`."""
    t = np.asarray(z, dtype=np.complex128)[np.asarray(F)]
    d1 = t[:, 1] - t[:, 0]
    d2 = t[:, 2] - t[:, 0]
    return 0.5 * (d1.real * d2.imag - d1.imag * d2.real)


def sphere_flip_faces(P, F):
    """`assemble.py:259-263`."""
    t = np.asarray(P)[np.asarray(F)]
    det = np.einsum("ij,ij->i", t[:, 0], np.cross(t[:, 1], t[:, 2]))
    return np.flatnonzero(det < 0)


def stereo_inverse(z):
    """Plane (+ infinity) to the unit sphere (`assemble.py:224-245`)."""
    z = np.atleast_1d(np.asarray(z, dtype=np.complex128))
    out = np.empty((len(z), 3))
    at_inf = np.isinf(z.real) | np.isinf(z.imag)
    out[at_inf] = (0.0, 0.0, 1.0)
    zf = z[~at_inf]
    big = np.abs(zf) > 1.0
    res = np.empty((len(zf), 3))
    zs = zf[~big]
    r2 = np.abs(zs) ** 2
    res[~big, 0] = 2 * zs.real / (1 + r2)
    res[~big, 1] = 2 * zs.imag / (1 + r2)
    res[~big, 2] = (r2 - 1) / (1 + r2)
    w = 1.0 / zf[big]
    w2 = np.abs(w) ** 2
    res[big, 0] = 2 * w.real / (1 + w2)
    res[big, 1] = -2 * w.imag / (1 + w2)
    res[big, 2] = (1 - w2) / (1 + w2)
    out[~at_inf] = res
    return out


class Stitched:
    def __init__(self, mode, coords, flipped, provenance, seam_max, diagnostics):
        self.mode = mode
        self.coords = coords
        self.flipped_faces = flipped
        self.provenance = provenance
        self.seam_max_dev = seam_max
        self.diagnostics = diagnostics


def stitch(n, F, vertex_maps, embeddings, mode, hard_tol=1e-6, circle_tol=1e-9):
    """Average seam copies and apply the mode's finish (`assemble.py:286-337`)."""
    acc = np.zeros(n, dtype=np.complex128)
    cnt = np.zeros(n)
    prov = np.full(n, -1, dtype=np.int64)
    spread = np.zeros(n)
    first = np.zeros(n, dtype=np.complex128)
    scale = 0.0
    for si, (vm, e) in enumerate(zip(vertex_maps, embeddings)):
        e = np.asarray(e, dtype=np.complex128)
        new = prov[vm] < 0
        prov[vm[new]] = si
        first[vm[new]] = e[new]
        spread[vm] = np.maximum(spread[vm], np.abs(e - first[vm]))
        acc[vm] += e
        cnt[vm] += 1.0
        scale = max(scale, float(np.max(np.abs(e))))
    if np.any(cnt == 0):
        raise OracleSolveError("some parent vertices received no coordinates")
    seam = float(np.max(spread))
    if scale > 0 and seam > hard_tol * scale:
        raise OracleSolveError(f"seam disagreement {seam:.3e} exceeds {hard_tol:g} x scale {scale:.3e}")
    coords = acc / cnt
    diag = {"seam_max_dev": seam, "scale": scale}
    if mode == "sphere":
        P = stereo_inverse(np.conj(coords))
        P /= np.linalg.norm(P, axis=1)[:, None]
        return Stitched(mode, P, sphere_flip_faces(P, F), prov, seam, diag)
    if mode == "disk":
        bl = boundary_loop_list(F)[0]
        dev = np.max(np.abs(np.abs(coords[bl]) - 1.0))
        if dev > circle_tol:
            raise OracleSolveError(f"disk boundary off the unit circle by {dev:.3e}")
        diag["boundary_circle_dev"] = float(dev)
    flips = np.flatnonzero(planar_signed_areas(coords, F) <= 0)
    return Stitched(mode, coords, flips, prov, seam, diag)


def _corner(u, v):
    nu = np.linalg.norm(u, axis=-1)
    nv = np.linalg.norm(v, axis=-1)
    with np.errstate(invalid="ignore", divide="ignore"):
        c = np.einsum("...i,...i->...", u, v) / (nu * nv)
    return np.arccos(np.clip(c, -1.0, 1.0)), (nu == 0) | (nv == 0)


def _angles(P, F):
    """`metrics.py:31-44`."""
    p = np.asarray(P)
    if np.iscomplexobj(p) or p.ndim == 1:
        p = np.column_stack([p.real, p.imag])
    tri = np.asarray(p, dtype=np.float64)[np.asarray(F)]
    ang = np.empty((len(tri), 3))
    bad = np.zeros((len(tri), 3), dtype=bool)
    for i in range(3):
        ang[:, i], bad[:, i] = _corner(tri[:, (i + 1) % 3] - tri[:, i],
                                       tri[:, (i + 2) % 3] - tri[:, i])
    return ang, bad


def _angles_sphere(P, F):
    """`metrics.py:47-58`."""
    tri = np.asarray(P, dtype=np.float64)[np.asarray(F)]
    ang = np.empty((len(tri), 3))
    bad = np.zeros((len(tri), 3), dtype=bool)
    for i in range(3):
        a = tri[:, i]
        b = tri[:, (i + 1) % 3]
        c = tri[:, (i + 2) % 3]
        tb = b - np.einsum("ij,ij->i", b, a)[:, None] * a
        tc = c - np.einsum("ij,ij->i", c, a)[:, None] * a
        ang[:, i], bad[:, i] = _corner(tb, tc)
    return ang, bad


def angle_distortion(V, F, coords, mode):
    """Per-corner (param - original) angle in degrees + validity
    (`metrics.py:61-75`); corner index = 3 * face + corner."""
    ref, bref = _angles(V, F)
    if mode == "sphere":
        new, bnew = _angles_sphere(coords, F)
    else:
        new, bnew = _angles(np.asarray(coords, dtype=np.complex128), F)
    return np.degrees(new - ref).ravel(), (~(bref | bnew)).ravel()


def _areas(coords, F, mode):
    if mode == "sphere":
        p = np.asarray(coords)[np.asarray(F)]
        return 0.5 * np.linalg.norm(np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), axis=1)
    z = np.asarray(coords, dtype=np.complex128)[np.asarray(F)]
    d1 = z[:, 1] - z[:, 0]
    d2 = z[:, 2] - z[:, 0]
    return 0.5 * np.abs(d1.real * d2.imag - d1.imag * d2.real)


def area_log_ratio(V, F, coords, mode):
    """`metrics.py:89-104`."""
    an = _areas(coords, F, mode)
    v = np.asarray(V)
    f = np.asarray(F)
    ar = 0.5 * np.linalg.norm(np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]]), axis=1)
    ok = an > 0
    d = np.zeros(len(ar))
    d[ok] = np.log((an / np.sum(an))[ok] / (ar / np.sum(ar))[ok])
    return d, ok


def summary_stats(values):
    """`metrics.py:114-126`."""
    v = np.asarray(values, dtype=np.float64)
    if v.size == 0:
        raise ValueError("cannot summarize an empty array")
    q25, q50, q75 = np.percentile(v, [25, 50, 75])
    return {"mean": float(np.mean(v)), "sd": float(np.std(v)),
            "median": float(q50), "iqr": float(q75 - q25)}


def histogram_abs(d, bin_width=0.1):
    """0.1-degree histogram of |d| (`metrics.py:140-149`)."""
    d = np.abs(d)
    if not d.size:
        return {"bin_width": bin_width, "start": 0.0, "counts": []}
    top = max(bin_width, float(np.max(d)))
    edges = np.arange(0.0, top + bin_width, bin_width)
    counts, _ = np.histogram(d, bins=edges)
    return {"bin_width": bin_width, "start": 0.0, "counts": counts.tolist()}


def distortion_summary(V, F, coords, mode, energy=None):
    """`distortion_report(...).to_dict()` (`metrics.py:140-176`)."""
    d, dv = angle_distortion(V, F, coords, mode)
    da, av = area_log_ratio(V, F, coords, mode)
    return {
        "angular_abs": summary_stats(np.abs(d[dv])),
        "area_abs": summary_stats(np.abs(da[av])),
        "angular_histogram": histogram_abs(d[dv]),
        "excluded_corners": int(np.sum(~dv)),
        "excluded_faces": int(np.sum(~av)),
        "conformal_energy": energy,
    }
