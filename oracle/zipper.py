"""Oracle: boundary welding by zipper maps (restates `welding.py:79-842`).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

A map log is a list of records `(kind, params)`; `_apply` dispatches on the
kind. Each kind restates one reference record class:

    "mob"   MobiusRec       welding.py:236-286   (a, b, c, d, axis, pins)
    "sqr"   SqrtRatioRec    welding.py:289-314   (z0, z1, branch)
    "open"  OpenRec         welding.py:317-384   (xi, branch)
    "close" CloseRec        welding.py:387-459   (ai, bi)
    "sq"    SquareMobiusRec welding.py:462-509   (q,)

Operand types (numpy complex128 scalars vs Python complex) follow the
reference expression by expression, because numpy and CPython use different
complex-division formulas; with identical types the oracle reproduces the
reference bit for bit (pinned by tests/test_oracle_pins.py).
"""

import numpy as np

FREE, UP, DOWN = 0, 1, -1
INF = np.complex128(complex(np.inf, 0.0))
HUGE = 1e100


class OracleWeldError(RuntimeError):
    pass


def _pts(z):
    return np.atleast_1d(np.asarray(z, dtype=np.complex128))


def _fin(z):
    return np.isfinite(z.real) & np.isfinite(z.imag)


def _isinf(z):
    z = np.asarray(z)
    return np.isinf(z.real) | np.isinf(z.imag)


def _inf1(z):
    return bool(np.isinf(np.real(z)) or np.isinf(np.imag(z)))


def _nan_guard(z, where):
    if np.isnan(z.real).any() or np.isnan(z.imag).any():
        raise OracleWeldError(f"numerical breakdown (NaN) during {where}")


def _maxabs(z):
    f = _fin(z)
    if not f.any():
        return 1.0
    s = float(np.max(np.abs(z[f])))
    return s if s > 0 else 1.0


# ---------------------------------------------------------------------------
# records


def mob(a, b, c, d, axis=False, pins=()):
    if a * d - b * c == 0:
        raise OracleWeldError("degenerate Mobius coefficients")
    return ("mob", (a, b, c, d, axis, tuple(pins)))


def _apply_mob(prm, z, s):
    a, b, c, d, axis, pins = prm
    w = np.empty_like(z)
    t = np.zeros_like(s)
    hit = np.zeros(z.shape, dtype=bool)
    for pz, pw, ps in pins:
        m = (z == pz) & ~hit
        w[m] = pw
        t[m] = ps
        hit |= m
    at_inf = _isinf(z) & ~hit
    if at_inf.any():
        w[at_inf] = a / c if c != 0 else INF
        if axis:
            t[at_inf] = s[at_inf]
        hit |= at_inf
    rest = ~hit
    if rest.any():
        zr = z[rest]
        num = a * zr + b
        den = c * zr + d
        w[rest] = np.where(den == 0, INF, num / np.where(den == 0, 1, den))
    if axis:
        tagged = (s != 0) & rest
        tf = tagged & _fin(w)
        on = 1j * w[tf].imag
        w[tf] = on
        t[tf] = np.where(on.imag > 0, UP, np.where(on.imag < 0, DOWN, s[tf]))
        ti = tagged & ~_fin(w)
        t[ti] = s[ti]
    return w, t


def _apply_sqr(prm, z, s):
    z0, z1, br = prm
    w = np.empty_like(z)
    t = np.zeros_like(s)
    hit = np.zeros(z.shape, dtype=bool)
    for pz, pw, ps in ((z0, INF, br), (z1, 0j, br), (INF, 1.0 + 0j, FREE)):
        m = (z == pz) & ~hit
        w[m] = pw
        t[m] = ps
        hit |= m
    rest = ~hit
    if rest.any():
        zr = z[rest]
        w[rest] = np.sqrt((zr - z1) / (zr - z0))
    return w, t


def _apply_open(prm, z, s):
    xi, br = prm
    xi = complex(xi)
    r2 = abs(xi) ** 2
    p = xi.real / r2
    q = xi.imag / r2
    w = np.empty_like(z)
    t = np.zeros_like(s)
    hit = z == xi
    w[hit] = 0j
    t[hit] = br
    tagged = (s != 0) & ~hit
    if tagged.any():
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            h = np.where(_isinf(z[tagged]), np.inf, z[tagged].imag)
            den = 1.0 - q * h
            h2 = np.where(den == 0, np.inf, p * h / np.where(den == 0, 1, den))
            h2 = np.where(np.isinf(h), (-p / q if q != 0 else np.inf), h2)
        vals = np.empty(h2.shape, dtype=np.complex128)
        tt = np.zeros(h2.shape, dtype=s.dtype)
        fm = np.isfinite(h2)
        vals[~fm] = INF
        tt[~fm] = s[tagged][~fm]
        sg = np.where(h2[fm] == 0, br, np.sign(h2[fm]))
        vals[fm] = sg * 1j * np.hypot(h2[fm], 1.0)
        tt[fm] = sg.astype(s.dtype)
        w[tagged] = vals
        t[tagged] = tt
        hit |= tagged
    rest = ~hit
    if rest.any():
        zr = z[rest]
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            zinf = _isinf(zr)
            den = 1.0 + q * 1j * zr
            Lz = np.where(den == 0, INF, p * zr / np.where(den == 0, 1, den))
            Lz = np.where(zinf, -(p / q) * 1j, Lz) if q != 0 else np.where(zinf, INF, Lz)
        lf = _fin(Lz)
        big = lf & (np.abs(Lz) > HUGE)
        small = lf & ~big
        vals = np.empty_like(Lz)
        vals[~lf] = INF
        vals[big] = np.where(Lz[big].real >= 0, Lz[big], -Lz[big])
        vals[small] = np.sqrt(Lz[small] * Lz[small] - 1.0)
        w[rest] = vals
    return w, t


def _apply_close(prm, z, s):
    a, b = prm
    c = -2 * a * b / (a - b)
    d = (a + b) / (a - b)
    w = np.empty_like(z)
    t = np.zeros_like(s)
    hit = np.zeros(z.shape, dtype=bool)
    for pz in (np.complex128(complex(0.0, a)), np.complex128(complex(0.0, b))):
        m = (z == pz) & ~hit
        w[m] = 0j
        hit |= m
    tagged = (s != 0) & ~hit
    if tagged.any():
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            h = np.where(_isinf(z[tagged]), np.inf, z[tagged].imag)
            den = c + d * h
            h2 = np.where(den == 0, np.inf, h / np.where(den == 0, 1, den))
            h2 = np.where(np.isinf(h), (1.0 / d if d != 0 else np.inf), h2)
        vals = np.empty(h2.shape, dtype=np.complex128)
        tt = np.zeros(h2.shape, dtype=s.dtype)
        gone = ~np.isfinite(h2)
        vals[gone] = INF
        tt[gone] = s[tagged][gone]
        stay = ~gone & (np.abs(h2) > 1)
        hs = h2[stay]
        with np.errstate(over="ignore"):
            mag = np.where(np.abs(hs) < HUGE, np.sqrt(np.maximum(hs * hs - 1.0, 0.0)), np.abs(hs))
        vals[stay] = np.sign(hs) * 1j * mag
        tt[stay] = np.where(hs > 0, UP, DOWN)
        off = ~gone & (np.abs(h2) <= 1)
        vals[off] = np.sqrt(np.maximum(1.0 - h2[off] * h2[off], 0.0))
        w[tagged] = vals
        t[tagged] = tt
        hit |= tagged
    rest = ~hit
    if rest.any():
        zr = z[rest]
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            zinf = _isinf(zr)
            den = c - d * 1j * zr
            T = np.where(den == 0, INF, zr / np.where(den == 0, 1, den))
            T = np.where(zinf, (1.0 / d) * 1j, T) if d != 0 else np.where(zinf, INF, T)
        tf = _fin(T)
        big = tf & (np.abs(T) > HUGE)
        small = tf & ~big
        vals = np.empty_like(T)
        vals[~tf] = INF
        vals[big] = np.where(T[big].real >= 0, T[big], -T[big])
        vals[small] = np.sqrt(T[small] * T[small] + 1.0)
        w[rest] = vals
    return w, t


def _apply_sq(prm, z, s):
    q = np.complex128(prm[0])
    qinf = _inf1(q)
    w = np.empty_like(z)
    t = np.zeros_like(s)
    hit = z == q
    w[hit] = INF
    if not qinf:
        zi = _isinf(z) & ~hit
        w[zi] = q * q
        hit |= zi
    tagged = (s != 0) & ~hit
    if tagged.any():
        h = z[tagged].imag
        if qinf:
            h2 = h
        else:
            den = 1.0 - h / q.imag
            with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
                h2 = np.where(den == 0, np.inf, h / np.where(den == 0, 1, den))
        with np.errstate(over="ignore"):
            w[tagged] = np.where(np.isfinite(h2), -(h2 * h2) + 0j, INF)
        hit |= tagged
    rest = ~hit
    if rest.any():
        zr = z[rest]
        if qinf:
            mm = zr
        else:
            den = 1.0 - zr / q
            mm = np.where(den == 0, INF, zr / np.where(den == 0, 1, den))
        with np.errstate(over="ignore", invalid="ignore"):
            vals = mm * mm
        vals[~_fin(vals)] = INF
        w[rest] = vals
    return w, t


_DISPATCH = {"mob": _apply_mob, "sqr": _apply_sqr, "open": _apply_open,
             "close": _apply_close, "sq": _apply_sq}


def _apply(rec, z, s):
    return _DISPATCH[rec[0]](rec[1], z, s)


def replay(log, points, sides=None):
    """Apply a record list to a point set (`welding.py:512-526`)."""
    z = _pts(points).copy()
    s = np.zeros(z.shape, dtype=np.int8) if sides is None else np.asarray(sides, dtype=np.int8).copy()
    for rec in log:
        z, s = _apply(rec, z, s)
    _nan_guard(z, "apply_log")
    return z, s


# ---------------------------------------------------------------------------
# Mobius helpers


def three_point(zs, ws):
    """Coefficients of the Mobius map z_i -> w_i (`welding.py:99-133`)."""
    zs = [np.complex128(v) for v in zs]
    ws = [np.complex128(v) for v in ws]
    for tri in (zs, ws):
        for i in range(3):
            for j in range(i + 1, 3):
                bi, bj = _inf1(tri[i]), _inf1(tri[j])
                if (bi and bj) or (not bi and not bj and tri[i] == tri[j]):
                    raise OracleWeldError("three-point Mobius needs distinct points")

    def std(z1, z2, z3):
        if _inf1(z1):
            return (0, z2 - z3, 1, -z3)
        if _inf1(z2):
            return (1, -z1, 1, -z3)
        if _inf1(z3):
            return (1, -z1, 0, z2 - z1)
        return (z2 - z3, -z1 * (z2 - z3), z2 - z1, -z3 * (z2 - z1))

    a1, b1, c1, d1 = std(*zs)
    a2, b2, c2, d2 = std(*ws)
    a = d2 * a1 - b2 * c1
    b = d2 * b1 - b2 * d1
    c = -c2 * a1 + a2 * c1
    d = -c2 * b1 + a2 * d1
    nrm = max(abs(a), abs(b), abs(c), abs(d))
    return (a / nrm, b / nrm, c / nrm, d / nrm)


def _walk_key(h):
    """Position along the imaginary-axis circle walking up from 0
    (`welding.py:169-176`)."""
    if np.isinf(h):
        return (1, 0.0)
    if h > 0:
        return (0, h)
    return (2, h)


# ---------------------------------------------------------------------------
# zipping (Algorithm 1)


def _zip(pts, s, k, br, collapse_tol=1e-13):
    """`welding.py:546-575`."""
    log = []
    if pts[0] == pts[1]:
        raise OracleWeldError("zip points 0 and 1 coincide")
    rec = ("sqr", (complex(pts[0]), complex(pts[1]), br))
    pts, s = _apply(rec, pts, s)
    log.append(rec)
    for j in range(2, k + 1):
        xi = complex(pts[j])
        if s[j] != 0 or _inf1(xi):
            raise OracleWeldError(f"zip point {j} left the right half-plane")
        if not xi.real > 0:
            raise OracleWeldError(f"zip point {j} landed on the imaginary axis "
                                  "(duplicate or non-Jordan input)")
        if abs(xi) < collapse_tol:
            raise OracleWeldError(f"zip points {j - 1} and {j} collapsed "
                                  f"(spacing below {collapse_tol:g} in the zip frame)")
        rec = ("open", (xi, br))
        pts, s = _apply(rec, pts, s)
        log.append(rec)
    _nan_guard(pts, "zipping")
    return pts, s, log


def half_unzip(points, k, br=UP):
    """Intermediate form (`welding.py:578-602`): returns (values, sides, log)."""
    pts = _pts(points).copy()
    if k < 1:
        raise OracleWeldError("zip count must be at least 1")
    if len(pts) < k + 1:
        raise OracleWeldError("need at least k + 1 points")
    s = np.zeros(len(pts), dtype=np.int8)
    pts, s, log = _zip(pts, s, k, br)
    w0 = np.complex128(pts[0])
    if not _inf1(w0):
        if w0 == 0:
            raise OracleWeldError("far end of the zip collapsed to 0")
        rec = mob(1, 0, -1 / w0, 1, axis=True,
                  pins=((w0, INF, br), (np.complex128(0), np.complex128(0), br)))
        pts, s = _apply(rec, pts, s)
        log.append(rec)
    _nan_guard(pts, "intermediate form")
    return pts, s, log


# ---------------------------------------------------------------------------
# partial / closed welding (Algorithm 2)


def _unit_frame(pts, tries=4):
    """`welding.py:609-625`."""
    f = _fin(pts)
    if not f.any():
        raise OracleWeldError("no finite boundary points")
    c = complex(np.mean(pts[f]))
    s = float(np.max(np.abs(pts[f] - c)))
    if s == 0:
        raise OracleWeldError("degenerate boundary (all points coincide)")
    for _ in range(tries):
        if not np.any(pts[f] == c):
            break
        c += s * (0.0137 + 0.00271j)
    else:
        raise OracleWeldError("could not place tracking origin off the boundary")
    return mob(1 / s, -c / s, 0, 1)


class WeldOut:
    def __init__(self, a, b, log_a, log_b, aux_a, aux_b, seam_error, k):
        self.a, self.b = a, b
        self.log_a, self.log_b = log_a, log_b
        self.aux_a, self.aux_b = aux_a, aux_b
        self.seam_error = seam_error
        self.k = k


def partial_weld(a_points, b_points, k, hard_tol=1e-6):
    """Algorithm 2 (`welding.py:640-731`)."""
    a = _pts(a_points)
    b = _pts(b_points)
    m = len(a) - 1
    n = len(b) - 1
    if k < 1 or k > min(m, n):
        raise OracleWeldError(f"shared prefix length k={k} out of range")
    fa = _unit_frame(a)
    fb = _unit_frame(b)
    an, _ = _apply(fa, a, np.zeros(len(a), dtype=np.int8))
    bn, _ = _apply(fb, b, np.zeros(len(b), dtype=np.int8))
    va, sa, la = half_unzip(np.concatenate([an, [np.complex128(0), INF]]), k, UP)
    vb, sb, lb = half_unzip(np.concatenate([bn, [np.complex128(0), INF]]), k, DOWN)
    log_a = [fa] + la
    log_b = [fb] + lb
    for j in range(k - 1, 0, -1):
        al = np.complex128(va[j])
        be = np.complex128(vb[j])
        if sa[j] == 0 or _inf1(al) or al.imag == 0:
            raise OracleWeldError(f"alignment point {j} (a side) left the imaginary axis")
        if sb[j] == 0 or _inf1(be) or be.imag == 0:
            raise OracleWeldError(f"alignment point {j} (b side) left the imaginary axis")
        if not _walk_key(al.imag) < _walk_key(be.imag):
            raise OracleWeldError(f"alignment points {j} not strictly ordered on the "
                                  "imaginary axis (invalid correspondence)")
        rec = ("close", (float(al.imag), float(be.imag)))
        va, sa = _apply(rec, va, sa)
        vb, sb = _apply(rec, vb, sb)
        log_a.append(rec)
        log_b.append(rec)
    qa, qb = np.complex128(va[0]), np.complex128(vb[0])
    if _inf1(qa) != _inf1(qb) or (not _inf1(qa) and abs(qa - qb) > 1e-9 * max(_maxabs(va), 1.0)):
        raise OracleWeldError("far ends of the two slits diverged")
    rec = ("sq", (INF if _inf1(qa) else qa,))
    va, sa = _apply(rec, va, sa)
    vb, sb = _apply(rec, vb, sb)
    log_a.append(rec)
    log_b.append(rec)
    za, zb = np.complex128(va[m + 1]), np.complex128(vb[n + 1])
    ia, ib = np.complex128(va[m + 2]), np.complex128(vb[n + 2])
    if _inf1(za) or _inf1(zb) or _inf1(ia) or _inf1(ib):
        raise OracleWeldError("tracking points degenerated during welding")
    zmid = 0.5 * (ia + ib)
    if za != zb and za != zmid and zb != zmid:
        co = three_point((za, zb, zmid), (-1.0, 1.0, INF))
    elif za != 0:
        co = (-1.0 / za, 0.0, 0.0, 1.0)
    else:
        co = (1.0, 0.0, 0.0, 1.0)
    rec = mob(*co)
    va, sa = _apply(rec, va, sa)
    vb, sb = _apply(rec, vb, sb)
    log_a.append(rec)
    log_b.append(rec)
    _nan_guard(va, "partial weld")
    _nan_guard(vb, "partial weld")
    with np.errstate(invalid="ignore"):
        gap = np.abs(va[:k + 1] - vb[:k + 1])
    gap[_isinf(va[:k + 1]) & _isinf(vb[:k + 1])] = 0.0
    seam = float(np.max(gap))
    scale = max(_maxabs(va), _maxabs(vb))
    if seam > hard_tol * scale:
        raise OracleWeldError(f"seam alignment error {seam:.3e} exceeds "
                              f"{hard_tol:g} x scale {scale:.3e}")
    return WeldOut(va[:m + 1], vb[:n + 1], log_a, log_b, va[m + 1:], vb[n + 1:], seam, k)


def closed_weld(a_points, b_points, hard_tol=1e-6):
    """Closed welding of two full cycles (`welding.py:734-763`)."""
    a = _pts(a_points)
    b = _pts(b_points)
    if len(a) != len(b):
        raise OracleWeldError("closed welding needs equal-length boundaries")
    if len(a) < 3:
        raise OracleWeldError("closed welding needs at least 3 boundary points")
    r = partial_weld(a, b, k=len(a) - 1, hard_tol=hard_tol)
    n = len(r.a)
    anchors = (r.a[0], r.a[n // 3], r.a[(2 * n) // 3])
    targets = tuple(np.exp(2j * np.pi * np.arange(3) / 3))
    rec = mob(*three_point(anchors, targets))
    va, _ = _apply(rec, np.concatenate([r.a, r.aux_a]), np.zeros(len(r.a) + 2, dtype=np.int8))
    vb, _ = _apply(rec, np.concatenate([r.b, r.aux_b]), np.zeros(len(r.b) + 2, dtype=np.int8))
    r.log_a.append(rec)
    r.log_b.append(rec)
    return WeldOut(va[:-2], vb[:-2], r.log_a, r.log_b, va[-2:], vb[-2:], r.seam_error, r.k)


# ---------------------------------------------------------------------------
# polygon helpers and the geodesic map to the circle


def _inside(poly, p):
    """Even-odd ray casting (`welding.py:770-778`)."""
    x, y = p.real, p.imag
    xs, ys = poly.real, poly.imag
    x2, y2 = np.roll(xs, -1), np.roll(ys, -1)
    cond = (ys > y) != (y2 > y)
    with np.errstate(divide="ignore", invalid="ignore"):
        xint = xs + (y - ys) / (y2 - ys) * (x2 - xs)
    return bool(np.sum(cond & (x < xint)) % 2)


def interior_point(poly):
    """`welding.py:781-796`."""
    poly = _pts(poly)
    c = complex(np.mean(poly))
    if _inside(poly, c):
        return c
    n = len(poly)
    for i in range(n):
        mid = 0.5 * (poly[i] + poly[(i + 1) % n])
        nrm = (poly[(i + 1) % n] - poly[i]) * 1j
        for t in (0.25, 0.05, 0.01):
            cand = mid + t * nrm
            if _inside(poly, cand):
                return complex(cand)
    raise OracleWeldError("could not locate a point inside the polygon")


def geodesic_to_circle(points, interior=None):
    """Boundary polygon onto the unit circle (`welding.py:803-842`)."""
    pts = _pts(points).copy()
    if len(pts) < 3:
        raise OracleWeldError("need at least 3 boundary points")
    if interior is None:
        interior = interior_point(pts)
    n = len(pts)
    pts = np.concatenate([pts, [np.complex128(interior)]])
    s = np.zeros(len(pts), dtype=np.int8)
    pts, s, log = _zip(pts, s, n - 1, UP)
    w0 = np.complex128(pts[0])
    rec = ("sq", (INF if _inf1(w0) else w0,))
    pts, s = _apply(rec, pts, s)
    log.append(rec)
    cay = mob(1, -1j, 1, 1j, pins=((INF, np.complex128(1.0), FREE),))
    pts, s = _apply(cay, pts, s)
    log.append(cay)
    al = np.complex128(pts[-1])
    if not abs(al) < 1:
        raise OracleWeldError("interior point left the unit disk during the geodesic mapping")
    cen = mob(1, -al, -np.conj(al), 1)
    pts, s = _apply(cen, pts, s)
    log.append(cen)
    pts = pts[:-1]
    _nan_guard(pts, "geodesic algorithm")
    err = np.max(np.abs(np.abs(pts) - 1.0))
    if err > 1e-9:
        raise OracleWeldError(f"boundary point left the unit circle by {err:.3e}")
    return pts, log
