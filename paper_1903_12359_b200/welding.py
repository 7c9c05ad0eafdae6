"""Conformal welding maps (drop-in for `welding.py`), executed on the device.

The record classes mirror `welding.py:236-509` and convert to the C ABI's
`pgcp_rec`; `partial_weld`, `closed_weld`, `geodesic_to_circle` and
`apply_log` run the CUDA weld engine (weld.cu). A few scalar helpers of the
reference API (`mobius_from_three_points`, `mobius_to_unit`,
`mobius_pair_align`, `opening_map`, `closing_map`, `cross_ratio`) are tiny
host formulas kept for API completeness; the pipeline never calls them.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .errors import WeldError

GENERIC = 0
UPPER = 1
LOWER = -1
INF = np.complex128(complex(np.inf, 0.0))

_VP, _I32, _I64, _D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
nat.register("pgcp_weld_schedule_run", [_VP, _I32, _VP, _VP, _VP, _VP, _D, _VP, _VP, _I64, _VP])
nat.register("pgcp_weld_schedule_prepare", [_I32, _VP, _VP, _VP, _VP, _VP, ctypes.POINTER(ctypes.c_void_p)])
nat.register("pgcp_weld_schedule_execute", [_VP, _VP, _D, _VP, _VP, _I64, _VP])
nat.register("pgcp_weld_schedule_free", [_VP], None)
nat.register("pgcp_weld_replay", [_VP, _I32, _VP, _VP, _I64, _VP])
nat.register("pgcp_weld_geodesic", [_VP, _VP, _I32, _VP, _VP, _VP, _I32, _VP, _VP])
nat.register("pgcp_polygon_interior", [_VP, _VP, _I32, ctypes.c_int, _VP, _VP])
nat.register("pgcp_inv_shift", [_VP, _VP, _I64, _D, _D, _D, _D, _VP])
nat.register("pgcp_weld_intermediate", [_VP, _VP, _I32, _I32, _I32, _VP, _I32, _VP, _VP])
nat.register("pgcp_gather_complex", [_VP, _VP, _VP, _I64, _VP])
nat.register("pgcp_scatter_complex", [_VP, _VP, _VP, _I64, _VP])


def _c2l(c):
    c = complex(c)
    return [c.real, c.imag]


def is_infinity(z):
    z = np.asarray(z)
    return np.isinf(z.real) | np.isinf(z.imag)


# ---------------------------------------------------------------------------
# records


@dataclass
class MobiusRec:
    a: complex
    b: complex
    c: complex
    d: complex
    axis: bool = False
    pins: tuple = ()

    def __post_init__(self):
        if complex(self.a) * complex(self.d) - complex(self.b) * complex(self.c) == 0:
            raise WeldError("degenerate Mobius coefficients")

    def to_dict(self):
        return {"kind": "mobius", "a": _c2l(self.a), "b": _c2l(self.b), "c": _c2l(self.c),
                "d": _c2l(self.d), "axis": self.axis}

    def _native(self, r):
        r.kind = 0
        r.flags = 1 if self.axis else 0
        vals = [complex(x) for x in (self.a, self.b, self.c, self.d)]
        for i, v in enumerate(vals):
            r.p[2 * i], r.p[2 * i + 1] = v.real, v.imag
        for k, (pz, pw, ps) in enumerate(self.pins):
            pz, pw = complex(pz), complex(pw)
            r.p[8 + 4 * k], r.p[9 + 4 * k], r.p[10 + 4 * k], r.p[11 + 4 * k] = pz.real, pz.imag, pw.real, pw.imag
            r.flags |= ((int(ps) & 0xff) << (16 + 8 * k))
        r.flags |= len(self.pins) << 8

    def apply(self, z, side):
        return _apply_recs([self], z, side)


@dataclass
class SqrtRatioRec:
    z0: complex
    z1: complex
    branch: int

    def to_dict(self):
        return {"kind": "sqrt_ratio", "z0": _c2l(self.z0), "z1": _c2l(self.z1), "branch": self.branch}

    def _native(self, r):
        r.kind = 1
        r.flags = int(self.branch) & 0xff
        z0, z1 = complex(self.z0), complex(self.z1)
        r.p[0], r.p[1], r.p[2], r.p[3] = z0.real, z0.imag, z1.real, z1.imag

    def apply(self, z, side):
        return _apply_recs([self], z, side)


@dataclass
class OpenRec:
    xi: complex
    branch: int

    def to_dict(self):
        return {"kind": "open", "xi": _c2l(self.xi), "branch": self.branch}

    def _native(self, r):
        r.kind = 2
        r.flags = int(self.branch) & 0xff
        xi = complex(self.xi)
        s2 = abs(xi) ** 2
        r.p[0], r.p[1], r.p[2], r.p[3] = xi.real, xi.imag, xi.real / s2, xi.imag / s2

    def apply(self, z, side):
        return _apply_recs([self], z, side)


@dataclass
class CloseRec:
    ai: float
    bi: float

    def to_dict(self):
        return {"kind": "close", "ai": self.ai, "bi": self.bi}

    def _native(self, r):
        a, b = float(self.ai), float(self.bi)
        r.kind = 3
        r.flags = 0
        r.p[0], r.p[1], r.p[2], r.p[3] = a, b, -2 * a * b / (a - b), (a + b) / (a - b)

    def apply(self, z, side):
        return _apply_recs([self], z, side)


@dataclass
class SquareMobiusRec:
    q: complex

    def to_dict(self):
        return {"kind": "square_mobius", "q": _c2l(self.q)}

    def _native(self, r):
        r.kind = 4
        r.flags = 0
        q = complex(self.q)
        r.p[0], r.p[1] = q.real, q.imag

    def apply(self, z, side):
        return _apply_recs([self], z, side)


def _s8(x):
    x &= 0xff
    return x - 256 if x > 127 else x


def _from_native(r):
    p = list(r.p)
    if r.kind == 0:
        npins = (r.flags >> 8) & 0xff
        pins = []
        for k in range(npins):
            side = _s8(r.flags >> (16 + 8 * k))
            pins.append((complex(p[8 + 4 * k], p[9 + 4 * k]), complex(p[10 + 4 * k], p[11 + 4 * k]), int(side)))
        rec = MobiusRec.__new__(MobiusRec)
        rec.a, rec.b, rec.c, rec.d = (complex(p[0], p[1]), complex(p[2], p[3]), complex(p[4], p[5]),
                                      complex(p[6], p[7]))
        rec.axis = bool(r.flags & 1)
        rec.pins = tuple(pins)
        return rec
    if r.kind == 1:
        return SqrtRatioRec(complex(p[0], p[1]), complex(p[2], p[3]), _s8(r.flags))
    if r.kind == 2:
        return OpenRec(complex(p[0], p[1]), _s8(r.flags))
    if r.kind == 3:
        return CloseRec(p[0], p[1])
    return SquareMobiusRec(complex(p[0], p[1]))


def _to_native(log):
    arr = (nat.Rec * max(len(log), 1))()
    for i, rec in enumerate(log):
        rec._native(arr[i])
    return arr


def _stream():
    from .device import stream_handle
    return stream_handle()


def _apply_recs(log, z, side):
    from .device import require_cuda, ptr
    require_cuda()
    zz = torch.as_tensor(np.atleast_1d(np.asarray(z, dtype=np.complex128)).copy()).cuda()
    ss = torch.as_tensor(np.asarray(side, dtype=np.int8).copy()).cuda() if side is not None else \
        torch.zeros(zz.shape, dtype=torch.int8, device=zz.device)
    arr = _to_native(log)
    nat.check(nat.lib().pgcp_weld_replay(arr, len(log), ptr(zz), ptr(ss), zz.numel(), _stream()))
    return zz.cpu().numpy(), ss.cpu().numpy()


def apply_log(log, points, sides=None):
    """Replay a record list on a point set (welding.py:512-526), on the device."""
    z = np.atleast_1d(np.asarray(points, dtype=np.complex128))
    s = np.zeros(z.shape, dtype=np.int8) if sides is None else np.asarray(sides, dtype=np.int8)
    if len(log) == 0:
        return z.copy(), s.copy()
    return _apply_recs(list(log), z, s)


def log_to_dicts(log):
    return [rec.to_dict() for rec in log]


def mobius_apply(coeffs, z):
    """(az + b)/(cz + d) with exact infinity/pole handling (welding.py:79-96)."""
    a, b, c, d = (complex(x) for x in coeffs)
    if a * d - b * c == 0:
        raise WeldError("degenerate Mobius coefficients (ad - bc = 0)")
    out, _ = _apply_recs([MobiusRec(a, b, c, d)], np.atleast_1d(np.asarray(z, dtype=np.complex128)), None)
    return out


# ---------------------------------------------------------------------------
# host scalar helpers of the API


def mobius_from_three_points(zs, ws):
    """Mobius map z_i -> w_i, normalised to unit max modulus (welding.py:99-133)."""
    zs = [np.complex128(z) for z in zs]
    ws = [np.complex128(w) for w in ws]
    inf = lambda v: bool(np.isinf(np.real(v)) or np.isinf(np.imag(v)))
    for trip in (zs, ws):
        for i in range(3):
            for j in range(i + 1, 3):
                if (inf(trip[i]) and inf(trip[j])) or (not inf(trip[i]) and not inf(trip[j])
                                                       and trip[i] == trip[j]):
                    raise WeldError("three-point Mobius needs distinct points")

    def std(z1, z2, z3):
        if inf(z1):
            return (0, z2 - z3, 1, -z3)
        if inf(z2):
            return (1, -z1, 1, -z3)
        if inf(z3):
            return (1, -z1, 0, z2 - z1)
        return (z2 - z3, -z1 * (z2 - z3), z2 - z1, -z3 * (z2 - z1))

    a1, b1, c1, d1 = std(*zs)
    a2, b2, c2, d2 = std(*ws)
    a, b = d2 * a1 - b2 * c1, d2 * b1 - b2 * d1
    c, d = -c2 * a1 + a2 * c1, -c2 * b1 + a2 * d1
    nrm = max(abs(a), abs(b), abs(c), abs(d))
    return (a / nrm, b / nrm, c / nrm, d / nrm)


def mobius_to_unit(xi):
    xi = complex(xi)
    if not np.isfinite(xi.real) or xi.real <= 0:
        raise WeldError("alignment target must lie strictly in the right half-plane")
    s = abs(xi) ** 2
    return (xi.real / s, 0.0, (xi.imag / s) * 1j, 1.0)


def mobius_pair_align(alpha, beta):
    a = complex(alpha).imag
    b = complex(beta).imag
    if not a > 0:
        raise WeldError("alpha must lie on the positive imaginary axis")
    if not b < 0:
        raise WeldError("beta must lie on the negative imaginary axis")
    c = -2 * a * b / (a - b)
    d = (a + b) / (a - b)
    return (1.0, 0.0, -d * 1j, c)


def _slit_sqrt(z, sign, branch):
    z = np.atleast_1d(np.asarray(z, dtype=np.complex128))
    out = np.empty_like(z)
    infm = is_infinity(z)
    out[infm] = INF
    r = np.sqrt(z[~infm] * z[~infm] + sign)
    on = r.real == 0
    r[on] = branch * 1j * np.abs(r[on].imag)
    out[~infm] = r
    return out


def opening_map(z, branch=UPPER):
    return _slit_sqrt(z, -1.0, branch)


def closing_map(z, branch=UPPER):
    return _slit_sqrt(z, 1.0, branch)


def cross_ratio(z1, z2, z3, z4):
    def diff(u, v):
        if np.isinf(np.real(u)) or np.isinf(np.real(v)):
            return None
        return complex(u) - complex(v)
    n1, n2, d1, d2 = diff(z1, z3), diff(z2, z4), diff(z1, z4), diff(z2, z3)
    num = (n1 if n1 is not None else 1) * (n2 if n2 is not None else 1)
    den = (d1 if d1 is not None else 1) * (d2 if d2 is not None else 1)
    return num / den


# ---------------------------------------------------------------------------
# welds on the device


@dataclass
class WeldResult:
    a: np.ndarray
    b: np.ndarray
    log_a: list
    log_b: list
    aux_a: np.ndarray
    aux_b: np.ndarray
    seam_error: float
    k: int


def run_schedule(tv, info, src, wb_off, wb, hard_tol, want_logs=False):
    """Run weld steps on the tracked values `tv` (CUDA complex tensor, in
    place). Returns (per-step out array, logs or None)."""
    from .device import ptr
    nsteps = len(info)
    info = np.ascontiguousarray(np.asarray(info, dtype=np.int32).reshape(-1, 6))
    src = np.ascontiguousarray(np.asarray(src, dtype=np.int32))
    wb_off = np.ascontiguousarray(np.asarray(wb_off, dtype=np.int64))
    wb = np.ascontiguousarray(np.asarray(wb, dtype=np.int32).reshape(-1, 2))
    out = np.zeros((max(nsteps, 1), 8))
    recs = None
    cap = 0
    if want_logs:
        cap = int(sum(2 * (2 * int(k) + 16) for k in info[:, 0]))
        recs = (nat.Rec * max(cap, 1))()
    st = nat.lib().pgcp_weld_schedule_run(ptr(tv), nsteps, info.ctypes.data, src.ctypes.data, wb_off.ctypes.data,
                                          wb.ctypes.data, float(hard_tol), out.ctypes.data, recs, cap, _stream())
    logs = None
    if want_logs and st == nat.OK:
        logs = []
        for i in range(nsteps):
            off = int(out[i, 7])
            k = int(info[i, 0])
            c = 2 * k + 16
            la = [_from_native(recs[off + j]) for j in range(int(out[i, 4]))]
            lb = [_from_native(recs[off + c + j]) for j in range(int(out[i, 5]))]
            logs.append((la, lb))
    nat.check(st)
    return out, logs


class PreparedSchedule:
    """A weld schedule whose host-side preparation and uploads are already
    done (pgcp_weld_schedule_prepare, on the current stream): `run(tv)` starts
    with the first weld launch. One run per object."""

    def __init__(self, info, src, wb_off, wb):
        self.nsteps = len(info)
        info = np.ascontiguousarray(np.asarray(info, dtype=np.int32).reshape(-1, 6))
        src = np.ascontiguousarray(np.asarray(src, dtype=np.int32))
        wb_off = np.ascontiguousarray(np.asarray(wb_off, dtype=np.int64))
        wb = np.ascontiguousarray(np.asarray(wb, dtype=np.int32).reshape(-1, 2))
        self._h = ctypes.c_void_p()
        nat.check(nat.lib().pgcp_weld_schedule_prepare(self.nsteps, info.ctypes.data, src.ctypes.data,
                                                       wb_off.ctypes.data, wb.ctypes.data, _stream(),
                                                       ctypes.byref(self._h)))

    def run(self, tv, hard_tol):
        """Weld the tracked values `tv` (CUDA complex tensor, in place) on the
        current stream; returns the per-step out array of `run_schedule`."""
        from .device import ptr
        out = np.zeros((max(self.nsteps, 1), 8))
        try:
            nat.check(nat.lib().pgcp_weld_schedule_execute(self._h, ptr(tv), float(hard_tol), out.ctypes.data, None, 0,
                                                           _stream()))
        finally:
            self.close()
        return out

    def close(self):
        if self._h:
            nat.lib().pgcp_weld_schedule_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


ARC_FROM_B = 1 << 24
CYC_A = 1 << 25
CYC_B = 1 << 26
SIDE_B = 1 << 31


def _pair(a_points, b_points, k, closed, hard_tol):
    from .device import device, require_cuda
    require_cuda()
    a = np.atleast_1d(np.asarray(a_points, dtype=np.complex128))
    b = np.atleast_1d(np.asarray(b_points, dtype=np.complex128))
    m, n = len(a) - 1, len(b) - 1
    if k < 1 or k > min(m, n):
        raise WeldError(f"shared prefix length k={k} out of range")
    tv = torch.as_tensor(np.concatenate([a, b])).to(device())
    ta = np.arange(m + 1)
    tb = np.arange(n + 1)
    code_a = np.where(ta <= k, ta + 1, 0) | CYC_A
    code_b = np.where(tb <= k, (tb + 1) | ARC_FROM_B, 0) | CYC_B | SIDE_B
    wb = np.concatenate([np.stack([ta, code_a], 1), np.stack([m + 1 + tb, code_b], 1)])
    info = [[k, int(closed), m + 1, n + 1, 0, 1]]
    src = np.concatenate([ta, m + 1 + tb])
    out, logs = run_schedule(tv, info, src, [0, len(wb)], wb.astype(np.int64).astype(np.int32), hard_tol,
                             want_logs=True)
    z = tv.cpu().numpy()
    la, lb = logs[0]
    # the tracking points (0, inf) enter after the prenormalizer (welding.py:664-665)
    aux_a, _ = apply_log(la[1:], np.array([0j, INF]))
    aux_b, _ = apply_log(lb[1:], np.array([0j, INF]))
    return WeldResult(z[:m + 1], z[m + 1:], la, lb, aux_a, aux_b, float(out[0, 0]), k)


def partial_weld(a_points, b_points, k, hard_tol=1e-6):
    """Algorithm 2 (welding.py:640-731) on the device."""
    return _pair(a_points, b_points, int(k), False, hard_tol)


def closed_weld(a_points, b_points, hard_tol=1e-6):
    """Closed welding of two full cycles (welding.py:734-763) on the device."""
    a = np.atleast_1d(np.asarray(a_points, dtype=np.complex128))
    b = np.atleast_1d(np.asarray(b_points, dtype=np.complex128))
    if len(a) != len(b):
        raise WeldError("closed welding needs equal-length boundaries")
    if len(a) < 3:
        raise WeldError("closed welding needs at least 3 boundary points")
    return _pair(a, b, len(a) - 1, True, hard_tol)


@dataclass
class IntermediateForm:
    values: np.ndarray
    sides: np.ndarray
    zipped_count: int
    log: list = field(default_factory=list)


def intermediate_form(points, k, branch=UPPER):
    """Half-unzip a boundary point sequence (welding.py:578-602) on the
    device: points 0..k onto the branch's half of the imaginary axis (point
    0 at infinity, point k at 0), the rest into the open right half-plane."""
    from .device import device, ptr, require_cuda
    require_cuda()
    br = UPPER if branch in (UPPER, "plus_i") else LOWER
    pts = torch.as_tensor(np.atleast_1d(np.asarray(points, dtype=np.complex128)).copy()).to(device())
    sides = torch.zeros(pts.shape, dtype=torch.int8, device=pts.device)
    cap = max(int(k), 1) + 1
    recs = (nat.Rec * cap)()
    nrec = ctypes.c_int32(0)
    nat.check(nat.lib().pgcp_weld_intermediate(ptr(pts), ptr(sides), pts.numel(), int(k), br, recs, cap,
                                               ctypes.byref(nrec), _stream()))
    log = [_from_native(recs[i]) for i in range(nrec.value)]
    return IntermediateForm(pts.cpu().numpy(), sides.cpu().numpy(), int(k), log)


def geodesic_to_circle(points, interior=None):
    """Jordan polygon onto the unit circle (welding.py:803-842) on the device.
    Returns (circle points, map log)."""
    from .device import device, ptr, require_cuda
    require_cuda()
    pts = np.atleast_1d(np.asarray(points, dtype=np.complex128))
    n = len(pts)
    if n < 3:
        raise WeldError("need at least 3 boundary points")
    tv = torch.as_tensor(pts).to(device())
    circ = torch.empty_like(tv)
    src = np.arange(n, dtype=np.int32)
    cap = n + 8
    recs = (nat.Rec * cap)()
    meta = np.zeros(8)
    it = None
    if interior is not None:
        c = complex(interior)
        it = (ctypes.c_double * 2)(c.real, c.imag)
    # geodesic_to_circle itself does not reorient (only the pipeline does):
    # pass a ccw polygon as the reference requires
    nat.check(nat.lib().pgcp_weld_geodesic(ptr(tv), src.ctypes.data, n, it, ptr(circ), recs, cap,
                                           meta.ctypes.data, _stream()))
    log = [_from_native(recs[i]) for i in range(int(meta[0]))]
    return circ.cpu().numpy(), log


def point_in_polygon(poly, p):
    x, y = p.real, p.imag
    xs, ys = poly.real, poly.imag
    x2, y2 = np.roll(xs, -1), np.roll(ys, -1)
    cond = (ys > y) != (y2 > y)
    with np.errstate(divide="ignore", invalid="ignore"):
        xint = xs + (y - ys) / (y2 - ys) * (x2 - xs)
    return bool(np.sum(cond & (x < xint)) % 2)


def polygon_interior_point(poly):
    """Centroid or edge-midpoint offset inside the polygon (welding.py:781-796),
    on the device."""
    from .device import device, ptr, require_cuda
    require_cuda()
    pts = np.atleast_1d(np.asarray(poly, dtype=np.complex128))
    tv = torch.as_tensor(pts).to(device())
    src = np.arange(len(pts), dtype=np.int32)
    out = np.zeros(2)
    nat.check(nat.lib().pgcp_polygon_interior(ptr(tv), src.ctypes.data, len(pts), 0, out.ctypes.data, _stream()))
    return complex(out[0], out[1])
