"""Oracle: quasi-conformal fold-over repair (restates `assemble.py:53-217`).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). numpy/scipy restatement
of the reference's `face_layout`, `beltrami_per_face`, `lbs_stiffness` and
`qc_correct`; the linear Beltrami systems go through scipy's `spsolve`
exactly as the reference calls it (SuperLU, `assemble.py:206`).
"""

import numpy as np
from scipy import sparse
from scipy.sparse.linalg import spsolve

MU_CAP = 0.95  # assemble.py:20


class OracleRepairError(RuntimeError):
    pass


def isometric_layout(V, F):
    """Per-face planar corners: 0, |e1|, (e2.e1 + i |e1 x e2|)/|e1|
    (assemble.py:53-67)."""
    V = np.asarray(V, dtype=np.float64)
    F = np.asarray(F)
    a = V[F[:, 1]] - V[F[:, 0]]
    b = V[F[:, 2]] - V[F[:, 0]]
    la = np.linalg.norm(a, axis=1)
    out = np.zeros((len(F), 3), dtype=np.complex128)
    out[:, 1] = la
    out[:, 2] = np.einsum("ij,ij->i", b, a) / la + 1j * (np.linalg.norm(np.cross(a, b), axis=1) / la)
    return out


def face_beltrami(src, dst):
    """mu = f_zbar / f_z of the affine map taking the (m, 3) corners `src` to
    `dst` per face (assemble.py:74-92); f_z == 0 -> inf."""
    s = np.asarray(src, dtype=np.complex128)
    t = np.asarray(dst, dtype=np.complex128)
    p, q = s[:, 1] - s[:, 0], s[:, 2] - s[:, 0]
    u, w = t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]
    det = p * np.conj(q) - np.conj(p) * q
    zero = np.flatnonzero(det == 0)
    if zero.size:
        raise OracleRepairError(f"degenerate source triangle {int(zero[0])} in Beltrami computation")
    fz = (u * np.conj(q) - np.conj(p) * w) / det
    fzb = (p * w - u * q) / det
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(fz == 0, np.inf, fzb / np.where(fz == 0, 1, fz))


def capped(mu, cap):
    """Magnitude capped at `cap`; non-finite coefficients become 0
    (assemble.py:193-200)."""
    mag = np.abs(mu)
    out = np.where(np.isfinite(mu), mu, 0.0)
    over = np.isfinite(mag) & (mag > cap)
    out[over] *= cap / mag[over]
    out[~np.isfinite(mag)] = 0.0
    return out


def beltrami_stiffness(z, F, mu):
    """Linear-element stiffness of div(A grad u) with the 2x2 tensor A of the
    Beltrami coefficient mu, absolute face areas (assemble.py:124-164)."""
    F = np.asarray(F)
    c = np.asarray(z, dtype=np.complex128)[F]
    r, t = mu.real, mu.imag
    den = np.maximum(1.0 - r * r - t * t, 1e-12)
    A11 = ((r - 1.0) ** 2 + t * t) / den
    A12 = -2.0 * t / den
    A22 = ((1.0 + r) ** 2 + t * t) / den
    d1, d2 = c[:, 1] - c[:, 0], c[:, 2] - c[:, 0]
    area = 0.5 * (d1.real * d2.imag - d1.imag * d2.real)
    wgt = np.maximum(np.abs(area), 1e-300)
    grad = []
    for i in range(3):
        e = c[:, (i + 2) % 3] - c[:, (i + 1) % 3]
        grad.append((-e.imag / (2.0 * area), e.real / (2.0 * area)))
    R, Cc, Vv = [], [], []
    for i in range(3):
        for j in range(3):
            (xi, yi), (xj, yj) = grad[i], grad[j]
            R.append(F[:, i])
            Cc.append(F[:, j])
            Vv.append((A11 * xi * xj + A12 * (xi * yj + yi * xj) + A22 * yi * yj) * wgt)
    n = len(np.atleast_1d(z))
    return sparse.csr_matrix((np.concatenate(Vv), (np.concatenate(R), np.concatenate(Cc))), shape=(n, n))


def planar_flips(z, F):
    t = np.asarray(z)[np.asarray(F)]
    d1, d2 = t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]
    return np.flatnonzero(0.5 * (d1.real * d2.imag - d1.imag * d2.real) <= 0)


def repair_folds(layout, F, z, fixed, max_iter=5, cap=MU_CAP):
    """qc_correct (assemble.py:174-217). Returns (z, iterations, cleared,
    remaining face indices, initial flips)."""
    z = np.array(z, dtype=np.complex128)
    fixed = np.asarray(fixed, dtype=np.int64)
    g = z[fixed].copy()
    F = np.asarray(F)
    n0 = len(planar_flips(z, F))
    if n0 == 0:
        return z, 0, True, np.zeros(0, dtype=np.int64), 0
    free = np.setdiff1d(np.arange(len(z)), fixed)
    left = None
    for it in range(1, max_iter + 1):
        K = beltrami_stiffness(z, F, capped(face_beltrami(z[F], layout), cap))
        Kf = K[free]
        Kff = Kf[:, free].tocsc()
        Kfb = Kf[:, fixed]
        x = spsolve(Kff, -(Kfb @ g.real))
        y = spsolve(Kff, -(Kfb @ g.imag))
        if not (np.all(np.isfinite(x)) and np.all(np.isfinite(y))):
            raise OracleRepairError("singular linear Beltrami system during repair")
        z = z.copy()
        z[free] = x + 1j * y
        left = planar_flips(z, F)
        if len(left) == 0:
            return z, it, True, np.zeros(0, dtype=np.int64), n0
    return z, max_iter, False, left, n0
