"""Oracle: cotangent Laplacian, DNCP free-boundary flattening, Dirichlet
harmonic extension (restates `flatten.py:28-188` and `assemble.py:23-50`).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import logging

import numpy as np
from scipy import sparse
from scipy.sparse.linalg import spsolve

log = logging.getLogger(__name__)

COT_LIMIT = 1e8  # flatten.py:21


class OracleSolveError(RuntimeError):
    pass


class OracleMeshError(ValueError):
    pass


def cot_half_weights(V, F):
    """(m, 3) array: 0.5 * cot of the angle at corner c of every face, the
    weight of the opposite edge (F[c+1], F[c+2]).

    Arithmetic as `flatten.py:39-53`: u1 = v_j - v_i, u2 = v_k - v_i,
    cot = einsum(u1, u2) / |cross(u1, u2)|, clamp |cot| <= 1e8.
    """
    V = np.asarray(V, dtype=np.float64)
    F = np.asarray(F, dtype=np.int64)
    out = np.empty((len(F), 3))
    for c in range(3):
        i, j, k = F[:, c], F[:, (c + 1) % 3], F[:, (c + 2) % 3]
        e1 = V[j] - V[i]
        e2 = V[k] - V[i]
        area2 = np.linalg.norm(np.cross(e1, e2), axis=1)
        zero = np.flatnonzero(area2 == 0)
        if zero.size:
            raise OracleMeshError(f"zero-area face {int(zero[0])} in cotangent weights")
        ct = np.einsum("ij,ij->i", e1, e2) / area2
        big = np.abs(ct) > COT_LIMIT
        if big.any():
            log.warning("clamping %d near-degenerate cotangents", int(big.sum()))
            ct = np.clip(ct, -COT_LIMIT, COT_LIMIT)
        out[:, c] = 0.5 * ct
    return out


def cotan_laplacian(V, F, n=None):
    """Canonical CSR cotangent Laplacian (PSD convention), `flatten.py:28-61`.

    The COO triplets are emitted in the reference's order (corner-major, then
    (j,k), (k,j), (j,j), (k,k) blocks) so scipy's duplicate summation sees the
    same operand order and the diagonals come out bit-identical.
    """
    F = np.asarray(F, dtype=np.int64)
    if n is None:
        n = len(V)
    w = cot_half_weights(V, F)
    r, c, v = [], [], []
    for corner in range(3):
        j = F[:, (corner + 1) % 3]
        k = F[:, (corner + 2) % 3]
        wc = w[:, corner]
        r.extend([j, k, j, k])
        c.extend([k, j, j, k])
        v.extend([-wc, -wc, wc, wc])
    return sparse.csr_matrix((np.concatenate(v), (np.concatenate(r), np.concatenate(c))),
                             shape=(n, n))


def area_form(n, loops):
    """2n x 2n matrix of the shoelace area quadratic form, `flatten.py:64-86`."""
    r, c, v = [], [], []
    for loop in loops:
        p = np.asarray(loop, dtype=np.int64)
        q = np.roll(p, -1)
        quarter = np.full(len(p), 0.25)
        r.extend([p, q + n, q, p + n])
        c.extend([q + n, p, p + n, q])
        v.extend([quarter, quarter, -quarter, -quarter])
    return sparse.csr_matrix((np.concatenate(v), (np.concatenate(r), np.concatenate(c))),
                             shape=(2 * n, 2 * n))


def half_perimeter_pins(loop, V):
    """Default pins (loop[0], loop[j]) with j the cumulative-arclength point
    nearest half the perimeter, `flatten.py:113-122`."""
    pts = np.asarray(V)[loop]
    seg = np.linalg.norm(np.roll(pts, -1, axis=0) - pts, axis=1)
    cum = np.concatenate([[0.0], np.cumsum(seg)])
    j = int(np.argmin(np.abs(cum[:-1] - cum[-1] / 2.0)))
    if j == 0:
        j = len(loop) // 2
    return int(loop[0]), int(loop[j])


def _shoelace(z, loops):
    tot = 0.0
    for loop in loops:
        w = z[loop]
        nxt = np.roll(w, -1)
        tot += 0.5 * np.sum(w.real * nxt.imag - w.imag * nxt.real)
    return tot


def conformal_energy(L, z, loops):
    """E_D - A (`flatten.py:89-110`)."""
    x, y = z.real, z.imag
    return 0.5 * (x @ (L @ x) + y @ (L @ y)) - _shoelace(z, loops)


def dncp_system(V, F, loop, pins=None, targets=(0j, 1 + 0j)):
    """Assemble the pinned DNCP system of `flatten.py:157-166`.

    Returns (L, Cff CSR, rhs, free index array, fixed array, fixed values,
    pins)."""
    n = len(V)
    if pins is None:
        pins = half_perimeter_pins(loop, V)
    p0, p1 = pins
    t0, t1 = complex(targets[0]), complex(targets[1])
    L = cotan_laplacian(V, F, n)
    M = area_form(n, [loop])
    C = sparse.block_diag([L, L], format="csr") - 2.0 * M
    fixed = np.array([p0, p1, p0 + n, p1 + n])
    fixed_vals = np.array([t0.real, t1.real, t0.imag, t1.imag])
    free = np.setdiff1d(np.arange(2 * n), fixed)
    Crows = C[free]
    Cff = Crows[:, free]
    rhs = -Crows[:, fixed] @ fixed_vals
    return L, Cff, rhs, free, fixed, fixed_vals, (int(p0), int(p1))


def dncp_flatten(V, F, loop, pins=None, targets=(0j, 1 + 0j), tol=1e-10):
    """DNCP free-boundary conformal flattening, `flatten.py:125-188`.

    `loop` is the single boundary loop (local indices, surface on the left).
    Returns the complex (n,) embedding.
    """
    n = len(V)
    loop = np.asarray(loop, dtype=np.int64)
    if pins is not None:
        p0, p1 = pins
        on = set(int(x) for x in loop)
        if p0 == p1 or p0 not in on or p1 not in on:
            raise OracleMeshError("pins must be two distinct boundary vertices")
    if complex(targets[0]) == complex(targets[1]):
        raise OracleMeshError("pin targets must be distinct")
    L, Cff, rhs, free, fixed, fixed_vals, _ = dncp_system(V, F, loop, pins, targets)
    A = Cff.tocsc()
    sol = spsolve(A, rhs)
    if not np.all(np.isfinite(sol)):
        raise OracleSolveError("singular constrained system in conformal flattening")
    res = np.linalg.norm(A @ sol - rhs)
    ref = np.linalg.norm(rhs)
    if ref > 0 and res > max(tol * ref, 1e3 * tol * np.linalg.norm(sol)):
        raise OracleSolveError(f"flattening residual {res:.3e} above tolerance")
    xy = np.empty(2 * n)
    xy[free] = sol
    xy[fixed] = fixed_vals
    z = xy[:n] + 1j * xy[n:]
    if _shoelace(z, [loop]) <= 0:
        raise OracleMeshError("flattening produced nonpositive signed area")
    ec = conformal_energy(L, z, [loop])
    if ec < -1e-8 * float(np.max(np.abs(z)) ** 2):
        raise OracleSolveError(f"conformal energy {ec:.3e} below lower bound")
    return z


def harmonic_system(V, F, bidx, bvals):
    """(L, Lii CSR, rhs complex, interior) of `assemble.py:34-41`."""
    n = len(V)
    L = cotan_laplacian(V, F, n)
    bidx = np.asarray(bidx, dtype=np.int64)
    interior = np.setdiff1d(np.arange(n), bidx)
    Lrows = L[interior]
    Lii = Lrows[:, interior]
    rhs = -(Lrows[:, bidx] @ np.asarray(bvals, dtype=np.complex128))
    return L, Lii, rhs, interior


def dirichlet_extend(V, F, bidx, bvals, tol=1e-10):
    """Harmonic extension of complex Dirichlet data, `assemble.py:23-50`."""
    n = len(V)
    bvals = np.asarray(bvals, dtype=np.complex128)
    if not np.all(np.isfinite(bvals.real) & np.isfinite(bvals.imag)):
        raise OracleSolveError("non-finite boundary data for harmonic solve")
    _, Lii, rhs, interior = harmonic_system(V, F, bidx, bvals)
    z = np.zeros(n, dtype=np.complex128)
    z[np.asarray(bidx, dtype=np.int64)] = bvals
    if len(interior) == 0:
        return z
    A = Lii.tocsc()
    sol = spsolve(A, rhs)
    if not np.all(np.isfinite(sol.real) & np.isfinite(sol.imag)):
        raise OracleSolveError("singular harmonic system")
    res = np.linalg.norm(A @ sol - rhs)
    ref = np.linalg.norm(rhs)
    if ref > 0 and res > max(tol * ref, 1e3 * tol * np.linalg.norm(sol)):
        raise OracleSolveError(f"harmonic residual {res:.3e} above tolerance")
    z[interior] = sol
    return z
