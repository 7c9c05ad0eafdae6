"""CPU study: PCG iteration counts (and SpMV counts) of the DNCP flatten
system of a cfg-2 subdomain under stronger preconditioners than k_pcg2's
additive two-level one:

  additive      M^-1 = I + Q,  Q = W^ E^-1 W^T       (k_pcg2 today)
  mult(s)       symmetric two-level V(1,1): Jacobi/Chebyshev pre-smoothing
                of degree s, coarse correction, post-smoothing
  sa-add        additive with the smoothed prolongator P = (I - w A) W^
  sa-mult(s)    multiplicative with P

    python tools/precond_study.py [subdomain]
"""
import os
import sys

import numpy as np
from scipy import sparse

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.laplace import dncp_system  # noqa: E402  (study tool)
from oracle.surface import split_mesh  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402
from deflation_study import aggregates, coarse_basis  # noqa: E402


def pcg(A, b, apply_m, x0=None, tol=1e-10, maxit=6000):
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - A @ x
    z = apply_m(r)
    p = z.copy()
    rz = r @ z
    bn = np.linalg.norm(b)
    for it in range(1, maxit + 1):
        q = A @ p
        al = rz / (p @ q)
        x += al * p
        r -= al * q
        if np.linalg.norm(r) <= tol * bn:
            return it
        z = apply_m(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return maxit


def lmax_est(A, n=30):
    v = np.random.default_rng(0).standard_normal(A.shape[0])
    for _ in range(n):
        v = A @ v
        v /= np.linalg.norm(v)
    return float(v @ (A @ v)) * 1.05


def cheb_smoother(A, deg, lmax, ratio=30.0):
    """Chebyshev polynomial approximating A^-1 on [lmax/ratio, lmax]."""
    lmin = lmax / ratio
    th = 0.5 * (lmax + lmin)
    de = 0.5 * (lmax - lmin)
    sig = th / de

    def apply(r):
        # standard Chebyshev iteration for A x = r from x = 0
        rho = 1.0 / sig
        x = r / th
        d = x.copy()
        res = r - A @ x
        for _ in range(deg - 1):
            rho_n = 1.0 / (2 * sig - rho)
            d = rho_n * rho * d + (2 * rho_n / de) * res
            x = x + d
            res = res - A @ d
            rho = rho_n
        return x
    return apply


def main():
    isub = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    V, F, cuts = gen.height_field_case(1024, 8)
    split = split_mesh(V, F, cuts)
    Vs, Fs, loop = split.sub_V[isub], split.sub_F[isub], split.loops[isub]
    n = len(Vs)
    _, C, rhs, free, _, _, _ = dncp_system(Vs, Fs, loop)
    d = C.diagonal()
    Ds = sparse.diags(1.0 / np.sqrt(d))
    A = (Ds @ C @ Ds).tocsr()
    bh = rhs / np.sqrt(d)
    agg, a, b = aggregates(Vs)
    W = coarse_basis(free, n, Vs, agg, a, b)
    Wh = (sparse.diags(np.sqrt(d)) @ W).tocsr()
    lmax = lmax_est(A)
    print(f"n={n} unknowns={A.shape[0]} coarse={W.shape[1]} lmax~{lmax:.3f}", flush=True)

    def coarse_op(P):
        E = (P.T @ A @ P).toarray()
        Ei = np.linalg.pinv(E, rcond=1e-12, hermitian=True)
        return lambda v: P @ (Ei @ (P.T @ v))

    Q = coarse_op(Wh)
    it = pcg(A, bh, lambda r: r + Q(r), x0=Q(bh))
    print(f"additive+x0: {it} it, {it} spmv", flush=True)

    om = 1.0 / lmax * 4 / 3
    Ps = (Wh - om * (A @ Wh)).tocsr()
    Qs = coarse_op(Ps)
    it = pcg(A, bh, lambda r: r + Qs(r), x0=Qs(bh))
    print(f"sa-additive+x0: {it} it, {it} spmv", flush=True)

    for name, QQ in (("plain", Q), ("sa", Qs)):
        for deg in (1, 2, 3, 4):
            S = cheb_smoother(A, deg, lmax)

            def mult(r, S=S, QQ=QQ):
                z = S(r)
                r1 = r - A @ z
                z = z + QQ(r1)
                r2 = r - A @ z
                return z + S(r2)
            it = pcg(A, bh, mult)
            spmv = it * (1 + 2 * deg + (1 if deg else 0))
            print(f"mult-{name} cheb{deg}: {it} it, ~{spmv} spmv", flush=True)


if __name__ == "__main__":
    main()
