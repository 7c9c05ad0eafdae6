"""CPU study: PCG iteration counts of the DNCP flatten system of cfg-2
subdomains under Jacobi, the additive two-level preconditioner k_pcg2 uses
(M^-1 = I + W E^-1 W^T on the Jacobi-scaled system) and deflation (DEF2:
x0 = Q b, z = (I - Q A) r, which keeps W^T r = 0).

The aggregates follow DESIGN.md section 4 (principal axes, G quantile strips
x G quantile cells, G = min(8, sqrt(n/128)), functions 1, u, v per aggregate,
applied to x and y), without the CTA-boundary splits.

    python tools/deflation_study.py [n_subdomains]
"""
import os
import sys

import numpy as np
from scipy import sparse
from scipy.sparse.linalg import splu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.laplace import dncp_system  # noqa: E402  (study tool: oracle as the system builder)
from oracle.surface import split_mesh  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402


def aggregates(P):
    n = len(P)
    G = max(1, min(8, int(np.sqrt(n / 128))))
    c = P - P.mean(0)
    _, _, vt = np.linalg.svd(c, full_matrices=False)
    a, b = c @ vt[0], c @ vt[1]
    strip = np.minimum((np.argsort(np.argsort(a)) * G) // n, G - 1)
    agg = np.empty(n, dtype=np.int64)
    for s in range(G):
        idx = np.nonzero(strip == s)[0]
        cell = np.minimum((np.argsort(np.argsort(b[idx])) * G) // len(idx), G - 1)
        agg[idx] = s * G + cell
    return agg, a, b


def coarse_basis(free, n, V, agg, a, b):
    """Real-form W: (1, u, v) per aggregate on the x and on the y block."""
    cols, rows, vals = [], [], []
    na = agg.max() + 1
    for k, f in enumerate(free):
        blk, vtx = divmod(f, n)
        g = agg[vtx]
        base = (g * 2 + blk) * 3
        for t, val in enumerate((1.0, a[vtx], b[vtx])):
            rows.append(k)
            cols.append(base + t)
            vals.append(val)
    W = sparse.csr_matrix((vals, (rows, cols)), shape=(len(free), na * 6))
    # centre/scale u, v per aggregate column for conditioning
    W = W.tocsc()
    keep = [j for j in range(W.shape[1]) if W[:, j].nnz > 0]
    return W[:, keep].tocsr()


def pcg(A, b, apply_m, x0=None, project=None, tol=1e-10, maxit=20000):
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - A @ x
    z = apply_m(r)
    if project is not None:
        z = project(z)
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
        if project is not None:
            z = project(z)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return maxit


def main():
    nsub = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    V, F, cuts = gen.height_field_case(1024, 8)
    split = split_mesh(V, F, cuts)
    for i in range(min(nsub, split.n_sub)):
        Vs, Fs, loop = split.sub_V[i], split.sub_F[i], split.loops[i]
        n = len(Vs)
        _, C, rhs, free, _, _, _ = dncp_system(Vs, Fs, loop)
        d = C.diagonal()
        Ds = sparse.diags(1.0 / np.sqrt(d))
        A = (Ds @ C @ Ds).tocsr()
        bh = rhs / np.sqrt(d)
        agg, a, b = aggregates(Vs)
        W = coarse_basis(free, n, Vs, agg, a, b)
        Wh = sparse.diags(np.sqrt(d)) @ W
        E = (Wh.T @ A @ Wh).toarray()
        Ei = np.linalg.pinv(E, rcond=1e-12, hermitian=True)
        Q = lambda v: Wh @ (Ei @ (Wh.T @ v))
        it_j = pcg(A, bh, lambda r: r)
        it_a = pcg(A, bh, lambda r: r + Q(r))
        it_d = pcg(A, bh, lambda r: r, x0=Q(bh), project=lambda z: z - Q(A @ z))
        it_ax = pcg(A, bh, lambda r: r + Q(r), x0=Q(bh))
        om = {w: pcg(A, bh, lambda r, w=w: r + w * Q(r)) for w in (0.5, 2.0, 4.0)}
        Ei32 = Ei.astype(np.float32).astype(np.float64)
        Q32 = lambda v: Wh @ (Ei32 @ (Wh.T @ v))
        it_d32 = pcg(A, bh, lambda r: r, x0=Q32(bh), project=lambda z: z - Q32(A @ z))
        print(f"subdomain {i}: n={n} coarse={W.shape[1]} jacobi={it_j} additive={it_a} additive+x0={it_ax} "
              f"additive(w)={om} deflated={it_d} deflated(fp32 E^-1)={it_d32}", flush=True)


if __name__ == "__main__":
    main()
