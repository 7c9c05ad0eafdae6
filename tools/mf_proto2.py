"""CPU study for the multifrontal solver: nested-dissection variants on a
subdomain system, numeric multifrontal Cholesky in numpy, checked against
SuperLU; prints separator / front sizes and real multiply-adds.

  split = morton : bisection of index ranges of a Morton order
          kd     : recursive median split along the longer bounding-box axis

    python tools/mf_proto2.py [subdomain] [grid] [blocks] [leaf]
"""
import os
import sys

import numpy as np
from scipy import sparse
from scipy.sparse.linalg import spsolve

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle.laplace import cotan_laplacian, half_perimeter_pins  # noqa: E402
from oracle.surface import split_mesh  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402
from mf_proto import morton  # noqa: E402


def nd_tree(A, P2, leaf, split):
    """Nodes of a nested dissection of the graph of A (m x m).
    Returns (list of pivot index arrays in postorder, parent list)."""
    m = A.shape[0]
    ptr, idx = A.indptr, A.indices
    nodes, parent = [], []

    def rec(verts, par_slot):
        # returns node id of this subtree's root
        if len(verts) <= leaf:
            nodes.append(np.sort(verts))
            parent.append(-1)
            return len(nodes) - 1
        if split == "kd":
            ext = P2[verts].max(0) - P2[verts].min(0)
            ax = int(np.argmax(ext))
            o = np.argsort(P2[verts, ax], kind="stable")
        else:
            q = P2[verts]
            lo, hi = q.min(0), q.max(0)
            qi = ((q - lo) / np.maximum(hi - lo, 1e-300) * 65535).astype(np.int64)
            o = np.argsort(morton(qi[:, 0], qi[:, 1]), kind="stable")
        vs = verts[o]
        h = len(vs) // 2
        left, right = vs[:h], vs[h:]
        inr = np.zeros(m, bool)
        inr[right] = True
        sep = np.array([v for v in left if inr[idx[ptr[v]:ptr[v + 1]]].any()], dtype=np.int64)
        insep = np.zeros(m, bool)
        insep[sep] = True
        left = left[~insep[left]]
        kids = []
        if len(left):
            kids.append(rec(left, None))
        if len(right):
            kids.append(rec(right, None))
        nodes.append(np.sort(sep))
        parent.append(-1)
        me = len(nodes) - 1
        for k in kids:
            parent[k] = me
        return me

    rec(np.arange(m), None)
    return nodes, parent


def multifrontal(A, b, nodes, parent):
    """Numeric multifrontal Cholesky + solve; returns x, real multiply-adds, max front."""
    m = A.shape[0]
    order = np.concatenate(nodes)
    eidx = np.empty(m, dtype=np.int64)
    eidx[order] = np.arange(m)
    Ap = A[order][:, order].tocsr()
    bp = b[order]
    cplx = np.iscomplexobj(A.data)
    off = np.cumsum([0] + [len(p) for p in nodes])
    children = [[] for _ in nodes]
    for k, p in enumerate(parent):
        if p >= 0:
            children[p].append(k)
    upd, ups, fac = [], {}, []
    madds, fmax = 0.0, 0
    for k in range(len(nodes)):
        P = np.arange(off[k], off[k + 1])
        top = off[k + 1] - 1
        s = set()
        for r in P:
            s.update(c for c in Ap.indices[Ap.indptr[r]:Ap.indptr[r + 1]] if c > top)
        for c in children[k]:
            s.update(x for x in upd[c] if x > top)
        U = np.array(sorted(s), dtype=np.int64)
        upd.append(U)
        S = np.concatenate([P, U])
        f, sp = len(S), len(P)
        fmax = max(fmax, f)
        loc = {g: i for i, g in enumerate(S)}
        Fm = np.zeros((f, f), complex if cplx else float)
        if sp:
            Fm[:sp, :] = Ap[P][:, S].toarray()
            Fm[:, :sp] = np.conj(Fm[:sp, :].T)
        for c in children[k]:
            ix = [loc[g] for g in upd[c]]
            Fm[np.ix_(ix, ix)] += ups.pop(c)
        u = f - sp
        if sp:
            Lpp = np.linalg.cholesky(Fm[:sp, :sp])
            Lup = np.linalg.solve(Lpp, Fm[:sp, sp:]).conj().T
        else:
            Lpp, Lup = np.zeros((0, 0)), np.zeros((u, 0))
        ups[k] = Fm[sp:, sp:] - Lup @ Lup.conj().T
        fac.append((Lpp, Lup))
        w = sp ** 3 / 6 + u * sp * sp / 2 + u * u * sp / 2
        madds += w * (4 if cplx else 1)
    y = bp.astype(complex).copy()
    for k in range(len(nodes)):
        P = np.arange(off[k], off[k + 1])
        Lpp, Lup = fac[k]
        if len(P):
            y[P] = np.linalg.solve(Lpp, y[P])
            if len(upd[k]):
                y[upd[k]] -= Lup @ y[P]
    for k in reversed(range(len(nodes))):
        P = np.arange(off[k], off[k + 1])
        Lpp, Lup = fac[k]
        if len(P):
            r = y[P] - (Lup.conj().T @ y[upd[k]] if len(upd[k]) else 0)
            y[P] = np.linalg.solve(Lpp.conj().T, r)
    x = np.empty(m, complex)
    x[order] = y
    return x, madds, fmax


def main():
    isub = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    grid = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    leaf = int(sys.argv[4]) if len(sys.argv) > 4 else 48
    V, F, cuts = gen.height_field_case(grid, blocks)
    split = split_mesh(V, F, cuts)
    Vs, Fs, loop = split.sub_V[isub], split.sub_F[isub], np.asarray(split.loops[isub])
    n = len(Vs)
    L = cotan_laplacian(Vs, Fs, n).tocsr()
    p0, p1 = half_perimeter_pins(loop, Vs)
    c = Vs - Vs.mean(0)
    _, _, vt = np.linalg.svd(c, full_matrices=False)
    P2 = np.stack([c @ vt[0], c @ vt[1]], 1)
    # flatten system over U = all but the pins
    U = np.setdiff1d(np.arange(n), [p0, p1])
    pos = np.full(n, -1)
    pos[U] = np.arange(len(U))
    H = L[U][:, U].astype(complex).tolil()
    b = -(L[U][:, [p0, p1]] @ np.array([0j, 1 + 0j]))
    t = {p0: 0j, p1: 1 + 0j}
    for k, v in enumerate(loop):
        if v in t:
            continue
        a, cc = loop[(k + 1) % len(loop)], loop[k - 1]
        if a in t:
            b[pos[v]] -= 0.5j * t[a]
        else:
            H[pos[v], pos[a]] += 0.5j
        if cc in t:
            b[pos[v]] += 0.5j * t[cc]
        else:
            H[pos[v], pos[cc]] -= 0.5j
    H = H.tocsr()
    ref = spsolve(H.tocsc(), b)
    onb = np.zeros(n, bool)
    onb[loop] = True
    I = np.nonzero(~onb)[0]
    Lii = L[I][:, I].tocsr()
    g = np.exp(2j * np.pi * np.arange(len(loop)) / len(loop))
    bI = -(L[I][:, loop] @ g)
    refI = spsolve(Lii.tocsc(), bI)
    for sp in ("morton", "kd"):
        nodes, parent = nd_tree(H, P2[U], leaf, sp)
        x, ma, fm = multifrontal(H, b, nodes, parent)
        e = np.max(np.abs(x - ref)) / np.max(np.abs(ref))
        big = sorted((len(p) for p in nodes), reverse=True)[:4]
        print(f"[{sp}] flatten full ND (complex): nodes {len(nodes)} top separators {big} max front {fm} "
              f"real madds {ma/1e6:.1f}M err {e:.1e}", flush=True)
        nodes, parent = nd_tree(Lii, P2[I], leaf, sp)
        x, ma2, fm = multifrontal(Lii, bI, nodes, parent)
        e = np.max(np.abs(x - refI)) / np.max(np.abs(refI))
        print(f"[{sp}] dirichlet ND (real): max front {fm} real madds {ma2/1e6:.1f}M err {e:.1e}; "
              f"total {(ma + ma2)/1e6:.1f}M", flush=True)


if __name__ == "__main__":
    main()
