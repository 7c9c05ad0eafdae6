"""CPU prototype of the batched multifrontal solver (direct.cu): geometric
nested dissection of a subdomain's interior by index-range bisection of a
Morton order, boundary loop eliminated last (complex root front), and the
numeric multifrontal factor / solves in numpy. Checks the DNCP flatten and
the Dirichlet solve against SuperLU and prints front sizes and flop counts.

    python tools/mf_proto.py [subdomain] [grid] [blocks] [leaf]
"""
import os
import sys
import time

import numpy as np
from scipy import sparse
from scipy.sparse.linalg import spsolve

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.laplace import cotan_laplacian, half_perimeter_pins  # noqa: E402
from oracle.surface import split_mesh  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402


def morton(ix, iy):
    def spread(x):
        x = x.astype(np.uint64) & np.uint64(0xFFFF)
        x = (x | (x << np.uint64(8))) & np.uint64(0x00FF00FF)
        x = (x | (x << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        x = (x | (x << np.uint64(2))) & np.uint64(0x33333333)
        x = (x | (x << np.uint64(1))) & np.uint64(0x55555555)
        return x
    return spread(ix) | (spread(iy) << np.uint64(1))


def nd_order(P2, interior, adj_ptr, adj_idx, leaf):
    """Index-range bisection of the Morton order of the interior vertices.
    Returns node_of (per interior position), depth, pos_of (vertex -> pos)."""
    nI = len(interior)
    lo, hi = P2[interior].min(0), P2[interior].max(0)
    q = ((P2[interior] - lo) / np.maximum(hi - lo, 1e-300) * 65535).astype(np.int64)
    key = morton(q[:, 0], q[:, 1])
    perm = np.argsort(key, kind="stable")
    verts = interior[perm]                 # pos -> vertex
    pos_of = np.full(len(P2), -1, dtype=np.int64)
    pos_of[verts] = np.arange(nI)
    depth = 0
    while (nI >> depth) > leaf:
        depth += 1
    node_of = np.zeros(nI, dtype=np.int64)  # 0: unassigned
    for lev in range(depth):
        # range of every position at this level
        for p in range(nI):
            if node_of[p]:
                continue
            a, b, h = 0, nI, 1
            for _ in range(lev):
                m = (a + b) // 2
                if p < m:
                    b, h = m, 2 * h
                else:
                    a, h = m, 2 * h + 1
            m = (a + b) // 2
            if p >= m:
                continue
            v = verts[p]
            for w in adj_idx[adj_ptr[v]:adj_ptr[v + 1]]:
                pw = pos_of[w]
                if pw >= m and pw < b and node_of[pw] == 0:
                    node_of[p] = h
                    break
    for p in range(nI):
        if node_of[p] == 0:
            a, b, h = 0, nI, 1
            for _ in range(depth):
                m = (a + b) // 2
                if p < m:
                    b, h = m, 2 * h
                else:
                    a, h = m, 2 * h + 1
            node_of[p] = h
    return node_of, depth, verts, pos_of


def postorder(depth):
    out = []

    def rec(h, lev):
        if lev < depth:
            rec(2 * h, lev + 1)
            rec(2 * h + 1, lev + 1)
        out.append(h)
    rec(1, 0)
    return out


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
    onb = np.zeros(n, bool)
    onb[loop] = True
    interior = np.nonzero(~onb)[0]
    bnd = np.array([v for v in loop if v not in (p0, p1)])
    # adjacency
    Lc = L.tocsr()
    adj_ptr, adj_idx = Lc.indptr, Lc.indices
    c = Vs - Vs.mean(0)
    _, _, vt = np.linalg.svd(c, full_matrices=False)
    P2 = np.stack([c @ vt[0], c @ vt[1]], 1)
    t0 = time.time()
    node_of, depth, verts, pos_of = nd_order(P2, interior, adj_ptr, adj_idx, leaf)
    print(f"n={n} interior={len(interior)} boundary unknowns={len(bnd)} depth={depth} ordering {time.time()-t0:.1f}s")
    post = postorder(depth)
    rank = {h: i for i, h in enumerate(post)}
    # elimination order: interior by (postorder rank of node, pos), then boundary
    key = np.array([rank[h] for h in node_of]) * (1 << 32) + np.arange(len(node_of))
    order_pos = np.argsort(key, kind="stable")
    elim = np.concatenate([verts[order_pos], bnd])      # elimination index -> vertex
    eidx = np.full(n, -1, dtype=np.int64)
    eidx[elim] = np.arange(len(elim))
    # the unknown system H over U = all but pins, permuted to elimination order
    U = elim
    nxt = np.roll(loop, -1)
    prv = np.roll(loop, 1)
    Luu = L[U][:, U].astype(complex).tolil()
    pins = {p0: 0j, p1: 1 + 0j}
    b = -(L[U][:, [p0, p1]] @ np.array([0j, 1 + 0j]))
    for k, v in enumerate(loop):
        if v in pins:
            continue
        r = eidx[v]
        a, cc = nxt[k], prv[k]
        if a in pins:
            b[r] -= 0.5j * pins[a]
        else:
            Luu[r, eidx[a]] += 0.5j
        if cc in pins:
            b[r] += 0.5j * pins[cc]
        else:
            Luu[r, eidx[cc]] -= 0.5j
    H = Luu.tocsr()
    ref = spsolve(H.tocsc(), b)
    # nodes: pivots per node (elimination indices), children
    nodes = post + [0]                     # 0 = complex boundary root
    piv = {h: [] for h in nodes}
    for p in order_pos:
        piv[node_of[p]].append(eidx[verts[p]])
    piv[0] = list(range(len(interior), len(elim)))
    parent = {h: (h // 2 if h > 1 else 0) for h in post}
    children = {h: [] for h in nodes}
    for h in post:
        children[parent[h]].append(h)
    # symbolic: struct = pivots + update set (ancestor elimination indices)
    Hc = H.tocsr()
    upd = {}
    first = {}
    for h in nodes:
        s = set()
        lo = min(piv[h]) if piv[h] else 0
        top = max(piv[h]) if piv[h] else -1
        for r in piv[h]:
            for cidx in Hc.indices[Hc.indptr[r]:Hc.indptr[r + 1]]:
                if cidx > top:
                    s.add(int(cidx))
        for ch in children[h]:
            s.update(x for x in upd[ch] if x > top)
        upd[h] = sorted(s)
        first[h] = lo
    # numeric
    fronts = {}
    flops = 0
    fmax = 0
    ups = {}
    Lfac = {}
    for h in nodes:
        P = piv[h]
        S = P + upd[h]
        f = len(S)
        fmax = max(fmax, f)
        loc = {g: i for i, g in enumerate(S)}
        Fm = np.zeros((f, f), complex)
        sub = Hc[P][:, S].toarray()
        Fm[:len(P), :] += sub
        Fm[:, :len(P)] = np.conj(Fm[:len(P), :].T)
        for ch in children[h]:
            idx = [loc[g] for g in upd[ch]]
            Fm[np.ix_(idx, idx)] += ups[ch]
            del ups[ch]
        s = len(P)
        if s:
            Lpp = np.linalg.cholesky(Fm[:s, :s])
            Lup = np.linalg.solve(Lpp, Fm[:s, s:]).conj().T
        else:
            Lpp = np.zeros((0, 0), complex)
            Lup = np.zeros((f, 0), complex)
        ups[h] = Fm[s:, s:] - Lup @ Lup.conj().T
        Lfac[h] = (Lpp, Lup)
        u = f - s
        flops += s ** 3 / 3 + u * s * s + u * u * s
    # solve
    y = b.astype(complex).copy()
    for h in nodes:
        P = piv[h]
        Lpp, Lup = Lfac[h]
        yp = np.linalg.solve(Lpp, y[P]) if P else y[P]
        y[P] = yp
        if upd[h]:
            y[upd[h]] -= Lup @ yp
    x = y.copy()
    for h in reversed(nodes):
        P = piv[h]
        Lpp, Lup = Lfac[h]
        rhs = x[P] - (Lup.conj().T @ x[upd[h]] if upd[h] else 0)
        if P:
            x[P] = np.linalg.solve(Lpp.conj().T, rhs)
    err = np.max(np.abs(x - ref)) / np.max(np.abs(ref))
    res = np.linalg.norm(H @ x - b) / np.linalg.norm(b)
    sizes = sorted(((len(piv[h]), len(upd[h])) for h in nodes), key=lambda t: -(t[0] + t[1]))
    print(f"nodes={len(nodes)} max front={fmax} multiply-adds={flops/1e6:.1f}M (complex)")
    print("largest fronts (pivots, update):", sizes[:8])
    print(f"flatten: rel err vs SuperLU {err:.2e}, residual {res:.2e}")
    # Dirichlet solve with the leading (interior) block of the same factor
    g = np.exp(2j * np.pi * np.arange(len(loop)) / len(loop))
    bI = -(L[elim[:len(interior)]][:, loop] @ g)
    refI = spsolve(L[elim[:len(interior)]][:, elim[:len(interior)]].tocsc(), bI)
    y = np.zeros(len(elim), complex)
    y[:len(interior)] = bI
    for h in post:
        Lpp, Lup = Lfac[h]
        yp = np.linalg.solve(Lpp, y[piv[h]]) if piv[h] else y[piv[h]]
        y[piv[h]] = yp
        if upd[h]:
            y[upd[h]] -= Lup @ yp
    y[len(interior):] = 0
    for h in reversed(post):
        Lpp, Lup = Lfac[h]
        rhs = y[piv[h]] - (Lup.conj().T @ y[upd[h]] if upd[h] else 0)
        if piv[h]:
            y[piv[h]] = np.linalg.solve(Lpp.conj().T, rhs)
    errI = np.max(np.abs(y[:len(interior)] - refI)) / np.max(np.abs(refI))
    print(f"dirichlet: rel err vs SuperLU {errI:.2e}")


if __name__ == "__main__":
    main()
