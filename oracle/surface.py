"""Oracle: mesh topology and partition (restates `mesh.py:113-223` and
`partition.py:48-137`). TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from dataclasses import dataclass, field

import numpy as np
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components

from .laplace import OracleMeshError


class OraclePartitionError(ValueError):
    pass


def directed_edges(F):
    """All 3m directed edges in the block order (0,1), (1,2), (2,0) of
    `mesh.py:113-116`."""
    F = np.asarray(F, dtype=np.int64)
    return np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]])


def boundary_edges(F):
    """Directed edges whose reverse is absent, in directed-edge order
    (`mesh.py:146-154`)."""
    de = directed_edges(F)
    if len(de) == 0:
        return de
    n = int(de.max()) + 1
    fwd = de[:, 0] * n + de[:, 1]
    rev = de[:, 1] * n + de[:, 0]
    return de[~np.isin(rev, fwd)]


def boundary_loop_list(F):
    """Boundary loops walked from each not-yet-visited boundary vertex in
    increasing order, surface on the left (`mesh.py:174-203`)."""
    bde = boundary_edges(F)
    src = bde[:, 0]
    if len(np.unique(src)) != len(src):
        # first repeated source in directed-edge order, as the dict insert does
        seen = set()
        for a in src.tolist():
            if a in seen:
                raise OracleMeshError(f"pinched boundary at vertex {a}")
            seen.add(a)
    nxt = dict(zip(src.tolist(), bde[:, 1].tolist()))
    loops = []
    seen = set()
    for s in sorted(nxt):
        if s in seen:
            continue
        cyc = [s]
        seen.add(s)
        cur = nxt[s]
        while cur != s:
            if cur in seen or cur not in nxt:
                raise OracleMeshError(f"boundary traversal failed at vertex {cur}")
            cyc.append(cur)
            seen.add(cur)
            cur = nxt[cur]
        loops.append(np.array(cyc, dtype=np.int64))
    return loops


def unique_edge_count(F):
    de = np.sort(directed_edges(F), axis=1)
    if len(de) == 0:
        return 0
    return len(np.unique(de, axis=0))


def topology_class(n_vertices, F):
    """(chi, n_loops, class) as `validate_topology` (`mesh.py:206-223`)."""
    chi = n_vertices - unique_edge_count(F) + len(F)
    try:
        nl = len(boundary_loop_list(F))
    except OracleMeshError:
        return chi, -1, "unsupported"
    if chi == 1 and nl == 1:
        return chi, nl, "disk_type"
    if chi == 2 and nl == 0:
        return chi, nl, "sphere_type"
    return chi, nl, "unsupported"


def normalize_cuts(F, cuts):
    """Sorted-pair cut set; duplicates and non-edges rejected
    (`partition.py:48-59`). Returned in input order."""
    cuts = np.asarray(cuts, dtype=np.int64).reshape(-1, 2)
    norm = np.sort(cuts, axis=1)
    if len(norm) and len(np.unique(norm, axis=0)) != len(norm):
        raise OraclePartitionError("duplicate cut edges")
    if len(norm):
        de = np.sort(directed_edges(F), axis=1)
        n = int(max(de.max(), norm.max())) + 1
        ek = np.unique(de[:, 0] * n + de[:, 1])
        ck = norm[:, 0] * n + norm[:, 1]
        bad = ~np.isin(ck, ek)
        if bad.any():
            e = norm[np.flatnonzero(bad)[0]]
            raise OraclePartitionError(f"cut pair {(int(e[0]) + 1, int(e[1]) + 1)} is not a mesh edge")
    return norm


@dataclass
class SplitResult:
    V: np.ndarray
    F: np.ndarray
    sub_V: list                  # per submesh local vertex positions
    sub_F: list                  # per submesh local faces (int64)
    vertex_maps: list            # local -> parent (sorted)
    face_assignment: np.ndarray  # parent face -> submesh id
    cuts: np.ndarray
    loops: list = field(default_factory=list)            # local boundary loop
    boundary_cycles: list = field(default_factory=list)  # parent ids

    @property
    def n_sub(self):
        return len(self.sub_F)


def face_components(F, cut_norm):
    """Face labels of the adjacency graph minus cut edges
    (`partition.py:100-117`)."""
    F = np.asarray(F, dtype=np.int64)
    m = len(F)
    de = directed_edges(F)
    face = np.concatenate([np.arange(m)] * 3)
    lo = de.min(axis=1)
    hi = de.max(axis=1)
    n = int(F.max()) + 1
    key = lo * n + hi
    order = np.argsort(key, kind="stable")
    ks = key[order]
    pair = np.flatnonzero(ks[1:] == ks[:-1])
    ckeys = cut_norm[:, 0] * n + cut_norm[:, 1] if len(cut_norm) else np.zeros(0, np.int64)
    keep = ~np.isin(ks[pair], ckeys)
    fa = face[order][pair[keep]]
    fb = face[order][pair[keep] + 1]
    g = coo_matrix((np.ones(2 * len(fa)), (np.concatenate([fb, fa]), np.concatenate([fa, fb]))),
                   shape=(m, m))
    return connected_components(g, directed=False)


def split_mesh(V, F, cuts):
    """Partition along cut edges into disk-type submeshes
    (`partition.py:94-137`)."""
    V = np.asarray(V, dtype=np.float64)
    F = np.asarray(F, dtype=np.int64)
    cut_norm = normalize_cuts(F, cuts)
    ncomp, labels = face_components(F, cut_norm)
    sub_V, sub_F, vmaps, loops, cycles = [], [], [], [], []
    nvert = len(V)
    # faces grouped by label, each group in increasing face order (= F[labels == ci])
    order = np.argsort(labels, kind="stable")
    bounds = np.searchsorted(labels[order], np.arange(ncomp + 1))
    remap = np.full(nvert, -1, dtype=np.int64)
    for ci in range(ncomp):
        f = F[order[bounds[ci]:bounds[ci + 1]]]
        used = np.unique(f)
        remap[used] = np.arange(len(used))
        lf = remap[f]
        remap[used] = -1
        chi, nl, cls = topology_class(len(used), lf)
        if cls != "disk_type":
            raise OraclePartitionError(
                f"component {ci} is {cls} (chi={chi}, {nl} loops); adjust the cut set")
        loop = boundary_loop_list(lf)[0]
        sub_V.append(V[used])
        sub_F.append(lf)
        vmaps.append(used)
        loops.append(loop)
        cycles.append(used[loop])
    return SplitResult(V, F, sub_V, sub_F, vmaps, labels.astype(np.int64), cut_norm,
                       loops, cycles)


def single_domain(V, F):
    """The K = 1 'partition' `parameterize` uses without cuts
    (`pipeline.py:143-150`)."""
    V = np.asarray(V, dtype=np.float64)
    F = np.asarray(F, dtype=np.int64)
    loop = boundary_loop_list(F)[0]
    return SplitResult(V, F, [V], [F], [np.arange(len(V))],
                       np.zeros(len(F), dtype=np.int64), np.zeros((0, 2), np.int64),
                       [loop], [loop])
