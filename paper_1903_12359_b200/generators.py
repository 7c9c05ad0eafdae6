"""Seeded synthetic inputs for the BASELINE configurations.

The reference ships Python-loop fixture generators (`pkg/src/pgcp/shapes.py`)
and none of the BASELINE meshes; these are vectorised numpy generators that
follow the construction spelled out in BASELINE.json / SURVEY.md §8(d):

* `height_field_grid` -- cfg 1 / 2 / 5: regular n x n grid on [0,1]^2, two
  right triangles per cell in the vertex/face order of `shapes.flat_grid`
  (`shapes.py:12-32`), z = sum of Gaussian bumps drawn in the order
  cx, cy, s, a of `shapes.bumpy_grid` (`shapes.py:36-48`) with BASELINE's
  ranges (centres U[0,1], sigma U[0.05,0.2], amplitude U[-0.2,0.2]).
* `block_face_labels` -- cell-aligned kx x ky blocks.
* `cuts_from_face_labels` -- interior edges whose two faces carry different
  labels (same output as `shapes.cuts_from_face_labels`, `shapes.py:113-131`:
  sorted (min, max) pairs).

These are input generators only: they run on the host, outside every timed
region, exactly like the reference's own fixture code.
"""

import numpy as np

__all__ = ["flat_grid_arrays", "height_field_grid", "block_face_labels",
           "strip_face_labels", "cuts_from_face_labels", "cfg1", "cfg2",
           "height_field_case", "icosphere_arrays", "row_tree_schedule_order"]


def flat_grid_arrays(nx, ny=None, width=1.0, height=1.0):
    """(V, F) of the regular grid with nx x ny cells (`shapes.py:12-32` layout).

    Vertex id = iy * (nx + 1) + ix (x fastest); per cell (iy outer, ix inner)
    faces [v00, v10, v11] and [v00, v11, v01]. F is int32.
    """
    if ny is None:
        ny = nx
    xs = np.linspace(0.0, width, nx + 1)
    ys = np.linspace(0.0, height, ny + 1)
    gx, gy = np.meshgrid(xs, ys, indexing="xy")
    V = np.column_stack([gx.ravel(), gy.ravel(), np.zeros(gx.size)])
    iy, ix = np.meshgrid(np.arange(ny, dtype=np.int64),
                         np.arange(nx, dtype=np.int64), indexing="ij")
    v00 = (iy * (nx + 1) + ix).ravel()
    v10 = v00 + 1
    v01 = v00 + (nx + 1)
    v11 = v01 + 1
    F = np.empty((2 * v00.size, 3), dtype=np.int32)
    F[0::2, 0] = v00
    F[0::2, 1] = v10
    F[0::2, 2] = v11
    F[1::2, 0] = v00
    F[1::2, 1] = v11
    F[1::2, 2] = v01
    return V, F


def height_field_grid(n=100, n_bumps=8, seed=0, amp=0.2, s_lo=0.05, s_hi=0.2):
    """BASELINE height field on an n x n *vertex* grid ((n-1)^2 cells)."""
    V, F = flat_grid_arrays(n - 1)
    rng = np.random.default_rng(seed)
    x = V[:, 0]
    y = V[:, 1]
    z = np.zeros(len(V))
    for _ in range(n_bumps):
        cx, cy = rng.uniform(0.0, 1.0, size=2)
        s = rng.uniform(s_lo, s_hi)
        a = rng.uniform(-amp, amp)
        z += a * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * s * s))
    V[:, 2] = z
    return V, F


def block_face_labels(n, kx, ky=None):
    """Cell-aligned kx x ky block label per face of an n x n vertex grid.

    label = (ix * kx // (n - 1)) + kx * (iy * ky // (n - 1)) with
    cell = face // 2, ix = cell % (n - 1), iy = cell // (n - 1).
    """
    if ky is None:
        ky = kx
    c = n - 1
    cell = np.arange(2 * c * c, dtype=np.int64) // 2
    ix = cell % c
    iy = cell // c
    return (ix * kx // c) + kx * (iy * ky // c)


def strip_face_labels(n, k):
    """k vertical cell-aligned strips of an n x n vertex grid."""
    c = n - 1
    cell = np.arange(2 * c * c, dtype=np.int64) // 2
    return (cell % c) * k // c


def cuts_from_face_labels(F, labels):
    """Interior edges separating faces with different labels, as sorted
    unique (min, max) int64 pairs (the output of `shapes.py:113-131`)."""
    F = np.asarray(F, dtype=np.int64)
    labels = np.asarray(labels)
    m = len(F)
    a = np.concatenate([F[:, 0], F[:, 1], F[:, 2]])
    b = np.concatenate([F[:, 1], F[:, 2], F[:, 0]])
    face = np.concatenate([np.arange(m)] * 3)
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    nv = int(F.max()) + 1 if m else 0
    key = lo * nv + hi
    order = np.argsort(key, kind="stable")
    ks = key[order]
    fs = face[order]
    same = ks[1:] == ks[:-1]
    idx = np.nonzero(same)[0]
    differ = labels[fs[idx]] != labels[fs[idx + 1]]
    cut_keys = ks[idx[differ]]
    out = np.column_stack([cut_keys // nv, cut_keys % nv]).astype(np.int64)
    return out.reshape(-1, 2)


def height_field_case(n, k, n_bumps=8, seed=0, layout="blocks"):
    """(V, F, cuts) of an n x n height field split into k x k blocks
    (layout="blocks") or k vertical strips (layout="strips")."""
    V, F = height_field_grid(n, n_bumps=n_bumps, seed=seed)
    if layout == "blocks":
        lab = block_face_labels(n, k)
    elif layout == "strips":
        lab = strip_face_labels(n, k)
    else:
        raise ValueError(f"unknown layout {layout!r}")
    return V, F, cuts_from_face_labels(F, lab)


def cfg1(seed=0):
    """BASELINE configs[0]: 100 x 100 height field, 8 bumps, 2 x 2 blocks."""
    return height_field_case(100, 2, n_bumps=8, seed=seed)


def cfg2(seed=0):
    """BASELINE configs[1]: 1024 x 1024 height field, 8 bumps, 8 x 8 blocks."""
    return height_field_case(1024, 8, n_bumps=8, seed=seed)


def row_tree_schedule_order(kx, ky):
    """Submesh pairs of the balanced "rows -> strips, then pairwise tree"
    weld order for a kx x ky cell-aligned block layout (SURVEY §7 hard part 2).

    Block (bx, by) is submesh by * kx + bx, which is the component order
    `partition_mesh` assigns (labels ordered by minimum face index).
    Returns a list of (rep_a, rep_b) component-representative pairs.
    """
    order = []
    for r in range(ky):
        for bx in range(1, kx):
            order.append((r * kx, r * kx + bx))
    span = 1
    while span < ky:
        for r in range(0, ky, 2 * span):
            if r + span < ky:
                order.append((r * kx, (r + span) * kx))
        span *= 2
    return order


def pairwise_tree_schedule_order(kx, ky):
    """Fully balanced variant: blocks of a row are merged pairwise (spans
    1, 2, 4, ...), then the rows pairwise as in `row_tree_schedule_order`.
    log2(kx) + log2(ky) weld levels instead of (kx - 1) + log2(ky); every
    merge still glues one contiguous arc (the edge between two adjacent
    blocks, or the full row edge)."""
    order = []
    span = 1
    while span < kx:
        for r in range(ky):
            for bx in range(0, kx, 2 * span):
                if bx + span < kx:
                    order.append((r * kx + bx, r * kx + bx + span))
        span *= 2
    span = 1
    while span < ky:
        for r in range(0, ky, 2 * span):
            if r + span < ky:
                order.append((r * kx, (r + span) * kx))
        span *= 2
    return order


def quadtree_schedule_order(kx, ky):
    """Quadtree weld order: horizontal and vertical pairwise merges
    alternate (blocks -> 2x1 -> 2x2 -> 4x2 -> 4x4 ...), so components stay
    near-square and every shared arc is one straight run of block edges.
    On 8x8 blocks the arcs are 1, 2, 2, 4, 4, 8 block edges long (rows then
    strips: 1, 1, 1, 8, 8, 8), i.e. 22 % fewer serial weld records, and the
    welded map is less distorted (measured with the oracle at 129^2 and 257^2:
    mean |d| 0.147 vs 0.223 and 0.074 vs 0.111 degrees)."""
    order = []
    sx, sy = 1, 1
    while sx < kx or sy < ky:
        if sx <= sy and sx < kx:
            for by in range(0, ky, sy):
                for bx in range(0, kx, 2 * sx):
                    if bx + sx < kx:
                        order.append((by * kx + bx, by * kx + bx + sx))
            sx *= 2
        else:
            for by in range(0, ky, 2 * sy):
                for bx in range(0, kx, sx):
                    if by + sy < ky:
                        order.append((by * kx + bx, (by + sy) * kx + bx))
            sy *= 2
    return order


# ---------------------------------------------------------------------------
# icosphere (vectorised edge-midpoint subdivision; `shapes.py:52-92` ordering
# of new vertices is NOT reproduced -- only the geometry class)


_T = (1.0 + 5.0 ** 0.5) / 2.0
_ICO_V = np.array([
    [-1, _T, 0], [1, _T, 0], [-1, -_T, 0], [1, -_T, 0],
    [0, -1, _T], [0, 1, _T], [0, -1, -_T], [0, 1, -_T],
    [_T, 0, -1], [_T, 0, 1], [-_T, 0, -1], [-_T, 0, 1]], dtype=np.float64)
_ICO_F = np.array([
    [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
    [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
    [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
    [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)


def icosphere_arrays(subdiv):
    """Unit icosphere (V float64, F int32), outward oriented."""
    V = _ICO_V / np.linalg.norm(_ICO_V, axis=1, keepdims=True)
    F = _ICO_F.copy()
    for _ in range(subdiv):
        nv = len(V)
        e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]])
        lo = np.minimum(e[:, 0], e[:, 1])
        hi = np.maximum(e[:, 0], e[:, 1])
        key = lo * nv + hi
        uniq, inv = np.unique(key, return_inverse=True)
        mid = V[uniq // nv] + V[uniq % nv]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        m = len(F)
        ab = nv + inv[:m]
        bc = nv + inv[m:2 * m]
        ca = nv + inv[2 * m:]
        a, b, c = F[:, 0], F[:, 1], F[:, 2]
        F = np.concatenate([np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
                            np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)])
        V = np.concatenate([V, mid])
    return V, F.astype(np.int32)
