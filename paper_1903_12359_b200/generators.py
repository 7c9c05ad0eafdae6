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


def jittered_grid_case(n, jitter=0.45, amp=0.1, sigma=0.1, seed=0, n_bumps=3, strips=0):
    """(V, F, cuts) of an n x n grid whose interior vertices are displaced in
    the plane by up to `jitter` cells (uniform, seeded) and lifted by
    `n_bumps` Gaussian bumps of amplitude `amp`, width `sigma`, centres in
    [0.2, 0.8]^2. The obtuse triangles give negative cotangent weights, so
    the harmonic maps fold and the pipeline's fold-over repair
    (pipeline.py:88-102) runs. strips > 1: that many vertical strips
    (cuts), else one domain (cuts = None)."""
    V, F = flat_grid_arrays(n - 1)
    rng = np.random.default_rng(seed)
    h = 1.0 / (n - 1)
    x, y = V[:, 0], V[:, 1]
    inner = (x > 1e-9) & (x < 1 - 1e-9) & (y > 1e-9) & (y < 1 - 1e-9)
    V[inner, :2] += rng.uniform(-jitter * h, jitter * h, (int(inner.sum()), 2))
    for _ in range(n_bumps):
        cx, cy = rng.uniform(0.2, 0.8, 2)
        V[:, 2] += amp * np.exp(-((V[:, 0] - cx) ** 2 + (V[:, 1] - cy) ** 2) / (2 * sigma ** 2))
    cuts = cuts_from_face_labels(F, strip_face_labels(n, strips)) if strips > 1 else None
    return V, F, cuts


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


# ---------------------------------------------------------------------------
# BASELINE cfg 3 (Delaunay disk) and cfg 4 (spherical-harmonic icosphere).
# The construction details BASELINE leaves open are pinned here and listed in
# the noise smoothing (mean over the 16 nearest neighbours), the
# interior radius margin (interior points stay inside the 256-gon, so the
# convex hull is exactly the boundary circle's polygon), the harmonic field
# normalisation (max |f| = 1) and the k-means setup (scikit-learn, n_init=1).

def _kmeans_labels(X, k, seed):
    from sklearn.cluster import KMeans
    km = KMeans(n_clusters=k, random_state=seed, n_init=1, max_iter=50).fit(X)
    return km.cluster_centers_


def _face_labels_nearest(centroids, centers):
    from scipy.spatial import cKDTree
    return cKDTree(centers).query(centroids)[1].astype(np.int64)


def delaunay_disk(n_points=500_000, n_boundary=256, seed=0, noise=0.02):
    """cfg 3 mesh: n_boundary points on the unit circle, the rest uniform in
    the disk (r = sqrt(U)), Delaunay-triangulated (CCW), lifted to
    z = 0.5 (1 - r^2) + noise * (N(0,1) averaged over 16 nearest points)."""
    from scipy.spatial import Delaunay, cKDTree
    rng = np.random.default_rng(seed)
    nin = n_points - n_boundary
    margin = np.cos(np.pi / n_boundary) * (1.0 - 1e-4)
    r = np.sqrt(rng.uniform(0.0, 1.0, nin)) * margin
    th = rng.uniform(0.0, 2.0 * np.pi, nin)
    tb = 2.0 * np.pi * np.arange(n_boundary) / n_boundary
    xy = np.concatenate([np.stack([np.cos(tb), np.sin(tb)], 1), np.stack([r * np.cos(th), r * np.sin(th)], 1)])
    F = Delaunay(xy).simplices.astype(np.int64)
    a, b, c = xy[F[:, 0]], xy[F[:, 1]], xy[F[:, 2]]
    neg = ((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])) < 0
    F[neg] = F[neg][:, [0, 2, 1]]
    rr = np.hypot(xy[:, 0], xy[:, 1])
    eta = rng.standard_normal(len(xy))
    nbr = cKDTree(xy).query(xy, k=16)[1]
    z = 0.5 * (1.0 - rr * rr) + noise * eta[nbr].mean(axis=1)
    V = np.column_stack([xy, z]).astype(np.float64)
    return V, F.astype(np.int32)


def repair_pinches(F, labels, n_vertices, max_rounds=20):
    """Make every label region a manifold surface: a vertex where one label
    touches in two or more separate fans (label changes around the vertex
    exceed its distinct labels) takes the majority label for all its faces;
    repeated until no such vertex is left."""
    F = np.asarray(F, dtype=np.int64)
    labels = np.asarray(labels, dtype=np.int64).copy()
    m = len(F)
    de = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]])
    fid = np.tile(np.arange(m), 3)
    key = np.minimum(de[:, 0], de[:, 1]) * n_vertices + np.maximum(de[:, 0], de[:, 1])
    order = np.argsort(key, kind="stable")
    ks = key[order]
    pair = np.nonzero(ks[1:] == ks[:-1])[0]
    f1, f2 = fid[order[pair]], fid[order[pair + 1]]      # interior edges: their two faces
    ev = np.stack([ks[pair] // n_vertices, ks[pair] % n_vertices], 1)
    vf = np.repeat(np.arange(m), 3)
    vv = F.reshape(-1)
    for _ in range(max_rounds):
        chg = labels[f1] != labels[f2]
        changes = np.bincount(ev[chg].ravel(), minlength=n_vertices)
        pairs = np.unique(vv * (labels.max() + 1) + labels[vf])
        distinct = np.bincount(pairs // (labels.max() + 1), minlength=n_vertices)
        bnd = np.zeros(n_vertices, dtype=bool)
        single = np.ones(len(key), dtype=bool)
        single[order[pair]] = False
        single[order[pair + 1]] = False
        bnd[de[single].ravel()] = True
        # interior vertex: changes == distinct (cyclic) when each label is one fan
        # (one label: 0 changes); boundary vertex: changes == distinct - 1
        expect = np.where(bnd, distinct - 1, np.where(distinct > 1, distinct, 0))
        bad = np.nonzero(changes > expect)[0]
        if len(bad) == 0:
            return labels
        for v in bad:
            fs = vf[vv == v]
            vals, cnt = np.unique(labels[fs], return_counts=True)
            labels[fs] = vals[np.argmax(cnt)]
    return labels


def cfg3(seed=0, n_points=500_000, n_clusters=128):
    """BASELINE cfg 3: Delaunay disk, 128 k-means subdomains on xy (face
    centroid -> nearest centre, pinched regions repaired), disk mode."""
    V, F = delaunay_disk(n_points, 256, seed)
    cent = V[F].mean(axis=1)[:, :2]
    centers = _kmeans_labels(V[:, :2], n_clusters, seed)
    labels = repair_pinches(F, _face_labels_nearest(cent, centers), len(V))
    return V, F, cuts_from_face_labels(F, labels)


def real_sph_harm_field(P, degree=8, seed=0):
    """sum_{l<=degree, m} c_lm Y_lm(P) with c_lm ~ N(0,1) (seeded), real
    orthonormal harmonics, normalised to max |f| = 1 over the points P."""
    from scipy.special import sph_harm_y
    rng = np.random.default_rng(seed)
    x, y, z = P[:, 0], P[:, 1], P[:, 2]
    theta = np.arccos(np.clip(z / np.linalg.norm(P, axis=1), -1.0, 1.0))
    phi = np.arctan2(y, x)
    f = np.zeros(len(P))
    for l in range(degree + 1):
        for m in range(-l, l + 1):
            Y = sph_harm_y(l, abs(m), theta, phi)
            if m < 0:
                Yr = np.sqrt(2.0) * (-1.0) ** m * Y.imag
            elif m == 0:
                Yr = Y.real
            else:
                Yr = np.sqrt(2.0) * (-1.0) ** m * Y.real
            f += rng.standard_normal() * Yr
    return f / np.max(np.abs(f))


def harmonic_sphere(subdiv=9, amp=0.3, degree=8, seed=0):
    """cfg 4 mesh: icosphere with radius 1 + amp * f(direction)."""
    V, F = icosphere_arrays(subdiv)
    f = real_sph_harm_field(V, degree, seed)
    return V * (1.0 + amp * f)[:, None], F


def cfg4(seed=0, subdiv=9, n_clusters=256):
    """BASELINE cfg 4: spherical-harmonic icosphere (subdivision 9), 256
    k-means subdomains on the unit directions, sphere mode."""
    V, F = harmonic_sphere(subdiv, 0.3, 8, seed)
    U = V / np.linalg.norm(V, axis=1, keepdims=True)
    centers = _kmeans_labels(U, n_clusters, seed)
    cent = U[F].mean(axis=1)
    labels = repair_pinches(F, _face_labels_nearest(cent, centers), len(V))
    return V, F, cuts_from_face_labels(F, labels)

