"""Interior reconstruction and global assembly (drop-in for `assemble.py`).

`harmonic_solve` runs on the device (pcg.cu); the quasi-conformal fold-over
repair (`face_layout`, `beltrami_per_face`, `qc_correct`,
assemble.py:53-217) runs on the device as well (repair.cu), batched over
every folded submesh by the pipeline; `stitch_global` is the device stitch
(metrics.cu).
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .errors import SolveError

MU_CAP = 0.95  # assemble.py:20


def harmonic_solve(mesh, boundary_idx, boundary_vals, residual_tol=1e-10, rtol=1e-10):
    """Dirichlet harmonic extension (assemble.py:23-50) on the device."""
    n = mesh.n_vertices
    bidx = np.asarray(boundary_idx, dtype=np.int64)
    bvals = np.asarray(boundary_vals, dtype=np.complex128)
    if not np.all(np.isfinite(bvals.real) & np.isfinite(bvals.imag)):
        raise SolveError("non-finite boundary data for harmonic solve")
    z = np.zeros(n, dtype=np.complex128)
    z[bidx] = bvals
    if len(np.setdiff1d(np.arange(n), bidx)) == 0:
        return z
    b = mesh.batch()
    info = b.info()
    if info[nat.INFO_SUM_N] != n:
        raise SolveError("singular harmonic system (unreferenced vertices)")
    if info[nat.INFO_K] == 1:
        gid = bidx
    else:  # parent -> local-vertex ids (each vertex lies in one component)
        vmap = b.host(nat.ARR_VMAP, torch.int32)
        inv = np.empty(n, dtype=np.int64)
        inv[vmap] = np.arange(len(vmap))
        gid = inv[bidx]
    zz, _ = b.harmonic(gid.astype(np.int32), bvals, rtol=rtol, contract_tol=residual_tol)
    out = zz.cpu().numpy()
    if info[nat.INFO_K] != 1:
        vmap = b.host(nat.ARR_VMAP, torch.int32)
        res = np.empty(n, dtype=np.complex128)
        res[vmap] = out
        out = res
    return out


def signed_areas(coords, faces):
    z = np.asarray(coords, dtype=np.complex128)[np.asarray(faces)]
    d1 = z[:, 1] - z[:, 0]
    d2 = z[:, 2] - z[:, 0]
    return 0.5 * (d1.real * d2.imag - d1.imag * d2.real)


def stereographic_inverse(z):
    """Plane (+inf) -> unit sphere, 0 -> south pole (assemble.py:224-245)."""
    z = np.atleast_1d(np.asarray(z, dtype=np.complex128))
    out = np.empty((len(z), 3))
    infm = np.isinf(z.real) | np.isinf(z.imag)
    out[infm] = (0.0, 0.0, 1.0)
    zf = z[~infm]
    big = np.abs(zf) > 1.0
    res = np.empty((len(zf), 3))
    zs = zf[~big]
    s = np.abs(zs) ** 2
    res[~big, 0] = 2 * zs.real / (1 + s)
    res[~big, 1] = 2 * zs.imag / (1 + s)
    res[~big, 2] = (s - 1) / (1 + s)
    w = 1.0 / zf[big]
    sw = np.abs(w) ** 2
    res[big, 0] = 2 * w.real / (1 + sw)
    res[big, 1] = -2 * w.imag / (1 + sw)
    res[big, 2] = (1 - sw) / (1 + sw)
    out[~infm] = res
    return out


def stereographic_project(p):
    """Unit sphere -> plane, north pole -> infinity (assemble.py:248-256)."""
    p = np.atleast_2d(np.asarray(p, dtype=np.float64))
    den = 1.0 - p[:, 2]
    out = np.empty(len(p), dtype=np.complex128)
    pole = den == 0
    out[pole] = complex(np.inf, 0.0)
    out[~pole] = (p[~pole, 0] + 1j * p[~pole, 1]) / den[~pole]
    return out


def spherical_flips(points3, faces):
    p = np.asarray(points3)[np.asarray(faces)]
    det = np.einsum("ij,ij->i", p[:, 0], np.cross(p[:, 1], p[:, 2]))
    return np.nonzero(det < 0)[0]


@dataclass
class GlobalParam:
    mode: str
    coords: np.ndarray
    flipped_faces: np.ndarray
    provenance: np.ndarray
    seam_max_dev: float = 0.0
    diagnostics: dict = field(default_factory=dict)

    @property
    def uv(self):
        z = np.asarray(self.coords, dtype=np.complex128)
        return np.column_stack([z.real, z.imag])


# ---------------------------------------------------------------------------
# Fold-over repair (assemble.py:53-217), on the device


def _stream():
    from .device import stream_handle
    return stream_handle()


def _p(t):
    from .device import ptr
    return ptr(t)


def face_layout(mesh):
    """Isometric per-face 2D coordinates of a 3D mesh, (m, 3) complex: corner
    0 at the origin, corner 1 on the positive real axis (assemble.py:53-67)."""
    from .device import device, to_dev
    V = to_dev(np.asarray(mesh.vertices, dtype=np.float64), torch.float64)
    F = to_dev(np.asarray(mesh.faces), torch.int32)
    m = int(F.shape[0])
    out = torch.empty((m, 3), dtype=torch.complex128, device=device())
    nat.check(nat.lib().pgcp_face_layout(_p(V), _p(F), m, _p(out), _stream()))
    return out.cpu().numpy()


def beltrami_per_face(source, target, faces=None):
    """Per-face Beltrami coefficient of the piecewise-linear map source ->
    target (assemble.py:74-92): per-vertex complex coordinates with `faces`,
    or (m, 3) per-face corner arrays. SolveError on a degenerate source
    triangle; fz == 0 gives inf."""
    from .device import device, to_dev
    src = to_dev(np.asarray(source, dtype=np.complex128).reshape(-1), torch.complex128)
    tgt = to_dev(np.asarray(target, dtype=np.complex128).reshape(-1), torch.complex128)
    if faces is not None:
        fd = to_dev(np.asarray(faces), torch.int32).reshape(-1)
        m = fd.numel() // 3
        sf = tf = fd
    else:
        m = src.numel() // 3
        sf = tf = None
    mu = torch.empty(m, dtype=torch.complex128, device=device())
    if m == 0:
        return mu.cpu().numpy()
    bad = ctypes.c_int64(-1)
    nat.check(nat.lib().pgcp_beltrami(_p(src), _p(sf) if sf is not None else None, _p(tgt),
                                      _p(tf) if tf is not None else None, m, _p(mu), ctypes.byref(bad), _stream()))
    return mu.cpu().numpy()


@dataclass
class BijectivityReport:
    bad_faces: np.ndarray
    max_mu: float
    threshold: float

    @property
    def ok(self):
        return len(self.bad_faces) == 0


def check_bijectivity(mu, threshold=0.99):
    """Faces whose Beltrami magnitude reaches `threshold` (folded or nearly),
    non-finite magnitudes counted as infinite (assemble.py:116-121)."""
    mag = np.abs(np.asarray(mu))
    mag[~np.isfinite(mag)] = np.inf
    return BijectivityReport(np.flatnonzero(mag >= threshold), float(mag.max()) if mag.size else 0.0, threshold)


def lbs_stiffness(coords, faces, mu):
    """Stiffness matrix (scipy CSR, n x n) of the divergence-form operator
    whose solutions have Beltrami coefficient mu (per face) on the planar
    mesh, linear elements, absolute face areas (assemble.py:124-164). The
    element rows are assembled on the device on the mesh's own CSR pattern."""
    from scipy import sparse
    from .device import DeviceBatch, device, ptr, stream_handle, to_dev
    z = np.atleast_1d(np.asarray(coords, dtype=np.complex128))
    n = len(z)
    F = np.asarray(faces)
    b = DeviceBatch(np.column_stack([z.real, z.imag, np.zeros(n)]), F, no_cuts=True)
    b.laplacian()
    vmap = b.host(nat.ARR_VMAP, torch.int32).astype(np.int64)
    zl = to_dev(z[vmap], torch.complex128)
    mud = to_dev(np.asarray(mu, dtype=np.complex128), torch.complex128)
    nnz = b.info()[nat.INFO_NNZ_L]
    kval = torch.empty(nnz, dtype=torch.float64, device=device())
    nat.check(nat.lib().pgcp_batch_lbs_stiffness(b.h, ptr(zl), ptr(mud), ptr(kval), stream_handle()))
    rp = b.host(nat.ARR_L_ROWPTR, torch.int64)
    col = b.host(nat.ARR_L_COL, torch.int32).astype(np.int64)
    val = kval.cpu().numpy()
    rows = np.repeat(vmap, np.diff(rp))
    return sparse.csr_matrix((val, (rows, vmap[col])), shape=(n, n))


@dataclass
class RepairReport:
    iterations: int
    cleared: bool
    remaining_faces: np.ndarray
    initial_flips: int


def qc_correct(layout, faces, embedding, fixed_idx, max_iter=5, cap=MU_CAP):
    """Remove fold-overs from a planar embedding by quasi-conformal
    composition (assemble.py:174-217), on the device: repeatedly solve the
    linear Beltrami equation whose coefficient is the capped inverse Beltrami
    coefficient (embedding -> layout), holding `fixed_idx` at the embedding's
    values, until no face has signed area <= 0 or `max_iter` is reached.
    Returns (embedding, RepairReport)."""
    from .device import DeviceBatch, to_dev
    emb = np.array(embedding, dtype=np.complex128)
    F = np.asarray(faces)
    fixed = np.asarray(fixed_idx, dtype=np.int64)
    flips0 = int(np.count_nonzero(signed_areas(emb, F) <= 0))
    if flips0 == 0:
        return emb, RepairReport(0, True, np.array([], dtype=np.int64), 0)
    lay = np.asarray(layout, dtype=np.complex128).reshape(-1, 3)
    beltrami_per_face(emb[F], lay)  # the reference's first-iteration check: degenerate -> SolveError
    n = len(emb)
    V3 = np.column_stack([emb.real, emb.imag, np.zeros(n)])
    b = DeviceBatch(V3, F, no_cuts=True)
    if b.info()[nat.INFO_SUM_N] != n:
        raise SolveError("singular linear Beltrami system during repair (unreferenced vertices)")
    # single domain: local ids are parent ids (every vertex referenced)
    z = to_dev(emb, torch.complex128)
    rows, flipped = b.qc_repair(fixed.astype(np.int32), z, layout=lay, max_iter=max_iter, cap=cap,
                                want_flipped=True)
    _, iters, cleared, _ = rows[0]
    remaining = np.flatnonzero(flipped.cpu().numpy()).astype(np.int64) if not cleared else \
        np.array([], dtype=np.int64)
    return z.cpu().numpy(), RepairReport(int(iters), bool(cleared), remaining, flips0)


def stitch_global(partition, embeddings, mode, snap_tol=1e-8, hard_tol=1e-6, boundary_circle_tol=1e-9):
    """Combine per-submesh embeddings into one coordinate per parent vertex
    (assemble.py:286-337) with the device stitch: seam copies averaged and
    checked against hard_tol x scale, disk boundary on the unit circle,
    sphere finish, flips."""
    from .device import device, to_dev
    b = partition.batch
    z = to_dev(np.concatenate([np.asarray(e, dtype=np.complex128) for e in embeddings]), torch.complex128)
    dev = device()
    n, m = b.n, b.m
    coords = torch.empty(n, dtype=torch.complex128, device=dev)
    sphere = torch.empty((n, 3), dtype=torch.float64, device=dev) if mode == "sphere" else None
    prov = torch.empty(n, dtype=torch.int32, device=dev)
    flip = torch.empty(m, dtype=torch.uint8, device=dev)
    stats = np.zeros(8)
    mcode = {"free": 0, "disk": 1, "sphere": 2}[mode]
    nat.check(nat.lib().pgcp_batch_stitch(b.h, _p(z), mcode, hard_tol, boundary_circle_tol, _p(coords),
                                          _p(sphere) if sphere is not None else None, _p(prov), _p(flip),
                                          stats.ctypes.data, _stream()))
    diag = {"seam_max_dev": float(stats[0]), "scale": float(stats[1])}
    if mode == "disk":
        diag["boundary_circle_dev"] = float(stats[2])
    out = (sphere if mode == "sphere" else coords).cpu().numpy()
    flipped = np.flatnonzero(flip.cpu().numpy()).astype(np.int64)
    return GlobalParam(mode, out, flipped, prov.cpu().numpy().astype(np.int64), float(stats[0]), diag)
