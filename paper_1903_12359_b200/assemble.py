"""Interior reconstruction and global assembly (drop-in for `assemble.py`).

`harmonic_solve` runs on the device (pcg.cu). The quasi-conformal repair
(`assemble.py:105-217`) is out of scope: the pipeline reports
flips instead of repairing them.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .errors import SolveError


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
