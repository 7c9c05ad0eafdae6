"""Free-boundary conformal flattening (drop-in for `flatten.py`).

`cotangent_laplacian` and `flatten_free_boundary` run on the device
(laplace.cu K1/K2, pcg.cu K3); `area_matrix` and the energy helpers are the
small host-side forms the reference API exposes.
"""

import logging

import numpy as np
import torch
from scipy import sparse

from . import _native as nat
from .errors import MeshError, SolveError
from .mesh import boundary_loops

logger = logging.getLogger(__name__)

COT_CLAMP = 1e8


def _single_domain(mesh):
    b = mesh.batch()
    info = b.info()
    if info[nat.INFO_K] != 1 or info[nat.INFO_SUM_N] != mesh.n_vertices:
        return b, False
    return b, True


def cotangent_laplacian(mesh):
    """Canonical CSR cotangent Laplacian (flatten.py:28-61), built on the
    device: structural zeros kept, int32 sorted indices."""
    b = mesh.batch()
    ncl = b.laplacian()
    if ncl:
        logger.warning("clamping %d near-degenerate cotangents", ncl)
    n = mesh.n_vertices
    rp = b.host(nat.ARR_L_ROWPTR, torch.int64)
    col = b.host(nat.ARR_L_COL, torch.int32)
    val = b.host(nat.ARR_L_VAL, torch.float64)
    b_single = _single_domain(mesh)[1]
    if b_single:
        return sparse.csr_matrix((val, col, rp.astype(np.int32)), shape=(n, n))
    # several components / unreferenced vertices: map local -> parent ids
    vmap = b.host(nat.ARR_VMAP, torch.int32).astype(np.int64)
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    comp = np.repeat(np.arange(len(voff) - 1), np.diff(voff))
    rows = np.repeat(vmap, np.diff(rp))
    cols = vmap[voff[np.repeat(comp, np.diff(rp))] + col]
    return sparse.csr_matrix((val, (rows, cols)), shape=(n, n))


def area_matrix(mesh, loops=None):
    """Shoelace area form on boundary edges (flatten.py:64-86)."""
    n = mesh.n_vertices
    if loops is None:
        loops = boundary_loops(mesh)
    r, c, v = [], [], []
    for loop in loops:
        p = np.asarray(loop, dtype=np.int64)
        q = np.roll(p, -1)
        quarter = np.full(len(p), 0.25)
        r.extend([p, q + n, q, p + n])
        c.extend([q + n, p, p + n, q])
        v.extend([quarter, quarter, -quarter, -quarter])
    if not r:
        return sparse.csr_matrix((2 * n, 2 * n))
    return sparse.csr_matrix((np.concatenate(v), (np.concatenate(r), np.concatenate(c))),
                             shape=(2 * n, 2 * n))


def dirichlet_energy(L, z):
    x, y = z.real, z.imag
    return 0.5 * (x @ (L @ x) + y @ (L @ y))


def boundary_signed_area(z, loops):
    total = 0.0
    for loop in loops:
        w = z[loop]
        total += 0.5 * np.sum(w.real * np.roll(w, -1).imag - w.imag * np.roll(w, -1).real)
    return total


def conformal_energy(mesh, z, L=None, loops=None):
    """E_C = E_D - A (flatten.py:104-110). Without explicit L/loops the
    device computes it (laplace.cu k_energy)."""
    if L is None and loops is None:
        b, single = _single_domain(mesh)
        if single:
            zt = torch.as_tensor(np.asarray(z, dtype=np.complex128)).to(b.V.device)
            return float(b.energy(zt).sum())
    if L is None:
        L = cotangent_laplacian(mesh)
    if loops is None:
        loops = boundary_loops(mesh)
    z = np.asarray(z, dtype=np.complex128)
    return dirichlet_energy(L, z) - boundary_signed_area(z, loops)


def default_pins(loop, vertices):
    """Half-perimeter pins (flatten.py:113-122). Host form of the API helper;
    the pipeline uses the device version (laplace.cu k_default_pins)."""
    pts = np.asarray(vertices)[loop]
    seg = np.linalg.norm(np.roll(pts, -1, axis=0) - pts, axis=1)
    cum = np.concatenate([[0.0], np.cumsum(seg)])
    j = int(np.argmin(np.abs(cum[:-1] - cum[-1] / 2.0)))
    if j == 0:
        j = len(loop) // 2
    return int(loop[0]), int(loop[j])


def flatten_free_boundary(mesh, pins=None, pin_targets=(0.0 + 0.0j, 1.0 + 0.0j), residual_tol=1e-10,
                          rtol=1e-10):
    """DNCP free-boundary conformal flattening (flatten.py:125-188) on the
    device. Returns the (n,) complex embedding."""
    b, single = _single_domain(mesh)
    info = b.info()
    nl = info[nat.INFO_PARENT_LOOPS]
    if info[nat.INFO_K] != 1 or nl != 1:
        got = nl if nl >= 0 else "several"
        raise MeshError(f"flattening needs one boundary loop, got {got}")
    if not single:
        raise SolveError("singular constrained system in conformal flattening "
                         "(unreferenced vertices)")
    if complex(pin_targets[0]) == complex(pin_targets[1]):
        raise MeshError("pin targets must be distinct")
    z, _ = b.flatten(pins=None if pins is None else [list(pins)], targets=pin_targets, rtol=rtol,
                     contract_tol=residual_tol)
    return z.cpu().numpy()
