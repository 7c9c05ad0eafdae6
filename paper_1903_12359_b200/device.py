"""Device plumbing: torch allocations/streams around the native batch.

PyTorch is used only for device memory, streams and (in dist.py)
torch.distributed; every computation is a libpgcp_b200 kernel.
"""

import ctypes
import threading
import warnings

import numpy as np
import torch

from . import _native as nat
from .errors import SolveError

_DT = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32,
       np.dtype(np.int64): torch.int64, np.dtype(np.complex128): torch.complex128,
       np.dtype(np.uint8): torch.uint8, np.dtype(np.int8): torch.int8}


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1903_12359_b200 needs a CUDA device (no CPU fallback)")
    nat.lib()


def device():
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def to_dev(a, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (no copy if already there)."""
    if isinstance(a, torch.Tensor):
        t = a
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if not t.is_cuda:
            t = t.to(device(), non_blocking=False)
        return t.contiguous()
    arr = np.ascontiguousarray(a)
    if dtype is None:
        dtype = _DT[arr.dtype]
    with warnings.catch_warnings():
        # frozen (read-only) mesh arrays: the tensor is only a copy source
        warnings.simplefilter("ignore", UserWarning)
        host = torch.from_numpy(arr)
    return host.to(device=device(), dtype=dtype)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)


class _CudaArray:
    """__cuda_array_interface__ view of batch-owned device memory; keeps the
    owner alive for as long as the view lives."""

    def __init__(self, p, n, typestr, owner):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(p or 0), False), "version": 3, "strides": None}


_TYPESTR = {torch.int32: "<i4", torch.int64: "<i8", torch.float64: "<f8"}


class DeviceBatch:
    """A device-resident partition of one mesh into disk-type submeshes plus
    everything derived from it (Laplacians, solver systems)."""

    def __init__(self, V, F, cuts=None, no_cuts=False, stream=None, validate_only=False, base=None):
        """A partition of (V, F) along `cuts` (or the whole mesh). With
        `validate_only` only the parent mesh is validated and its topology
        built (TriMesh's check); with `base` (such a batch, or any other of
        the same mesh) the partition starts from base's topology."""
        require_cuda()
        self.stream = stream
        self.V = to_dev(V, torch.float64)
        self.F = to_dev(F, torch.int32)
        self.n = int(self.V.shape[0])
        self.m = int(self.F.shape[0])
        if cuts is not None and len(cuts):
            self.cuts = to_dev(cuts, torch.int64).reshape(-1, 2)
            ncuts = int(self.cuts.shape[0])
        else:
            self.cuts = None
            ncuts = 0
        flags = nat.BATCH_NO_CUTS if (no_cuts or ncuts == 0) else 0
        if validate_only:
            flags |= nat.BATCH_VALIDATE_ONLY
        h = ctypes.c_void_p()
        if base is not None:
            nat.check(nat.lib().pgcp_batch_create_from(base.h, ptr(self.cuts), ncuts, flags, stream_handle(stream),
                                                       ctypes.byref(h)))
        else:
            nat.check(nat.lib().pgcp_batch_create(ptr(self.V), ptr(self.F), self.n, self.m, ptr(self.cuts), ncuts,
                                                  flags, stream_handle(stream), ctypes.byref(h)))
        self.h = h
        self._info = None
        self._cache = {}
        self._lock = threading.Lock()

    # -- lifetime
    def release_solvers(self, which=3):
        """Free the last flatten (bit 0) / harmonic (bit 1) solver systems
        (factors and workspaces) once their results are consumed."""
        if getattr(self, "h", None) is not None and self.h.value:
            nat.check(nat.lib().pgcp_batch_release_solvers(self.h, which))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            nat.lib().pgcp_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- queries
    def info(self):
        buf = (ctypes.c_int64 * nat.INFO_COUNT)()
        nat.check(nat.lib().pgcp_batch_info(self.h, buf, nat.INFO_COUNT))
        return list(buf)

    @property
    def K(self):
        return self.info()[nat.INFO_K]

    def array(self, which, dtype):
        p = ctypes.c_void_p()
        cnt = ctypes.c_int64()
        nat.check(nat.lib().pgcp_batch_array(self.h, which, ctypes.byref(p), ctypes.byref(cnt)))
        if cnt.value == 0:
            return torch.empty(0, dtype=dtype, device=device())
        return torch.as_tensor(_CudaArray(p.value, cnt.value, _TYPESTR[dtype], self), device=device())

    def host(self, which, dtype):
        return self.array(which, dtype).cpu().numpy()

    def local_faces(self):
        K = self.K
        off = (ctypes.c_int64 * (K + 1))()
        faces = torch.empty((self.m, 3), dtype=torch.int32, device=device())
        nat.check(nat.lib().pgcp_batch_local_faces(self.h, off, ptr(faces), stream_handle(self.stream)))
        return np.frombuffer(off, dtype=np.int64).copy(), faces

    # -- compute
    def laplacian(self):
        """Build (once) the cotangent Laplacians of every submesh. Guarded: a
        rebuild replaces device arrays other streams may be reading."""
        with self._lock:
            if "lap" not in self._cache:
                cl = ctypes.c_int64()
                nat.check(nat.lib().pgcp_batch_laplacian(self.h, ctypes.byref(cl), stream_handle(self.stream)))
                self._cache["lap"] = int(cl.value)
            return self._cache["lap"]

    def default_pins(self):
        nat.check(nat.lib().pgcp_batch_default_pins(self.h, stream_handle(self.stream)))
        return self.host(nat.ARR_PINS, torch.int32).reshape(-1, 2)

    @staticmethod
    def _opts(rtol, contract_tol, maxit, cluster, solver="default"):
        """solver: "default" (the multifrontal direct solver unless maxit > 0
        or PGCP_SOLVER=pcg), "direct" or "pcg"."""
        o = nat.SolveOpts()
        o.rtol = rtol
        o.contract_tol = contract_tol
        o.maxit = maxit
        o.cluster = cluster
        o.solver = nat.SOLVERS[solver] if isinstance(solver, str) else int(solver)
        return o

    def _comps(self, comps):
        if comps is None:
            return None, 0, self.K
        arr = (ctypes.c_int32 * len(comps))(*[int(c) for c in comps])
        return arr, len(comps), len(comps)

    def flatten(self, comps=None, pins=None, targets=(0j, 1 + 0j), rtol=1e-10, contract_tol=1e-10,
                maxit=0, cluster=0, out=None, solver="default"):
        """DNCP flattening of the listed submeshes -> complex tensor over all
        local vertices (sum_n), plus per-submesh solve stats."""
        self.laplacian()
        carr, nc, nslot = self._comps(comps)
        z = out if out is not None else torch.zeros(self.info()[nat.INFO_SUM_N], dtype=torch.complex128,
                                                    device=device())
        if comps is not None and nc == 0:  # an empty shard (more ranks than submeshes)
            self.last_stats = []
            return z, []
        parr = None
        if pins is not None:
            flat = np.asarray(pins, dtype=np.int32).ravel()
            parr = (ctypes.c_int32 * len(flat))(*flat.tolist())
        t = (ctypes.c_double * 4)(complex(targets[0]).real, complex(targets[0]).imag,
                                  complex(targets[1]).real, complex(targets[1]).imag)
        stats = (nat.SolveStat * max(nslot, 1))()
        st = nat.lib().pgcp_batch_flatten(self.h, carr, nc, parr, t, ctypes.byref(self._opts(rtol, contract_tol, maxit, cluster, solver)),
                                          ptr(z), stats, stream_handle(self.stream))
        self.last_stats = [_stat(s) for s in stats[:nslot]]
        nat.check(st)
        return z, self.last_stats

    def harmonic(self, fixed_gid, fixed_val, comps=None, rtol=1e-10, contract_tol=1e-10, maxit=0,
                 cluster=0, out=None, solver="default"):
        self.laplacian()
        carr, nc, nslot = self._comps(comps)
        fg = to_dev(fixed_gid, torch.int32)
        fv = to_dev(fixed_val, torch.complex128)
        z = out if out is not None else torch.zeros(self.info()[nat.INFO_SUM_N], dtype=torch.complex128,
                                                    device=device())
        if comps is not None and nc == 0:
            self.last_stats = []
            return z, []
        stats = (nat.SolveStat * max(nslot, 1))()
        st = nat.lib().pgcp_batch_harmonic(self.h, carr, nc, ptr(fg), ptr(fv), int(fg.numel()),
                                           ctypes.byref(self._opts(rtol, contract_tol, maxit, cluster, solver)), ptr(z),
                                           stats, stream_handle(self.stream))
        self.last_stats = [_stat(s) for s in stats[:nslot]]
        nat.check(st)
        return z, self.last_stats

    def harmonic_prepare(self, fixed_gid, comps=None, rtol=1e-10, contract_tol=1e-10, maxit=0, cluster=0,
                         stream=None, solver="default"):
        """First half of `harmonic`: everything that does not depend on the
        fixed values (may run on another stream while those are computed)."""
        self.laplacian()
        carr, nc, nslot = self._comps(comps)
        fg = to_dev(fixed_gid, torch.int32)
        self._prep = (comps, nslot, int(fg.numel()))
        if comps is not None and nc == 0:
            return
        nat.check(nat.lib().pgcp_batch_harmonic_prepare(
            self.h, carr, nc, ptr(fg), int(fg.numel()),
            ctypes.byref(self._opts(rtol, contract_tol, maxit, cluster, solver)),
            stream_handle(stream if stream is not None else self.stream)))

    def harmonic_solve(self, fixed_val, rtol=1e-10, contract_tol=1e-10, maxit=0, cluster=0, out=None,
                       solver="default"):
        """Second half of `harmonic` (after `harmonic_prepare`)."""
        comps, nslot, nfixed = self._prep
        fv = to_dev(fixed_val, torch.complex128)
        if int(fv.numel()) != nfixed:
            raise ValueError(f"{fv.numel()} fixed values for {nfixed} fixed vertices")
        z = out if out is not None else torch.zeros(self.info()[nat.INFO_SUM_N], dtype=torch.complex128,
                                                    device=device())
        if comps is not None and len(comps) == 0:
            self.last_stats = []
            return z, []
        stats = (nat.SolveStat * max(nslot, 1))()
        st = nat.lib().pgcp_batch_harmonic_solve(self.h, ptr(fv), nfixed,
                                                 ctypes.byref(self._opts(rtol, contract_tol, maxit, cluster, solver)),
                                                 ptr(z), stats, stream_handle(self.stream))
        self.last_stats = [_stat(s) for s in stats[:nslot]]
        nat.check(st)
        return z, self.last_stats

    def qc_repair(self, fixed_gid, z, comps=None, layout=None, max_iter=5, cap=0.95, rtol=1e-10,
                  contract_tol=1e-10, cluster=0, want_flipped=False):
        """Quasi-conformal fold-over repair (qc_correct, assemble.py:174-217)
        of the listed submeshes, in place on the local-vertex embedding z.
        Returns per submesh (flips_before, iterations, cleared, flips_after)
        and, if asked, the per-parent-face flags of faces still folded."""
        self.laplacian()
        carr, nc, nslot = self._comps(comps)
        fg = to_dev(fixed_gid, torch.int32)
        lay = to_dev(layout, torch.complex128) if layout is not None else None
        info = (ctypes.c_int32 * (4 * max(nslot, 1)))()
        flipped = torch.zeros(self.m, dtype=torch.uint8, device=device()) if want_flipped else None
        if comps is not None and nc == 0:
            return [], flipped
        nat.check(nat.lib().pgcp_batch_qc_repair(
            self.h, carr, nc, ptr(lay) if lay is not None else None, ptr(fg), int(fg.numel()), int(max_iter),
            float(cap), ctypes.byref(self._opts(rtol, contract_tol, 0, cluster)), ptr(z), info,
            ptr(flipped) if flipped is not None else None, stream_handle(self.stream)))
        rows = np.frombuffer(info, dtype=np.int32)[:4 * nslot].reshape(-1, 4)
        return [tuple(int(v) for v in r) for r in rows], flipped

    def export_system(self, which, comp):
        """(scipy CSR, rhs) of the last flatten (0: C_ff) / harmonic (1: L_II) system."""
        from scipy import sparse
        dims = (ctypes.c_int64 * 2)()
        L = nat.lib()
        nat.check(L.pgcp_batch_export_system(self.h, which, comp, dims, None, None, None, None,
                                             stream_handle(self.stream)))
        rows, nnz = dims[0], dims[1]
        indptr = np.empty(rows + 1, np.int32)
        indices = np.empty(nnz, np.int32)
        data = np.empty(nnz, np.float64)
        rhs = np.empty(rows if which == 0 else 2 * rows, np.float64)
        nat.check(L.pgcp_batch_export_system(self.h, which, comp, dims, indptr.ctypes.data, indices.ctypes.data,
                                             data.ctypes.data, rhs.ctypes.data, stream_handle(self.stream)))
        if which == 1:
            rhs = rhs.view(np.complex128)
        return sparse.csr_matrix((data, indices, indptr), shape=(rows, rows)), rhs

    def last_solve(self, which):
        """PCG kernel time (CUDA events), iterations and compulsory bytes of
        the last flatten (0) / harmonic (1) solve."""
        out = (ctypes.c_double * 19)()
        nat.check(nat.lib().pgcp_batch_last_solve(self.h, which, out, 19))
        r = {"kernel_ms": out[0], "iters_sum": out[1], "iters_max": out[2], "bytes": out[3],
             "stored_entries": out[4], "rows": out[5], "cluster": int(out[6]), "submeshes": int(out[7]),
             "ref_bytes": out[8], "coarse_ms": out[9], "solver": "direct" if out[10] else "pcg",
             "borrowed": out[10] == 2}
        if out[10]:
            r.update({"fmas": out[11], "factor_ms": out[12], "solve_ms": out[13], "max_front": int(out[14]),
                      "front_bytes": out[15], "nodes": int(out[16]), "levels": int(out[17]),
                      "numeric_ms": out[18]})
        return r

    def energy(self, z):
        out = (ctypes.c_double * self.K)()
        nat.check(nat.lib().pgcp_batch_conformal_energy(self.h, ptr(z), out, stream_handle(self.stream)))
        return np.array(out[:])


def _stat(s):
    return {"iters": s.iters, "status": s.status, "relres": s.relres, "true_res": s.true_res,
            "bnorm": s.bnorm, "xnorm": s.xnorm}


def solve_error_from(stats):
    bad = [s for s in stats if s["status"] != 0]
    if bad:
        raise SolveError(f"solve failed: {bad[0]}")
