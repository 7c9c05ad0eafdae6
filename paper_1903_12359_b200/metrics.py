"""Distortion measurement (drop-in for `metrics.py`), computed on the device
(metrics.cu): corner angles, angular and area distortion, the report's
summaries. The Mobius area post-optimisation (`metrics.py:183-270`) is out
of scope."""

import ctypes
import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat

_VP, _I64, _D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
nat.register("pgcp_distortion", [_VP, _VP, _I64, _I64, _VP, ctypes.c_int, _VP, _VP, _VP, _VP, _I64, _VP])
nat.register("pgcp_distortion_ex", [_VP, _VP, _I64, _I64, _VP, ctypes.c_int, _VP, nat.REDUCE_FN, _VP, _VP, _VP, _VP,
                                    _VP, _I64, _VP])

SUMMARY_COUNT = 16


def _param_coords(param):
    mode = getattr(param, "mode", None)
    coords = getattr(param, "coords", param)
    if mode is None:
        arr = np.asarray(coords) if not isinstance(coords, torch.Tensor) else coords
        mode = "sphere" if (arr.ndim == 2 and arr.shape[1] == 3) else "free"
    return coords, mode


class DeviceDistortion:
    """Raw device outputs of pgcp_distortion."""

    def __init__(self, V, F, coords, mode, hist=True, face_mask=None, reduce=None):
        """face_mask / reduce: the sharded form (pgcp_distortion_ex): this
        rank's faces, and the pgcp_reduce_fn summing over ranks."""
        from .device import device, ptr, stream_handle, to_dev
        sphere = mode == "sphere"
        Vd = to_dev(V, torch.float64)
        Fd = to_dev(np.asarray(F, dtype=np.int32) if not isinstance(F, torch.Tensor) else F, torch.int32)
        if isinstance(coords, torch.Tensor):
            cd = coords.to(device()).contiguous()
        else:
            cd = to_dev(np.asarray(coords, dtype=np.float64 if sphere else np.complex128))
        m = int(Fd.shape[0])
        n = int(Vd.shape[0])
        self.d = torch.empty(3 * m, dtype=torch.float64, device=device())
        self.valid = torch.empty(3 * m, dtype=torch.uint8, device=device())
        self.summary = np.zeros(SUMMARY_COUNT)
        cap = 0
        h = None
        if hist:
            cap = 1 << 20
            h = np.zeros(cap, dtype=np.uint64)
        if face_mask is None and reduce is None:
            nat.check(nat.lib().pgcp_distortion(ptr(Vd), ptr(Fd), n, m, ptr(cd), int(sphere), ptr(self.d),
                                                ptr(self.valid), self.summary.ctypes.data,
                                                h.ctypes.data if h is not None else None, cap, stream_handle()))
        else:
            nat.check(nat.lib().pgcp_distortion_ex(ptr(Vd), ptr(Fd), n, m, ptr(cd), int(sphere),
                                                   ptr(face_mask) if face_mask is not None else None,
                                                   reduce if reduce is not None else nat.REDUCE_FN(), None,
                                                   ptr(self.d), ptr(self.valid), self.summary.ctypes.data,
                                                   h.ctypes.data if h is not None else None, cap, stream_handle()))
        nb = int(self.summary[11])
        self.hist = h[:nb].tolist() if (h is not None and self.summary[12] > 0) else []

    def stats(self, which):
        o = 0 if which == "angular" else 4
        s = self.summary
        return {"mean": float(s[o]), "sd": float(s[o + 1]), "median": float(s[o + 2]), "iqr": float(s[o + 3])}


def angular_distortion(mesh, param):
    """Per-corner (param - original) angle in degrees + validity mask
    (metrics.py:61-75)."""
    coords, mode = _param_coords(param)
    dd = DeviceDistortion(mesh.vertices, mesh.faces, coords, mode, hist=False)
    return dd.d.cpu().numpy(), dd.valid.cpu().numpy().astype(bool)


def area_distortion(mesh, param):
    """Per-face log of the normalised area ratio (metrics.py:89-104), on the
    device; faces of zero parametric area are invalid (d = 0)."""
    from .device import device, ptr, stream_handle, to_dev
    coords, mode = _param_coords(param)
    sphere = mode == "sphere"
    Vd = to_dev(np.asarray(mesh.vertices, dtype=np.float64), torch.float64)
    Fd = to_dev(np.asarray(mesh.faces), torch.int32)
    cd = coords.to(device()).contiguous() if isinstance(coords, torch.Tensor) else \
        to_dev(np.asarray(coords, dtype=np.float64 if sphere else np.complex128))
    m = int(Fd.shape[0])
    d = torch.empty(m, dtype=torch.float64, device=device())
    valid = torch.empty(m, dtype=torch.uint8, device=device())
    nat.check(nat.lib().pgcp_area_distortion(ptr(Vd), ptr(Fd), int(Vd.shape[0]), m, ptr(cd), int(sphere), ptr(d),
                                             ptr(valid), stream_handle()))
    return d.cpu().numpy(), valid.cpu().numpy().astype(bool)


def _corner_angles(points, faces, kind):
    from .device import device, ptr, stream_handle, to_dev
    F = to_dev(np.asarray(faces), torch.int32)
    P = to_dev(points)
    m = int(F.shape[0])
    ang = torch.empty((m, 3), dtype=torch.float64, device=device())
    bad = torch.empty((m, 3), dtype=torch.uint8, device=device())
    nat.check(nat.lib().pgcp_corner_angles(ptr(P), kind, ptr(F), m, ptr(ang), ptr(bad), stream_handle()))
    return ang.cpu().numpy(), bad.cpu().numpy().astype(bool)


def corner_angles(points, faces):
    """(m, 3) corner angles of a planar (complex or 2D) or 3D vertex array and
    the degeneracy mask (metrics.py:31-44), on the device."""
    p = np.asarray(points)
    if np.iscomplexobj(p) or p.ndim == 1:
        return _corner_angles(np.asarray(p, dtype=np.complex128), faces, 0)
    p = np.ascontiguousarray(p, dtype=np.float64)
    return _corner_angles(p, faces, 1 if p.shape[1] == 2 else 2)


def corner_angles_sphere(points, faces):
    """Spherical corner angles through the tangent-plane projection of the
    edges (metrics.py:47-58), on the device."""
    return _corner_angles(np.ascontiguousarray(points, dtype=np.float64), faces, 3)


def summarize(values):
    """Mean, population sd, median, IQR with linear interpolation
    (metrics.py:114-126)."""
    v = np.asarray(values, dtype=np.float64)
    if v.size == 0:
        raise ValueError("cannot summarize an empty array")
    q25, q50, q75 = np.percentile(v, [25, 50, 75])
    return {"mean": float(np.mean(v)), "sd": float(np.std(v)), "median": float(q50), "iqr": float(q75 - q25)}


@dataclass
class DistortionReport:
    angular: object
    area: object
    angular_stats: dict
    area_stats: dict
    excluded_corners: int
    excluded_faces: int
    conformal_energy: float = None
    extra: dict = field(default_factory=dict)
    histogram: list = None

    def to_dict(self, histogram_bin=0.1):
        return {
            "angular_abs": self.angular_stats,
            "area_abs": self.area_stats,
            "angular_histogram": {"bin_width": histogram_bin, "start": 0.0,
                                  "counts": list(self.histogram or [])},
            "excluded_corners": self.excluded_corners,
            "excluded_faces": self.excluded_faces,
            "conformal_energy": self.conformal_energy,
            **self.extra,
        }

    def to_json(self, path):
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(self.to_dict(), fh, indent=2)


def distortion_report(mesh, param, energy=None, V=None, F=None, face_mask=None, reduce=None):
    """Device distortion report (metrics.py:165-176). The per-corner values
    stay on the device (`report.angular` is a CUDA tensor of the valid |d|
    entries' source array and mask)."""
    coords, mode = _param_coords(param)
    Vs = V if V is not None else mesh.vertices
    Fs = F if F is not None else mesh.faces
    dd = DeviceDistortion(Vs, Fs, coords, mode, hist=True, face_mask=face_mask, reduce=reduce)
    s = dd.summary
    return DistortionReport(angular=dd.d, area=None, angular_stats=dd.stats("angular"),
                            area_stats=dd.stats("area"), excluded_corners=int(s[8]),
                            excluded_faces=int(s[9]), conformal_energy=energy, histogram=dd.hist)
