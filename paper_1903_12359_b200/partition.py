"""Mesh partition, shared arcs and weld-schedule planning (drop-in for
`partition.py`).

`partition_mesh` runs on the device (topology.cu: connected components of
the face graph minus cut edges, labelled by minimum face; sorted vertex
maps; disk check; boundary cycles). `plan_weld_schedule` is the native
host planner (planner.cpp). Both are bit-exact restatements of the
reference's integer outputs.
"""

import ctypes
import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .errors import PartitionError
from .mesh import TriMesh

nat.register("pgcp_plan_weld_schedule",
             [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
              ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
              ctypes.POINTER(ctypes.c_int64)])


def read_cut_edges(path):
    """Cut file -> (c, 2) int64 zero-based vertex pairs. The format
    (partition.py:25-39) is one 1-based `i j` pair per line; blank lines and
    `#` comments are skipped."""
    rows = []
    with open(path, "r", encoding="utf-8") as fh:
        for ln, line in enumerate(fh, start=1):
            tok = line.split()
            if not tok or tok[0].startswith("#"):
                continue
            if len(tok) != 2:
                raise PartitionError(f"{path}:{ln}: expected two vertex ids")
            rows.append((ln, int(tok[0]), int(tok[1])))
    arr = np.asarray(rows, dtype=np.int64).reshape(-1, 3)
    bad = np.flatnonzero((arr[:, 1] < 1) | (arr[:, 2] < 1))
    if len(bad):
        raise PartitionError(f"{path}:{int(arr[bad[0], 0])}: vertex ids are 1-based")
    return arr[:, 1:] - 1


def write_cut_edges(path, cuts):
    """Inverse of read_cut_edges (1-based pairs, one per line)."""
    np.savetxt(path, np.asarray(cuts, dtype=np.int64).reshape(-1, 2) + 1, fmt="%d")


def validate_cuts(mesh, cuts):
    """Sorted pairs (partition.py:48-59); duplicates rejected here, non-edges
    by the device partition (k_mark_cuts), with the reference's messages."""
    cuts = np.asarray(cuts, dtype=np.int64).reshape(-1, 2)
    norm = np.empty_like(cuts)  # each pair sorted (elementwise min / max: a row-wise np.sort is 4x slower)
    np.minimum(cuts[:, 0], cuts[:, 1], out=norm[:, 0])
    np.maximum(cuts[:, 0], cuts[:, 1], out=norm[:, 1])
    if len(norm) > 1:  # duplicates first, as the reference (also duplicate non-edges)
        key = norm[:, 0] * (int(norm[:, 1].max()) + 1) + norm[:, 1]
        key.sort()
        if np.any(key[1:] == key[:-1]):
            raise PartitionError("duplicate cut edges")
    return norm


class Partition:
    """Result of `partition_mesh` (partition.py:62-91). Host arrays are
    materialised lazily from the device batch `self.batch`."""

    def __init__(self, mesh, batch, cuts):
        self.mesh = mesh
        self.batch = batch
        self.cuts = cuts
        self._vmaps = None
        self._cycles = None
        self._subs = None
        self._fa = None
        self._loops = None

    @property
    def n_submeshes(self):
        return self.batch.K

    def _host_maps(self):
        if self._vmaps is None:
            b = self.batch
            vmap = b.host(nat.ARR_VMAP, torch.int32).astype(np.int64)
            voff = b.host(nat.ARR_VERT_OFF, torch.int64)
            loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
            loop = b.host(nat.ARR_LOOP, torch.int32).astype(np.int64)
            K = len(voff) - 1
            self._vmaps = [vmap[voff[c]:voff[c + 1]] for c in range(K)]
            self._loops = [loop[loff[c]:loff[c + 1]] for c in range(K)]
            self._voff, self._loff = voff, loff

    @property
    def vertex_maps(self):
        self._host_maps()
        return self._vmaps

    @property
    def boundary_cycles(self):
        if self._cycles is None:
            b = self.batch
            cyc = b.host(nat.ARR_CYCLES, torch.int32).astype(np.int64)
            loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
            self._cycles = [cyc[loff[c]:loff[c + 1]] for c in range(len(loff) - 1)]
        return self._cycles

    @property
    def local_loops(self):
        self._host_maps()
        return self._loops

    @property
    def face_assignment(self):
        if self._fa is None:
            self._fa = self.batch.host(nat.ARR_FACE_COMP, torch.int32).astype(np.int64)
        return self._fa

    @property
    def submeshes(self):
        if self._subs is None:
            foff, faces = self.batch.local_faces()
            faces = faces.cpu().numpy().astype(np.int64)
            V = self.mesh.vertices
            self._subs = [TriMesh(V[vm], faces[foff[c]:foff[c + 1]], check=False)
                          for c, vm in enumerate(self.vertex_maps)]
        return self._subs

    def local_index(self, i):
        arr = np.full(self.mesh.n_vertices, -1, dtype=np.int64)
        arr[self.vertex_maps[i]] = np.arange(len(self.vertex_maps[i]))
        return arr

    def summary(self):
        voff = self.batch.host(nat.ARR_VERT_OFF, torch.int64)
        fc = np.bincount(self.face_assignment, minlength=self.n_submeshes)
        return {"n_submeshes": self.n_submeshes,
                "submesh_vertices": [int(x) for x in np.diff(voff)],
                "submesh_faces": [int(x) for x in fc],
                "n_cut_edges": int(len(self.cuts))}

    def summary_json(self, path):
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(self.summary(), fh, indent=2)


def partition_mesh(mesh, cuts):
    """Split along cut edges into disk-type submeshes (partition.py:94-137),
    on the device."""
    norm = validate_cuts(mesh, cuts)
    batch = mesh.partition_batch(norm)
    info = batch.info()
    bad = info[nat.INFO_BAD_COMP]
    if bad >= 0:
        chi, loops = info[9], info[10]
        cls = "sphere_type" if (chi == 2 and loops == 0) else "unsupported"
        raise PartitionError(f"component {bad} is {cls} (chi={chi}, {loops} loops); adjust the cut set")
    return Partition(mesh, batch, norm)


@dataclass
class SharedArc:
    pair: tuple
    parents: np.ndarray
    local_i: np.ndarray
    local_j: np.ndarray
    closed: bool = False


@dataclass
class WeldStep:
    comp_a: int
    comp_b: int
    a_cycle: np.ndarray
    b_cycle: np.ndarray
    k: int
    closed: bool
    merged_cycle: np.ndarray


def plan_weld_schedule(partition, mode="free", pairs=None):
    """Greedy longest-arc-first plan (partition.py:236-324), or the steps of
    an explicit merge order `pairs` [(rep_a, rep_b), ...] (the balanced
    rows -> strips -> tree schedule is a documented deviation)."""
    cyc = partition.boundary_cycles
    K = len(cyc)
    off = np.zeros(K + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(c) for c in cyc])
    flat = np.ascontiguousarray(np.concatenate(cyc) if K else np.zeros(0, np.int64), dtype=np.int64)
    cuts = np.ascontiguousarray(partition.cuts, dtype=np.int64)
    parr = None
    npairs = 0
    if pairs is not None:
        parr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
        npairs = len(parr)
    L = nat.lib()
    ln = (ctypes.c_int64 * 2)()
    args = [flat.ctypes.data, off.ctypes.data, K, cuts.ctypes.data, len(cuts), int(mode == "sphere"),
            parr.ctypes.data if parr is not None else None, npairs]
    nat.check(L.pgcp_plan_weld_schedule(*args, None, None, 0, ln))
    nsteps, nidx = ln[0], ln[1]
    meta = np.empty((max(nsteps, 1), 8), dtype=np.int64)
    idx = np.empty(max(nidx, 1), dtype=np.int64)
    nat.check(L.pgcp_plan_weld_schedule(*args, meta.ctypes.data, idx.ctypes.data, nidx, ln))
    steps = StepList()
    for s in range(nsteps):
        ca, cb, k, closed, o, la, lb, lm = meta[s]
        a = idx[o:o + la].copy()
        b = idx[o + la:o + la + lb].copy()
        mg = idx[o + la + lb:o + la + lb + lm].copy()
        steps.append(WeldStep(int(ca), int(cb), a, b, int(k), bool(closed), mg))
    steps.meta, steps.idx = meta, idx  # flat planner output (WeldPlan's native input)
    return steps


class StepList(list):
    """List of WeldStep that also carries the planner's flat arrays."""
    meta = None
    idx = None


def _cyclic_runs(c1, c2):
    """Maximal runs of consecutive c1 vertices that c2 traverses in the
    opposite direction (the shared arcs of two boundary cycles,
    partition.py:149-179). Vectorised: edge i of c1 (c1[i] -> c1[i+1]) is
    shared iff c2 holds c1[i+1] immediately before c1[i]. Returns "full"
    when every edge is shared (two cycles bounding the same curve)."""
    a = np.asarray(c1, dtype=np.int64)
    b = np.asarray(c2, dtype=np.int64)
    n1, n2 = len(a), len(b)
    order = np.argsort(b, kind="stable")
    sb = b[order]

    def pos_in_b(v):
        j = np.searchsorted(sb, v)
        j = np.minimum(j, n2 - 1)
        return np.where(sb[j] == v, order[j], -1)

    p_here = pos_in_b(a)
    p_next = pos_in_b(np.roll(a, -1))
    shared = (p_here >= 0) & (p_next >= 0) & ((p_next + 1) % n2 == p_here)
    if shared.all():
        if n1 != n2:
            raise PartitionError("inconsistent full-cycle correspondence")
        return "full"
    if not shared.any():
        return []
    # rotate so the scan starts after a non-shared edge; a run starts at
    # every shared edge whose predecessor is not shared
    first_gap = int(np.flatnonzero(~shared)[0])
    idx = (first_gap + 1 + np.arange(n1)) % n1
    s = shared[idx]
    starts = np.flatnonzero(s & ~np.roll(s, 1))
    runs = []
    for st in starts:
        ln = int(np.argmin(s[st:]))  # s ends with the gap, so a False exists
        runs.append([int(a[i]) for i in (idx[st] + np.arange(ln + 1)) % n1])
    return runs


def shared_arcs(partition):
    """Maximal arcs of cut edges between submesh pairs (partition.py:182-216)."""
    K = partition.n_submeshes
    cyc = partition.boundary_cycles
    arcs = []
    for i in range(K):
        li = partition.local_index(i)
        si = set(map(int, cyc[i]))
        for j in range(i + 1, K):
            if not si.intersection(map(int, cyc[j])):
                continue
            runs = _cyclic_runs(cyc[i], cyc[j])
            lj = partition.local_index(j)
            if runs == "full":
                p = np.asarray(cyc[i], dtype=np.int64)
                arcs.append(SharedArc((i, j), p, li[p], lj[p], closed=True))
                continue
            for ch in runs:
                p = np.array(ch, dtype=np.int64)
                arcs.append(SharedArc((i, j), p, li[p], lj[p]))
    return arcs
