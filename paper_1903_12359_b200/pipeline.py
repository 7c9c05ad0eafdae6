"""End-to-end PGCP on the device (drop-in for `pipeline.py`).

parameterize (pipeline.py:119-271) keeps every array on the GPU:
  partition   topology.cu          one DeviceBatch: components, vertex maps, loops
  plan        planner.cpp          host, integer-exact (boundary cycles only)
  flatten     laplace.cu + pcg.cu  K1/K2 + batched cluster PCG over all submeshes
  weld        weld.cu              tracked boundary values, schedule levels
  boundary    weld.cu              disk: geodesic map; sphere: exterior inversion
  harmonic    pcg.cu               batched cluster PCG with the welded boundary
  stitch      metrics.cu           seam averaging, sphere finish, flips
  metrics     metrics.cu           energy, angular/area distortion report
Host work is bookkeeping over boundary-cycle ids (the weld write-back lists)
and the final device -> host copy of the coordinates.
"""

import ctypes
import json
import os
import sys
import threading
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .assemble import GlobalParam
from .errors import PartitionError, SolveError, ValidationError, WeldError
from .mesh import TriMesh, load_obj, validate_topology, write_obj_with_param
from .partition import Partition, plan_weld_schedule, read_cut_edges, validate_cuts
from .welding import (ARC_FROM_B, CYC_A, CYC_B, SIDE_B, PreparedSchedule, _from_native, run_schedule)


@dataclass
class RunConfig:
    input: str = None
    cuts: str = None
    mode: str = "free"             # free | disk | sphere
    workers: int = 1
    out: str = None
    report: str = None
    mobius_area: bool = False
    seed: int = 0
    snap_tol: float = 1e-8
    hard_tol: float = 1e-6
    beltrami_threshold: float = 0.99
    repair_iters: int = 5
    # B200 additions (named options; defaults keep the reference behaviour)
    schedule: str = "greedy"       # greedy (reference planner) | pairs (explicit merge order)
    pairs: list = None
    rtol: float = 1e-10            # PCG recurrence tolerance
    cluster: int = 0               # CTAs per subdomain (0 = auto)
    keep_device: bool = False      # leave coords on the device (no final D2H)

    def validate(self):
        if self.mode not in ("free", "disk", "sphere"):
            raise ValidationError(f"unknown mode {self.mode!r}")
        if self.workers < 1:
            raise ValidationError("worker count must be >= 1")
        if self.schedule not in ("greedy", "pairs"):
            raise ValidationError(f"unknown schedule {self.schedule!r}")


@dataclass
class RunReport:
    mode: str = ""
    n_vertices: int = 0
    n_faces: int = 0
    n_submeshes: int = 0
    submesh_sizes: list = field(default_factory=list)
    timings: dict = field(default_factory=dict)
    seam_residuals: list = field(default_factory=list)
    repairs: list = field(default_factory=list)
    flips: int = 0
    distortion: dict = field(default_factory=dict)
    ok: bool = False
    mobius_info: dict = None
    bench: dict = None
    solver: dict = None

    def to_dict(self):
        return {k: v for k, v in self.__dict__.items() if v is not None}

    def to_json(self, path):
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(self.to_dict(), fh, indent=2)


class _Clock:
    """Stage timer: host wall time around device work, synchronised."""

    def __init__(self, timings, sync=True):
        self.t = timings
        self.sync = sync
        self.t0 = None

    def start(self):
        if self.sync:
            torch.cuda.synchronize()
        self.t0 = time.perf_counter()

    def stop(self, name):
        if self.sync:
            torch.cuda.synchronize()
        self.t[name] = self.t.get(name, 0.0) + time.perf_counter() - self.t0


def _ptr(t):
    from .device import ptr
    return ptr(t)


def _stream():
    from .device import stream_handle
    return stream_handle()


nat.register("pgcp_weld_plan",
             [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
              ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
              ctypes.POINTER(ctypes.c_int64)])


class WeldPlan:
    """Bookkeeping of a weld schedule over the tracked boundary slots.

    Slot s is one entry of one submesh's boundary loop (submesh order, loop
    order), i.e. the (component, parent id) value the reference keeps in its
    per-component dicts (pipeline.py:174-204). For every step the plan lists
    the slots of a_cycle / b_cycle (phase-1 inputs) and the write-back code of
    every slot of the two components (native: planner.cpp pgcp_weld_plan)."""

    def __init__(self, cycles, steps, n_parent):
        K = len(cycles)
        nb = np.array([len(c) for c in cycles], dtype=np.int64)
        self.loop_off = np.zeros(K + 1, dtype=np.int64)
        self.loop_off[1:] = np.cumsum(nb)
        self.slot_parent = np.ascontiguousarray(np.concatenate(cycles).astype(np.int64)) if K else \
            np.zeros(0, np.int64)
        self.slot_sub = np.repeat(np.arange(K), nb)
        self.n_parent = n_parent
        self._table = None
        meta, idx = getattr(steps, "meta", None), getattr(steps, "idx", None)
        ns = len(steps)
        if meta is None:
            meta = np.zeros((max(ns, 1), 8), dtype=np.int64)
            parts, o = [], 0
            for q, st in enumerate(steps):
                la, lb, lm = len(st.a_cycle), len(st.b_cycle), len(st.merged_cycle)
                meta[q] = (st.comp_a, st.comp_b, st.k, int(st.closed), o, la, lb, lm)
                parts += [st.a_cycle, st.b_cycle, st.merged_cycle]
                o += la + lb + lm
            idx = np.ascontiguousarray(np.concatenate(parts).astype(np.int64)) if parts else np.zeros(1, np.int64)
        L = nat.lib()
        lens = (ctypes.c_int64 * 2)()
        args = [self.slot_parent.ctypes.data, self.loop_off.ctypes.data, K, meta.ctypes.data, idx.ctypes.data, ns,
                int(n_parent)]
        nat.check(L.pgcp_weld_plan(*args, None, None, None, None, None, lens))
        self.info = np.zeros((max(ns, 1), 6), dtype=np.int32)
        self.src = np.zeros(max(lens[0], 1), dtype=np.int32)
        self.wb_off = np.zeros(ns + 1, dtype=np.int64)
        self.wb = np.zeros((max(lens[1], 1), 2), dtype=np.int32)
        ext = np.zeros(max(K, 1), dtype=np.int32)
        nat.check(L.pgcp_weld_plan(*args, self.info.ctypes.data, self.src.ctypes.data, self.wb_off.ctypes.data,
                                   self.wb.ctypes.data, ext.ctypes.data, lens))
        self.info = self.info[:ns]
        self.src = self.src[:lens[0]]
        self.wb = self.wb[:lens[1]]
        if ns and steps[-1].closed:
            self.exterior_candidates = ([int(i) for i in np.nonzero(ext[:K] == 1)[0]],
                                        [int(i) for i in np.nonzero(ext[:K] == 2)[0]])

    def slots_of(self, subs):
        return np.concatenate([np.arange(self.loop_off[i], self.loop_off[i + 1]) for i in subs]) \
            if len(subs) else np.zeros(0, np.int64)

    def any_slot_of_parents(self, parents):
        if self._table is None:
            self._table = np.full(self.n_parent, -1, dtype=np.int64)
            self._table[self.slot_parent] = np.arange(len(self.slot_parent))
        return self._table[np.asarray(parents, dtype=np.int64)]


def _poly_area(z):
    return 0.5 * float(np.sum(z.real * np.roll(z, -1).imag - z.imag * np.roll(z, -1).real))


def parameterize(mesh, cuts=None, mode="free", workers=1, seed=0, mobius_area=False, config=None,
                 schedule=None, pairs=None, keep_device=False, shard=None):
    """Global conformal parameterization (pipeline.py:119-271) on the device.

    Same signature and results as the reference; `schedule`/`pairs` select
    the documented balanced weld order (config.schedule="pairs"). `shard`
    (dist.Shard) splits the flatten/harmonic solves across ranks: each rank
    solves its own subdomains and one sum-all-reduce per stage assembles the
    boundary values / embeddings (dist.py)."""
    from .device import device, require_cuda
    require_cuda()
    cfg = config or RunConfig(mode=mode, workers=workers, seed=seed, mobius_area=mobius_area)
    if schedule is not None:
        cfg.schedule = schedule
    if pairs is not None:
        cfg.pairs = pairs
        cfg.schedule = "pairs"
    if keep_device:
        cfg.keep_device = True
    cfg.validate()
    mode = cfg.mode
    report = RunReport(mode=mode, n_vertices=mesh.n_vertices, n_faces=mesh.n_faces)
    timings = report.timings
    clk = _Clock(timings)
    dev = device()

    # ---- partition (+ parent topology) ----------------------------------------
    clk.start()
    V, F = mesh.device_arrays()
    have_cuts = cuts is not None and len(cuts) > 0
    if have_cuts:
        norm = validate_cuts(mesh, cuts)
        batch = mesh.partition_batch(norm)
    else:
        norm = np.zeros((0, 2), np.int64)
        batch = mesh.batch()
    info = batch.info()
    chi, nl = info[nat.INFO_PARENT_CHI], info[nat.INFO_PARENT_LOOPS]
    cls = "disk_type" if (chi == 1 and nl == 1) else ("sphere_type" if (chi == 2 and nl == 0) else "unsupported")
    if mode in ("free", "disk") and cls != "disk_type":
        raise ValidationError(f"mode {mode!r} needs a disk-type mesh, got {cls}")
    if mode == "sphere" and cls != "sphere_type":
        raise ValidationError(f"sphere mode needs a genus-0 closed mesh, got {cls}")
    if not have_cuts and mode == "sphere":
        raise ValidationError("sphere mode requires a cut set (K >= 2)")
    if have_cuts and info[nat.INFO_BAD_COMP] >= 0:
        c_chi, c_loops = info[9], info[10]
        ccls = "sphere_type" if (c_chi == 2 and c_loops == 0) else "unsupported"
        raise PartitionError(f"component {info[nat.INFO_BAD_COMP]} is {ccls} (chi={c_chi}, {c_loops} loops); "
                             "adjust the cut set")
    part = Partition(mesh, batch, norm)
    K = info[nat.INFO_K]
    report.n_submeshes = K
    voff = batch.host(nat.ARR_VERT_OFF, torch.int64)
    report.submesh_sizes = [int(x) for x in np.diff(voff)]
    welds = not (K == 1 and mode == "free")
    if welds:  # host copies the planner needs, taken before the solve is queued
        cycles = part.boundary_cycles
        loop_local = batch.host(nat.ARR_LOOP, torch.int32).astype(np.int64)
    clk.stop("partition")

    own = shard.comps(report.submesh_sizes) if (shard is not None and K > 1) else None

    # ---- local free-boundary flattening (all submeshes, one launch), with the
    # host-side weld planning (planner.cpp, weld plan) overlapped on this thread
    clk.start()
    fres = {}
    # the flatten runs on a high-priority stream; the harmonic system (which
    # depends only on which vertices are fixed) is prepared meanwhile on a
    # normal-priority stream, on the SMs the flatten's cluster waves leave idle
    hi, lo = _streams(dev)
    cur = torch.cuda.current_stream()
    # the Laplacian both streams read is built once, here, before the flatten
    # worker thread and the harmonic preparation start using the batch
    batch.laplacian()
    hi.wait_stream(cur)
    lo.wait_stream(cur)
    overlap_prep = welds and os.environ.get("PGCP_OVERLAP_HPREP", "1") != "0"
    # where the harmonic preparation (the Dirichlet factorization) overlaps:
    # the flatten (default) or, with PGCP_HPREP_AT=weld, the weld (the weld
    # then runs on the high-priority stream). cfg 2, end of round 2: beside the
    # weld the flatten runs at its standalone 10.7 ms (12.4 with the
    # preparation beside it), but the weld's latency-bound record chain slows
    # from 5.4 to 8.8 ms: 25.5 ms per step against 23.5, so the default stays.
    prep_at_weld = overlap_prep and os.environ.get("PGCP_HPREP_AT", "flatten") == "weld"

    def _flatten():
        try:
            torch.cuda.set_device(dev)  # the current device is per host thread
            with torch.cuda.stream(hi):
                fres["out"] = batch.flatten(comps=own, rtol=cfg.rtol, cluster=cfg.cluster)
        except BaseException as exc:  # re-raised on the caller's thread
            fres["err"] = exc

    # three host threads hand the GIL back and forth around their native
    # calls (flatten, Dirichlet preparation, planning): with the default 5 ms
    # switch interval a thread returning from a call can wait that long
    swi = sys.getswitchinterval()
    if os.environ.get("PGCP_SWITCH_INTERVAL", "1") != "0":
        sys.setswitchinterval(1e-4)
    worker = threading.Thread(target=_flatten, name="pgcp-flatten")
    worker.start()
    # the Dirichlet preparation needs only the fixed vertices (every loop
    # vertex, in slot order = submesh order, loop order): it starts now, in
    # its own thread, beside the flatten and the host-side planning
    hprep = {}
    pworker = None
    if welds:
        nbl = np.array([len(c) for c in cycles], dtype=np.int64)
        loop_gid_host = (voff[np.repeat(np.arange(K), nbl)] + loop_local).astype(np.int32)
    if overlap_prep and not prep_at_weld:
        def _hprep_early():
            try:
                torch.cuda.set_device(dev)
                t_h = time.perf_counter()
                with torch.cuda.stream(lo):
                    lg = torch.as_tensor(loop_gid_host).to(dev)
                    batch.harmonic_prepare(lg, comps=own, rtol=cfg.rtol, cluster=cfg.cluster, stream=lo)
                hprep["t"] = time.perf_counter() - t_h
                hprep["gid"] = lg
            except BaseException as exc:
                hprep["err"] = exc

        pworker = threading.Thread(target=_hprep_early, name="pgcp-harmonic-prepare")
        pworker.start()
    steps, plan, perr, sched = [], None, None, None
    t_plan = time.perf_counter()
    try:
        if have_cuts:
            steps = plan_weld_schedule(part, mode, pairs=cfg.pairs if cfg.schedule == "pairs" else None)
        if welds:
            plan = WeldPlan(cycles, steps, mesh.n_vertices)
            # the weld's host-side preparation and uploads, here (this thread
            # would only wait for the flatten) instead of at the head of the
            # weld stage; on this thread's stream, which is idle meanwhile
            if len(steps) and os.environ.get("PGCP_WELD_PREPARE", "1") != "0":
                sched = PreparedSchedule(plan.info, plan.src, plan.wb_off, plan.wb)
        timings["plan (overlapped)"] = time.perf_counter() - t_plan
    except BaseException as exc:
        perr = exc
    worker.join()
    # the preparation is joined here, before the weld: letting it run on into
    # the weld was measured to starve the weld's cluster kernels now and then
    # (one cfg-2 step in ten: weld 9 -> 63 ms)
    if pworker is not None:
        pworker.join()
        if "err" in hprep and perr is None:
            perr = hprep["err"]
        if "t" in hprep:
            timings["harmonic prepare (overlapped)"] = hprep["t"]
    sys.setswitchinterval(swi)
    cur.wait_stream(hi)
    cur.wait_stream(lo)
    if "err" in fres:
        raise fres["err"]
    if perr is not None:
        raise perr
    pworker = None
    z0, fst = fres["out"]
    clk.stop("flatten")
    report.solver = {"flatten_iters": [s["iters"] for s in fst], "flatten": batch.last_solve(0)}
    if own is not None:
        report.solver["shard"] = own

    if not welds:
        embeddings = z0
    else:
        # ---- welding on tracked boundary values ---------------------------------
        clk.start()
        loop_gid = torch.as_tensor(loop_gid_host).to(dev)
        hworker = None
        if prep_at_weld:
            lo.wait_stream(cur)

            def _hprep():
                try:
                    torch.cuda.set_device(dev)
                    t_h = time.perf_counter()
                    with torch.cuda.stream(lo):
                        batch.harmonic_prepare(loop_gid, comps=own, rtol=cfg.rtol, cluster=cfg.cluster, stream=lo)
                    hprep["t"] = time.perf_counter() - t_h
                except BaseException as exc:
                    hprep["err"] = exc

            hworker = threading.Thread(target=_hprep, name="pgcp-harmonic-prepare")
            hworker.start()
        # with the preparation beside it, the weld runs on the high-priority
        # stream: its cluster launches get the SMs the factorization frees
        wstream = hi if ((hworker is not None or pworker is not None)
                         and os.environ.get("PGCP_WELD_HI", "1") != "0") else cur
        if wstream is not cur:
            wstream.wait_stream(cur)
        try:
            with torch.cuda.stream(wstream):
                if own is None:
                    tv = torch.empty(len(plan.slot_parent), dtype=torch.complex128, device=dev)
                    nat.check(nat.lib().pgcp_gather_complex(_ptr(z0), _ptr(loop_gid), _ptr(tv), tv.numel(),
                                                            _stream()))
                else:  # the one exchange: all-gather of every rank's boundary-loop values
                    own_slots, tv = _exchange_boundary(shard, plan, loop_gid_host, z0, dev)
                out = None
                if len(steps):
                    if sched is not None:
                        out = sched.run(tv, cfg.hard_tol)
                    else:
                        out, _ = run_schedule(tv, plan.info, plan.src, plan.wb_off, plan.wb, cfg.hard_tol)
                    report.seam_residuals = [float(x) for x in out[:, 1]]
        except BaseException:
            for w in (hworker, pworker):  # never leave the preparation running on the batch
                if w is not None:
                    w.join()
            raise
        if wstream is not cur:
            cur.wait_stream(wstream)
        exterior = []
        if len(steps) and steps[-1].closed:
            A, B = plan.exterior_candidates
            exterior = B if out[-1, 2] > 0 else A
        clk.stop("weld")
        for w in (hworker, pworker):
            if w is not None:
                w.join()
                cur.wait_stream(lo)
                if "err" in hprep:
                    raise hprep["err"]
                timings["harmonic prepare (overlapped)"] = hprep["t"]

        if mode == "disk":
            clk.start()
            gc = steps[-1].merged_cycle if steps else cycles[0]
            _geodesic_boundary(plan, tv, gc)
            clk.stop("boundary_map")

        # ---- harmonic reconstruction with the welded boundary --------------------
        clk.start()
        center = None
        if mode == "sphere" and exterior:
            seam_slots = plan.any_slot_of_parents(steps[-1].a_cycle).astype(np.int32)
            c = np.zeros(2)
            rev = int(out[-1, 2] < 0)
            nat.check(nat.lib().pgcp_polygon_interior(_ptr(tv), seam_slots.ctypes.data, len(seam_slots), rev,
                                                      c.ctypes.data, _stream()))
            center = complex(c[0], c[1])
            ext_slots = torch.as_tensor(plan.slots_of(exterior).astype(np.int32)).to(dev)
            nat.check(nat.lib().pgcp_inv_shift(_ptr(tv), _ptr(ext_slots), ext_slots.numel(), 0.0, 0.0,
                                               center.real, center.imag, _stream()))
        # sharded: the other ranks' subdomains stay NaN here (never solved on
        # this rank; stitch and metrics skip them) except their boundary
        # loops, filled below with the welded values
        zout = None
        if own is not None:
            zout = torch.full((int(voff[-1]),), complex(float("nan"), float("nan")), dtype=torch.complex128,
                              device=dev)
        if overlap_prep:
            z, hst = batch.harmonic_solve(tv, rtol=cfg.rtol, cluster=cfg.cluster, out=zout)
        else:
            z, hst = batch.harmonic(loop_gid, tv, comps=own, rtol=cfg.rtol, cluster=cfg.cluster, out=zout)
        report.solver["harmonic_iters"] = [s["iters"] for s in hst]
        report.solver["harmonic"] = batch.last_solve(1)
        # fold-over repair of the submeshes whose harmonic map flipped faces
        # (pipeline.py:88-102, per submesh before the exterior map-back),
        # batched over every folded submesh on the device (repair.cu)
        report.repairs = _repair(batch, loop_gid, z, own, K, cfg, shard)
        # the factors (GBs at cfg 2/5) are not needed past this point;
        # PGCP_RELEASE_SOLVERS=1 frees them here (measured: e2e steps become
        # erratic, so by default they go with the batch)
        if os.environ.get("PGCP_RELEASE_SOLVERS", "0") == "1":
            batch.release_solvers()
        if own is not None:
            # the other ranks' boundary loops hold the welded values (their
            # Dirichlet data), so every seam copy is known here
            _fill_foreign_loops(tv, z, own_slots, loop_gid_host, dev)
        if center is not None:
            gids = np.concatenate([np.arange(voff[i], voff[i + 1]) for i in exterior]).astype(np.int32)
            gt = torch.as_tensor(gids).to(dev)
            nat.check(nat.lib().pgcp_inv_shift(_ptr(z), _ptr(gt), gt.numel(), center.real, center.imag, 0.0, 0.0,
                                               _stream()))
        embeddings = z
        clk.stop("harmonic")

    # ---- stitch ---------------------------------------------------------------
    clk.start()
    smaps = _shard_maps(batch, own, dev) if own is not None else None
    gp, flip = _stitch(batch, embeddings, mode, cfg, mesh, smaps)
    clk.stop("stitch")
    return _finish(mesh, batch, embeddings, gp, report, cfg, clk, shard if own is not None else None, smaps, own)


def _exchange_boundary(shard, plan, loop_gid_host, z0, dev):
    """SURVEY §8(e)'s only data-path collective: every rank packs the
    boundary-loop values of its own submeshes (slot order) and one
    all-gather hands every rank every block; a scatter puts them into the
    tracked-value vector (padding lands in a dummy slot past the end)."""
    nslot = len(plan.slot_parent)
    own_slots, smap, blk = shard.slot_layout(plan.loop_off)
    send = torch.zeros(blk, dtype=torch.complex128, device=dev)
    if len(own_slots):
        idx = torch.as_tensor(loop_gid_host[own_slots]).to(dev)
        nat.check(nat.lib().pgcp_gather_complex(_ptr(z0), _ptr(idx), _ptr(send), len(own_slots), _stream()))
    recv = torch.empty(shard.world * blk, dtype=torch.complex128, device=dev)
    shard.all_gather_(send, recv)
    tv_ext = torch.empty(nslot + 1, dtype=torch.complex128, device=dev)
    sm = torch.as_tensor(smap).to(dev)
    nat.check(nat.lib().pgcp_scatter_complex(_ptr(recv), _ptr(sm), _ptr(tv_ext), recv.numel(), _stream()))
    return own_slots, tv_ext[:nslot]


def _fill_foreign_loops(tv, z, own_slots, loop_gid_host, dev):
    """z on the boundary loops of other ranks' submeshes := their welded
    Dirichlet values (what their harmonic solves hold fixed)."""
    mine = np.zeros(len(loop_gid_host), dtype=bool)
    mine[own_slots] = True
    foreign = np.flatnonzero(~mine).astype(np.int32)
    if not len(foreign):
        return
    src = torch.as_tensor(foreign).to(dev)
    dst = torch.as_tensor(loop_gid_host[foreign]).to(dev)
    tmp = torch.empty(len(foreign), dtype=torch.complex128, device=dev)
    nat.check(nat.lib().pgcp_gather_complex(_ptr(tv), _ptr(src), _ptr(tmp), len(foreign), _stream()))
    nat.check(nat.lib().pgcp_scatter_complex(_ptr(tmp), _ptr(dst), _ptr(z), len(foreign), _stream()))


nat.register("pgcp_batch_shard_maps", [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p])
nat.register("pgcp_batch_stitch_ex", [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p])


def _shard_maps(batch, own, dev):
    """(face mask, own parent vertices, count) of this rank's submeshes."""
    mask = torch.empty(batch.m, dtype=torch.uint8, device=dev)
    ov = torch.empty(max(batch.n, 1), dtype=torch.int32, device=dev)
    cnt = ctypes.c_int64()
    arr = (ctypes.c_int32 * max(len(own), 1))(*[int(c) for c in own])
    nat.check(nat.lib().pgcp_batch_shard_maps(batch.h, arr, len(own), _ptr(mask), _ptr(ov), ctypes.byref(cnt),
                                              _stream()))
    return mask, ov[:cnt.value], int(cnt.value)


def _repair(batch, loop_gid, z, own, K, cfg, shard):
    """Per-submesh flip check and qc_correct of the folded ones
    (pipeline.py:88-102) -> the reference's report.repairs entries
    (pipeline.py:258-260). Remaining faces are local face indices (faces of
    a submesh in increasing parent-face order, partition.py:121-126)."""
    from .assemble import MU_CAP
    rows, _ = batch.qc_repair(loop_gid, z, comps=own, max_iter=cfg.repair_iters, cap=MU_CAP, rtol=cfg.rtol,
                              cluster=cfg.cluster)
    comps = list(range(K)) if own is None else list(own)
    info = np.zeros((K, 4), dtype=np.int64)
    for c, r in zip(comps, rows):
        info[c] = r
    if shard is not None and own is not None:  # every rank reports every submesh
        t = torch.as_tensor(info, device=z.device)
        shard.sum_(t)
        info = t.cpu().numpy()
    remaining = {}
    # submeshes still folded after the repair, over every rank's submeshes
    stuck_all = [c for c in range(K) if info[c, 1] > 0 and not info[c, 2]]
    stuck = [c for c in stuck_all if c in set(comps)]
    if stuck:
        _, flipped = batch.qc_repair(loop_gid, z, comps=stuck, max_iter=0, cap=MU_CAP, want_flipped=True)
        fl = flipped.cpu().numpy().astype(bool)
        fc = batch.host(nat.ARR_FACE_COMP, torch.int32)
        for c in stuck:
            pf = np.flatnonzero(fc == c)
            remaining[c] = [int(x) for x in np.flatnonzero(fl[pf])]
    if shard is not None and own is not None and stuck_all:  # the owners' lists, to every rank
        for part in shard.gather_objects(remaining):
            remaining.update(part)
    out = []
    for c in range(K):
        before, iters, cleared = int(info[c, 0]), int(info[c, 1]), bool(info[c, 2])
        e = {"flips_before": before, "repair_iterations": iters, "cleared": cleared}
        if before:
            e["remaining"] = remaining.get(c, [])
        e["submesh"] = c
        out.append(e)
    return out


_STREAMS = {}


def _streams(dev):
    """(high-priority, normal-priority) streams per device, kept for the life
    of the process (scratch allocated on them is freed on them)."""
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _STREAMS:
        lo_p, hi_p = torch.cuda.Stream.priority_range()
        _STREAMS[key] = (torch.cuda.Stream(device=dev, priority=hi_p), torch.cuda.Stream(device=dev, priority=lo_p))
    return _STREAMS[key]


def _geodesic_boundary(plan, tv, gc):
    """Disk mode (pipeline.py:216-235): map the global boundary onto the unit
    circle and push every other tracked point through the same log."""
    from .device import device
    dev = device()
    src = plan.any_slot_of_parents(gc).astype(np.int32)
    n = len(src)
    circ = torch.empty(n, dtype=torch.complex128, device=dev)
    cap = n + 8
    recs = (nat.Rec * cap)()
    meta = np.zeros(8)
    nat.check(nat.lib().pgcp_weld_geodesic(_ptr(tv), src.ctypes.data, n, None, _ptr(circ), recs, cap,
                                           meta.ctypes.data, _stream()))
    nrec = int(meta[0])
    # every slot whose parent is on the global cycle gets its circle value
    pos = np.full(plan.n_parent, -1, dtype=np.int64)
    pos[np.asarray(gc, dtype=np.int64)] = np.arange(n)
    sp = pos[plan.slot_parent]
    on = np.nonzero(sp >= 0)[0]
    off = np.nonzero(sp < 0)[0]
    if len(off):
        idx = torch.as_tensor(off.astype(np.int32)).to(dev)
        tmp = torch.empty(len(off), dtype=torch.complex128, device=dev)
        nat.check(nat.lib().pgcp_gather_complex(_ptr(tv), _ptr(idx), _ptr(tmp), len(off), _stream()))
        nat.check(nat.lib().pgcp_weld_replay(recs, nrec, _ptr(tmp), None, len(off), _stream()))
        nat.check(nat.lib().pgcp_scatter_complex(_ptr(tmp), _ptr(idx), _ptr(tv), len(off), _stream()))
    if len(on):
        src_on = torch.as_tensor(sp[on].astype(np.int32)).to(dev)
        dst_on = torch.as_tensor(on.astype(np.int32)).to(dev)
        tmp = torch.empty(len(on), dtype=torch.complex128, device=dev)
        nat.check(nat.lib().pgcp_gather_complex(_ptr(circ), _ptr(src_on), _ptr(tmp), len(on), _stream()))
        nat.check(nat.lib().pgcp_scatter_complex(_ptr(tmp), _ptr(dst_on), _ptr(tv), len(on), _stream()))


def _stitch(batch, z, mode, cfg, mesh, smaps=None):
    from .device import device
    dev = device()
    n, m = batch.n, batch.m
    coords = torch.empty(n, dtype=torch.complex128, device=dev)
    sphere = torch.empty((n, 3), dtype=torch.float64, device=dev) if mode == "sphere" else None
    prov = torch.empty(n, dtype=torch.int32, device=dev)
    flip = torch.empty(m, dtype=torch.uint8, device=dev)
    stats = np.zeros(8)
    mcode = {"free": 0, "disk": 1, "sphere": 2}[mode]
    if smaps is None:
        st = nat.lib().pgcp_batch_stitch(batch.h, _ptr(z), mcode, cfg.hard_tol, 1e-9, _ptr(coords),
                                         _ptr(sphere) if sphere is not None else None, _ptr(prov), _ptr(flip),
                                         stats.ctypes.data, _stream())
    else:  # sharded: flips of own faces; the seam check waits for the global scale (_finish)
        st = nat.lib().pgcp_batch_stitch_ex(batch.h, _ptr(z), mcode, float("inf"), 1e-9, _ptr(smaps[0]),
                                            _ptr(coords), _ptr(sphere) if sphere is not None else None, _ptr(prov),
                                            _ptr(flip), stats.ctypes.data, _stream())
    nat.check(st)
    nflip = int(stats[3])
    flipped = np.nonzero(flip.cpu().numpy())[0] if nflip else np.zeros(0, dtype=np.int64)
    diag = {"seam_max_dev": float(stats[0]), "scale": float(stats[1])}
    if mode == "disk":
        diag["boundary_circle_dev"] = float(stats[2])
    out = sphere if mode == "sphere" else coords
    gp = GlobalParam(mode, out, flipped, prov, float(stats[0]), diag)
    gp._device = True
    gp._nflip_local = nflip
    return gp, flip


def _finish(mesh, batch, embeddings, gp, report, cfg, clk, shard=None, smaps=None, own=None):
    """Energy, distortion report, acceptance flags (pipeline.py:274-297).
    Sharded: this rank measures its own faces; the global quantities are
    summed over ranks (dist.py) and the result's D2H covers only this
    rank's own vertices."""
    from .metrics import distortion_report
    clk.start()
    energy = None
    e_sub = batch.energy(embeddings) if gp.mode in ("free", "disk") else None
    nflip = int(len(gp.flipped_faces))
    if shard is None:
        if e_sub is not None:
            energy = float(e_sub.sum())
    else:
        # flips, energy and every rank's seam scale in one small all-reduce
        vec = np.zeros(2 + shard.world)
        vec[0] = gp._nflip_local
        vec[1] = float(e_sub[list(own)].sum()) if e_sub is not None and len(own) else 0.0
        vec[2 + shard.rank] = gp.diagnostics["scale"]
        t = torch.as_tensor(vec, device=embeddings.device)
        shard.sum_(t)
        vec = t.cpu().numpy()
        nflip = int(round(vec[0]))
        energy = float(vec[1]) if e_sub is not None else None
        scale = float(vec[2:].max())
        gp.diagnostics["scale"] = scale
        if scale > 0 and gp.seam_max_dev > cfg.hard_tol * scale:
            raise SolveError(f"seam disagreement {gp.seam_max_dev:.3e} exceeds {cfg.hard_tol:g} x scale "
                             f"{scale:.3e} (welding bug upstream)")
    V, F = mesh.device_arrays()
    pending = None
    if not cfg.keep_device:
        # the result's D2H runs on a copy stream while the metrics kernels run
        if smaps is None:
            pending = (_to_host_async(gp.coords), _to_host_async(gp.provenance.to(torch.int64)))
        else:  # this rank's own vertices only
            ov = smaps[1]
            pending = (_to_host_async(_rows(gp.coords, ov)), _to_host_async(_rows(gp.provenance, ov).to(torch.int64)),
                       _to_host_async(ov))
    if shard is None:
        dist = distortion_report(mesh, gp, energy=energy, V=V, F=F)
    else:
        dist = distortion_report(mesh, gp, energy=energy, V=V, F=F, face_mask=smaps[0], reduce=shard.reduce_fn())
        report.solver["exchanged_bytes"] = shard.exchanged_bytes
    clk.stop("metrics")
    if cfg.mobius_area:
        report.mobius_info = {"pre": None, "post": None, "improved": False,
                              "note": "Mobius area optimisation is out of scope on this path"}
    report.flips = nflip
    report.distortion = dist.to_dict()
    seam_ok = all(r <= cfg.snap_tol for r in report.seam_residuals)
    report.ok = report.flips == 0 and seam_ok
    if cfg.keep_device:
        if smaps is not None:
            gp.diagnostics["own_vertices"] = smaps[1]
        return gp, report
    # hand back host arrays, as the reference's GlobalParam holds numpy
    clk.start()
    if smaps is None:
        gp.coords = _host_result(pending[0])
        gp.provenance = _host_result(pending[1])  # widened on the device
    else:
        ov = _host_result(pending[2]).astype(np.int64)
        vals, prov = _host_result(pending[0]), _host_result(pending[1])
        full = np.full((mesh.n_vertices,) + vals.shape[1:], np.nan, dtype=vals.dtype)
        full[ov] = vals
        pv = np.full(mesh.n_vertices, -1, dtype=np.int64)
        pv[ov] = prov
        gp.coords, gp.provenance = full, pv
        gp.diagnostics["own_vertices"] = ov
        report.solver["d2h_bytes"] = int(vals.nbytes + prov.nbytes + 4 * len(ov))
    clk.stop("d2h")
    return gp, report


def _rows(t, idx):
    """t[idx] on the device (planar coordinates through the library's
    gather kernel; sphere rows and provenance through torch's index_select)."""
    if t.dtype == torch.complex128 and t.dim() == 1:
        out = torch.empty(idx.numel(), dtype=t.dtype, device=t.device)
        nat.check(nat.lib().pgcp_gather_complex(_ptr(t), _ptr(idx), _ptr(out), idx.numel(), _stream()))
        return out
    return t.index_select(0, idx.long())


_COPY_STREAMS = {}


def _to_host_async(t):
    """Queue a device -> pinned-host copy of t on a per-device copy stream,
    ordered after the work queued so far on the current stream."""
    dev = t.device
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = torch.cuda.Stream(device=dev)
    cs = _COPY_STREAMS[dev]
    cs.wait_stream(torch.cuda.current_stream(dev))
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    with torch.cuda.stream(cs):
        h.copy_(t, non_blocking=True)
        t.record_stream(cs)
        ev = torch.cuda.Event()
        ev.record(cs)
    return h, ev


def _host_result(pending):
    h, ev = pending
    ev.synchronize()
    return h.numpy()


def run_pipeline(config):
    config.validate()
    if not config.input:
        raise ValidationError("missing input mesh path")
    mesh = load_obj(config.input)
    cuts = read_cut_edges(config.cuts) if config.cuts else None
    gp, report = parameterize(mesh, cuts=cuts, config=config)
    if config.out:
        coords = gp.coords if gp.mode == "sphere" else gp.uv
        write_obj_with_param(config.out, mesh, coords)
    if config.report:
        report.to_json(config.report)
    return gp, report


def benchmark_subdomains(mesh, n_values, mode="free", repeats=3, workers=None, cut_files=None, seed=0):
    """T_n, S_n = T_2/T_n, E_n = S_n/(n/2) over subdomain counts
    (pipeline.py:320-361); strip cuts by face-centroid quantiles."""
    from .generators import cuts_from_face_labels
    n_values = sorted(set(int(n) for n in n_values))
    if any(n < 2 for n in n_values):
        raise ValidationError("subdomain counts must be >= 2")
    if 2 not in n_values:
        n_values = [2] + n_values
    T = {}
    for idx, n in enumerate(n_values):
        if cut_files:
            cuts = read_cut_edges(cut_files[idx])
        else:
            cent = mesh.vertices[mesh.faces].mean(axis=1)[:, 0]
            qs = np.quantile(cent, np.linspace(0, 1, n + 1)[1:-1])
            cuts = cuts_from_face_labels(mesh.faces, np.searchsorted(qs, cent, side="right"))
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            gp, rep = parameterize(mesh, cuts=cuts, mode=mode, seed=seed)
            times.append(time.perf_counter() - t0)
            if not rep.ok:
                raise SolveError(f"benchmark run with n={n} subdomains failed acceptance (flips={rep.flips})")
        T[n] = float(np.median(times))
    bench = {"n": n_values, "T_n": {str(n): T[n] for n in n_values},
             "S_n": {str(n): T[2] / T[n] for n in n_values},
             "E_n": {str(n): (T[2] / T[n]) / (n / 2.0) for n in n_values}, "repeats": repeats}
    out = RunReport(mode=mode, n_vertices=mesh.n_vertices, n_faces=mesh.n_faces)
    out.bench = bench
    out.ok = True
    out.timings = {f"T_{n}": T[n] for n in n_values}
    return out
