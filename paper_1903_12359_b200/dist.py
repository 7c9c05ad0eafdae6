"""Multi-GPU PGCP: subdomain sharding across ranks (SURVEY.md §8 row e).

The reference parallelises with one process per subdomain solve
(`pipeline._run_tasks`, pipeline.py:105-109), while the partition, weld loop
and stitch stay serial in the driver process. Here one process drives one
GPU, and the data plane is the one SURVEY §8(e) specifies:

  partition        every rank (replicated, deterministic)
  flatten          rank r solves only its own subdomains (LPT shard)
  exchange         ONE all-gather (NCCL over NVLink) of the boundary-loop
                   values of every rank's subdomains: each rank packs its
                   own slots, and a scatter puts the gathered blocks into the
                   tracked-value vector in slot order (Σnb x 16 B in total)
  weld / boundary  every rank (replicated: the record chain is serial and
                   identical inputs give identical outputs)
  harmonic/repair  rank r solves (and repairs) only its own subdomains; the
                   welded Dirichlet values are already known to every rank,
                   so every seam copy of every parent vertex is known too
  stitch/metrics   every rank stitches all seam vertices and its own
                   interiors, and measures only its own faces; the report's
                   global quantities (flip count, energy, repair info, seam
                   scale; the distortion sums, exact order statistics and
                   histogram counts) are summed over ranks with small
                   all-reduces (a few KB to ~0.1 MB, `pgcp_reduce_fn`)
  result           per-rank D2H of the rank's own vertices (no collective);
                   `gather_coords` assembles the full UV on one rank if asked

Every rank returns the same RunReport; GlobalParam.coords holds this rank's
own vertices (every seam vertex included) and NaN elsewhere.
"""

import ctypes
import json
import os
import statistics
import time
import traceback

import numpy as np
import torch
import torch.distributed as dist


def subdomain_cost(n):
    """Relative solve cost of an n-vertex subdomain: CG iterations grow like
    sqrt(n) (2-D Laplacian, condition ~ n), each costs O(n)."""
    return float(n) ** 1.5


def lpt_shards(sizes, world):
    """Longest-processing-time assignment of subdomains to `world` ranks.
    Deterministic: ties broken by subdomain id, then by rank. Returns one
    sorted list of subdomain ids per rank."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    order = sorted(range(len(sizes)), key=lambda i: (-subdomain_cost(sizes[i]), i))
    load = [0.0] * world
    out = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        out[r].append(i)
        load[r] += subdomain_cost(sizes[i])
    return [sorted(s) for s in out]


from ._native import REDUCE_FN  # noqa: E402

_RED_TYPESTR = {0: "<f8", 1: "<i4", 2: "<i8"}  # u32 / u64 sums are summed as their signed views (same bits)


class Shard:
    """Rank-local view of the sharded pipeline (pass as parameterize(shard=))."""

    def __init__(self, group=None):
        if not dist.is_available() or not dist.is_initialized():
            raise RuntimeError("Shard needs an initialised torch.distributed process group")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.exchanged_bytes = 0
        self.shards = None
        self._cfn = None

    def comps(self, sizes):
        """This rank's submeshes (LPT over every rank; all ranks agree)."""
        self.shards = lpt_shards(list(sizes), self.world)
        return self.shards[self.rank]

    # -- the boundary exchange ------------------------------------------------
    def slot_layout(self, loop_off):
        """(own slots, scatter map of the gathered buffer, block length).
        Rank r's block holds the slots of its submeshes in slot order,
        padded to the longest block; the map sends every gathered entry to
        its slot, padding to the dummy slot Σnb."""
        nslot = int(loop_off[-1])
        per = [np.concatenate([np.arange(loop_off[c], loop_off[c + 1]) for c in sh]).astype(np.int64)
               if len(sh) else np.zeros(0, np.int64) for sh in self.shards]
        blk = max(1, max(len(p) for p in per))
        smap = np.full(self.world * blk, nslot, dtype=np.int32)
        for r, p in enumerate(per):
            smap[r * blk:r * blk + len(p)] = p
        return per[self.rank], smap, blk

    def all_gather_(self, send, recv):
        """recv[r * len(send):(r + 1) * len(send)] = rank r's send."""
        sv, rv = torch.view_as_real(send) if send.is_complex() else send, \
            torch.view_as_real(recv) if recv.is_complex() else recv
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(rv, sv, group=self.group)
        else:  # gloo (CPU tests, the one-GPU two-rank test): the list form
            dist.all_gather(list(rv.chunk(self.world)), sv, group=self.group)
        self.exchanged_bytes += rv.numel() * rv.element_size()
        return recv

    # -- small reductions -------------------------------------------------------
    def sum_(self, t):
        """In-place sum over ranks (complex tensors as their real view)."""
        v = torch.view_as_real(t) if t.is_complex() else t
        dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
        self.exchanged_bytes += v.numel() * v.element_size()
        return t

    def reduce_fn(self):
        """pgcp_reduce_fn for the native sharded metrics: an all-reduce of a
        device buffer on the current stream (NCCL orders it there)."""
        if self._cfn is None:
            from .device import _CudaArray, device

            def fn(buf, count, dtype, op, user, stream):
                try:
                    t = torch.as_tensor(_CudaArray(buf, count, _RED_TYPESTR[dtype], None), device=device())
                    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM, group=self.group)
                    self.exchanged_bytes += t.numel() * t.element_size()
                    return 0
                except BaseException:  # reported by the native caller as a failed reduction
                    traceback.print_exc()
                    return 1

            self._cfn = REDUCE_FN(fn)
        return self._cfn

    def gather_objects(self, obj):
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out


def gather_coords(gp, shard, dst=0):
    """Assemble the full parameterization on rank `dst` from every rank's
    own vertices (each rank holds NaN elsewhere). Not part of the timed
    pipeline: the product returns each rank's share by a per-rank D2H."""
    own = np.asarray(gp.diagnostics["own_vertices"])
    vals = np.asarray(gp.coords)[own]
    parts = shard.gather_objects((own, vals))
    if shard.rank != dst:
        return None
    full = np.array(gp.coords, copy=True)
    for o, v in parts:
        full[o] = v
    return full


def parameterize_distributed(mesh, cuts=None, mode="free", group=None, **kw):
    """`parameterize` with the subdomain solves sharded over the ranks of
    `group`; every rank returns the same RunReport and a GlobalParam with
    its own vertices (`gather_coords` assembles the whole map)."""
    from .pipeline import parameterize
    return parameterize(mesh, cuts, mode, shard=Shard(group), **kw)


def _max_over_ranks(x, dev):
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x, dev):
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def bench_distributed(args, V, F, cuts, pairs, metric, unit, workload):
    """bench.py at N > 1 (torchrun, one rank per GPU, NCCL): strong scaling of
    the cfg-2 pipeline. Device time per step is the max over ranks of CUDA
    event time; rank 0 prints the JSON line."""
    import paper_1903_12359_b200 as pg
    from . import _native as nat
    import bench as B

    if "RANK" not in os.environ:  # a single process outside torchrun (PGCP_BENCH_DIST=1)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(port))
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    try:
        lib = nat.lib()
        n = len(V)
        mesh_dev = pg.TriMesh(V, F)
        mesh_dev.device_arrays()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        shard = Shard()

        def step():
            return pg.parameterize(mesh_dev, cuts, "free", pairs=pairs, keep_device=True, shard=shard)

        for _ in range(args.warmup):
            gp, rep = step()
        if rep.flips:
            raise RuntimeError("warm-up run produced flips")
        stream = torch.cuda.current_stream()
        sampler = B.ClockSampler(local) if rank == 0 else None
        dist.barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.start()
        l0 = lib.pgcp_launch_count()
        ms_steps, num_ms, num_fmas = [], [], []  # the direct solver's numeric phase of this rank's flatten
        for _ in range(args.steps):
            flush.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gp, rep = step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms_steps.append(_max_over_ranks(e0.elapsed_time(e1), dev))
            fl = rep.solver["flatten"]
            if fl.get("solver") != "direct":
                raise RuntimeError("the bench measures the default (direct) solver")
            num_ms.append(fl["numeric_ms"])
            num_fmas.append(fl["fmas"])
        dist.barrier()
        torch.cuda.synchronize()
        launches = _sum_over_ranks(lib.pgcp_launch_count() - l0, dev)
        clocks = sampler.stop() if sampler else None
        ms = statistics.mean(ms_steps)
        value = n / (ms / 1e3)

        e2e = None
        if not args.no_e2e:
            Vn = torch.from_numpy(np.ascontiguousarray(V)).pin_memory().numpy()
            Fn = torch.from_numpy(np.ascontiguousarray(F.astype(np.int32))).pin_memory().numpy()
            Cn = torch.from_numpy(np.ascontiguousarray(cuts)).pin_memory().numpy()
            h2d = Vn.nbytes + Fn.nbytes + Cn.nbytes
            d2h = 0
            et = []
            for i in range(args.warmup + args.steps):
                dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                mesh = pg.TriMesh(Vn, Fn)
                gp, rep = parameterize_distributed(mesh, Cn, "free", pairs=pairs)
                d2h = rep.solver.get("d2h_bytes", 0)  # this rank's own vertices (coords, provenance, ids)
                torch.cuda.synchronize()
                dt = _max_over_ranks(time.perf_counter() - t0, dev)
                if i >= args.warmup:
                    et.append(dt)
            e = statistics.mean(et)
            e2e = {"value": n / e, "unit": unit, "ms_per_step": 1e3 * e, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h)}

        peak, peak_src = B.measured_peak()
        fp64 = B.fp64_probe_tflops()
        numeric_ms = _max_over_ranks(statistics.mean(num_ms), dev)
        fmas_all = _sum_over_ranks(statistics.mean(num_fmas), dev)
        if rank == 0:
            # per-GPU average of the factorization flops over the slowest rank's numeric phase
            achieved = 2.0 * fmas_all / world / (numeric_ms / 1e3) / 1e12
            roof = {"bound": "fp64",
                    "kernel": "multifrontal numeric factorization of each rank's shard of the 64 cfg-2 DNCP "
                              "systems (bench.py's `roofline` at N = 1)",
                    "achieved": achieved, "peak": fp64, "unit": "TFLOP/s",
                    "frac": achieved / fp64 if fp64 else None,
                    "traffic": B.ncu_summary("r2_direct_ncu_summary_end.json").get("dram_bytes_per_factorization"),
                    "peak_source": "measured here: pgcp_fp64_probe on rank 0", "numeric_ms": numeric_ms,
                    "flops_per_step_all_ranks": 2.0 * fmas_all, "hbm_peak": peak, "hbm_peak_source": peak_src,
                    "note": "per-GPU average of the factorization flops over the slowest rank's numeric "
                            "phase; latency-bound small fronts (DESIGN.md section 4b); `traffic` is the "
                            "single-GPU capture"}
            line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                    "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                    "config": {"workload": workload, "n_vertices": n, "n_faces": int(len(F)),
                               "n_subdomains": 64, "l2": "flushed before every timed step (256 MiB write)",
                               "parallelism": f"subdomain shards over {world} GPUs (LPT): one NCCL all-gather "
                                              "of the boundary-loop values after the flatten, replicated weld, "
                                              "per-rank harmonic/stitch/metrics with small reductions, per-rank "
                                              "D2H of own vertices"},
                    "roofline": roof, "cpu_baseline": None, "e2e": e2e, "clocks": clocks,
                    "gpu_launches": int(launches), "exchanged_bytes_per_step": shard.exchanged_bytes
                    / max(1, args.warmup + args.steps),
                    "quality": {"flips": rep.flips, "angular_mean_deg": rep.distortion["angular_abs"]["mean"]}}
            print(json.dumps(line), flush=True)
        dist.barrier()
    finally:
        dist.destroy_process_group()
    return 0
