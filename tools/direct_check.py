"""GPU check of the multifrontal direct solver (direct.cu) against the PCG
path and the CPU oracle: per-subdomain flatten and Dirichlet solves on a
small case (vs SuperLU), then cfg 2 end to end (direct vs PCG UV, stage
times, factorization statistics).

    python tools/direct_check.py [grid] [blocks]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402


def small():
    import oracle
    V, F, cuts = gen.height_field_case(129, 4, seed=1)
    part = pg.partition_mesh(pg.TriMesh(V, F), cuts)
    b = part.batch
    b.laplacian()
    zd, std = b.flatten(solver="direct")
    sd = b.last_solve(0)
    zp, stp = b.flatten(solver="pcg")
    zd, zp = zd.cpu().numpy(), zp.cpu().numpy()
    print("direct stats:", {k: sd[k] for k in ("fmas", "factor_ms", "solve_ms", "max_front", "nodes", "levels")})
    print("status direct", [s["status"] for s in std][:8], "true_res", max(s["true_res"] for s in std))
    print("flatten direct vs pcg max |dz| / diam:", np.max(np.abs(zd - zp)) / (2 * np.max(np.abs(zp))))
    sp = oracle.split_mesh(V, F, cuts)
    off = np.concatenate([[0], np.cumsum([len(v) for v in sp.sub_V])])
    worst = 0
    for i in range(sp.n_sub):
        zr = oracle.dncp_flatten(sp.sub_V[i], sp.sub_F[i], sp.loops[i])
        diam = 2 * np.max(np.abs(zr - zr.mean()))
        worst = max(worst, np.max(np.abs(zd[off[i]:off[i + 1]] - zr)) / diam)
    print("flatten direct vs oracle (SuperLU) max err / diam:", worst)
    # Dirichlet: boundary values from the oracle flatten
    loops = [np.asarray(l) for l in sp.loops]
    gid = np.concatenate([off[i] + loops[i] for i in range(sp.n_sub)]).astype(np.int32)
    vals = np.concatenate([zd[off[i] + loops[i]] for i in range(sp.n_sub)])
    zh, sth = b.harmonic(gid, vals, solver="direct")
    print("harmonic stats:", {k: b.last_solve(1).get(k) for k in ("fmas", "factor_ms", "solve_ms", "max_front")})
    zh = zh.cpu().numpy()
    worst = 0
    loff = np.concatenate([[0], np.cumsum([len(l) for l in loops])])
    for i in range(sp.n_sub):
        zr = oracle.dirichlet_extend(sp.sub_V[i], sp.sub_F[i], loops[i], vals[loff[i]:loff[i + 1]])
        diam = 2 * np.max(np.abs(zr - zr.mean()))
        worst = max(worst, np.max(np.abs(zh[off[i]:off[i + 1]] - zr)) / diam)
    print("harmonic direct vs oracle max err / diam:", worst)


def cfg2(grid, blocks):
    V, F, cuts = gen.height_field_case(grid, blocks)
    pairs = gen.quadtree_schedule_order(blocks, blocks)
    out = {}
    for solver in ("direct", "pcg"):
        os.environ["PGCP_SOLVER"] = solver
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            gp, rep_ = pg.parameterize(pg.TriMesh(V, F), cuts, "free", pairs=pairs)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        out[solver] = np.asarray(gp.coords)
        st = rep_.stages_ms if hasattr(rep_, "stages_ms") else None
        print(f"[{solver}] wall {dt*1e3:.1f} ms, flips {rep_.flips}, mean |d| {rep_.distortion['angular_abs']['mean']:.6f}",
              flush=True)
        sv = rep_.solver
        for k in ("flatten", "harmonic"):
            d = sv.get(k, {})
            print(f"   {k}: " + ", ".join(f"{x}={d[x]:.4g}" if isinstance(d[x], float) else f"{x}={d[x]}"
                                      for x in d), flush=True)
        if hasattr(rep_, "timings"):
            print("   timings", rep_.timings)
    z0, z1 = out["direct"], out["pcg"]
    diam = 2 * np.max(np.abs(z1 - z1.mean()))
    print("cfg UV direct vs pcg max |dz| / diam:", np.max(np.abs(z0 - z1)) / diam)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    small()
    g = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cfg2(g, k)
