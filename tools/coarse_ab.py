"""A/B of the PCG preconditioner on cfg 2: Jacobi (PGCP_PCG_COARSE=0) vs
two-level (default). Prints stage times, iteration totals and the UV change."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

grid = int(os.environ.get("GRID", "1024"))
blocks = int(os.environ.get("BLOCKS", "8"))
V, F, cuts = gen.height_field_case(grid, blocks)
pairs = gen.quadtree_schedule_order(blocks, blocks)
mesh = pg.TriMesh(V, F)
res = {}
for mode in ["0", "1", "0", "1"]:
    os.environ["PGCP_PCG_COARSE"] = mode
    ts = {}
    for rep_i in range(3):
        gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
        for k, v in rep.timings.items():
            ts.setdefault(k, []).append(1e3 * v)
    z = gp.coords.cpu().numpy()
    fl, hm = rep.solver["flatten"], rep.solver["harmonic"]
    res[mode] = z
    print(f"coarse={mode}: " + " ".join(f"{k} {statistics.median(v):.1f}" for k, v in ts.items()),
          f"| flatten kernel {fl['kernel_ms']:.1f} ms iters sum {fl['iters_sum']:.0f} max {fl['iters_max']:.0f}",
          f"| harmonic kernel {hm['kernel_ms']:.1f} ms iters sum {hm['iters_sum']:.0f} max {hm['iters_max']:.0f}",
          f"| flips {rep.flips} mean {rep.distortion['angular_abs']['mean']:.9f}", flush=True)
d = np.abs(res["0"] - res["1"]).max() / (np.abs(res["0"]).max())
print("max |uv0 - uv1| / max|uv| =", d)
