"""Weld-stage time on cfg 2 for phase-1 launch shapes (PGCP_WELD_NT threads
per CTA, PGCP_WELD_PPT points per thread -> CTAs per cluster)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
mesh = pg.TriMesh(V, F)
ref = None
for nt, ppt in [(256, 1), (256, 2), (512, 1), (512, 2), (512, 4), (512, 8), (256, 4), (256, 16)]:
    os.environ["PGCP_WELD_NT"] = str(nt)
    os.environ["PGCP_WELD_PPT"] = str(ppt)
    ts = []
    for _ in range(4):
        gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
        ts.append(rep.timings["weld"] * 1e3)
    z = gp.coords.cpu().numpy()
    if ref is None:
        ref = z
    print(f"NT={nt} PPT={ppt}: weld {statistics.median(ts[1:]):.2f} ms  identical={np.array_equal(z, ref)}", flush=True)
