"""Weld-order A/B on cfg 2: stage times and distortion for the rows-as-chains,
pairwise-tree and quadtree orders."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

V, F, cuts = gen.height_field_case(1024, 8)
mesh = pg.TriMesh(V, F)
for name, pairs in [("rows-chain", gen.row_tree_schedule_order(8, 8)),
                    ("pairwise", gen.pairwise_tree_schedule_order(8, 8)),
                    ("quadtree", gen.quadtree_schedule_order(8, 8))]:
    ts = []
    for _ in range(3):
        gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
        ts.append(rep.timings)
    w = statistics.median(t["weld"] for t in ts) * 1e3
    tot = statistics.median(sum(t.values()) for t in ts) * 1e3
    d = rep.distortion["angular_abs"]
    print(f"{name:11s} weld {w:6.2f} ms total {tot:6.1f} ms | flips {rep.flips} mean {d['mean']:.6f} "
          f"sd {d['sd']:.6f} median {d['median']:.6f}", flush=True)
