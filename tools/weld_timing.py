import os, sys
sys.path.insert(0, os.getcwd())
os.environ.setdefault("PGCP_WELD_TIMING", "1")
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen
V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
mesh = pg.TriMesh(V, F)
for _ in range(2):
    gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
    print("weld ms", rep.timings["weld"] * 1e3, flush=True)
