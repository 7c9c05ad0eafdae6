"""cfg-2 pipeline a few times (warm-up + measured runs); also the launch
target for ncu captures of the weld kernels (k_phase1c / k_replay_slots)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
mesh = pg.TriMesh(V, F)
for _ in range(int(os.environ.get("REPS", "2"))):
    gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
    print({k: round(1e3 * v, 2) for k, v in rep.timings.items()}, flush=True)
