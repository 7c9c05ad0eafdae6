"""cProfile of the host side of parameterize on cfg 2 (value and e2e styles)."""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
mesh = pg.TriMesh(V, F)
pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)

def e2e():
    m = pg.TriMesh(V, F)
    gp, rep = pg.parameterize(m, cuts, "free", pairs=pairs)
    return rep

def val():
    gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
    return rep

for name, fn in (("value", val), ("e2e", e2e)):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pr = cProfile.Profile(); pr.enable(); rep = fn(); torch.cuda.synchronize(); pr.disable()
    print(f"=== {name}: {1e3*(time.perf_counter()-t0):.1f} ms; stages", {k: round(1e3*v, 1) for k, v in rep.timings.items()})
    s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue()[:6000])
