"""Weld-stage time on cfg 2 against the streamed replay's counter interval
(PGCP_WELD_PROG_EVERY) and with the serial replay (PGCP_WELD_STREAM=0)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
mesh = pg.TriMesh(V, F)
ref = None
for stream, every in [("1", 8), ("1", 16), ("1", 32), ("1", 64), ("1", 4), ("0", 8)]:
    os.environ["PGCP_WELD_STREAM"] = stream
    os.environ["PGCP_WELD_PROG_EVERY"] = str(every)
    ts = []
    for _ in range(5):
        gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
        ts.append(rep.timings["weld"] * 1e3)
    z = gp.coords.cpu().numpy()
    ref = z if ref is None else ref
    print(f"stream={stream} every={every}: weld {statistics.median(ts[1:]):.2f} ms identical={np.array_equal(z, ref)}",
          flush=True)
