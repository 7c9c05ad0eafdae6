"""A few cfg-2 parameterize calls with the bench's settings (stage timings
printed; PGCP_* switches from the environment)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402

torch.cuda.set_device(0)
V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
mesh = pg.TriMesh(V, F)
mesh.device_arrays()
import time  # noqa: E402
for i in range(int(os.environ.get("REPS", "4"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
    torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t0)
    print(f"wall {wall:.2f} ms", {k: round(1e3 * v, 2) for k, v in rep.timings.items()}, file=sys.stderr, flush=True)
