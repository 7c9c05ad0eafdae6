"""The bench's e2e leg with stage timings: TriMesh from pinned host arrays
+ parameterize + coordinates to the host, a few reps."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402

torch.cuda.set_device(0)
V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
Vn = torch.from_numpy(np.ascontiguousarray(V)).pin_memory().numpy()
Fn = torch.from_numpy(np.ascontiguousarray(F.astype(np.int32))).pin_memory().numpy()
Cn = torch.from_numpy(np.ascontiguousarray(cuts)).pin_memory().numpy()
for i in range(int(os.environ.get("REPS", "5"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mesh = pg.TriMesh(Vn, Fn)
    t1 = time.perf_counter()
    gp, rep = pg.parameterize(mesh, Cn, "free", pairs=pairs)
    t2 = time.perf_counter()
    c = gp.coords
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"e2e {1e3*(t3-t0):.2f} ms: TriMesh {1e3*(t1-t0):.2f} parameterize {1e3*(t2-t1):.2f} tail {1e3*(t3-t2):.2f}",
          {k: round(1e3 * v, 2) for k, v in rep.timings.items()}, file=sys.stderr, flush=True)
