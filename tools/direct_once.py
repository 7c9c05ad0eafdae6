"""One direct flatten + one Dirichlet solve of cfg 2 (for ncu launch lists)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import _native as nat  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402

torch.cuda.set_device(0)
V, F, cuts = gen.height_field_case(int(os.environ.get("GRID", 1024)), int(os.environ.get("BLOCKS", 8)))
part = pg.partition_mesh(pg.TriMesh(V, F), cuts)
b = part.batch
b.laplacian()
z, st = b.flatten(solver=os.environ.get("SOLVER", "direct"))
torch.cuda.synchronize()
if os.environ.get("HARMONIC", "1") == "1":
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
    lp = b.host(nat.ARR_LOOP, torch.int32)
    gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
    zh, sth = b.harmonic(gid, z.cpu().numpy()[gid], solver=os.environ.get("SOLVER", "direct"))
    torch.cuda.synchronize()
print("ok", b.last_solve(0)["solver"])
