"""Per-level timeline of the persistent substitution sweeps (k_solve_pers) on
cfg 2: flatten + Dirichlet solve twice, PGCP_DIRECT_SOLVE_TRACE on the
second pass (stderr).

    python tools/solve_trace.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import _native as nat  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402

torch.cuda.set_device(0)
V, F, cuts = gen.height_field_case(1024, 8)
b = pg.partition_mesh(pg.TriMesh(V, F), cuts).batch
b.laplacian()
voff = b.host(nat.ARR_VERT_OFF, torch.int64)
loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
lp = b.host(nat.ARR_LOOP, torch.int32)
gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
for rep in range(2):
    if rep == 1:
        os.environ["PGCP_DIRECT_SOLVE_TRACE"] = "1"
        print("=== flatten", file=sys.stderr, flush=True)
    z, st = b.flatten(solver="direct")
    torch.cuda.synchronize()
    if rep == 1:
        print("=== harmonic", file=sys.stderr, flush=True)
    zh, sth = b.harmonic(gid, z.cpu().numpy()[gid], solver="direct")
    torch.cuda.synchronize()
    print("solve ms", b.last_solve(0)["solve_ms"], b.last_solve(1)["solve_ms"], flush=True)
