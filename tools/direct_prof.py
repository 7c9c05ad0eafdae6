"""Standalone timing of the batched solves on cfg 2 (no pipeline overlap):
wall time of batch.flatten / harmonic_prepare / harmonic_solve with the
direct solver, plus the library's own split (PGCP_DIRECT_TIMING=1,
PGCP_PCG_TIMING=1 print to stderr).

    python tools/direct_prof.py [solver] [grid] [blocks]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import _native as nat  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402

solver = sys.argv[1] if len(sys.argv) > 1 else "direct"
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 8
torch.cuda.set_device(0)
V, F, cuts = gen.height_field_case(grid, blocks)
part = pg.partition_mesh(pg.TriMesh(V, F), cuts)
b = part.batch
b.laplacian()
voff = b.host(nat.ARR_VERT_OFF, torch.int64)
loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
lp = b.host(nat.ARR_LOOP, torch.int32)
gid = torch.tensor(np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32),
                   device="cuda")
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    z, st = b.flatten(solver=solver)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    b.harmonic_prepare(gid, solver=solver)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    zh, sth = b.harmonic_solve(z[gid.long()], solver=solver)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    fl, hm = b.last_solve(0), b.last_solve(1)
    print(f"rep {rep}: flatten {1e3*(t1-t0):.2f} ms (factor {fl.get('factor_ms', 0):.2f}, solve "
          f"{fl.get('solve_ms', fl['kernel_ms']):.2f}), harmonic prepare {1e3*(t2-t1):.2f} ms (factor "
          f"{hm.get('factor_ms', 0):.2f}), harmonic solve {1e3*(t3-t2):.2f} ms (solve {hm.get('solve_ms', hm['kernel_ms']):.2f})",
          file=sys.stderr, flush=True)
