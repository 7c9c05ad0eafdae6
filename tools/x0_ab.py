"""A/B of the coarse start (PGCP_PCG_X0) on cfg 2: flatten and harmonic
kernel time and PCG iterations. Run once per setting of the variable."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen, _native as nat

V, F, cuts = gen.height_field_case(1024, 8)
b = pg.partition_mesh(pg.TriMesh(V, F, check=False), cuts).batch
b.laplacian()
for rep in range(3):
    z, st = b.flatten()
    s = b.last_solve(0)
    print("x0", os.environ.get("PGCP_PCG_X0", "0"), "flatten kernel", round(s["kernel_ms"], 2), "ms",
          {k: v for k, v in s.items() if "iter" in k}, flush=True)
voff = b.host(nat.ARR_VERT_OFF, torch.int64); loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
lp = b.host(nat.ARR_LOOP, torch.int32)
gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
g = torch.as_tensor(gid).cuda()
vals = z[g.long()].clone()
for rep in range(3):
    b.harmonic_prepare(g)
    zh, sth = b.harmonic_solve(vals)
    s = b.last_solve(1)
    print("x0", os.environ.get("PGCP_PCG_X0", "0"), "harmonic kernel", round(s["kernel_ms"], 2), "ms",
          {k: v for k, v in s.items() if "iter" in k}, flush=True)
