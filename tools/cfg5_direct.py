"""cfg 5 (4096^2, 64 bumps, 16x16 blocks) with the direct solver: the flatten
and the Dirichlet solve of all 256 subdomains, timed, with factorization
statistics; a sample compared with the PCG path.

    python tools/cfg5_direct.py
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

torch.cuda.set_device(0)
V, F, cuts = gen.height_field_case(4096, 16, n_bumps=64, seed=0)
part = pg.partition_mesh(pg.TriMesh(V, F), cuts)
b = part.batch
b.laplacian()
voff = b.host(nat.ARR_VERT_OFF, torch.int64)
loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
lp = b.host(nat.ARR_LOOP, torch.int32)
gid = torch.tensor(np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32),
                   device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    z, st = b.flatten(solver="direct")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    zh, sth = b.harmonic(gid, z[gid.long()], solver="direct")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    fl, hm = b.last_solve(0), b.last_solve(1)
    assert all(x["status"] == 0 for x in st) and all(x["status"] == 0 for x in sth)
    print(f"rep {rep}: flatten {1e3*(t1-t0):.1f} ms (factor {fl['factor_ms']:.1f}, solve {fl['solve_ms']:.1f}, "
          f"FMAs {fl['fmas']:.3g}, max front {fl['max_front']}, fronts {fl['front_bytes']/1e9:.2f} GB), "
          f"harmonic {1e3*(t2-t1):.1f} ms (factor {hm['factor_ms']:.1f}, solve {hm['solve_ms']:.1f}, "
          f"fronts {hm['front_bytes']/1e9:.2f} GB); mem {torch.cuda.mem_get_info()[0]/1e9:.1f} GB free", flush=True)
zd = z.cpu().numpy()
zp, stp = b.flatten(solver="pcg")
zp = zp.cpu().numpy()
worst = 0
for c in range(0, b.K, 17):
    a_, e_ = zd[voff[c]:voff[c + 1]], zp[voff[c]:voff[c + 1]]
    worst = max(worst, np.max(np.abs(a_ - e_)) / (2 * np.max(np.abs(e_ - e_.mean()))))
print(f"direct vs pcg (every 17th subdomain): max err / diam {worst:.2e}; pcg kernel {b.last_solve(0)['kernel_ms']:.0f} ms")
