"""Standalone wall time of the harmonic preparation (pgcp_batch_harmonic_
prepare: unknown numbering, sliced ELL, Jacobi scaling, coarse space,
column encoding) on cfg 2, with nothing else on the GPU, and of the
flatten's system build for comparison."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen, _native as nat

V, F, cuts = gen.height_field_case(1024, 8)
b = pg.partition_mesh(pg.TriMesh(V, F, check=False), cuts).batch
b.laplacian()
z, st = b.flatten()
voff = b.host(nat.ARR_VERT_OFF, torch.int64)
loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
lp = b.host(nat.ARR_LOOP, torch.int32)
gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
g = torch.as_tensor(gid).cuda()
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b.harmonic_prepare(g)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    b.flatten()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    fl = b.last_solve(0)
    print(f"harmonic_prepare {1e3 * (t1 - t0):.2f} ms standalone; flatten call {1e3 * (t2 - t1):.2f} ms "
          f"(kernel {fl['kernel_ms']:.2f}, coarse setup {fl['coarse_ms']:.2f})", flush=True)
