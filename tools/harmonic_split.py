import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen, _native as nat
V, F, cuts = gen.height_field_case(1024, 8)
b = pg.partition_mesh(pg.TriMesh(V, F, check=False), cuts).batch
b.laplacian()
z, st = b.flatten()
voff = b.host(nat.ARR_VERT_OFF, torch.int64); loff = b.host(nat.ARR_LOOP_OFF, torch.int64); lp = b.host(nat.ARR_LOOP, torch.int32)
gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
g = torch.as_tensor(gid).cuda()
vals = z[g.long()].clone()
for it in range(4):
    b.harmonic_prepare(g)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    zh, sth = b.harmonic_solve(vals)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    rows, _ = b.qc_repair(g, zh)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"harmonic_solve {1e3*(t1-t0):.2f} ms (kernel {b.last_solve(1)['kernel_ms']:.2f})  flip check {1e3*(t2-t1):.2f} ms", flush=True)
