"""Run the cfg-2 DNCP flatten (and a harmonic solve) a few times; profiling
helper for ncu and PGCP_PCG_TIMING=1 phase timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen
from paper_1903_12359_b200 import _native as nat

grid = int(os.environ.get("GRID", "1024"))
blocks = int(os.environ.get("BLOCKS", "8"))
reps = int(os.environ.get("REPS", "1"))
V, F, cuts = gen.height_field_case(grid, blocks)
mesh = pg.TriMesh(V, F, check=False)
part = pg.partition_mesh(mesh, cuts)
b = part.batch
b.laplacian()
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    z, st = b.flatten(cluster=int(os.environ.get("CLUSTER", "0")))
    torch.cuda.synchronize()
    print("flatten", round(1e3 * (time.perf_counter() - t0), 2), "ms", b.last_solve(0), flush=True)
    if r == 0 and os.environ.get("ITERS"):
        print("iters by slot", [s["iters"] for s in st], flush=True)
if os.environ.get("HARMONIC"):
    loop_gid = []
    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
    loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
    lp = b.host(nat.ARR_LOOP, torch.int32)
    import numpy as np
    for c in range(b.K):
        loop_gid.append(voff[c] + lp[loff[c]:loff[c + 1]])
    gid = np.concatenate(loop_gid).astype(np.int32)
    vals = z[torch.as_tensor(gid, device=z.device).long()]
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        zh, sth = b.harmonic(gid, vals)
        torch.cuda.synchronize()
        print("harmonic", round(1e3 * (time.perf_counter() - t0), 2), "ms", b.last_solve(1), flush=True)
