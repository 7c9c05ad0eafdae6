import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen
V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
Vn = torch.from_numpy(np.ascontiguousarray(V)).pin_memory().numpy()
Fn = torch.from_numpy(np.ascontiguousarray(F.astype(np.int32))).pin_memory().numpy()
Cn = torch.from_numpy(np.ascontiguousarray(cuts)).pin_memory().numpy()
for it in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    mesh = pg.TriMesh(Vn, Fn)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    gp, rep = pg.parameterize(mesh, Cn, "free", pairs=pairs)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"TriMesh {1e3*(t1-t0):.2f} ms  parameterize {1e3*(t2-t1):.2f} ms  stages {{{', '.join(f'{k}: {v*1e3:.2f}' for k, v in rep.timings.items())}}}", flush=True)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m2 = pg.TriMesh(Vn, Fn, check=False)
    m2.device_arrays()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    m2.batch()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"H2D {1e3*(t1-t0):.2f} ms  validation batch {1e3*(t2-t1):.2f} ms", flush=True)
