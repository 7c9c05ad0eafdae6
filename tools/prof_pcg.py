"""Run the cfg-2 DNCP flatten once (profiling helper for ncu)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

grid = int(os.environ.get("GRID", "1024"))
blocks = int(os.environ.get("BLOCKS", "8"))
which = os.environ.get("WHICH", "flatten")
V, F, cuts = gen.height_field_case(grid, blocks)
mesh = pg.TriMesh(V, F, check=False)
part = pg.partition_mesh(mesh, cuts)
b = part.batch
b.laplacian()
torch.cuda.synchronize()
t0 = time.perf_counter()
z, st = b.flatten(cluster=int(os.environ.get("CLUSTER", "0")))
torch.cuda.synchronize()
print("flatten", time.perf_counter() - t0, b.last_solve(0))
