"""Flatten kernel time of the first n cfg-2 subdomains (the per-GPU share at
64/n GPUs) for the automatic cluster shape and forced 4 / 8 / 16 CTAs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

V, F, cuts = gen.height_field_case(1024, 8)
b = pg.partition_mesh(pg.TriMesh(V, F, check=False), cuts).batch
b.laplacian()
for n in (8, 16, 32, 64):
    row = []
    for cl in (0, 4, 8, 16):
        b.flatten(comps=list(range(n)), cluster=cl)
        r = b.flatten(comps=list(range(n)), cluster=cl) and b.last_solve(0)
        row.append(f"c{cl or 'auto'}={r['cluster']}:{r['kernel_ms']:.1f}ms")
    print(n, "subdomains:", "  ".join(row), flush=True)
