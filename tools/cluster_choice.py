"""Flatten kernel time of the first n cfg-2 subdomains (the per-GPU share at
64/n GPUs) for the automatic cluster shape and forced cluster sizes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

V, F, cuts = gen.height_field_case(1024, 8)
b = pg.partition_mesh(pg.TriMesh(V, F, check=False), cuts).batch
b.laplacian()
sizes = [int(x) for x in os.environ.get("SIZES", "0,4,6,8,10,12,16").split(",")]
for n in [int(x) for x in os.environ.get("COUNTS", "8,16,32,64").split(",")]:
    row = []
    for cl in sizes:
        try:
            b.flatten(comps=list(range(n)), cluster=cl)
            b.flatten(comps=list(range(n)), cluster=cl)
            r = b.last_solve(0)
            row.append(f"c{cl or 'auto'}={r['cluster']}:{r['kernel_ms']:.1f}ms/{int(r['iters_sum'])}it")
        except Exception as e:
            row.append(f"c{cl}: {type(e).__name__}")
    print(n, "subdomains:", "  ".join(row), flush=True)
