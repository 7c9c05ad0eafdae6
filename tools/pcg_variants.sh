#!/bin/bash
# PCG kernel variants on cfg 2 (one subdomain and all 64)
for v in 0 1 2 3 4; do
  echo "variant $v"
  PGCP_PCG_VARIANT=$v PGCP_PCG_TIMING=1 python - <<'PY' 2>&1 | grep -E "timing|ms="
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen
V, F, cuts = gen.height_field_case(1024, 8)
b = pg.partition_mesh(pg.TriMesh(V, F, check=False), cuts).batch
b.laplacian()
for comps in ([0], None):
    b.flatten(comps=comps, cluster=4); r = b.last_solve(0)
    print(f"comps={'all' if comps is None else 1} ms={r['kernel_ms']:.2f} us/iter={1e3*r['kernel_ms']/r['iters_max']:.2f}", flush=True)
PY
done
