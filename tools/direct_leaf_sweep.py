"""Leaf-size sweep of the direct solver on the cfg-2 flatten and Dirichlet
systems: factorization FMAs, factor / solve time (PGCP_DIRECT_LEAF).

    python tools/direct_leaf_sweep.py 16 24 32 48 64
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402

torch.cuda.set_device(0)
V, F, cuts = gen.height_field_case(int(os.environ.get("GRID", 1024)), int(os.environ.get("BLOCKS", 8)))
part = pg.partition_mesh(pg.TriMesh(V, F), cuts)
b = part.batch
b.laplacian()
z0 = None
for leaf in sys.argv[1:] or ["48"]:
    os.environ["PGCP_DIRECT_LEAF"] = leaf
    for rep in range(3):
        z, st = b.flatten(solver="direct")
        torch.cuda.synchronize()
    d = b.last_solve(0)
    zz = z.cpu().numpy()
    if z0 is None:
        z0 = zz
    print(f"leaf {leaf}: FMAs {d['fmas']:.3g} factor {d['factor_ms']:.2f} ms solve {d['solve_ms']:.2f} ms "
          f"max front {d['max_front']} nodes {d['nodes']} levels {d['levels']} front GB {d['front_bytes']/1e9:.2f} "
          f"max|dz| vs first {np.max(np.abs(zz - z0)):.2e}", flush=True)
