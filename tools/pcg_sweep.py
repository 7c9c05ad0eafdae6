"""Per-iteration PCG latency: one subdomain alone vs all, by cluster size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

V, F, cuts = gen.height_field_case(int(os.environ.get("GRID", "1024")), int(os.environ.get("BLOCKS", "8")))
part = pg.partition_mesh(pg.TriMesh(V, F, check=False), cuts)
b = part.batch
b.laplacian()
for which in ("flatten", "harmonic"):
    for comps in ([0], [0, 1, 2, 3], None):
        for cl in (4, 8, 16):
            try:
                if which == "flatten":
                    b.flatten(comps=comps, cluster=cl)
                    r = b.last_solve(0)
                else:
                    import numpy as np
                    from paper_1903_12359_b200 import _native as nat
                    voff = b.host(nat.ARR_VERT_OFF, torch.int64)
                    loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
                    loop = b.host(nat.ARR_LOOP, torch.int32)
                    K = len(voff) - 1
                    gid = np.concatenate([voff[c] + loop[loff[c]:loff[c + 1]] for c in range(K)]).astype(np.int32)
                    vals = torch.ones(len(gid), dtype=torch.complex128)
                    b.harmonic(gid, vals, comps=comps, cluster=cl)
                    r = b.last_solve(1)
                n = "all" if comps is None else len(comps)
                print(f"{which:8s} comps={n:>3} cluster={r['cluster']:2d} ms={r['kernel_ms']:8.2f} "
                      f"iters_max={r['iters_max']:6.0f} us/iter(max)={1e3*r['kernel_ms']/r['iters_max']:7.2f}", flush=True)
            except Exception as e:
                print(which, comps, cl, "ERR", str(e)[:100])
