"""cfg-5 subdomains that are hard for the coarse space: iterations per
preconditioner variant (PGCP_PCG_COARSE, PGCP_COARSE_FP64)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen
V, F, cuts = gen.height_field_case(4096, 16, n_bumps=64, seed=0)
mesh = pg.TriMesh(V, F)
part = pg.partition_mesh(mesh, cuts)
b = part.batch
b.laplacian()
comps = [int(x) for x in os.environ.get("COMPS", "14,15,16").split(",")]
for coarse, fp64 in (("1", "0"), ("1", "1"), ("0", "0")):
    os.environ["PGCP_PCG_COARSE"] = coarse
    os.environ["PGCP_COARSE_FP64"] = fp64
    try:
        z, st = b.flatten(comps=comps, maxit=int(os.environ.get("MAXIT", "30000")))
        ok = "ok"
    except Exception as e:
        ok = f"FAIL {str(e)[:70]}"
        st = b.last_stats
    fl = b.last_solve(0)
    print(f"coarse {coarse} fp64 {fp64}: kernel {fl['kernel_ms']:.0f} ms",
          [(s["iters"], f"{s['relres']:.1e}") for s in st], ok, flush=True)
