"""Large subdomains (cfg-5 size, ~66K vertices each) on a 2049^2 grid, 8x8
blocks: convergence and timing of both preconditioners."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

grid = int(os.environ.get("GRID", "2049"))
blocks = int(os.environ.get("BLOCKS", "8"))
V, F, cuts = gen.height_field_case(grid, blocks, n_bumps=64, seed=0)
mesh = pg.TriMesh(V, F)
part = pg.partition_mesh(mesh, cuts)
b = part.batch
b.laplacian()
for mode in os.environ.get("MODES", "1,0").split(","):
    os.environ["PGCP_PCG_COARSE"] = mode
    t0 = time.perf_counter()
    try:
        z, st = b.flatten(maxit=int(os.environ.get("MAXIT", "20000")))
        ok = "ok"
    except Exception as e:
        ok = f"FAIL {e}"
        st = b.last_stats
    fl = b.last_solve(0)
    its = sorted(s["iters"] for s in st)
    print(f"coarse={mode}: {1e3 * (time.perf_counter() - t0):.0f} ms kernel {fl['kernel_ms']:.1f} ms cluster {fl['cluster']}"
          f" iters min/med/max {its[0]}/{its[len(its) // 2]}/{its[-1]} {ok}", flush=True)
    bad = [(i, s['iters'], s['relres']) for i, s in enumerate(st) if s["status"] != 0]
    if bad:
        print("  failing:", bad[:5], flush=True)
