"""Full-size parity check: cfg 2 (1024^2, 8x8 blocks, tree schedule) on the
device vs the CPU oracle (SuperLU solves, numpy welds). Prints the UV error
relative to the parameterization's diameter for both preconditioners and the
distortion statistics. Test infrastructure (imports oracle/)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

grid = int(os.environ.get("GRID", "1024"))
blocks = int(os.environ.get("BLOCKS", "8"))
V, F, cuts = gen.height_field_case(grid, blocks)
pairs = gen.quadtree_schedule_order(blocks, blocks)
t0 = time.perf_counter()
ref = oracle.run_parameterize(V, F, cuts, "free", workers=os.cpu_count() or 1, schedule="pairs", pairs=pairs)
print(f"oracle {time.perf_counter() - t0:.1f} s", flush=True)
zr = np.asarray(ref["coords"])
diam = 2 * np.max(np.abs(zr - zr.mean()))
mesh = pg.TriMesh(V, F)
for mode in ("0", "1"):
    os.environ["PGCP_PCG_COARSE"] = mode
    gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs)
    z = np.asarray(gp.coords)
    err = np.max(np.abs(z - zr)) / diam
    d, dr = rep.distortion["angular_abs"], ref["distortion"]["angular_abs"]
    print(f"coarse={mode}: uv err/diam {err:.3e}  flips {rep.flips}  mean {d['mean']:.9f} (oracle {dr['mean']:.9f})"
          f"  sd {d['sd']:.9f} (oracle {dr['sd']:.9f})", flush=True)
