"""Record the first CG coefficients (alpha, rr, beta) and the final iteration
count of every subdomain's DNCP flatten (PGCP_PCG_HIST) on cfg-2-shaped
height fields with several seeds: data for an iteration-count predictor
(launch order of the flatten clusters)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = os.environ.setdefault("PGCP_PCG_HIST", "gpurun_out/hist.bin")
if os.path.exists(out):
    os.remove(out)
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

for seed in range(int(os.environ.get("SEEDS", "4"))):
    V, F, cuts = gen.height_field_case(1024, 8, seed=seed)
    b = pg.partition_mesh(pg.TriMesh(V, F, check=False), cuts).batch
    b.laplacian()
    z, st = b.flatten()
    print("seed", seed, "kernel", round(b.last_solve(0)["kernel_ms"], 2), "ms", flush=True)
