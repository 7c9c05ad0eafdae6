"""Stage-wise cfg 5 (4096^2, 64 bumps, 16x16 blocks): the flatten of all 256
subdomains (the HBM-bound regime: ~1.2 GB of matrices, larger than L2).
Prints kernel time, iterations and the SURVEY 8(d) algorithmic bandwidth."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

V, F, cuts = gen.height_field_case(4096, 16, n_bumps=64, seed=0)
mesh = pg.TriMesh(V, F)
t0 = time.perf_counter()
part = pg.partition_mesh(mesh, cuts)
b = part.batch
b.laplacian()
print(f"partition + laplacian {1e3 * (time.perf_counter() - t0):.0f} ms, K {b.K}", flush=True)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
for _ in range(2):
    t0 = time.perf_counter()
    z, st = b.flatten()
    dt = time.perf_counter() - t0
    fl = b.last_solve(0)
    its = sorted(s["iters"] for s in st)
    gbs = fl["ref_bytes"] / (fl["kernel_ms"] / 1e3) / 1e9
    print(f"flatten {1e3 * dt:.0f} ms, kernel {fl['kernel_ms']:.0f} ms, cluster {fl['cluster']}, iters "
          f"min/med/max {its[0]}/{its[len(its) // 2]}/{its[-1]}, algorithmic {gbs:.0f} GB/s = {gbs / peak:.2f} of HBM "
          f"peak, device-model {fl['bytes'] / (fl['kernel_ms'] / 1e3) / 1e9:.0f} GB/s", flush=True)
