"""cfg 5 (4096^2 height field, 64 bumps, 16x16 blocks) through the device
pipeline: stage times, solver stats, quality."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen

t0 = time.perf_counter()
V, F, cuts = gen.height_field_case(4096, 16, n_bumps=64, seed=0)
print(f"generate {time.perf_counter() - t0:.1f} s: n {len(V)} m {len(F)} cuts {len(cuts)}", flush=True)
mesh = pg.TriMesh(V, F)
pairs = gen.quadtree_schedule_order(16, 16)
for _ in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
    dt = time.perf_counter() - t0
    fl, hm = rep.solver["flatten"], rep.solver["harmonic"]
    print(f"total {1e3 * dt:.0f} ms ({len(V) / dt / 1e6:.2f} M vert/s)", {k: round(1e3 * v, 1) for k, v in rep.timings.items()},
          f"| flatten kernel {fl['kernel_ms']:.1f} ms iters max {fl['iters_max']:.0f} cluster {fl['cluster']}"
          f" GB/s {fl['bytes'] / fl['kernel_ms'] / 1e6:.0f}",
          f"| harmonic kernel {hm['kernel_ms']:.1f} ms | flips {rep.flips} mean {rep.distortion['angular_abs']['mean']:.6f}",
          flush=True)
