"""Stage-wise measurements at full BASELINE size for cfg 3 (Delaunay disk,
500K points, 128 k-means subdomains) and cfg 4 (icosphere-9 with a degree-8
spherical-harmonic radius, 2.6M vertices, 256 subdomains): partition,
flatten and Dirichlet-solve kernel times and the SURVEY 8(d) bandwidth. The
reference does not weld these layouts end to end."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1903_12359_b200 as pg
from paper_1903_12359_b200 import generators as gen
from paper_1903_12359_b200 import _native as nat

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
which = sys.argv[1:] or ["cfg3", "cfg4"]
for name in which:
    t0 = time.perf_counter()
    V, F, cuts = gen.cfg3() if name == "cfg3" else gen.cfg4()
    print(f"{name}: generated in {time.perf_counter() - t0:.1f} s, n {len(V)} m {len(F)} cuts {len(cuts)}", flush=True)
    mesh = pg.TriMesh(V, F)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        part = pg.partition_mesh(mesh, cuts)
        b = part.batch
        b.laplacian()
        torch.cuda.synchronize()
        tp = time.perf_counter() - t0
        t0 = time.perf_counter()
        z, st = b.flatten()
        tf = time.perf_counter() - t0
        fl = b.last_solve(0)
        voff = b.host(nat.ARR_VERT_OFF, torch.int64)
        loff = b.host(nat.ARR_LOOP_OFF, torch.int64)
        lp = b.host(nat.ARR_LOOP, torch.int32)
        gid = np.concatenate([voff[c] + lp[loff[c]:loff[c + 1]] for c in range(b.K)]).astype(np.int32)
        t0 = time.perf_counter()
        zh, sth = b.harmonic(gid, z[torch.as_tensor(gid, device=z.device).long()])
        th = time.perf_counter() - t0
        hm = b.last_solve(1)
        its = sorted(s["iters"] for s in st)
        print(f"  K {b.K}: partition+laplacian {1e3 * tp:.0f} ms | flatten {1e3 * tf:.0f} ms (kernel "
              f"{fl['kernel_ms']:.0f}, cluster {fl['cluster']}, iters med/max {its[len(its) // 2]}/{its[-1]}, "
              f"{fl['ref_bytes'] / fl['kernel_ms'] / 1e6:.0f} GB/s = {fl['ref_bytes'] / fl['kernel_ms'] / 1e6 / peak:.2f}"
              f" of peak) | harmonic {1e3 * th:.0f} ms (kernel {hm['kernel_ms']:.0f})", flush=True)
