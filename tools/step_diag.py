"""Per-step diagnostics of the bench's two legs (device-resident `value` loop
and the host-buffer `e2e` loop): wall time, stage timings, workspace-cache
growth (pgcp_workspace_stats), Python GC pauses and torch's reserved memory.
Used to find the multi-10-ms outlier steps. MODE=value|e2e|both, REPS=N."""
import gc
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import _native as nat  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402

torch.cuda.set_device(0)
V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
reps = int(os.environ.get("REPS", "20"))
mode = os.environ.get("MODE", "both")

gc_ms = [0.0]
_gc_t = [0.0]


def _gc_cb(phase, info):
    if phase == "start":
        _gc_t[0] = time.perf_counter()
    else:
        gc_ms[0] += 1e3 * (time.perf_counter() - _gc_t[0])


gc.callbacks.append(_gc_cb)


def ws():
    out = (ctypes_d * 4)()
    nat.check(nat.lib().pgcp_workspace_stats(out, 4))
    return list(out)


import ctypes  # noqa: E402
ctypes_d = ctypes.c_double


def run(label, fn):
    walls = []
    for i in range(reps):
        w0, g0 = ws(), gc_ms[0]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = fn()
        torch.cuda.synchronize()
        wall = 1e3 * (time.perf_counter() - t0)
        w1 = ws()
        walls.append(wall)
        print(f"{label} {i:2d} wall {wall:7.2f} ms | ws slots {int(w1[0])} {w1[1] / 1e9:.2f} GB "
              f"grows +{int(w1[2] - w0[2])} ({w1[3] - w0[3]:.1f} ms) | gc {gc_ms[0] - g0:.1f} ms | "
              f"torch reserved {torch.cuda.memory_reserved() / 1e9:.2f} GB |",
              {k: round(1e3 * v, 2) for k, v in rep.timings.items()}, file=sys.stderr, flush=True)
    w = np.array(walls[3:])
    print(f"{label}: median {np.median(w):.2f} mean {w.mean():.2f} max {w.max():.2f} ms", file=sys.stderr, flush=True)


if mode in ("value", "both"):
    mesh_dev = pg.TriMesh(V, F)
    mesh_dev.device_arrays()
    state = {}

    def step_value():
        state["gp"], rep = pg.parameterize(mesh_dev, cuts, "free", pairs=pairs, keep_device=True)
        return rep
    run("value", step_value)
    state.clear()
    del mesh_dev

if mode in ("e2e", "both"):
    Vn = torch.from_numpy(np.ascontiguousarray(V)).pin_memory().numpy()
    Fn = torch.from_numpy(np.ascontiguousarray(F.astype(np.int32))).pin_memory().numpy()
    Cn = torch.from_numpy(np.ascontiguousarray(cuts)).pin_memory().numpy()
    st = {}

    def step_e2e():
        mesh = pg.TriMesh(Vn, Fn)
        st["gp"], rep = pg.parameterize(mesh, Cn, "free", pairs=pairs)
        _ = st["gp"].coords
        return rep
    run("e2e", step_e2e)
