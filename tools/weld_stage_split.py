"""Where the cfg-2 weld stage's time goes: host-side timers around each part
of the stage as parameterize runs it (gather, schedule run, result handling),
next to the library's per-level device times (PGCP_WELD_TIMING=1).

    python tools/weld_stage_split.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PGCP_WELD_TIMING", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402
from paper_1903_12359_b200 import pipeline as pl  # noqa: E402
from paper_1903_12359_b200 import welding as wd  # noqa: E402

V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
mesh = pg.TriMesh(V, F)
orig = wd.run_schedule


def timed(tv, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig(tv, *a, **k)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"run_schedule: call {1e3 * (t1 - t0):.3f} ms, +sync {1e3 * (t2 - t1):.3f} ms", flush=True)
    return r


pl.run_schedule = timed
_run = wd.PreparedSchedule.run


def timed_run(self, tv, hard_tol):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = _run(self, tv, hard_tol)
    print(f"PreparedSchedule.run: {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
    return r


wd.PreparedSchedule.run = timed_run
for _ in range(3):
    gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True)
    print("weld stage ms", rep.timings["weld"] * 1e3, flush=True)
