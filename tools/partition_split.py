"""Host-side split of the cfg-2 partition stage (pipeline.py's first block):
validate_cuts, the device partition, info / offsets reads, boundary cycles.

    python tools/partition_split.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import _native as nat  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402
from paper_1903_12359_b200.partition import Partition, validate_cuts  # noqa: E402

V, F, cuts = gen.height_field_case(1024, 8)
mesh = pg.TriMesh(V, F)
mesh.device_arrays()
acc = {}


def lap(name, t0):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    acc[name] = acc.get(name, 0.0) + 1e3 * (t1 - t0)
    return t1


N = 10
for i in range(N + 3):
    if i == 3:
        acc.clear()
    torch.cuda.synchronize()
    t = time.perf_counter()
    norm = validate_cuts(mesh, cuts)
    t = lap("validate_cuts", t)
    batch = mesh.partition_batch(norm)
    t = lap("partition_batch", t)
    info = batch.info()
    t = lap("info", t)
    part = Partition(mesh, batch, norm)
    voff = batch.host(nat.ARR_VERT_OFF, torch.int64)
    t = lap("Partition + vert_off", t)
    cycles = part.boundary_cycles
    t = lap("boundary_cycles", t)
    loop_local = batch.host(nat.ARR_LOOP, torch.int32).astype(np.int64)
    t = lap("loop read", t)
    batch.laplacian()
    t = lap("laplacian", t)
print({k: round(v / N, 3) for k, v in acc.items()}, "sum", round(sum(acc.values()) / N, 3))
