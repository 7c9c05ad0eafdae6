"""Stage timings of the sharded pipeline (NCCL, world size 1 on one GPU) next
to the single-GPU pipeline on cfg 2: what the sharding's own steps cost
(boundary exchange, foreign-loop fill, shard maps, reduced metrics).

    python tools/dist_stage_split.py
"""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402
from paper_1903_12359_b200.dist import Shard  # noqa: E402

with socket.socket() as sk:
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
V, F, cuts = gen.height_field_case(1024, 8)
pairs = gen.quadtree_schedule_order(8, 8)
mesh = pg.TriMesh(V, F)
mesh.device_arrays()
import time  # noqa: E402

from paper_1903_12359_b200 import pipeline as pl  # noqa: E402
from paper_1903_12359_b200.device import DeviceBatch  # noqa: E402

split = {}


def timed(label, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        split[label] = split.get(label, 0.0) + 1e3 * (time.perf_counter() - t0)
        return r
    return w


pl._repair = timed("_repair", pl._repair)
pl._fill_foreign_loops = timed("_fill_foreign_loops", pl._fill_foreign_loops)
pl._exchange_boundary = timed("_exchange_boundary", pl._exchange_boundary)
pl._shard_maps = timed("_shard_maps", pl._shard_maps)
DeviceBatch.harmonic_solve = timed("harmonic_solve", DeviceBatch.harmonic_solve)
DeviceBatch.qc_repair = timed("qc_repair", DeviceBatch.qc_repair)

for name, kw in (("single", {}), ("sharded", {"shard": Shard()})):
    split.clear()
    acc = {}
    for i in range(8):
        gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs, keep_device=True, **kw)
        if i >= 3:
            for k, v in rep.timings.items():
                acc[k] = acc.get(k, 0.0) + 1e3 * v / 5
    print(name, {k: round(v, 2) for k, v in acc.items()}, "sum (non-overlapped)",
          round(sum(v for k, v in acc.items() if "overlapped" not in k), 2), flush=True)
    print("   per call (8 runs):", {k: round(v / 8, 2) for k, v in split.items()}, flush=True)
dist.destroy_process_group()
