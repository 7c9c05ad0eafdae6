"""Leak check: live DeviceBatch objects across parameterize calls and who
holds them (GPU)."""
import gc
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1903_12359_b200 as pg  # noqa: E402
from paper_1903_12359_b200 import generators as gen  # noqa: E402
from paper_1903_12359_b200.device import DeviceBatch  # noqa: E402

torch.cuda.set_device(0)
V, F, cuts = gen.height_field_case(257, 4)
pairs = gen.quadtree_schedule_order(4, 4)


def live():
    return [o for o in gc.get_objects() if type(o) is DeviceBatch]


for i in range(5):
    mesh = pg.TriMesh(V, F)
    gp, rep = pg.parameterize(mesh, cuts, "free", pairs=pairs)
    print("step", i, "live DeviceBatch", len(live()), flush=True)
gc.collect()
objs = live()
print("after gc.collect: live", len(objs))
for b in objs:
    refs = [type(r).__name__ for r in gc.get_referrers(b) if r is not objs]
    print("  batch", hex(id(b)), "held by", refs)
    for r in gc.get_referrers(b):
        if r is objs or type(r).__name__ in ("frame",):
            continue
        if type(r).__name__ not in ("TriMesh",):
            for r2 in gc.get_referrers(r)[:3]:
                if r2 is not objs:
                    print("     ", type(r).__name__, "<-", type(r2).__name__, str(r2)[:90])
del objs
