"""L2 read-bandwidth probe sweep (buffer size, loads in flight): the
denominator bench.py's roofline uses for the L2-bound PCG kernel."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench as B
from paper_1903_12359_b200 import _native as nat

dev = torch.device("cuda", 0)
for u in ("4", "8"):  # default kernel: 4
    os.environ["PGCP_L2_PROBE_U"] = u
    for mib in (16, 32, 48, 64, 80, 96):
        print(f"U={u} {mib:3d} MiB: {B.l2_probe_gbs(dev, mib=mib):8.0f} GB/s", flush=True)
