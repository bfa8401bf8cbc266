"""Short bench-shaped run for ncu captures (2 cold scans, fixed tuned-like configs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.synth import lidar_scan

net = NetworkRunner(minkunet18(), dtype=torch.float16)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
for seed in range(int(os.environ.get("SCANS", 2))):
    s = lidar_scan(200_000, seed=seed + 1)
    cs = sk.CoordSet.create(torch.from_numpy(s).cuda())
    f = torch.randn(len(s), 4, device="cuda").half()
    net.forward(cs, f)
torch.cuda.synchronize()
print("done")
