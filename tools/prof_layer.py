"""Run one layer's forward a few times (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import uniform_voxels, lidar_scan

C = int(os.environ.get("C", 64))
S = int(os.environ.get("SPLITS", 1))
KIND = int(os.environ.get("KIND", 2))
coords = torch.from_numpy(lidar_scan() if os.environ.get("SCAN") == "lidar" else uniform_voxels(127_000, 64, 1)).cuda()
c = sk.CoordSet.create(coords)
m = sk.build_kmap(c, c, 3, 1)
x = torch.randn(m.n_in, C, device="cuda").half()
w = (torch.randn(27, C, C, device="cuda") / 40).half()
cfg = sk.DataflowConfig(KIND, S, sk.tile_large())
for _ in range(int(os.environ.get("REPS", 3))):
    y = sk.conv_forward(m, x, w, cfg)
torch.cuda.synchronize()
print("done", m.n_in, m.total_pairs())
