import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import lidar_scan
C = int(os.environ.get("C", 96))
c = sk.CoordSet.create(torch.from_numpy(lidar_scan()).cuda())
m = sk.build_kmap(c, c, 3, 1)
x = torch.randn(m.n_in, C, device="cuda").half()
dy = torch.randn(m.n_out, C, device="cuda").half()
cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
for _ in range(3):
    sk.conv_wgrad(m, x, dy, cfg)
torch.cuda.synchronize(); print("done", m.total_pairs())
