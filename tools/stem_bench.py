import os, sys
sys.path.insert(0, "/root/repo")
import torch, numpy as np
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import lidar_scan
c = sk.CoordSet.create(torch.from_numpy(lidar_scan()).cuda())
m = sk.build_kmap(c, c, 3, 1)
x = torch.randn(m.n_in, 4, device="cuda").half()
w = (torch.randn(27, 4, 32, device="cuda") / 10).half()
cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
for _ in range(3): y = sk.conv_forward(m, x, w, cfg)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): y = sk.conv_forward(m, x, w, cfg)
e.record(); torch.cuda.synchronize(); print("ms per call", s.elapsed_time(e) / 20)
