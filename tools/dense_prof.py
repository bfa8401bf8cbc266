"""One identity-map (K=1) layer shape through sk200's dense path, for ncu:
python tools/dense_prof.py C_IN C_OUT [reps] [rows]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import lidar_scan

ci, co = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
c = torch.from_numpy(lidar_scan(200_000, seed=1)).cuda()
cs = sk.CoordSet.create(c)
m = sk.build_kmap(cs, cs, 1, 1)
x = torch.randn(cs.n, ci, device="cuda").half()
w = (torch.randn(1, ci, co, device="cuda") / 10).half()
y = torch.empty(cs.n, co, device="cuda").half()
cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
for _ in range(reps):
    sk.conv_forward(m, x, w, cfg, out=y)
torch.cuda.synchronize()
