"""Stem layer (4 -> 32, K=3 submanifold) on the lidar scan: device time per
call of the small-C_in path (k_conv_small_cin), GPU sleep ahead of the events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import lidar_scan
c = sk.CoordSet.create(torch.from_numpy(lidar_scan(200_000, seed=1)).cuda())
m = sk.build_kmap(c, c, 3, 1)
x = torch.randn(m.n_in, 4, device="cuda").half()
w = (torch.randn(27, 4, 32, device="cuda") / 10).half()
y = torch.empty(m.n_out, 32, device="cuda").half()
cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
ts = []
for i in range(23):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000)
    a.record(); sk.conv_forward(m, x, w, cfg, out=y); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
print(f"stem 4->32 on {m.n_out} voxels: {np.median(ts[3:])*1e3:.1f} us (incl. the per-call weight transpose)")
