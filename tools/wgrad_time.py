"""k_wgrad_tc device time on the lidar scan's K=3 map for several widths."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import lidar_scan
c = sk.CoordSet.create(torch.from_numpy(lidar_scan(200_000, seed=1)).cuda())
m = sk.build_kmap(c, c, 3, 1)
cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
for C in (32, 64, 96, 128, 256):
    x = torch.randn(m.n_in, C, device="cuda").half()
    dy = torch.randn(m.n_out, C, device="cuda").half()
    ts = []
    for i in range(13):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record(); sk.conv_wgrad(m, x, dy, cfg); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    t = np.median(ts[3:])
    print(f"wgrad C={C}: {t*1e3:.1f} us, {2*m.total_pairs()*C*C/t/1e9:.1f} TFLOP/s", flush=True)
