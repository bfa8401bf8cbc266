"""K=1 stride-1 (identity map) layers: sk200 k_dense_tc vs a torch (cuBLAS)
GEMM of the same shape, device time per call (GPU sleep ahead of the start
event hides host launch overhead)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import lidar_scan


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100_000)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


c = torch.from_numpy(lidar_scan(200_000, seed=1)).cuda()
cs = sk.CoordSet.create(c)
m = sk.build_kmap(cs, cs, 1, 1)
n = cs.n
for ci, co in [(32, 96), (96, 96), (32, 32), (64, 128), (128, 128), (128, 256), (256, 256)]:
    x = torch.randn(n, ci, device="cuda").half()
    w = (torch.randn(1, ci, co, device="cuda") / 10).half()
    y = torch.empty(n, co, device="cuda").half()
    cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
    t_sk = timeit(lambda: sk.conv_forward(m, x, w, cfg, out=y))
    w2 = w[0]
    t_th = timeit(lambda: torch.matmul(x, w2, out=y))
    byts = n * (ci + co) * 2
    print(f"n={n} {ci}->{co}: sk {t_sk*1e3:7.1f} us ({byts/t_sk/1e6:6.0f} GB/s)  "
          f"cuBLAS {t_th*1e3:7.1f} us ({byts/t_th/1e6:6.0f} GB/s)")
