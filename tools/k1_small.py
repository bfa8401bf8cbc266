"""K=1 identity-map layers at the deep MinkUNet levels (few rows): sk200
k_dense_tc device time per call vs cuBLAS (torch.matmul) and the minimum
(launch + fixed latency) of an empty torch kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import random_instance_coords


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for n_pts, ci, co in [(600, 256, 256), (3000, 128, 256), (3000, 256, 256), (14000, 64, 128),
                      (14000, 128, 128), (55000, 32, 96)]:
    c = random_instance_coords(1, n_pts, -40, 40)
    cs = sk.CoordSet.create(c)
    m = sk.build_kmap(cs, cs, 1, 1)
    n = cs.n
    x = torch.randn(n, ci, device="cuda").half()
    w = (torch.randn(1, ci, co, device="cuda") / 10).half()
    y = torch.empty(n, co, device="cuda").half()
    cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
    t_sk = timeit(lambda: sk.conv_forward(m, x, w, cfg, out=y))
    w2 = w[0]
    t_th = timeit(lambda: torch.matmul(x, w2, out=y))
    print(f"n={n} {ci}->{co}: sk {t_sk*1e3:6.1f} us  cuBLAS {t_th*1e3:6.1f} us", flush=True)
z = torch.empty(1, device="cuda")
print(f"empty kernel: {timeit(lambda: z.add_(1))*1e3:.1f} us")
