"""A/B of TilePreset variants on single lidar-scan layers (C_in -> C_out)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import lidar_scan


def timeit(fn, warm=3, reps=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


c = sk.CoordSet.create(torch.from_numpy(lidar_scan(200_000, seed=1)).cuda())
m = sk.build_kmap(c, c, 3, 1)
tiles = {"large": sk.tile_large(), "m256": sk.TilePreset(256, 0, 0, 128, 4),
         "k32": sk.TilePreset(128, 0, 32, 128, 4), "tma": sk.TilePreset(128, 0, 0, 128, 1),
         "m64": sk.TilePreset(64, 0, 0, 128, 4), "m64k32": sk.TilePreset(64, 0, 32, 128, 4)}
for ci, co in [(96, 96), (32, 96), (64, 64), (128, 128)]:
    x = torch.randn(m.n_in, ci, device="cuda").half()
    w = (torch.randn(27, ci, co, device="cuda") / 40).half()
    y = torch.empty(m.n_out, co, device="cuda").half()
    res = {}
    for name, t in tiles.items():
        cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, t)
        res[name] = round(timeit(lambda: sk.conv_forward(m, x, w, cfg, out=y)) * 1e3, 1)
    print(f"{ci}->{co}: {res}", flush=True)
