"""Kernel-map build timing, block-index vs hash query, at the 1M C5 point
and the MinkUNet lidar scan (CUDA events; create = copy + hash insert)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import sweep_cloud, lidar_scan

ctx = sk.Context.get()
for name, c in (("1M", sweep_cloud(160_000, seed=1, tiles=10)), ("lidar", lidar_scan(200_000, seed=1))):
    coords = torch.from_numpy(c).cuda()
    for thr in (1, 1 << 30):
        ctx.set_kmap_block_rows(thr)
        ins, qry = [], []
        for _ in range(6):
            a, b, e = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record()
            cs = sk.CoordSet.create(coords)
            b.record()
            m = sk.build_kmap(cs, cs, 3, 1)
            e.record()
            torch.cuda.synchronize()
            ins.append(a.elapsed_time(b)); qry.append(b.elapsed_time(e))
            del m, cs
        ti, tq = statistics.median(ins[1:]), statistics.median(qry[1:])
        n = coords.shape[0]
        print(f"{name} n={n} {'block   ' if thr == 1 else 'hash    '}: create {ti*1e3:6.1f} us  "
              f"query {tq*1e3:6.1f} us  -> {208*n/((ti+tq)*1e-3)/1e9:6.0f} GB/s (208 B/voxel)")
ctx.set_kmap_block_rows(1 << 18)
