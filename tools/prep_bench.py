"""split_and_sort + pad (sk_kmap_prepare) device time on the lidar scan's
K=3 submanifold map, per split count (fresh map each time; CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import lidar_scan

c = torch.from_numpy(lidar_scan(200_000, seed=1)).cuda()
for splits in (1, 2, 3, 4):
    ts = []
    for rep in range(8):
        cs = sk.CoordSet.create(c)
        m = sk.build_kmap(cs, cs, 3, 1)
        m.os()  # materialise the map
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)  # host launch overhead hides behind it
        a.record()
        m.prepare(splits, 128)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"n={cs.n} splits={splits}: prepare {np.median(ts[2:])*1e3:7.1f} us (median of 6)")
