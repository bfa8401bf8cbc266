"""Per-group kernel-map cost of a cold MinkUNet forward (tuned configs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.synth import lidar_scan
net = NetworkRunner(minkunet18(), dtype=torch.float16)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
scans = [lidar_scan(200_000, seed=s) for s in (1, 2, 3, 4)]
f = [torch.randn(len(s), 4, device="cuda").half() for s in scans]
cs0 = sk.CoordSet.create(torch.from_numpy(scans[0]).cuda())
net.tune(cs0, f[0], training=0, warmup=1, runs=3)
for i in (1, 2, 3):
    cs = sk.CoordSet.create(torch.from_numpy(scans[i]).cuda())
    _, st = net.forward(cs, f[i], stats=True)
mp, kr = np.asarray(st["mapping_ms"]), np.asarray(st["kernel_ms"])
print("total mapping %.3f ms, kernels %.3f ms" % (mp.sum(), kr.sum()))
for g in range(net.num_groups):
    names = [net.layers[i].name for i in net.groups()[g]]
    print(f"g{g:2d} map {mp[g]:.3f} conv {kr[g]:.3f}  {net.config(g).name():32s} {names[:4]}")
