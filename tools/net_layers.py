"""Per-layer GPU time of MinkUNet (cold = first forward on a new scan, warm = cached)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.synth import lidar_scan
import bench
net = NetworkRunner(minkunet18(), dtype=torch.float16)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, int(os.environ.get("SPLITS", 1)), sk.tile_large()))
scans = [lidar_scan(200_000, seed=s) for s in (1, 2, 3)]
f = [torch.randn(len(s), 4, device="cuda").half() for s in scans]
cs0 = sk.CoordSet.create(torch.from_numpy(scans[0]).cuda()); net.forward(cs0, f[0])
if os.environ.get("TUNE"):
    net.tune(cs0, f[0], training=0, warmup=1, runs=3)
    print("tuned:", [net.config(g).name() for g in range(net.num_groups)])
cs = sk.CoordSet.create(torch.from_numpy(scans[1]).cuda())
cold, mp = net.forward_profiled(cs, f[1])
warm, _ = net.forward_profiled(cs, f[1])
pairs = bench.layer_pairs(sk, net, cs)
print(f"cold total {cold.sum():.3f} ms (maps {mp:.3f}), warm total {warm.sum():.3f} ms")
rows = []
for i, l in enumerate(net.layers):
    fl = 2.0 * pairs[i] * l.c_in * l.c_out
    rows.append((warm[i], i, l, fl))
for w, i, l, fl in sorted(rows, key=lambda r: -r[0])[:30]:
    print(f"{l.name:9s} g{net.group_of_layer(i):2d} K{l.kernel} s{l.stride} {l.kind[:6]} {l.c_in:3d}->{l.c_out:3d} "
          f"pairs={pairs[i]:8d} cold={cold[i]:.3f} warm={w:.3f} ms  {fl/w/1e9 if w else 0:6.1f} TF/s")
