"""Per-group / per-layer time breakdown of the MinkUNet bench workload."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.synth import lidar_scan
import bench

splits = int(os.environ.get("SPLITS", 1))
scan = lidar_scan(200_000, seed=1)
c = torch.from_numpy(scan).cuda()
f = torch.randn(len(scan), 4, device="cuda").half()
net = NetworkRunner(minkunet18(), dtype=torch.float16)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, splits, sk.tile_large()))
cs = sk.CoordSet.create(c)
for _ in range(3):
    net.forward(cs, f)
_, st = net.forward(cs, f, stats=True)
pairs = bench.layer_pairs(sk, net, cs)
groups = net.groups()
tot = 0
for g, ls in enumerate(groups):
    fl = sum(2.0 * pairs[i] * net.layers[i].c_in * net.layers[i].c_out for i in ls)
    k = st["kernel_ms"][g]
    tot += k
    L = net.layers[ls[0]]
    print(f"g{g:2d} n_layers={len(ls):2d} K={L.kernel} s={L.stride} {L.name:8s} ch={sorted(set((net.layers[i].c_in, net.layers[i].c_out) for i in ls))} "
          f"pairs={pairs[ls[0]]:8d} GFLOP={fl/1e9:7.2f} kernel_ms={k:6.3f} TF/s={fl/k/1e9:6.1f} map_ms={st['mapping_ms'][g]:.3f}")
print("kernel total ms", tot, "map total", st["mapping_ms"].sum())
