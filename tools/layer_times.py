"""Per-layer kernel time of a tuned MinkUNet forward (warm maps, CUDA events
per layer, no per-layer sync) with algorithmic TFLOP/s."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.synth import lidar_scan
net = NetworkRunner(minkunet18(), dtype=torch.float16, weight_seed=3)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
tc = torch.from_numpy(lidar_scan(200_000, seed=900_000)).cuda()
net.tune(sk.CoordSet.create(tc), torch.randn(len(tc), 4, device="cuda").half(), training=0, warmup=1, runs=3)
c = torch.from_numpy(lidar_scan(200_000, seed=1)).cuda()
cs = sk.CoordSet.create(c)
f = torch.randn(cs.n, 4, device="cuda").half()
for _ in range(3):
    net.forward(cs, f)
lm = np.zeros(net.num_layers)
for _ in range(5):
    l, _ = net.forward_profiled(cs, f)
    lm += l / 5
pairs = bench.layer_pairs(sk, net, cs)
rows = []
for i, L in enumerate(net.layers):
    fl = 2.0 * pairs[i] * L.c_in * L.c_out
    rows.append((lm[i], i, L.name, net.group_of_layer(i), L.c_in, L.c_out, L.kernel, pairs[i], fl / lm[i] / 1e9 if lm[i] else 0))
print(f"total {lm.sum():.3f} ms")
for r in sorted(rows, reverse=True)[:30]:
    print(f"{r[0]*1e3:7.1f} us  L{r[1]:2d} {r[2]:10s} g{r[3]:2d} {r[4]:3d}->{r[5]:3d} K{r[6]} pairs {r[7]:8d}  {r[8]:6.1f} TF/s  {net.config(r[3]).name()}")
