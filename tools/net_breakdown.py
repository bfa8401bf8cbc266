"""Per-group time breakdown of the MinkUNet bench workload: algorithmic FLOPs,
kernel ms (CUDA events per layer), TFLOP/s and the fraction of the measured
bf16 peak, map-build ms. TUNE=1 (default) tunes per group like bench.py.

  python tools/net_breakdown.py [--out profiles/r01_group_roofline.md]"""
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
if os.environ.get("TUNE", "1") == "1":
    tc = torch.from_numpy(lidar_scan(200_000, seed=900_000)).cuda()
    net.tune(sk.CoordSet.create(tc), torch.randn(len(tc), 4, device="cuda").half(), training=0,
             warmup=1, runs=3)
peak = bench.peaks().get("bf16_tflops", 1652.8)
cs = sk.CoordSet.create(c)
for _ in range(3):
    net.forward(cs, f)
_, st = net.forward(cs, f, stats=True)
pairs = bench.layer_pairs(sk, net, cs)
groups = net.groups()
tot = 0
lines = ["# MinkUNet-18 per map group: algorithmic FLOPs vs kernel time (one B200)", "",
         f"tools/net_breakdown.py; lidar scan {len(scan)} voxels, fp16 in / fp32 acc, tuned per "
         f"group; kernel ms from CUDA events per layer (warm maps); peak = {peak} TFLOP/s "
         "(MEASURED_PEAKS bf16). FLOPs = 2*pairs*C_in*C_out (padding not credited).", "",
         "| group | layers | K | s | first layer | (C_in, C_out) | pairs (first layer) | GFLOP | "
         "dataflow | kernel ms | TFLOP/s | frac | map ms |", "|" + "---|" * 13]
for g, ls in enumerate(groups):
    fl = sum(2.0 * pairs[i] * net.layers[i].c_in * net.layers[i].c_out for i in ls)
    k = st["kernel_ms"][g]
    tot += k
    L = net.layers[ls[0]]
    chans = sorted(set((net.layers[i].c_in, net.layers[i].c_out) for i in ls))
    lines.append(f"| {g} | {len(ls)} | {L.kernel} | {L.stride} | {L.name} | {chans} | {pairs[ls[0]]} | "
                 f"{fl / 1e9:.2f} | {net.config(g).name()} | {k:.3f} | {fl / k / 1e9:.1f} | "
                 f"{fl / k / 1e9 / peak:.3f} | {st['mapping_ms'][g]:.3f} |")
allfl = sum(2.0 * pairs[i] * l.c_in * l.c_out for i, l in enumerate(net.layers))
lines += ["", f"kernels {tot:.3f} ms, {allfl / tot / 1e9:.1f} TFLOP/s over the network "
          f"({allfl / tot / 1e9 / peak:.3f} of peak); map build {st['mapping_ms'].sum():.3f} ms"]
txt = "\n".join(lines) + "\n"
print(txt)
if "--out" in sys.argv:
    open(sys.argv[sys.argv.index("--out") + 1], "w").write(txt)
