"""One tuned cold MinkUNet forward after warmup (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.synth import lidar_scan
net = NetworkRunner(minkunet18(), dtype=torch.float16)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
scans = [lidar_scan(200_000, seed=s) for s in (1, 2, 3)]
f = [torch.randn(len(s), 4, device="cuda").half() for s in scans]
if os.environ.get("TUNE", "1") == "1":
    cs0 = sk.CoordSet.create(torch.from_numpy(scans[0]).cuda())
    net.tune(cs0, f[0], training=0, warmup=1, runs=3)
cs = sk.CoordSet.create(torch.from_numpy(scans[1]).cuda()); net.forward(cs, f[1])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
cs = sk.CoordSet.create(torch.from_numpy(scans[2]).cuda()); y, _ = net.forward(cs, f[2])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
