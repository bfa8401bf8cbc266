"""One tuned cold SECOND-encoder forward after warmup (for ncu launch lists:
ncu --profile-from-start off ... python tools/one_forward_second.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.models import second_encoder
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.synth import waymo_scan
net = NetworkRunner(second_encoder(), dtype=torch.float16)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
scans = [waymo_scan(seed=s) for s in (1, 2, 3)]
f = [torch.randn(len(s), 4, device="cuda").half() for s in scans]
cs0 = sk.CoordSet.create(torch.from_numpy(scans[0]).cuda())
net.tune(cs0, f[0], training=0, warmup=1, runs=3)
cs = sk.CoordSet.create(torch.from_numpy(scans[1]).cuda()); net.forward(cs, f[1])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
cs = sk.CoordSet.create(torch.from_numpy(scans[2]).cuda()); y, _ = net.forward(cs, f[2])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", cs.n)
