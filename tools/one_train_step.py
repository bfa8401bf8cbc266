"""One MinkUNet training step (batch 2 scans, fwd + dgrad + wgrad + SGD) after
warmup, profiler-start gated (for ncu launch lists of the backward)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.dist import DataParallelTrainer
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner
net = NetworkRunner(minkunet18(), dtype=torch.float16, weight_seed=3)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
scans = bench.make_scans(6, 77)
rng = np.random.default_rng(0)
data = [(torch.from_numpy(c).cuda(), torch.from_numpy(rng.standard_normal((len(c), 4)).astype(np.float16)).cuda(),
         torch.from_numpy(rng.standard_normal((len(c), 96)).astype(np.float16)).cuda()) for c in scans]
if os.environ.get("TUNE", "1") == "1":
    cs0 = sk.CoordSet.create(data[0][0])
    net.tune(cs0, data[0][1], training=1, warmup=1, runs=3)
tr = DataParallelTrainer(net, lr=1e-3, momentum=0.9)
def step(k):
    scenes = [(sk.CoordSet.create(c), x, t) for c, x, t in data[2 * k:2 * k + 2]]
    return tr.train_step(scenes, 2)
step(0); step(1); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step(2); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
