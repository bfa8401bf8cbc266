import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.network import NetworkRunner
scans = bench.make_scans(5, 1)
dc = [torch.from_numpy(c).cuda() for c in scans]
df = [torch.randn(len(c), 4, device="cuda").half() for c in scans]
net = NetworkRunner(bench.model_for("infer"), dtype=torch.float16, weight_seed=3)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for i in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cs = sk.CoordSet.create(dc[i])
        t1 = time.perf_counter()
        print(f"py create {1e6*(t1-t0):.1f} us", file=sys.stderr)
        net.forward(cs, df[i])
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"py forward returned {1e6*(t2-t1):.1f} us, done {1e6*(t3-t1):.1f}", file=sys.stderr)
