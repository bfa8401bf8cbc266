"""Where does a cold scan's time go? (host-timed with syncs; diagnostic only)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.synth import lidar_scan

net = NetworkRunner(minkunet18(), dtype=torch.float16)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
scans = [lidar_scan(200_000, seed=s) for s in range(1, 8)]
dc = [torch.from_numpy(s).cuda() for s in scans]
df = [torch.randn(len(s), 4, device="cuda").half() for s in scans]
def T():
    torch.cuda.synchronize(); return time.perf_counter()
for i in range(len(scans)):
    t0 = T()
    cs = sk.CoordSet.create(dc[i]); t1 = T()
    y, st = net.forward(cs, df[i], stats=True); t2 = T()
    y, _ = net.forward(cs, df[i]); t3 = T()
    # isolated pieces on a fresh set
    cs2 = sk.CoordSet.create(dc[i]); t4 = T()
    o = sk.build_out_coords(cs2, 2); t5 = T()
    m = sk.build_kmap(cs2, cs2, 3, 1); t6 = T()
    m.prepare(1, 128); t7 = T()
    m.prepare(2, 128); t8 = T()
    mt = sk.build_kmap(cs2, o, 3, 2).transpose(); t9 = T()
    print(f"scan{i}: create {1e3*(t1-t0):.2f} cold_fwd(stats) {1e3*(t2-t1):.2f} "
          f"[map {st['mapping_ms'].sum():.2f} kern {st['kernel_ms'].sum():.2f}] warm_fwd {1e3*(t3-t2):.2f} | "
          f"create {1e3*(t4-t3):.2f} down {1e3*(t5-t4):.2f} subm_query {1e3*(t6-t5):.2f} "
          f"prep_s1 {1e3*(t7-t6):.2f} prep_s2 {1e3*(t8-t7):.2f} strided+T {1e3*(t9-t8):.2f}")
