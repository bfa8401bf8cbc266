"""Repeatability of the e2e ScanPipeline window (bench.py's e2e leg) in one
process: W workers, pinned host scans, L2 flush inside the window."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.pipeline import ScanPipeline, replicate
W = int(os.environ.get("W", 6))
scans = bench.make_scans(23, 1)
rng = np.random.default_rng(0)
feats = [rng.standard_normal((len(c), 4)).astype(np.float16) for c in scans]
net = NetworkRunner(bench.model_for("infer"), dtype=torch.float16, weight_seed=3)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
tc = torch.from_numpy(bench.make_scans(1, 900_000)[0]).cuda()
net.tune(sk.CoordSet.create(tc), torch.randn(len(tc), 4, device="cuda").half(), training=0, warmup=1, runs=3)
hs = [(torch.from_numpy(c).pin_memory(), torch.from_numpy(f).pin_memory()) for c, f in zip(scans, feats)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
pipe = ScanPipeline(replicate(net, W), max(len(c) for c in scans), 4)
pipe.run(hs)
torch.cuda.synchronize()
for rep in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    pipe.run(hs[3:], before_scan=lambda i: flush.zero_())
    b.record()
    torch.cuda.synchronize()
    print(f"W={W} rep {rep}: {20 / (a.elapsed_time(b) / 1e3):7.1f} scans/s  host {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
