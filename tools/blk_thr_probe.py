"""W=1 cold MinkUNet latency vs the block-index query threshold
(sk_ctx_set_kmap_block_rows): events per scan, L2 flush outside."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.network import NetworkRunner
scans = bench.make_scans(12, 1)
rng = np.random.default_rng(0)
dc = [torch.from_numpy(c).cuda() for c in scans]
df = [torch.from_numpy(rng.standard_normal((len(c), 4)).astype(np.float16)).cuda() for c in scans]
net = NetworkRunner(bench.model_for("infer"), dtype=torch.float16, weight_seed=3)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
tcs = sk.CoordSet.create(dc[0]); net.tune(tcs, df[0], training=0, warmup=1, runs=3)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
yout = torch.empty(max(len(c) for c in scans), net.layer_shapes[-1][2], dtype=torch.float16, device="cuda")
s = torch.cuda.Stream()
for rep in range(3):
    for thr in (1 << 19, 1 << 16, 1 << 14):
        sk.Context.get().set_kmap_block_rows(thr)
        with torch.cuda.stream(s):
            for i in range(4):
                net.forward(sk.CoordSet.create(dc[i]), df[i], out=yout)
            torch.cuda.synchronize()
            ts = []
            for i in range(3, 12):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); net.forward(sk.CoordSet.create(dc[i]), df[i], out=yout); b.record()
                b.synchronize(); ts.append(a.elapsed_time(b))
        print(f"thr {thr:7d}: mean {np.mean(ts):.3f} median {np.median(ts):.3f} min {np.min(ts):.3f} ms", flush=True)
