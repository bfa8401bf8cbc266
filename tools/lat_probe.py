"""Per-scan latency (events per scan, flush outside) on the legacy default
stream vs a created stream, overlapped map build on/off."""
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
NOOUT = os.environ.get("NOOUT") == "1"


def fwd(i):
    if NOOUT:
        return net.forward(sk.CoordSet.create(dc[i]), df[i])
    return net.forward(sk.CoordSet.create(dc[i]), df[i], out=yout)


def lat(stream):
    with torch.cuda.stream(stream):
        for i in range(12):
            fwd(i)
        torch.cuda.synchronize()
        ts = []
        for i in range(3, 12):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fwd(i); b.record()
            b.synchronize(); ts.append(a.elapsed_time(b))
        return np.mean(ts), np.min(ts), np.max(ts)
for ov in (False, True):
    net.set_overlap(ov)
    for name, s in (("default", torch.cuda.default_stream()), ("created", torch.cuda.Stream())):
        r = lat(s)
        print(f"overlap={ov} {name:8s} mean {r[0]:.3f} min {r[1]:.3f} max {r[2]:.3f} ms")
