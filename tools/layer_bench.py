"""Single-layer timing (C1 / C5 sweep points): kmap build, prepare, and each
dataflow's fwd/dgrad/wgrad with CUDA events. Not the driver bench (bench.py)."""
import argparse
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import uniform_voxels, lidar_scan


def timeit(fn, warm=3, reps=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scan", default="c1")
    ap.add_argument("--c", type=int, nargs="+", default=[64])
    ap.add_argument("--k", type=int, default=3)
    a = ap.parse_args()
    coords = uniform_voxels(127_000, 64, 1) if a.scan == "c1" else lidar_scan()
    dc = torch.from_numpy(coords).cuda()
    n = len(coords)
    res = {"n": n}

    def kmap_once():
        c = sk.CoordSet.create(dc)
        m = sk.build_kmap(c, c, a.k, 1)
        return m
    res["kmap_ms"] = timeit(kmap_once)
    c = sk.CoordSet.create(dc)
    m = sk.build_kmap(c, c, a.k, 1)
    res["pairs"] = m.total_pairs()
    for C in a.c:
        x = torch.randn(n, C, device="cuda").half()
        w = (torch.randn(m.num_offsets, C, C, device="cuda") / 40).half()
        flops = 2.0 * res["pairs"] * C * C
        for cfg in [sk.DataflowConfig(sk.GATHER_GEMM_SCATTER), sk.DataflowConfig(sk.FETCH_ON_DEMAND)] + \
                [sk.DataflowConfig(sk.IMPLICIT_GEMM, s, sk.tile_large()) for s in range(4)]:
            t = timeit(lambda: sk.conv_forward(m, x, w, cfg))
            res[f"C{C}_fwd_{cfg.name()}_ms"] = t
            res[f"C{C}_fwd_{cfg.name()}_TFLOPs"] = flops / t / 1e9
        cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
        t = timeit(lambda: sk.conv_dgrad(m, x, w, cfg))
        res[f"C{C}_dgrad_ig1_ms"] = t
        t = timeit(lambda: sk.conv_wgrad(m, x, x, cfg))
        res[f"C{C}_wgrad_ms"] = t
        res[f"C{C}_wgrad_TFLOPs"] = flops / t / 1e9
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
