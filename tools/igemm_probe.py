"""Gathered-GEMM probe: per-layer implicit-GEMM timing on the MinkUNet lidar
scan against the padding-aware tensor bound. For each C: algorithmic TFLOP/s
(2*pairs*C^2), fraction of the measured peak, rows the MMA actually processes
(sum over 256-row items of 256 x popcount(item OR-mask)), cycles per 256-row
column step per SM, and the MMA-only time those rows need at peak.

  python tools/igemm_probe.py [--c 32 64 96 128 256] [--splits 1] [--dgrad]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import lidar_scan


def timeit(fn, warm=3, reps=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100_000)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def item_rows(m, splits, item=256):
    tot = 0
    for (_b, _e, ent, _orow, masks) in m.split(splits, 128):
        n = len(ent)
        for t in range(0, n, item):
            mm = np.bitwise_or.reduce(masks[t:t + item], axis=0)
            tot += item * sum(bin(int(x)).count("1") for x in mm)
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c", type=int, nargs="+", default=[32, 64, 96, 128, 256])
    ap.add_argument("--splits", type=int, nargs="+", default=[1])
    ap.add_argument("--dgrad", action="store_true")
    ap.add_argument("--json", default=None)
    ap.add_argument("--cta-k", type=int, default=0, help="TilePreset cta_k (0 auto, 32 = 32-channel stages)")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("bf16_tflops", 1675.9)
    coords = lidar_scan(200_000, seed=1)
    c = sk.CoordSet.create(torch.from_numpy(coords).cuda())
    m = sk.build_kmap(c, c, 3, 1)
    pairs = m.total_pairs()
    n = len(coords)
    out = {"n": n, "pairs": pairs, "rows": []}
    g = torch.Generator(device="cuda").manual_seed(0)
    for s in a.splits:
        rows = item_rows(m, s)
        for C in a.c:
            x = torch.randn(n, C, device="cuda", generator=g).half()
            w = (torch.randn(27, C, C, device="cuda", generator=g) / 40).half()
            cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, s, sk.TilePreset(128, 0, a.cta_k, 128, 4))
            fl = 2.0 * pairs * C * C
            t = timeit(lambda: sk.conv_forward(m, x, w, cfg))
            steps = rows / 256
            rec = {"C": C, "splits": s, "pad": rows / pairs, "fwd_ms": t,
                   "tflops": fl / t / 1e9, "frac": fl / t / 1e9 / peak,
                   "cyc_per_step": t * 1e-3 * 1.965e9 * 148 / steps,
                   "mma_bound_ms": 2.0 * rows * C * C / (peak * 1e12) * 1e3}
            if a.dgrad:
                td = timeit(lambda: sk.conv_dgrad(m, x, w, cfg))
                rec["dgrad_ms"] = td
            out["rows"].append(rec)
            print(json.dumps(rec), flush=True)
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
