"""BASELINE configs[4] layer sweep: C in {16,32,64,128,256}, 10k-1M voxels,
K in {3,5}, stride 1 (submanifold), stride 2 and transposed stride 2; every
fixed dataflow of the reference's default_space (tuner.cpp:9-26) against the
per-layer best ("autotuned"). Synthetic planar-patch scans (SURVEY §8(d) C5
recipe: gen_cloud(planar_patches, n, extent 2.0) at 2.5 cm; 1M = 10 disjoint
tiles of the n=160k recipe). fp16 in, fp32 accumulate, CUDA events, warm maps
(map build timed separately). Writes a markdown table (stdout or --out).

  python tools/sweep.py [--quick] [--out profiles/r01_layer_sweep.md]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import planar_patches, quantize


def scan(n_points, seed=1):
    if n_points <= 160_000:
        return quantize(planar_patches(n_points, seed, 2.0), [0.025] * 3)
    tiles = []
    for t in range(int(round(n_points / 160_000))):
        c = quantize(planar_patches(160_000, seed + t, 2.0), [0.025] * 3)
        c[:, 1] += 200 * t
        tiles.append(c)
    return np.concatenate(tiles)


def timeit(fn, warm=2, reps=5):
    """Device time of fn: a ~50 us GPU sleep is queued ahead of the start event
    so the host's Python/ctypes/launch overhead overlaps it instead of being
    counted (it dominated layers under ~50 us)."""
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


def space():
    """The tuner's whole space: the reference's 12 dataflow configs
    (tuner.cpp:9-26) then the B200 kernel variants (sk_tune_space_entry)."""
    from paper_2311_12862_b200.network import default_space
    return default_space()


PEAK = 1675.9  # MEASURED_PEAKS.json bf16_tflops (burst), overridden in main()


def main():
    global PEAK
    try:
        import json
        PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        pass
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="fewer points (CI / smoke)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    sizes = [16_000, 160_000] if a.quick else [16_000, 160_000, 1_600_000]
    chans = [32, 128] if a.quick else [16, 32, 64, 128, 256]
    kernels = [3] if a.quick else [3, 5]
    modes = ["s1", "s2", "t2"]
    rows = []
    for n_pts in sizes:
        coords = scan(n_pts)
        c = sk.CoordSet.create(torch.from_numpy(coords).cuda())
        down = sk.build_out_coords(c, 2)
        for K in kernels:
            maps = {}
            for mode in modes:
                if mode == "s1":
                    maps[mode] = sk.build_kmap(c, c, K, 1)
                elif mode == "s2":
                    maps[mode] = sk.build_kmap(c, down, K, 2)
                else:
                    maps[mode] = sk.build_kmap(down, c, K, 2, transposed=True)
            for mode in modes:
                m = maps[mode]
                pairs = m.total_pairs()
                for C in chans:
                    if C == 256 and n_pts > 200_000 and K == 5:
                        continue  # > 30 s of sweep for one point
                    x = torch.randn(m.n_in, C, device="cuda").half()
                    w = (torch.randn(m.num_offsets, C, C, device="cuda") / np.sqrt(C * 27)).half()
                    flops = 2.0 * pairs * C * C
                    res = {}
                    for cfg in space():
                        res[cfg.name()] = timeit(lambda: sk.conv_forward(m, x, w, cfg))
                    best = min(res, key=res.get)
                    rows.append((len(coords), K, mode, C, pairs, res, best, flops))
                    print(f"N={len(coords)} K={K} {mode} C={C} pairs={pairs} best={best} "
                          f"{res[best]:.4f} ms {flops / res[best] / 1e9:.1f} TF/s", flush=True)
    names = [cfg.name() for cfg in space()]
    lines = ["# Layer sweep (BASELINE configs[4]): forward ms per dataflow, fp16 in / fp32 acc",
             "", "tools/sweep.py on one B200; warm maps; device time per call (a GPU sleep "
             "ahead of the start event hides host launch overhead); algorithmic TFLOP/s = "
             "2*pairs*C^2 / best time (padded MACs not credited).", "",
             "| N | K | mode | C | pairs | " + " | ".join(n.replace("implicit_gemm_", "ig_")
                                                      .replace("_offline", "") for n in names)
             + " | autotuned (best) | TF/s | frac | best / default GGS |",
             "|" + "---|" * (len(names) + 10)]
    for n, K, mode, C, pairs, res, best, flops in rows:
        lines.append(f"| {n} | {K} | {mode} | {C} | {pairs} | "
                     + " | ".join(f"{res[nm]:.4f}" for nm in names)
                     + f" | {best.replace('implicit_gemm_', 'ig_').replace('_offline', '')} "
                       f"{res[best]:.4f} | {flops / res[best] / 1e9:.1f} | {flops / res[best] / 1e9 / PEAK:.3f} | "
                       f"{res[best] / res[names[0]]:.2f} |")
    txt = "\n".join(lines) + "\n"
    if a.out:
        open(a.out, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
