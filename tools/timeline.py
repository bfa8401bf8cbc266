"""Device timeline of one cold MinkUNet forward (overlapped map build, as the
bench's latency pass runs it) from the CUDA activity trace (torch.profiler /
CUPTI): span, busy time (union of kernel intervals), idle gaps, and the time
per kernel class (conv / dense / map / other).

  python tools/timeline.py [--json out.json]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.network import NetworkRunner


def classify(name):
    if "k_gconv" in name or "small_cin" in name:
        return "conv"
    if "k_dense_tc" in name:
        return "dense"
    if name.startswith("void sk::") or "sk::" in name or "k_" in name:
        return "map"
    return "other"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--scans", type=int, default=3)
    a = ap.parse_args()
    scans = bench.make_scans(a.scans + 2, 1)
    rng = np.random.default_rng(0)
    dc = [torch.from_numpy(c).cuda() for c in scans]
    df = [torch.from_numpy(rng.standard_normal((len(c), 4)).astype(np.float16)).cuda() for c in scans]
    net = NetworkRunner(bench.model_for("infer"), dtype=torch.float16, weight_seed=3)
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
    net.tune(sk.CoordSet.create(dc[0]), df[0], training=0, warmup=1, runs=3)
    st = torch.cuda.Stream()
    yout = torch.empty(max(len(c) for c in scans), net.layer_shapes[-1][2], dtype=torch.float16,
                       device="cuda")
    with torch.cuda.stream(st):
        net.forward(sk.CoordSet.create(dc[1]), df[1], out=yout)
    torch.cuda.synchronize()
    res = []
    for i in range(2, 2 + a.scans):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            with torch.cuda.stream(st):
                net.forward(sk.CoordSet.create(dc[i]), df[i], out=yout)
            torch.cuda.synchronize()
        ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
        iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
        if not iv:
            continue
        t0, t1 = iv[0][0], max(e[1] for e in iv)
        busy, cur_s, cur_e = 0.0, None, None
        gaps = []
        for s, e, _n in iv:
            if cur_e is None or s > cur_e:
                if cur_e is not None:
                    busy += cur_e - cur_s
                    gaps.append(s - cur_e)
                cur_s, cur_e = s, e
            else:
                cur_e = max(cur_e, e)
        busy += cur_e - cur_s
        # gaps > 3 us with the kernels around them
        gl, end_max, prev = [], None, None
        for s_, e_, n in iv:
            if end_max is not None and s_ - end_max > 3:
                short = lambda x: x.replace("void ", "").replace("sk::(anonymous namespace)::", "").split("<")[0].split("(")[0][:24]
                gl.append((round(s_ - end_max, 1), short(prev), short(n), round(end_max - t0, 1)))
            if end_max is None or e_ > end_max:
                end_max, prev = e_, n
        cls = {}
        for s, e, n in iv:
            c = classify(n)
            cls[c] = cls.get(c, 0.0) + (e - s)
        names = {}
        for s_, e_, n in iv:
            k = n.replace("void ", "").replace("sk::(anonymous namespace)::", "").replace("sk::", "")
            k = k.split("<")[0].split("(")[0][-40:]
            names[k] = names.get(k, 0.0) + (e_ - s_)
        ms = sorted(round(e_ - s_, 1) for s_, e_, n in iv if "Memset" in n)
        gaps = np.array(gaps) if gaps else np.zeros(1)
        inst = [(round(e_ - s_, 1), n.replace("void ", "").replace("sk::(anonymous namespace)::", "").split("(")[0][:40])
                for s_, e_, n in iv]
        r = {"instances": inst, "gap_list": gl, "memsets_us": ms, "span_us": t1 - t0, "busy_us": busy, "idle_us": (t1 - t0) - busy,
             "kernels": len(iv), "gaps_over_5us": int((gaps > 5).sum()),
             "largest_gaps_us": sorted(gaps.tolist())[-8:], "by_class_us": cls,
             "by_kernel_us": dict(sorted(((k, round(v, 1)) for k, v in names.items()),
                                         key=lambda kv: -kv[1]))}
        res.append(r)
        print(json.dumps(r))
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
