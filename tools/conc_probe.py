"""Repeatability of the MinkUNet window timings: serial vs W concurrent
workers (threads x streams x runners), with and without the in-window L2
flush, each repeated to expose run-to-run spread.

  python tools/conc_probe.py [--steps 12] [--reps 3]
"""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.network import NetworkRunner
from paper_2311_12862_b200.pipeline import replicate


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-tune", action="store_true")
    ap.add_argument("--workers", type=int, nargs="+", default=[1, 2, 3])
    a = ap.parse_args()
    if os.environ.get("NO_GC"):
        import gc
        gc.disable()
    n = a.steps
    scans = bench.make_scans(n, 1)
    rng = np.random.default_rng(0)
    feats = [rng.standard_normal((len(c), 4)).astype(np.float16) for c in scans]
    net = NetworkRunner(bench.model_for("infer"), dtype=torch.float16, weight_seed=3)
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
    if not a.no_tune:
        tscan = bench.make_scans(1, 900_000)[0]
        tcs = sk.CoordSet.create(torch.from_numpy(tscan).cuda())
        tf = torch.from_numpy(rng.standard_normal((len(tscan), 4)).astype(np.float16)).cuda()
        net.tune(tcs, tf, training=0, warmup=1, runs=3)
    dev_c = [torch.from_numpy(c).cuda() for c in scans]
    dev_f = [torch.from_numpy(f).cuda() for f in feats]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    nets = replicate(net, max(a.workers))
    if os.environ.get("OVERLAP") == "1":
        for r in nets:
            r.set_overlap(True)
    streams = [torch.cuda.Stream() for _ in range(max(a.workers))]
    if os.environ.get("GC_FREEZE"):
        import gc
        gc.collect()
        gc.freeze()  # setup objects leave the collector's generations

    log = []
    traced = []

    def run(W, flushing):
        log.clear()
        cur = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(cur)

        def worker(w):
            with torch.cuda.stream(streams[w]):
                streams[w].wait_event(start)
                for i in range(w, n, W):
                    t0 = time.perf_counter()
                    if flushing:
                        flush.zero_()
                    t1 = time.perf_counter()
                    cs = sk.CoordSet.create(dev_c[i])
                    t2 = time.perf_counter()
                    nets[w].forward(cs, dev_f[i])
                    t3 = time.perf_counter()
                    log.append((w, i, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2)))
        if W == 1:
            worker(0)
        else:
            th = [threading.Thread(target=worker, args=(w,)) for w in range(W)]
            for t in th:
                t.start()
            for t in th:
                t.join()
        for s in streams[:W]:
            cur.wait_stream(s)

    for W in a.workers:
        run(W, True)
    torch.cuda.synchronize()
    for W in a.workers:
        for flushing in (True,):
            res = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                prof = None
                if os.environ.get("TRACE_SLOW") and not traced:
                    from torch.profiler import ProfilerActivity, profile
                    prof = profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA])
                    prof.__enter__()
                t0 = time.perf_counter()
                e0.record()
                run(W, flushing)
                e1.record()
                torch.cuda.synchronize()
                if prof is not None:
                    prof.__exit__(None, None, None)
                    if e0.elapsed_time(e1) / n > 5.0:
                        prof.export_chrome_trace(os.environ["TRACE_SLOW"])
                        traced.append(1)
                        print("   traced a slow rep", flush=True)
                res.append((e0.elapsed_time(e1) / n, 1e3 * (time.perf_counter() - t0) / n))
                if res[-1][0] > 3.0 * min(r[0] for r in res) or res[-1][0] > 6:
                    worst = sorted(log, key=lambda r: -max(r[2:]))[:4]
                    print("   slow rep: worst calls (w, i, flush ms, create ms, forward ms):",
                          [(w_, i_, round(a_, 2), round(b_, 2), round(c_, 2)) for w_, i_, a_, b_, c_ in worst])
            print(f"W={W} flush={int(flushing)}: " +
                  "  ".join(f"{d:6.3f} (host {h:6.3f})" for d, h in res) + "  ms/scan", flush=True)


if __name__ == "__main__":
    main()
