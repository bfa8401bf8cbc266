"""Where the end-to-end (host buffers) MinkUNet step spends its time beyond
the device-resident step: times variants of bench.py's e2e_step with the same
L2 flush between steps, plus the host-side wall time per call.

  python tools/e2e_probe.py [--steps 10]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.network import NetworkRunner


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    n = a.steps + 3
    scans = bench.make_scans(n, 1)
    rng = np.random.default_rng(0)
    feats = [rng.standard_normal((len(c), 4)).astype(np.float16) for c in scans]
    net = NetworkRunner(bench.model_for("infer"), dtype=torch.float16, weight_seed=3)
    tscan = bench.make_scans(1, 900_000)[0]
    tcs = sk.CoordSet.create(torch.from_numpy(tscan).cuda())
    tf = torch.from_numpy(rng.standard_normal((len(tscan), 4)).astype(np.float16)).cuda()
    net.tune(tcs, tf, training=0, warmup=1, runs=3)
    dev_c = [torch.from_numpy(c).cuda() for c in scans]
    dev_f = [torch.from_numpy(f).cuda() for f in feats]
    host_c = [torch.from_numpy(c).pin_memory() for c in scans]
    host_f = [torch.from_numpy(f).pin_memory() for f in feats]
    out_pinned = torch.empty(max(len(c) for c in scans) * net.layers[-1].c_out,
                             dtype=torch.float16).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def fwd(c, f):
        cs = sk.CoordSet.create(c)
        y, _ = net.forward(cs, f)
        return y

    def d2h(y):
        out_pinned[:y.numel()].view_as(y).copy_(y, non_blocking=True)

    variants = {
        "device step": lambda i: fwd(dev_c[i], dev_f[i]),
        "h2d only": lambda i: (host_c[i].cuda(non_blocking=True), host_f[i].cuda(non_blocking=True)),
        "h2d + step": lambda i: fwd(host_c[i].cuda(non_blocking=True),
                                    host_f[i].cuda(non_blocking=True)),
        "step + d2h": lambda i: d2h(fwd(dev_c[i], dev_f[i])),
        "e2e (h2d + step + d2h)": lambda i: d2h(fwd(host_c[i].cuda(non_blocking=True),
                                                    host_f[i].cuda(non_blocking=True))),
    }
    from paper_2311_12862_b200.pipeline import ScanPipeline
    pipe = ScanPipeline(net, max(len(c) for c in scans), 4)
    hs = [(host_c[i], host_f[i]) for i in range(n)]

    def window(fn, label):
        fn(warm=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        fn(warm=False)
        e1.record()
        torch.cuda.synchronize()
        print(f"{label:34s} window {e0.elapsed_time(e1) / (n - 3):7.3f} ms/scan  "
              f"host {1e3 * (time.perf_counter() - t0) / (n - 3):7.3f}")

    def serial(flushing, copies):
        def fn(warm):
            for i in (range(3) if warm else range(3, n)):
                if flushing:
                    flush.zero_()
                if copies:
                    d2h(fwd(host_c[i].cuda(non_blocking=True), host_f[i].cuda(non_blocking=True)))
                else:
                    fwd(dev_c[i], dev_f[i])
        return fn

    def piped(flushing):
        def fn(warm):
            pipe.run(hs[:3] if warm else hs[3:],
                     before_scan=(lambda i: flush.zero_()) if flushing else None)
        return fn

    window(serial(True, False), "serial device step, flush")
    window(serial(False, False), "serial device step, no flush")
    window(serial(True, True), "serial e2e, flush")
    window(piped(True), "ScanPipeline, flush")
    window(piped(False), "ScanPipeline, no flush")
    window(piped(True), "ScanPipeline, flush (again)")
    # W host threads, each with its own NetworkRunner (same configs) on its
    # own CUDA stream: one runner's sync bubbles are filled by the other's work
    import threading
    for W in (2, 3):
        nets = [net]
        for _ in range(W - 1):
            n2 = NetworkRunner(bench.model_for("infer"), dtype=torch.float16, weight_seed=3)
            for g in range(net.num_groups):
                n2.set_config(g, net.config(g))
            nets.append(n2)
        streams = [torch.cuda.Stream() for _ in range(W)]

        def conc(flushing, idxs):
            start = torch.cuda.Event()
            start.record()

            def worker(w):
                with torch.cuda.stream(streams[w]):
                    torch.cuda.current_stream().wait_event(start)
                    for i in idxs[w::W]:
                        if flushing:
                            flush.zero_()
                        cs = sk.CoordSet.create(dev_c[i])
                        nets[w].forward(cs, dev_f[i])
            th = [threading.Thread(target=worker, args=(w,)) for w in range(W)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            for st_ in streams:
                torch.cuda.current_stream().wait_stream(st_)

        for flushing in (True, False):
            conc(flushing, list(range(3 * W)))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            conc(flushing, list(range(3, n)))
            e1.record()
            torch.cuda.synchronize()
            print(f"{W} threads x streams, flush={flushing}: window "
                  f"{e0.elapsed_time(e1) / (n - 3):7.3f} ms/scan")
    if os.environ.get("E2E_TRACE"):
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            pipe.run(hs[3:7], before_scan=lambda i: flush.zero_())
            torch.cuda.synchronize()
        prof.export_chrome_trace(os.environ["E2E_TRACE"])
    print(f"y dtype {fwd(dev_c[0], dev_f[0]).dtype}, voxels {np.mean([len(c) for c in scans]):.0f}")
    for name, fn in variants.items():
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        ev, host = [], []
        for i in range(3, n):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t0 = time.perf_counter()
            fn(i)
            host.append(time.perf_counter() - t0)
            e1.record()
            ev.append((e0, e1))
        torch.cuda.synchronize()
        ms = [x.elapsed_time(y) for x, y in ev]
        print(f"{name:28s} device {np.mean(ms):7.3f} ms/step (min {np.min(ms):.3f})   "
              f"host {1e3 * np.mean(host):7.3f} ms/call")


if __name__ == "__main__":
    main()
