"""Driver bench: MinkUNet-18 inference on SemanticKITTI-shaped synthetic scans
(BASELINE.json configs[1]) on sk200, or the reference's CPU NetworkRunner
(`--impl reference`).

One step = one NEW ~125k-voxel scan through the whole network, cold: its
coordinate hash, every group's kernel maps (downsample, query, transpose,
split/sort) and all 77 convolutions (fp16 in, fp32 accumulate). Scans are
distinct per step (seeded planar-patch clouds, 5 cm voxels), so nothing is
cached across steps; L2 (126 MB) is flushed between timed steps.

Prints ONE JSON line (rank 0). Under torchrun each rank runs its own scans
(scene-sharded data parallelism, no collective: weak scaling); the timed
region is bracketed by barrier + synchronize and the max over ranks is taken.

  value       scans/s over all ranks, inputs already in HBM, --concurrency
              (default 8) scans in flight per GPU; config.latency_ms_per_scan
              is the one-scan-at-a-time latency
  e2e         scans/s through the public API (pipeline.ScanPipeline) from
              pinned HOST coords+feats to the output features in pinned host
              memory: every scan's H2D and D2H inside one timed window,
              overlapped with neighbouring scans' forwards on copy streams
  roofline    dominant kernel group (implicit GEMM convs): algorithmic
              2*pairs*C_in*C_out FLOPs / CUDA-event time vs measured bf16 peak
  cpu_baseline  the compiled reference (oracle/_ref) NetworkRunner::forward on
              the same scan spec, all host cores, rank 0 only
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "MinkUNet ms/scan & scans/s (1–8 B200); spconv TFLOP/s, kmap GB/s vs roofline"
WORKLOAD = ("MinkUNet-18 inference (SURVEY App. B skeleton: 77 convs, 14 map groups) on a "
            "SemanticKITTI-shaped synthetic LiDAR scan (planar_patches n=200k, extent 4, "
            "5 cm voxels, 124,756 voxels at seed 1: exact gen_cloud restatement), 4 input channels, fp16 in / fp32 accumulate, cold "
            "maps per scan")


WORKLOAD_SECOND = ("SECOND/CenterPoint sparse 3D encoder (SURVEY App. A: subm 4->16, 16->16, three "
                   "[s2 conv + 2 subm] stages at 32/64/64, s2 conv 64->128; kernel maps reused "
                   "across each stride level) on a Waymo-shaped synthetic scan (planar_patches "
                   "n=275k, extent 8, voxel 0.1x0.1x0.15 m, 149,357 voxels at seed 1), fp16 in / fp32 "
                   "accumulate, cold maps per scan")


def model_for(workload):
    from paper_2311_12862_b200.models import minkunet18, second_encoder
    return second_encoder() if workload == "second" else minkunet18()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "fallback": True}


def make_scans(count, seed0, n_points=200_000, workload="infer"):
    from paper_2311_12862_b200.synth import lidar_scan, waymo_scan
    if workload == "second":
        return [waymo_scan(seed=seed0 + i) for i in range(count)]
    return [lidar_scan(n_points, seed=seed0 + i) for i in range(count)]


class ClockSampler:
    def __init__(self, gpu_index=0):
        self.proc = None
        self.path = f"/tmp/sk_clocks_{os.getpid()}.csv"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_time(coords, feats, threads, max_steps=1, workload="infer"):
    """Reference NetworkRunner::forward (cold) on the host cores; seconds/scan."""
    from oracle.oracle import Reference
    from paper_2311_12862_b200.models import spec_text
    ref = Reference()
    times = []
    for i in range(max_steps):
        net = ref.network(3, spec_text(model_for(workload)), prec=0, threads=threads, weight_seed=3)
        net.set_input(coords[i % len(coords)], feats[i % len(feats)].astype(np.float64), prec=0)
        t0 = time.perf_counter()
        net.forward()
        times.append(time.perf_counter() - t0)
    return times


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank, world):
    """--impl reference: the compiled reference on the box's host cores, on
    the very scans the sk200 arm times (rank 0's seeds warmup+1 ...)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    wl = args.workload if args.workload == "second" else "infer"
    k = max(1, min(args.steps, 4))
    scans = make_scans(args.warmup + k, 1, workload=wl)[args.warmup:]
    feats = bench_feats(scans, args.warmup, 0)
    feats = [f.astype(np.float32) for f in feats]
    # bounded sample: full cold scans, as many as fit ~120 s (at least 1)
    t_one = cpu_reference_time(scans, feats, threads, 1, wl)[0]
    n = max(1, min(args.steps, int(120.0 / max(t_one, 1e-3))))
    times = [t_one] + (cpu_reference_time(scans[1:] + scans[:1], feats[1:] + feats[:1], threads,
                                          n - 1, wl) if n > 1 else [])
    sec = statistics.median(times)
    value = 1.0 / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "scans/s",
        "n_gpus": world, "steps": len(times), "steps_requested": args.steps, "warmup": 0,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD_SECOND if wl == "second" else WORKLOAD,
                   "voxels_per_scan": int(np.mean([len(c) for c in scans])),
                   "scans": f"the sk200 arm's timed scans {args.warmup}..{args.warmup + k - 1} "
                            "(gen_cloud seeds warmup+1..)",
                   "impl_detail": "compiled reference NetworkRunner::forward, default GGS "
                                  "assignment, f32, cold maps"},
        "cpu_baseline": {"value": value, "unit": "scans/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{len(times)} cold {'SECOND encoder' if wl == 'second' else 'MinkUNet-18'} scans (median)"},
        "e2e": {"value": value, "unit": "scans/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_feats(scans, first_index, rank):
    """4-channel N(0,1) fp16 features of scan i, seeded by (rank, global scan
    index) so both arms read identical inputs."""
    return [np.random.default_rng([rank, first_index + i]).standard_normal((len(c), 4))
            .astype(np.float16) for i, c in enumerate(scans)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sk200", choices=["sk200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--splits", type=int, default=1)
    ap.add_argument("--workload", default="infer", choices=["infer", "second", "train"],
                    help="infer: configs[1] MinkUNet inference (default); second: configs[2] "
                         "SECOND encoder inference; train: configs[3] mixed-precision DP "
                         "training step, global batch 8 scans")
    ap.add_argument("--concurrency", type=int, default=8,
                    help="scans in flight (host threads x CUDA streams x NetworkRunners); "
                         "1 = one scan at a time")
    ap.add_argument("--no-tune", action="store_true",
                    help="skip the per-group autotuner; use implicit GEMM --splits everywhere")
    ap.add_argument("--tune", default=os.environ.get("SK_BENCH_TUNE"), choices=["warm", "cold"],
                    help="warm: the reference tuner (probes on cached maps); cold: every probe "
                         "builds the maps of a fresh copy of the tuning scan (sk_net_set_tune_cold). "
                         "Default: cold for the map-bound SECOND encoder (0.65-0.70 -> 0.55-0.58 "
                         "ms per scan), warm for MinkUNet (within noise either way)")
    args = ap.parse_args()
    if args.tune is None:
        args.tune = "cold" if args.workload == "second" else "warm"

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.workload == "train":
        return run_train(args, rank, world, local)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2311_12862_b200 import _lib, sparse as sk
    from paper_2311_12862_b200.models import minkunet18
    from paper_2311_12862_b200.network import NetworkRunner

    n_scans = args.warmup + args.steps
    wl = args.workload
    scans = make_scans(n_scans, 1 + rank * 10000, workload=wl)
    rng = np.random.default_rng(rank)
    feats = bench_feats(scans, 0, rank)
    net = NetworkRunner(model_for(wl), dtype=torch.float16, weight_seed=3)
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, args.splits, sk.tile_large()))
    dev_coords = [torch.from_numpy(c).cuda() for c in scans]
    dev_feats = [torch.from_numpy(f).cuda() for f in feats]
    tuned = None
    if not args.no_tune:
        # per-group autotuner (tune_inference, tuner.cpp:134-160) on a separate
        # sample scan; the chosen configs then serve every timed scan
        tscan = make_scans(1, 900_000 + rank, workload=wl)[0]
        tcs = sk.CoordSet.create(torch.from_numpy(tscan).cuda())
        tf = torch.from_numpy(rng.standard_normal((len(tscan), 4)).astype(np.float16)).cuda()
        t0 = time.perf_counter()
        net.set_tune_cold(args.tune == "cold")
        lat, _ = net.tune(tcs, tf, training=0, warmup=1, runs=3)
        net.set_tune_cold(False)
        tuned = {"tune_s": time.perf_counter() - t0, "tuned_forward_ms": lat, "tune": args.tune,
                 "configs": [net.config(g).name() for g in range(net.num_groups)]}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()

    yout = torch.empty(max(len(c) for c in scans), net.layer_shapes[-1][2], dtype=torch.float16,
                       device="cuda")

    def step(i):
        cs = sk.CoordSet.create(dev_coords[i])
        y, _ = net.forward(cs, dev_feats[i], out=yout)
        return y

    def timed(fn, idxs):
        ev = []
        for i in idxs:
            flush.zero_()  # outside the timed window: L2 flush
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn(i)
            b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev)

    # per-scan latency: one scan at a time, CUDA events around each scan, L2
    # flushed outside the events
    for i in range(n_scans):  # every scan once: all buffer size classes seen
        step(i)
    torch.cuda.synchronize()
    lat_ms = timed(step, range(args.warmup, n_scans)) / args.steps

    # throughput (value): W scans in flight, one host thread + NetworkRunner +
    # CUDA stream per worker (pipeline.replicate: same weights and configs);
    # one event window over the K timed scans, L2 flush before every scan
    # INSIDE the window
    from paper_2311_12862_b200.pipeline import ScanPipeline, replicate
    W = max(1, args.concurrency)
    nets = replicate(net, W)
    wstreams = [torch.cuda.Stream() for _ in range(W)]
    # per-worker output buffers: no allocator call per scan (a cudaMalloc for a
    # new size class stalls the whole device for milliseconds)
    c_out = net.layer_shapes[-1][2]
    wout = [torch.empty(max(len(c) for c in scans), c_out, dtype=torch.float16, device="cuda")
            for _ in range(W)]

    calls = []  # host ms per (create, forward): stall diagnostics on stderr

    def concurrent(idxs):
        calls.clear()
        cur = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(cur)

        def worker(w):
            torch.cuda.set_device(local)
            with torch.cuda.stream(wstreams[w]):
                wstreams[w].wait_event(start)
                for i in idxs[w::W]:
                    t0 = time.perf_counter()
                    flush.zero_()
                    cs = sk.CoordSet.create(dev_coords[i])
                    t1 = time.perf_counter()
                    nets[w].forward(cs, dev_feats[i], out=wout[w])
                    calls.append((1e3 * (t1 - t0), 1e3 * (time.perf_counter() - t1), w, i))
        th = [threading.Thread(target=worker, args=(w,)) for w in range(W)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for st_ in wstreams:
            cur.wait_stream(st_)

    concurrent(list(range(n_scans)))  # every scan once: all buffer size classes seen
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    time.sleep(0.3)  # let the sampler start before the load
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.lib().sk_kernel_launches()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record()
    concurrent(list(range(args.warmup, n_scans)))
    eb.record()
    torch.cuda.synchronize()
    t_ms = ea.elapsed_time(eb)
    clk = clocks.stop()
    slow = sorted(calls, key=lambda c: -max(c[0], c[1]))[:3]
    print(f"[bench] window {t_ms / args.steps:.3f} ms/scan; slowest host calls "
          f"(create ms, forward ms, worker, scan): {[tuple(round(x, 2) for x in c) for c in slow]}",
          file=sys.stderr)
    launches = _lib.lib().sk_kernel_launches() - launches0
    if world > 1:
        t = torch.tensor([t_ms, lat_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms, lat_ms = float(t[0].item()), float(t[1].item())
    total_scans = args.steps * world
    value = total_scans / (t_ms / 1e3)
    ms_per_step = t_ms / args.steps

    # ---- e2e through the public API with pinned host buffers ----
    host_c = [torch.from_numpy(c).pin_memory() for c in scans]
    host_f = [torch.from_numpy(f).pin_memory() for f in feats]
    h2d = int(np.mean([c.numel() * 4 + f.numel() * 2 for c, f in zip(host_c, host_f)]))
    # ScanPipeline with the same W workers: H2D of a worker's next scan and
    # D2H of its previous one ride their own streams under its forward; one
    # window from the first H2D to the last D2H landing in pinned host memory,
    # L2 flush before every scan INSIDE it
    pipe = ScanPipeline(nets, max(len(c) for c in scans), 4, streams=wstreams)
    e2e_scans = [(host_c[i], host_f[i]) for i in range(n_scans)]
    for _ in range(2):  # every scan twice (size classes, steady state), then the timed pass
        pipe.run(e2e_scans)
    torch.cuda.synchronize()
    pipe.reset_counters()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record()
    pipe.run(e2e_scans[args.warmup:], before_scan=lambda i: flush.zero_())
    eb.record()
    torch.cuda.synchronize()
    e2e_ms = ea.elapsed_time(eb)
    d2h = int(pipe.d2h_bytes / args.steps)
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = total_scans / (e2e_ms / 1e3)

    # ---- roofline of the dominant kernel group (per-group CUDA-event timing) ----
    cs = sk.CoordSet.create(dev_coords[0])
    _, st = net.forward(cs, dev_feats[0], stats=True)
    kmap_ms = float(np.sum(st["mapping_ms"]))
    group_flops = np.zeros(net.num_groups)
    pairs_by_layer = layer_pairs(sk, net, cs)
    for li, lay in enumerate(net.layers):
        group_flops[net.group_of_layer(li)] += 2.0 * pairs_by_layer[li] * lay.c_in * lay.c_out
    kr = st["kernel_ms"]
    g_dom = int(np.argmax(kr))
    pk = peaks()
    achieved = group_flops[g_dom] / (kr[g_dom] / 1e3) / 1e12
    net_tflops = group_flops.sum() / (float(np.sum(kr)) / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath) and wl == "infer":  # the capture is of MinkUNet's group-0 kernel
        traffic = json.load(open(tpath)).get("dominant_dram_bytes_per_launch")

    kmap_roof = kmap_roofline(sk, pk) if rank == 0 else None

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            t = cpu_reference_time(scans[args.warmup:args.warmup + 1],
                                   [f.astype(np.float32) for f in feats[args.warmup:args.warmup + 1]],
                                   threads, 1, wl)
            cpu = {"value": 1.0 / t[0], "unit": "scans/s", "cores": threads, "kind": "reference",
                   "cpu_model": cpu_model(),
                   "sample": f"1 cold {'SECOND encoder' if wl == 'second' else 'MinkUNet-18'} "
                             "forward on the first timed scan, f32, compiled reference "
                             "NetworkRunner (default GGS assignment)"}
        except Exception as e:  # reported, never fatal for the GPU line
            cpu = {"value": None, "unit": "scans/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "scans/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_SECOND if wl == "second" else WORKLOAD,
                       "voxels_per_scan": int(np.mean([len(c) for c in scans])),
                       "parallelism": f"scene-sharded dp{world} (no collective)",
                       "concurrency": f"{W} scans in flight per GPU ({W} host threads x "
                                      f"{W} CUDA streams x {W} NetworkRunners)",
                       "latency_ms_per_scan": lat_ms,
                       "dataflow": (tuned if tuned else
                                    f"implicit_gemm s{args.splits} (all groups, untuned)"),
                       "l2": "flushed (256 MB write) before every scan, inside the timed "
                             "window (latency: outside the per-scan events)",
                       "network_flops_per_scan": float(group_flops.sum()),
                       "network_tflops_kernels_only": net_tflops,
                       "kmap_ms_per_scan": kmap_ms},
            "roofline": {"bound": "tensor", "achieved": achieved,
                         "peak": pk.get("bf16_tflops", 1590.0), "unit": "TFLOP/s",
                         "frac": achieved / pk.get("bf16_tflops", 1590.0), "traffic": traffic,
                         "kernel": f"k_gconv_tc, map group {g_dom} "
                                   f"({', '.join(net.layers[i].name for i in net.groups()[g_dom][:3])}...)",
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)"
                                        if "fallback" not in pk else "fallback"},
            "roofline_kmap": kmap_roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "scans/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "pipeline.ScanPipeline: pinned host scans -> H2D (copy-in stream) "
                            "-> CoordSet.create + NetworkRunner.forward -> D2H to pinned host "
                            "(copy-out stream); one CUDA-event window over all timed scans, "
                            "L2 flush inside it"},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_train(args, rank, world, local):
    """configs[3]: MinkUNet mixed-precision training step (fwd + dgrad + wgrad),
    global batch 8 scans dealt scene-by-scene to the ranks, bucketed NCCL
    all-reduce of fp32 weight gradients overlapping the backward (strong
    scaling: the global batch is fixed)."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2311_12862_b200 import _lib, sparse as sk
    from paper_2311_12862_b200.dist import DataParallelTrainer, shard_scenes
    from paper_2311_12862_b200.models import minkunet18
    from paper_2311_12862_b200.network import NetworkRunner
    B = 8
    batches = [make_scans(B, 100 * s + 1) for s in range(args.warmup + args.steps)]
    net = NetworkRunner(minkunet18(), dtype=torch.float16, weight_seed=3)
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
    tuned = None
    if not args.no_tune:
        # tune_training (tuner.cpp:162-220, workload_pattern: forward, dgrad and
        # wgrad configs per group) on a separate sample scan, before the trainer
        # snapshots the weights
        tscan = make_scans(1, 900_000 + rank)[0]
        tcs = sk.CoordSet.create(torch.from_numpy(tscan).cuda())
        tf = torch.from_numpy(np.random.default_rng(7).standard_normal((len(tscan), 4))
                              .astype(np.float16)).cuda()
        t0 = time.perf_counter()
        lat, _ = net.tune(tcs, tf, training=1, warmup=1, runs=3)
        tuned = {"tune_s": time.perf_counter() - t0, "tuned_train_ms_per_scan": lat,
                 "configs": {ph: [net.config(g, ph).name() for g in range(net.num_groups)]
                             for ph in ("forward", "dgrad", "wgrad")}}
    tr = DataParallelTrainer(net, lr=1e-3, momentum=0.9, replicas=max(1, args.concurrency))
    rng = np.random.default_rng(rank)
    prepared = []
    for scans in batches:
        mine = shard_scenes([len(c) for c in scans], rank, world)
        prepared.append([(torch.from_numpy(scans[i]).cuda(),
                          torch.from_numpy(rng.standard_normal((len(scans[i]), 4))
                                           .astype(np.float16)).cuda(),
                          torch.from_numpy(rng.standard_normal((len(scans[i]), 96))
                                           .astype(np.float16)).cuda()) for i in mine])

    def step(i):
        scenes = [(sk.CoordSet.create(c), x, t) for c, x, t in prepared[i]]
        return tr.train_step(scenes, B)

    # e2e: the same steps from pinned HOST scans (coords, feats, targets) copied
    # in every step and the loss read back every step
    host = [[(c.cpu().pin_memory(), x.cpu().pin_memory(), t.cpu().pin_memory()) for c, x, t in pb]
            for pb in prepared]
    dev_slots = [[(torch.empty_like(c, device="cuda"), torch.empty_like(x, device="cuda"),
                   torch.empty_like(t, device="cuda")) for c, x, t in pb] for pb in host]
    h2d_bytes = [sum(c.numel() * c.element_size() + x.numel() * x.element_size() +
                     t.numel() * t.element_size() for c, x, t in pb) for pb in host]
    loss_host = torch.empty((), dtype=torch.float32).pin_memory()

    def step_e2e(i):
        scenes = []
        for (hc, hx, ht), (dc_, dx_, dt_) in zip(host[i], dev_slots[i]):
            dc_.copy_(hc, non_blocking=True)
            dx_.copy_(hx, non_blocking=True)
            dt_.copy_(ht, non_blocking=True)
            scenes.append((sk.CoordSet.create(dc_), dx_, dt_))
        loss = tr.train_step(scenes, B)
        loss_host.copy_(loss.float(), non_blocking=True)
        return loss

    # warm pass over every batch: the torch allocator (loss temporaries, per
    # replica stream) and the block cache see every size class before the
    # timed steps (a cudaMalloc mid-window stalls the whole device)
    for i in range(args.warmup + args.steps):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.lib().sk_kernel_launches()
    clocks = ClockSampler(local)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(args.warmup, args.warmup + args.steps):
        step(i)
    b.record()
    torch.cuda.synchronize()
    launches1 = _lib.lib().sk_kernel_launches()
    clk = clocks.stop()
    t_ms = a.elapsed_time(b)
    # e2e window (host data in, loss out, every step)
    for i in range(min(2, args.warmup)):
        step_e2e(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a.record()
    for i in range(args.warmup, args.warmup + args.steps):
        step_e2e(i)
    b.record()
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([t_ms, e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms, e2e_ms = float(t[0].item()), float(t[1].item())
    value = B * args.steps / (t_ms / 1e3)
    # roofline: every conv's algorithmic fwd + dgrad + wgrad FLOPs
    # (3 x 2 * pairs * C_in * C_out per scan) over the whole step, against the
    # sustained bf16 peak (a step is seconds-long at the power cap)
    pk = peaks()
    step_flops = 0.0
    for c, _x, _t in prepared[args.warmup]:
        cs = sk.CoordSet.create(c)
        pr = layer_pairs(sk, net, cs)
        step_flops += sum(3 * 2.0 * pr[i] * l.c_in * l.c_out for i, l in enumerate(net.layers))
    step_flops *= world  # every rank's scenes of the global batch (weak: B fixed)
    peak_s = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    ach = step_flops / (t_ms / args.steps * 1e-3) / 1e12
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        c0, x0, _ = prepared[args.warmup][0]
        from oracle.oracle import Reference
        from paper_2311_12862_b200.models import spec_text
        ref = Reference()
        rn = ref.network(3, spec_text(minkunet18()), prec=0, threads=threads, weight_seed=3)
        rn.set_input(c0.cpu().numpy(), x0.float().cpu().numpy().astype(np.float64), prec=0)
        t0 = time.perf_counter()
        rn.measure(fwd=True, dgrad=True, wgrad=True)
        sec = time.perf_counter() - t0
        cpu = {"value": 1.0 / sec, "unit": "scans/s", "cores": threads, "kind": "reference",
               "cpu_model": cpu_model(),
               "sample": "1 scan: compiled reference NetworkRunner::measure_ms (forward + dgrad "
                         "+ wgrad sweeps, f32, default GGS) on the first timed batch's first scan"}
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "scans/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic",
            "config": {"workload": "MinkUNet-18 mixed-precision training step (fwd + dgrad + "
                                   "wgrad, SGD), global batch 8 synthetic ~128k-voxel scans, "
                                   "scene-sharded DP with bucketed NCCL all-reduce",
                       "global_batch": B, "parallelism": f"dp{world}",
                       "concurrency": f"{len(tr.nets)} runner replicas per GPU (host threads x "
                                      "CUDA streams), gradients folded before the last scene",
                       "params": int(net.num_params),
                       "dataflow": tuned if tuned else "implicit_gemm s1 (all groups, untuned)"},
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak_s, "unit": "TFLOP/s",
                         "frac": ach / peak_s, "traffic": None,
                         "kernel": "whole training step: every conv's fwd + dgrad + wgrad "
                                   "(3 x 2*pairs*C_in*C_out per scan), all kernels in the step",
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained"},
            "cpu_baseline": cpu,
            "e2e": {"value": B * args.steps / (e2e_ms / 1e3), "unit": "scans/s",
                    "h2d_bytes_per_step": int(h2d_bytes[args.warmup]), "d2h_bytes_per_step": 4,
                    "path": "pinned host coords / feats / targets -> device every step, "
                            "CoordSet.create + DataParallelTrainer.train_step, loss -> pinned host"},
            "gpu_launches": int(launches1 - launches0),
            "clocks": clk}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def kmap_roofline(sk, pk):
    """Kernel-map build on the C5 1M-voxel sweep point (10 disjoint tiles of
    the planar n=160k / 2.5 cm recipe): coordinate set creation
    (copy + hash insert) and the K=3 submanifold map (block-index query at
    this size: k_block_claim + k_block_fill + k_kmap_query_blk; OS, masks). Algorithmic bytes are SURVEY §8(d)'s contract: 100 + 4*K^D =
    208 B per voxel (coords, the table charged at 2N x 16 B for the insert and
    again for the query, out coords, OS and masks)."""
    import torch
    from paper_2311_12862_b200.synth import sweep_cloud
    coords = torch.from_numpy(sweep_cloud(160_000, seed=1, tiles=10)).cuda()
    n = coords.shape[0]
    ins, qry = [], []
    for _ in range(5):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        cs = sk.CoordSet.create(coords)  # copy + hash insert (+ range check read)
        b.record()
        m = sk.build_kmap(cs, cs, 3, 1)  # block index + query: OS, masks
        c.record()
        torch.cuda.synchronize()
        ins.append(a.elapsed_time(b))
        qry.append(b.elapsed_time(c))
        del m, cs
    t_ins, t_q = statistics.median(ins[1:]), statistics.median(qry[1:])
    kd = 27
    algo = (100 + 4 * kd) * n
    achieved = algo / ((t_ins + t_q) * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("kmap_dram_bytes_per_build")
    return {"bound": "hbm", "achieved": achieved, "peak": pk.get("hbm_gbs", 6650.0),
            "unit": "GB/s", "frac": achieved / pk.get("hbm_gbs", 6650.0), "traffic": traffic,
            "voxels": int(n), "insert_ms": t_ins, "query_ms": t_q,
            "algorithmic_bytes": int(algo),
            "bytes_contract": "SURVEY 8(d): 208 B/voxel at K=3 (table at 2N x 16 B)",
            "kernel": "k_coords_check + k_block_claim + k_block_fill + k_kmap_query_blk<3> "
                      "(1M-voxel C5 sweep point)"}


def layer_pairs(sk, net, cs):
    """Pairs per layer from the cached maps (sync; outside timed regions)."""
    sets = {}
    pairs = []
    for li, lay in enumerate(net.layers):
        src = cs if not lay.inputs else sets[lay.inputs[0]]
        if lay.kind == "conv":
            out = sk.build_out_coords(src, lay.stride)
            m = sk.build_kmap(src, out, lay.kernel, lay.stride)
            sets[lay.name] = out
        else:
            j = [l.name for l in net.layers].index(lay.transpose_of)
            jl = net.layers[j]
            jsrc = cs if not jl.inputs else sets[jl.inputs[0]]
            m = sk.build_kmap(jsrc, sets[jl.name], jl.kernel, jl.stride)
            sets[lay.name] = jsrc
        pairs.append(m.total_pairs())
    return pairs


if __name__ == "__main__":
    main()
