"""W=1 forward: per-stream kernel intervals from a CUPTI (chrome) trace, and
where the conv stream waited: idle intervals on the conv stream while the map
stream was busy (the map build on the critical path) vs. both idle."""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.network import NetworkRunner

scans = bench.make_scans(4, 1)
dc = [torch.from_numpy(c).cuda() for c in scans]
df = [torch.randn(len(c), 4, device="cuda").half() for c in scans]
net = NetworkRunner(bench.model_for("infer"), dtype=torch.float16, weight_seed=3)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
net.tune(sk.CoordSet.create(dc[0]), df[0], training=0, warmup=1, runs=3)
net.set_pdl(False)  # true kernel durations
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    net.forward(sk.CoordSet.create(dc[1]), df[1])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    with torch.cuda.stream(st):
        net.forward(sk.CoordSet.create(dc[2]), df[2])
    torch.cuda.synchronize()
path = os.path.join(tempfile.gettempdir(), "sk_trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
by = {}
for e in ev:
    by.setdefault(e["args"].get("stream", -1), []).append((e["ts"], e["ts"] + e["dur"], e["name"]))
t0 = min(s for v in by.values() for s, _, _ in v)
conv_stream = max(by, key=lambda k: sum(1 for s, e, n in by[k] if "k_gconv" in n or "k_dense" in n))
print("streams:", {k: len(v) for k, v in by.items()}, "conv stream", conv_stream)
cv = sorted(by[conv_stream])
others = sorted(x for k, v in by.items() if k != conv_stream for x in v)
def busy_other(a, b):
    tot = 0.0
    for s, e, n in others:
        lo, hi = max(a, s), min(b, e)
        if hi > lo:
            tot += hi - lo
    return tot
span = cv[-1][1] - t0
idle_conv = []
prev_end = t0
for s, e, n in cv:
    if s > prev_end + 0.5:
        idle_conv.append((prev_end - t0, s - prev_end, busy_other(prev_end, s), n))
    prev_end = max(prev_end, e)
tot_idle = sum(g for _, g, _, _ in idle_conv)
tot_map_busy = sum(b for _, _, b, _ in idle_conv)
print(f"span {span:.0f} us; conv stream busy {sum(e - s for s, e, _ in cv):.0f} us; idle {tot_idle:.0f} us "
      f"(map stream busy during it: {tot_map_busy:.0f} us)")
for t, g, b, n in sorted(idle_conv, key=lambda x: -x[1])[:15]:
    print(f"  at {t:7.0f} us: conv idle {g:6.1f} us, map busy {b:6.1f} us, next {n.split('(')[0][-50:]}")
