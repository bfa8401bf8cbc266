"""One C1-shaped implicit-GEMM forward (fp16) for the SK_CONV_TRACE build:
SK_TRACE=path writes CTA 0's per-step clock64 timeline. argv: C, splits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import uniform_voxels
C = int(sys.argv[1]) if len(sys.argv) > 1 else 64
splits = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = torch.from_numpy(uniform_voxels(127_000, 64, 1)).cuda()
cs = sk.CoordSet.create(c)
m = sk.build_kmap(cs, cs, 3, 1)
x = torch.randn(cs.n, C, device="cuda").half()
w = (torch.randn(27, C, C, device="cuda") / 40).half()
cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, splits, sk.tile_large())
y = torch.empty(cs.n, C, device="cuda").half()
trace = os.environ.pop("SK_TRACE", None)
for _ in range(3):
    sk.conv_forward(m, x, w, cfg, out=y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    sk.conv_forward(m, x, w, cfg, out=y)
b.record(); b.synchronize()
print(f"C={C} splits={splits} n={cs.n} pairs={m.total_pairs()} {a.elapsed_time(b)/10*1e3:.1f} us/call")
if trace:
    os.environ["SK_TRACE"] = trace
    sk.conv_forward(m, x, w, cfg, out=y)
    torch.cuda.synchronize()
