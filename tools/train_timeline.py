"""Device time by kernel of one training step (DataParallelTrainer, one runner,
4 scenes, tuned-free IGEMM s1) from the CUDA activity trace."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import bench
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.dist import DataParallelTrainer
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner
net = NetworkRunner(minkunet18(), dtype=torch.float16, weight_seed=3)
net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
net.set_pdl(False)  # CUPTI durations of early-launched kernels would include their wait
tr = DataParallelTrainer(net, lr=1e-3, momentum=0.9, replicas=1)
scans = bench.make_scans(4, 1)
rng = np.random.default_rng(0)
data = [(torch.from_numpy(c).cuda(), torch.from_numpy(rng.standard_normal((len(c), 4)).astype(np.float16)).cuda(),
         torch.from_numpy(rng.standard_normal((len(c), 96)).astype(np.float16)).cuda()) for c in scans]
def step():
    tr.train_step([(sk.CoordSet.create(c), x, t) for c, x, t in data], 4)
for _ in range(2):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    k = e.name.replace("void ", "").replace("sk::(anonymous namespace)::", "").replace("sk::", "")
    k = k.split("<")[0].split("(")[0][:40]
    tot[k] = tot.get(k, 0.0) + (e.time_range.end - e.time_range.start)
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{v:9.1f} us {100 * v / s:5.1f}%  {k}")
print(f"total {s:.1f} us")
