"""Small MinkUNet forward + backward through the runner (PDL, overlapped map
build, one-tile items, im2col stem, 3-CTA and 2/3-CTA wgrad paths), for
compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.models import minkunet18
from paper_2311_12862_b200.network import NetworkRunner, default_space
from paper_2311_12862_b200.synth import lidar_scan
coords = lidar_scan(6000, seed=3)
c = torch.from_numpy(coords).cuda()
x = torch.randn(len(coords), 4, device="cuda").half()
net = NetworkRunner(minkunet18(), dtype=torch.float16, weight_seed=2)
space = default_space()
for cfg in (space[11], space[12], space[15], space[18], space[20]):  # s4 large, s1 m256, s1 k32, s1 m64, s3 m64
    net.set_all(cfg)
    y, _ = net.forward(sk.CoordSet.create(c), x)
    g = torch.zeros(net.num_params, device="cuda")
    net.backward(torch.ones_like(y), g)
    torch.cuda.synchronize()
    print(cfg.name(), float(y.float().abs().sum()), float(g.abs().sum()), flush=True)
print("done")
