"""1M-voxel submanifold kmap build (for ncu). argv[1] (optional): the
context's bucketed-query row threshold (default: the library's)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import sweep_cloud
if len(sys.argv) > 1:
    sk.Context.get().set_kmap_block_rows(int(sys.argv[1]))
coords = torch.from_numpy(sweep_cloud(160_000, seed=1, tiles=10)).cuda()
for _ in range(3):
    cs = sk.CoordSet.create(coords)
    m = sk.build_kmap(cs, cs, 3, 1)
torch.cuda.synchronize()
print("done", coords.shape[0])
