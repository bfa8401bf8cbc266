"""1M-voxel submanifold kmap build (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import planar_patches, quantize
tiles = []
for t in range(10):
    c = quantize(planar_patches(160_000, 1 + t, 2.0), [0.025] * 3)
    c[:, 1] += 200 * t
    tiles.append(c)
coords = torch.from_numpy(np.concatenate(tiles)).cuda()
for _ in range(3):
    cs = sk.CoordSet.create(coords)
    m = sk.build_kmap(cs, cs, 3, 1)
torch.cuda.synchronize()
print("done", coords.shape[0])
