"""Kernel-map build timing on the 1M-voxel C5 sweep point (bench.kmap_roofline)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2311_12862_b200 import sparse as sk
print(json.dumps(bench.kmap_roofline(sk, bench.peaks())))
