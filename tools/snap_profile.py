"""Run a few SNAP steps (for ncu launch lists / captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 40
r = bench.snap_run(cells, 2, 1, torch.device("cuda", 0))
print(r)
