"""cProfile of bench.lj_e2e (public API end to end) to see where the non-step time goes."""
import cProfile, pstats, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
bench.lj_e2e("full", 80, 100, dev)          # warm (allocator, library load)
pr = cProfile.Profile()
pr.enable()
r = bench.lj_e2e("full", 80, 100, dev)
pr.disable()
print(r)
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
