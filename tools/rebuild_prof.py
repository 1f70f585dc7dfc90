"""cProfile of the engine's rebuild path (migrate + build) at the bench size, GPU-synchronised."""
import cProfile, pstats, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2508_13523_b200.driver import RunConfig, Simulation
dev = torch.device("cuda", 0)
sim = Simulation(RunConfig(list_style="full", newton=False, device=dev), log=None)
sim.execute(bench.lj_script(80))
sim._ensure_system(); sim._forces_device()
for _ in range(3):
    sim._rebuild_lists()
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
for _ in range(10):
    sim._rebuild_lists()
torch.cuda.synchronize()
print("rebuild wall ms:", (time.perf_counter() - t0) * 100)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    sim._rebuild_lists()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(45)
