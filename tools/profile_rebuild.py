"""cProfile of the host side of the MD loop incl. rebuilds (diagnostic)."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_13523_b200.driver import RunConfig, Simulation
import bench

dev = torch.device("cuda", 0)
sim = Simulation(RunConfig(list_style="full", newton=False, device=dev), log=None)
sim.execute(bench.lj_script(80))
sim._ensure_system(); sim._forces_device()
for _ in range(5):
    sim.step_device()
torch.cuda.synchronize()
orig = sim._rebuild_lists
times = []
def timed():
    torch.cuda.synchronize(); a = time.perf_counter(); orig(); torch.cuda.synchronize(); times.append(time.perf_counter() - a)
sim._rebuild_lists = timed
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
for _ in range(30):
    sim.step_device()
torch.cuda.synchronize()
pr.disable()
print("30 steps wall", time.perf_counter() - t0, "rebuild times ms", [round(1e3 * t, 2) for t in times],
      "caps", [nl.alloc_cap for nl in sim.lists], [nl.max_count for nl in sim.lists])
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
