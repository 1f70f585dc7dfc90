"""cProfile of the bench's end-to-end `run 100` (host arrays -> thermo + snapshots), GPU-synchronised."""
import cProfile, gc, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2508_13523_b200.driver import RunConfig, Simulation

dev = torch.device("cuda", 0)


def one(prof=None):
    sim = Simulation(RunConfig(list_style="full", newton=False, skin=bench.LJ["skin"], device=dev), log=None)
    sim.execute(bench.lj_script(80, style_newton_thermo=100))
    gc.collect()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if prof:
        prof.enable()
    sim.run_nve(100)
    torch.cuda.synchronize()
    if prof:
        prof.disable()
    return (time.perf_counter() - t0) * 1e3


for _ in range(2):
    print("warm e2e ms:", one())
pr = cProfile.Profile()
print("profiled e2e ms:", one(pr))
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(40)
