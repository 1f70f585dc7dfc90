"""Host-side timing of the e2e path's pieces (no profiler): run_nve(100) from host arrays,
and the upload / download helpers on arrays of the e2e size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2508_13523_b200 import memspace
from paper_2508_13523_b200.driver import RunConfig, Simulation

dev = torch.device("cuda", 0)


def one(steps=100):
    sim = Simulation(RunConfig(list_style="full", newton=False, skin=bench.LJ["skin"], device=dev), log=None)
    sim.execute(bench.lj_script(80, style_newton_thermo=100))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.run_nve(steps)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


for k in range(4):
    print(f"run_nve(100) {one():.2f} ms")
print(f"run_nve(0) {one(0):.2f} ms")
a = np.random.default_rng(0).random((2048000, 4))
for k in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d = memspace.upload(a, dev); torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = memspace.download(d)
    t2 = time.perf_counter()
    print(f"upload 65.5 MB {1e3 * (t1 - t0):.2f} ms, download {1e3 * (t2 - t1):.2f} ms")
print("threads", torch.get_num_threads(), "cpus", os.cpu_count())


def phases():
    import math
    sim = Simulation(RunConfig(list_style="full", newton=False, skin=bench.LJ["skin"], device=dev), log=None)
    sim.execute(bench.lj_script(80, style_newton_thermo=100))
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    with torch.cuda.device(dev):
        from paper_2508_13523_b200.domain import RankedSystem
        sim.system = RankedSystem.distribute(sim.box, 1, sim._positions, sim._velocities, device=dev)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        sim._ensure_system()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        e = sim._forces_device()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        float(e.item()); sim._kinetic()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        snap = sim.system.gather_positions_async()
        snap()
        t.append(time.perf_counter())
    names = ["distribute (upload x, v)", "build_all", "forces", "thermo", "snapshot"]
    print("  ".join(f"{n} {1e3 * (b - a):.2f}" for n, a, b in zip(names, t, t[1:])))


for k in range(3):
    phases()
