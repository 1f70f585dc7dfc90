"""Host-side trace of one engine rebuild (2M-atom melt): wall time between
consecutive library calls / torch ops, GPU idle excluded (the device is
synchronised before each rebuild).  Shows which Python segments keep the GPU
waiting in the rebuild sequence (profiles/*_lj_timeline.txt gaps)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_13523_b200 import _lib
from paper_2508_13523_b200.driver import RunConfig, Simulation
import bench

dev = torch.device("cuda", 0)
sim = Simulation(RunConfig(list_style="full", newton=False, device=dev), log=None)
sim.execute(bench.lj_script(80))
sim._ensure_system(); sim._forces_device()
sim.advance(12)
torch.cuda.synchronize()
lib = _lib.lib()
T = []


class Proxy:
    def __getattr__(self, n):
        f = getattr(lib, n)
        if not n.startswith("mdkk_"):
            return f

        def w(*a):
            T.append((time.perf_counter(), n))
            return f(*a)
        return w


_lib._lib = Proxy()
for rep in range(3):
    torch.cuda.synchronize()
    T.clear()
    t0 = time.perf_counter()
    sim._rebuild_lists(defer=True)
    t1 = time.perf_counter()
    sim._forces_device()
    sim._settle_lists()
    torch.cuda.synchronize()
    if rep == 2:
        prev = t0
        for t, n in T:
            print(f"{(t - prev) * 1e6:8.1f} us before {n}")
            prev = t
        print(f"{(t1 - prev) * 1e6:8.1f} us to the end of _rebuild_lists; total host {(t1 - t0) * 1e6:.1f} us")

if "--cprofile" in sys.argv:
    # where the host time between the library calls goes (function-level, one rebuild)
    import cProfile, pstats
    for rep in range(3):
        torch.cuda.synchronize()
        pr = cProfile.Profile()
        pr.enable()
        sim._rebuild_lists(defer=True)
        sim._forces_device()
        pr.disable()
        sim._settle_lists()
        torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)

if "--fine" in sys.argv:
    # entry / exit stamps of the Python functions between the library calls
    import functools
    from paper_2508_13523_b200 import domain, neighbor
    from paper_2508_13523_b200.driver import simulation

    def stamp(owner, name):
        f = getattr(owner, name)

        @functools.wraps(f)
        def g(*a, **k):
            T.append((time.perf_counter(), f"> {name}"))
            r = f(*a, **k)
            T.append((time.perf_counter(), f"< {name}"))
            return r
        setattr(owner, name, g)
    for owner, names in ((domain.AtomStore, ["ensure_capacity", "_views", "device_wrote", "to_device"]),
                         (domain.RankedSystem, ["migrate", "_migrate_single", "_buf", "_combos"]),
                         (neighbor, ["build", "_recycled"]),
                         (neighbor.NeighborList, ["__init__"]),
                         (simulation.Simulation, ["_forces_device"])):
        for nm in names:
            if hasattr(owner, nm):
                stamp(owner, nm)
    simulation.build = neighbor.build
    for rep in range(3):
        torch.cuda.synchronize()
        T.clear()
        t0 = time.perf_counter()
        sim._rebuild_lists(defer=True)
        sim._forces_device()
        t1 = time.perf_counter()
        sim._settle_lists()
        torch.cuda.synchronize()
    prev = t0
    for t, n in T:
        print(f"{(t - prev) * 1e6:8.1f} us before {n}")
        prev = t
