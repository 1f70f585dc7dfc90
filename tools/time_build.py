"""Event-timed pieces of one rebuild on the 2M-atom melt (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_13523_b200 import _lib
from paper_2508_13523_b200.driver import RunConfig, Simulation
import bench

dev = torch.device("cuda", 0)
style = sys.argv[1] if len(sys.argv) > 1 else "full"
sim = Simulation(RunConfig(list_style=style, newton=(style == "half"), device=dev), log=None)
sim.execute(bench.lj_script(80))
sim._ensure_system(); sim._forces_device()
for _ in range(12):
    sim.step_device()
torch.cuda.synchronize()
lib = _lib.lib()
T = {}
orig = {name: getattr(lib, name) for name in ("mdkk_nbr_build", "mdkk_bin_atoms", "mdkk_halo_count", "mdkk_halo_fill",
                                             "mdkk_wrap", "mdkk_gather_rows4", "mdkk_lj_force", "mdkk_pack_shift")}
class Wrap:
    def __init__(self, name, fn): self.name, self.fn = name, fn
    def __call__(self, *a):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); r = self.fn(*a); e.record(); T.setdefault(self.name, []).append((s, e)); return r
class Proxy:
    def __getattr__(self, n):
        f = getattr(lib, n)
        return Wrap(n, f) if n in orig else f
_lib._lib = Proxy()
for _ in range(4):
    sim._rebuild_lists()
    sim._forces_device()
torch.cuda.synchronize()
for k, v in T.items():
    ms = [a.elapsed_time(b) for a, b in v]
    print(f"{k:22s} n={len(ms):3d} mean={np.mean(ms):8.3f} ms  min={np.min(ms):8.3f}")
print("cap", [nl.alloc_cap for nl in sim.lists], "max", [nl.max_count for nl in sim.lists])
