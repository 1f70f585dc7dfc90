"""Dump owned+ghost rows after a rebuild of the melting 2M system (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_13523_b200.driver import RunConfig, Simulation
import bench
dev = torch.device("cuda", 0)
sim = Simulation(RunConfig(list_style="full", newton=False, device=dev), log=None)
sim.execute(bench.lj_script(80))
sim._ensure_system(); sim._forces_device()
s = sim.system.stores[0]
np.savez_compressed("gpurun_out/state0.npz", x=s.x[: s.n_total, :3].cpu().numpy(), nl=s.n_local)
for _ in range(12):
    sim.step_device()
sim._rebuild_lists()
s = sim.system.stores[0]
np.savez_compressed("gpurun_out/state12.npz", x=s.x[: s.n_total, :3].cpu().numpy(), nl=s.n_local,
                    counts=sim.lists[0].counts)
