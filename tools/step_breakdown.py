"""Wall-clock breakdown of one LJ step's phases (host + device), synchronising between phases.

Diagnostic only (not the bench): shows where a step's time goes, including
host-side Python/launch overhead of the rebuild path.
"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_13523_b200.driver import RunConfig, Simulation
import bench

def main(cells=80, steps=30, style="full"):
    dev = torch.device("cuda", 0)
    sim = Simulation(RunConfig(list_style=style, newton=(style == "half"), device=dev), log=None)
    sim.execute(bench.lj_script(cells))
    sim._ensure_system(); sim._forces_device()
    for _ in range(3):
        sim.step_device()
    T = {}
    def t(name, fn):
        torch.cuda.synchronize(); a = time.perf_counter(); r = fn(); torch.cuda.synchronize()
        T.setdefault(name, []).append(time.perf_counter() - a); return r
    for _ in range(steps):
        need = t("kick_drift+check", sim._half_kick_drift)
        if need:
            t("rebuild.migrate", lambda: sim.system.migrate(sim.style.r_c + sim.config.skin))
            from paper_2508_13523_b200.neighbor import build
            def b():
                sim.lists = [build(s, sim.system.box, sim.style.r_c, sim.config.skin, style=sim._list_style,
                                   newton=sim.config.newton, cap_hint=sim._cap_hint) for s in sim.system.stores]
            t("rebuild.build", b)
        else:
            t("forward", sim.system.forward_comm)
        t("force", sim._forces_device)
        t("kick", sim._half_kick)
    for k, v in T.items():
        print(f"{k:20s} n={len(v):3d} mean={1e3*sum(v)/len(v):8.3f} ms total={1e3*sum(v):8.2f} ms")

if __name__ == "__main__":
    main(style=sys.argv[1] if len(sys.argv) > 1 else "full")
