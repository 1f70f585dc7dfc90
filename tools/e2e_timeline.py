"""GPU timeline of the bench's end-to-end `run 100` (host arrays in, thermo + snapshots out):
device busy vs idle and the largest idle gaps with the ops around them."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import bench
from paper_2508_13523_b200.driver import RunConfig, Simulation

dev = torch.device("cuda", 0)


def one():
    sim = Simulation(RunConfig(list_style="full", newton=False, skin=bench.LJ["skin"], device=dev), log=None)
    sim.execute(bench.lj_script(80, style_newton_thermo=100))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.run_nve(100)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


one(); one()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ms = one()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
k = sorted(({"name": e.name, "ts": e.time_range.start, "dur": e.time_range.end - e.time_range.start} for e in ev),
           key=lambda e: e["ts"])
span = k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]
iv, busy, cs, ce = sorted((e["ts"], e["ts"] + e["dur"]) for e in k), 0.0, None, None
for s0, e0 in iv:
    if ce is None or s0 > ce:
        if ce is not None:
            busy += ce - cs
        cs, ce = s0, e0
    else:
        ce = max(ce, e0)
busy += ce - cs
print(f"e2e wall {ms:.2f} ms; device span {span / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms, idle {(span - busy) / 1e3:.2f} ms")
gaps, end = [], k[0]["ts"] + k[0]["dur"]
for a, b in zip(k, k[1:]):
    end = max(end, a["ts"] + a["dur"])
    if b["ts"] > end:
        gaps.append((b["ts"] - end, a["name"][:45], b["name"][:45], (b["ts"] - k[0]["ts"]) / 1e3))
gaps.sort(reverse=True)
print("largest device-idle gaps (us, before -> after, at ms):")
for g in gaps[:20]:
    print(f"  {g[0]:9.1f}  {g[1]} -> {g[2]}  @{g[3]:.2f}")
if len(sys.argv) > 1 and sys.argv[1] == "--head":
    t0 = k[0]["ts"]
    print("first ops (start ms, dur us, name):")
    for e in k:
        if (e["ts"] - t0) / 1e3 > float(sys.argv[2] if len(sys.argv) > 2 else 9.0):
            break
        if e["dur"] > 20:
            print(f"  {(e['ts'] - t0) / 1e3:7.3f}  {e['dur']:8.1f}  {e['name'][:70]}")
