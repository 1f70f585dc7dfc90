"""GPU busy/idle timeline of the bench's LJ step loop (torch.profiler / CUPTI; no nsys needed).

Prints total wall, summed kernel time, and the largest idle gaps with the
CPU-side op that was running when each gap ended.
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import bench
from paper_2508_13523_b200.driver import RunConfig, Simulation

style = sys.argv[1] if len(sys.argv) > 1 else "full"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
loop = sys.argv[3] if len(sys.argv) > 3 else "advance"   # "advance" (the engine loop) or "step"
dev = torch.device("cuda", 0)
sim = Simulation(RunConfig(list_style=style, newton=(style == "half"), device=dev), log=None)
sim.execute(bench.lj_script(80))
sim._ensure_system(); sim._forces_device()
if loop == "advance":
    sim.advance(5)        # warm the fused loop's buffers outside the profile
else:
    for _ in range(5):
        sim.step_device()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=False) as prof:
    r0 = sim.n_rebuilds
    if loop == "advance":
        sim.advance(steps)
    else:
        for _ in range(steps):
            sim.step_device()
    torch.cuda.synchronize()
path = "gpurun_out/timeline.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy") and "dur" in e], key=lambda e: e["ts"])
t0, t1 = k[0]["ts"], k[-1]["ts"] + k[-1]["dur"]
busy = sum(e["dur"] for e in k)
print(f"{style}: steps={steps} rebuilds={sim.n_rebuilds - r0} wall(first->last kernel)={(t1 - t0) / 1e3:.3f} ms "
      f"kernel-busy={busy / 1e3:.3f} ms idle={(t1 - t0 - busy) / 1e3:.3f} ms")
gaps = []
for a, b in zip(k, k[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    if g > 0:
        gaps.append((g, a["name"][:40], b["name"][:40]))
gaps.sort(reverse=True)
tot = sum(g for g, *_ in gaps)
import collections
by = collections.Counter()
for g, a, b in gaps:
    by[(a, b)] += g
print("idle by (prev kernel -> next kernel), top 15:")
for (a, b), g in by.most_common(15):
    print(f"  {g / 1e3:8.3f} ms  {a} -> {b}")
cpu = collections.Counter()
for e in ev:
    if e.get("cat") == "cpu_op" and "dur" in e:
        cpu[e["name"][:50]] += e["dur"]
print("cpu ops (total us), top 15:")
for n, d in cpu.most_common(15):
    print(f"  {d / 1e3:8.3f} ms  {n}")
# per step: ops from one step delimiter to the next (the fused loop has no per-step
# verlet pass; each step starts with its speculative halo pack -- on one rank the pack
# rides in the previous force launch's reduction, k_reduce_pack, which then delimits)
delim = "k_verlet_first" if loop != "advance" else "k_pack_shift"
if loop == "advance" and any("k_reduce_pack" in e["name"] for e in k):
    delim = "k_reduce_pack"
starts = [n for n, e in enumerate(k) if delim in e["name"]]
rows = []
def _union(iv):
    tot, cur_s, cur_e = 0.0, None, None
    for s0, e0 in sorted(iv):
        if cur_e is None or s0 > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s0, e0
        else:
            cur_e = max(cur_e, e0)
    return tot + ((cur_e - cur_s) if cur_e is not None else 0.0)


for a, b in zip(starts, starts[1:]):
    ops = k[a:b]
    # device busy = union of the ops' intervals (side-stream copies overlap kernels);
    # idle = the step's span (to the next step's first op) minus that union
    busy = _union([(e["ts"], e["ts"] + e["dur"]) for e in ops])
    idle = max(0.0, (k[b]["ts"] - ops[0]["ts"]) - busy)
    rebuild = any("nbr_build" in e["name"] for e in ops)
    rows.append((rebuild, busy, idle, a, b))
for reb in (False, True):
    sel = [r for r in rows if r[0] == reb]
    if sel:
        print(f"{'rebuild' if reb else 'plain'} steps: n={len(sel)} busy={sum(r[1] for r in sel)/len(sel):.1f} us "
              f"idle={sum(r[2] for r in sel)/len(sel):.1f} us")
for reb in (False, True):
    sel = [r for r in rows if r[0] == reb]
    if not sel:
        continue
    _, _, _, a, b = sel[-1]
    print(("rebuild" if reb else "plain") + " step op sequence (gap before, duration, name):")
    for x, y in zip(k[a - 1:b], k[a:b + 1]):
        print(f"  gap {(y['ts'] - x['ts'] - x['dur']):8.1f} us  dur {y['dur']:8.1f} us  {y['name'][:70]}")
