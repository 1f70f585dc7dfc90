"""Distinct 128-byte position lines per warp gather (k_lj's L1 cost driver) for the
built full list of the 2M-atom melt, in the build's order and with each row sorted by j."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2508_13523_b200.driver import RunConfig, Simulation

dev = torch.device("cuda", 0)
sim = Simulation(RunConfig(list_style="full", newton=False, device=dev), log=None)
sim.execute(bench.lj_script(80))
sim._ensure_system(); sim._forces_device(); sim.advance(12)
torch.cuda.synchronize()
nl, s = sim.lists[0], sim.system.stores[0]
n, cap = s.n_local, nl.alloc_cap
ncl = (n + 31) // 32
t = nl.table_dev.reshape(-1)[: ncl * cap * 32].view(ncl, cap, 32).long()
cnt = nl.counts_dev[:n].long()
cntp = torch.zeros(ncl * 32, dtype=torch.long, device=dev); cntp[:n] = cnt
cntp = cntp.view(ncl, 32)
k = torch.arange(cap, device=dev).view(1, cap, 1)
valid = k < cntp.view(ncl, 1, 32)


def lines_per_pair(tab, quarter=False):
    line = torch.where(valid, tab >> 2, torch.full_like(tab, -1))
    g = line.view(ncl, cap, 4, 8) if quarter else line.view(ncl, cap, 1, 32)
    srt, _ = g.sort(dim=-1)
    distinct = ((srt[..., 1:] != srt[..., :-1]) & (srt[..., 1:] >= 0)).sum(-1) + (srt[..., 0] >= 0).long()
    return float(distinct.sum()) / float(cnt.sum())


print("n", n, "cap", cap, "mean count", float(cnt.float().mean()))
print("build order   lines/pair warp %.3f quarter %.3f" % (lines_per_pair(t), lines_per_pair(t, True)))
big = torch.iinfo(torch.long).max
ts, _ = torch.where(valid, t, torch.full_like(t, big)).sort(dim=1)
ts = torch.where(valid, ts, t)
print("j-sorted rows lines/pair warp %.3f quarter %.3f" % (lines_per_pair(ts), lines_per_pair(ts, True)))
# rows sorted by line then rank-aligned: entry order by (j >> 2)
tl_, _ = torch.where(valid, t >> 2, torch.full_like(t, big)).sort(dim=1)
