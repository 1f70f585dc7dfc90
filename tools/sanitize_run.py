"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

Covers every kernel family of the engine on small systems: neighbour build
(full / half, newton on / off), LJ force (atom + neighbour modes, Serial /
Duplicate strategies, the gated and fused-integration launches with rebuilds),
the counting sort, ghost exchange / forward / reverse comm with 2 in-process
ranks, SNAP 2J=8 (ui / yi / deidrj, staged path, descriptors), QEq.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import md
from paper_2508_13523_b200 import Box, Duplicate, LJCut, PairParams, RankedSystem, Serial, build_all, compute_pair
from paper_2508_13523_b200.driver import RunConfig, Simulation

melt = ("units lj\nboundary p p p\nlattice fcc 0.8442\ncreate_box 6 6 6\ncreate_atoms\nmass 1.0\n"
        "velocity 1.44 87287\npair_style lj/cut 2.5\npair_coeff 1.0 1.0\ntimestep 0.005\nthermo 10\nrun 30\n")
for style in ("full", "half"):
    for ranks in (1, 2):
        sim = Simulation(RunConfig(list_style=style, newton=(style == "half"), n_ranks=ranks), log=None)
        sim.execute(melt)
        print(style, ranks, "rebuilds", sim.results[-1].n_rebuilds, flush=True)
pos, L = md.random_config(400, 0.75, seed=3)
for style, newton in (("full", False), ("half", True), ("half", False)):
    system = RankedSystem.distribute(Box(L), 2, pos, np.zeros_like(pos))
    lists = build_all(system, 2.0, 0.3, style=style, newton=newton)
    for mode in ("atom", "neighbor"):
        for strat in (None, Serial(), Duplicate(copies=3)):
            compute_pair(LJCut(PairParams(1.0, 1.0, 2.0)), system, lists, mode=mode, strategy=strat)
    lists[0].pairs()
print("lj api ok", flush=True)
from paper_2508_13523_b200.snap import (SnapState, build_neighbor_map, compute_bi, compute_deidrj, compute_duidrj,
                                        compute_fused_deidrj, compute_ui, compute_yi, make_coupling_tables)
bpos, bl = md.lattice("bcc", 3.1803, (4, 4, 4))
bpos = md.jittered(bpos, 0.05, 2)
ssys = RankedSystem.distribute(Box(bl), 1, bpos, np.zeros_like(bpos))
(snl,) = build_all(ssys, 4.73, 0.3, style="full", newton=False)
st = ssys.stores[0]
nmap = build_neighbor_map(st, snl, 4.73)
state = SnapState(make_coupling_tables(4), st.n_local, np.linspace(0.05, 0.1, 55))
compute_ui(nmap, state)
compute_yi(state)
compute_fused_deidrj(nmap, state, st.n_total)
compute_deidrj(nmap, state, compute_duidrj(nmap, state), st.n_total)
compute_bi(state)
print("snap ok", flush=True)
from paper_2508_13523_b200.qeq import QeqParams, QeqSystem, build_matrix, solve_qeq
qpos, qL = md.random_config(60, 0.5, seed=12)
qsys = RankedSystem.distribute(Box(qL), 1, qpos, np.zeros_like(qpos))
(ql,) = build_all(qsys, 2.0, 0.3, style="full", newton=False)
H = build_matrix(qsys.stores[0], ql, QeqParams(gamma=0.8, eta=20.0, chi=-0.35, cutoff=2.0))
solve_qeq(QeqSystem(H, -0.35 + 0.1 * np.random.default_rng(1).normal(size=60), tol=1e-10))
torch.cuda.synchronize()
print("sanitize workload done")
